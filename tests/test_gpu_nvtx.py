"""NVTX ranges: every b2_bench call is an NVTX range
`b2.bench b=<B> ...` and the eager profile pass opens one range per op, so a
profiler can attribute kernels to the profiling cell that launched them.
Checked with ncu's NVTX filter: only kernels inside a matching range are
profiled, so a non-empty launch list proves the ranges exist (and an
excluded pattern proves the filter is real)."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = """
import sys
sys.path.insert(0, {root!r})
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
plan = R.Plan(zoo.build_plan("mlp", P.DT_BF16), P.DT_BF16)
plan.bench(4, n=3, warmup=1)
plan.profile_ops(4, iters=1)
plan.close()
print("nvtx-target ok")
"""


def _ncu() -> str:
    for cand in (shutil.which("ncu"), "/usr/local/cuda/bin/ncu"):
        if cand and Path(cand).exists():
            return cand
    pytest.fail("ncu not found on the GPU box")


def _profiled(include: str, tmp_path) -> tuple[int, str]:
    script = tmp_path / "nvtx_target.py"
    script.write_text(SCRIPT.format(root=str(ROOT)))
    env = {k: v for k, v in os.environ.items() if not k.startswith("B2_")}
    cmd = [_ncu(), "--nvtx", "--nvtx-include", include, "--metrics", "gpu__time_duration.sum",
           "--csv", sys.executable, str(script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    out = r.stdout + r.stderr
    assert "nvtx-target ok" in out, out[-2000:]
    return sum(1 for ln in out.splitlines() if "gpu__time_duration.sum" in ln), out


@pytest.mark.gpu
def test_nvtx_ranges_scope_the_profiled_kernels(gpu_required, tmp_path):
    n_bench, out = _profiled("regex:b2.bench.*/", tmp_path)
    assert n_bench > 0, out[-2000:]
    n_op, out = _profiled("regex:b2.profile_ops.*/", tmp_path)   # the eager per-op pass
    assert n_op > 0, out[-2000:]
    n_none, out = _profiled("regex:no-such-range.*/", tmp_path)
    assert n_none == 0, out[-2000:]
