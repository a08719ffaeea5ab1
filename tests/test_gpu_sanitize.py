"""compute-sanitizer over the tcgen05 / TMA / mbarrier pipelines.

Each case runs `tools/sanitize_target.py` (one graph forward + one eager
per-op pass of a model at a small batch) under one sanitizer tool and requires
a clean summary.  The shapes are chosen so every kernel family launches:
ResNet-50 b=16 (fused stem + max-pool, CTA-pair band conv, chained block
tails, single-CTA and CTA-pair GEMMs with TMA-prefetched residuals, split-K),
BERT b=2 (fused attention, LayerNorm, GELU), MobileNetV2 b=8 (depthwise
strips, narrow-K GEMMs, band stem).  `tools/sanitize.sh` runs the wider matrix
(VGG-16, fp32 3xTF32 plans) and keeps the logs.
"""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
TARGET = ROOT / "tools" / "sanitize_target.py"


def _sanitizer() -> str:
    for cand in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if cand and Path(cand).exists():
            return cand
    pytest.fail("compute-sanitizer not found on the GPU box")


CASES = [
    ("memcheck", "resnet50", 16),
    ("memcheck", "bert", 2),
    ("memcheck", "mobilenet_v2", 8),
    ("synccheck", "resnet50", 16),
    ("racecheck", "bert", 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("tool,model,batch", CASES)
def test_compute_sanitizer_clean(gpu_required, tool, model, batch):
    env = {k: v for k, v in os.environ.items() if not k.startswith("B2_")}   # default kernels
    cmd = [_sanitizer(), "--tool", tool, "--print-limit", "10", "--error-exitcode", "97",
           sys.executable, str(TARGET), model, str(batch)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "sanitize-target ok" in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    summary = [ln for ln in out.splitlines() if "SUMMARY" in ln]
    assert summary and all((" 0 errors" in ln or " 0 hazards" in ln) for ln in summary), summary
