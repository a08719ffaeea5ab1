"""The C-ABI library (include/b2.h) loads and exports every declared entry
point; no-GPU and malformed-plan paths fail loudly (no CPU fallback)."""
import re
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2006_05096_b200 import plan as P
from paper_2006_05096_b200 import runtime as R
from paper_2006_05096_b200 import zoo
from paper_2006_05096_b200.errors import LaunchFailure, PlanFormatError
from conftest import has_gpu

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "b2.h").read_text()
    return sorted(set(re.findall(r"B2_API\s+[\w\s\*]+?\b(b2_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = R.load_library()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(R.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", str(R.LIB_PATH)], capture_output=True,
                         text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_sm100a_code_present():
    sass = subprocess.run(["cuobjdump", "-sass", str(R.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_version():
    assert "sm_100a" in R.version()


def test_malformed_plan_rejected_before_device():
    with pytest.raises(PlanFormatError, match="magic"):
        R.Plan(b"XXXX" + b"\0" * 100)
    blob = bytearray(zoo.build_plan("mlp"))
    blob[200] ^= 0xFF
    with pytest.raises(PlanFormatError, match="CRC"):
        R.Plan(bytes(blob))


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_no_device_is_launch_failure():
    with pytest.raises(LaunchFailure, match="no CUDA device"):
        R.Plan(zoo.build_plan("mlp"))


def test_worker_exit_codes(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"garbage that is not a model")
    r = subprocess.run([sys.executable, "-m", "paper_2006_05096_b200.worker", "--model", str(bad)],
                       capture_output=True, cwd=ROOT, timeout=120)
    assert r.returncode == 2
    if not has_gpu():
        good = tmp_path / "mlp.plan"
        good.write_bytes(zoo.build_plan("mlp", P.DT_BF16))
        r = subprocess.run([sys.executable, "-m", "paper_2006_05096_b200.worker", "--model",
                            str(good)], capture_output=True, cwd=ROOT, timeout=120)
        assert r.returncode == 3 and b"no usable device" in r.stderr
