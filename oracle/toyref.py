"""ctypes wrapper of oracle/toyref.c (TEST INFRASTRUCTURE ONLY)."""
import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libtoyref.so"
ERRORS = {1: "bad magic", 2: "CRC mismatch", 3: "truncated", 4: "unsupported op", 5: "shape"}


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "toyref.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def forward(blob: bytes, x) -> np.ndarray:
    lib = ctypes.CDLL(str(build()))
    x = np.ascontiguousarray(x, dtype=np.float64)
    cap = x.shape[0] * 65536
    y = np.zeros(cap, dtype=np.float64)
    od = ctypes.c_int()
    rc = lib.toyref_forward(blob, ctypes.c_size_t(len(blob)), x.ctypes.data_as(ctypes.c_void_p),
                            x.shape[0], x.shape[1], y.ctypes.data_as(ctypes.c_void_p), cap,
                            ctypes.byref(od))
    if rc:
        raise ValueError(f"toyref: {ERRORS.get(rc, rc)}")
    return y[: x.shape[0] * od.value].reshape(x.shape[0], od.value)
