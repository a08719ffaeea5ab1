"""ctypes binding of libb2 (include/b2.h) — the Python side of the C-ABI boundary.

``Plan`` is what the b200 worker holds in place of the reference's
``MockServer`` (pkg/src/modelci/mockserve/server.py:91-134): create from a
variant blob, ``predict`` a batch, ``bench`` a sweep cell on the device.  Status
codes map onto the errors.py classes; a missing library or device is a loud
``LaunchFailure`` — there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from . import errors
from .plan import DT_BF16, DT_FP32, IN_TOKENS

LIB_PATH = Path(__file__).resolve().parent / "libb2.so"

B2_OK, B2_ERR_FORMAT, B2_ERR_UNSUPPORTED, B2_ERR_CUDA, B2_ERR_ARG, B2_ERR_NODEVICE, B2_ERR_FUSED = range(7)
DT_FROM_PLAN = -1

_lib = None
_lib_lock = threading.Lock()


def _declare(lib):
    c = ctypes
    P = c.c_void_p
    sig = {
        "b2_plan_create": (c.c_int, [P, c.c_size_t, c.c_int, c.POINTER(P)]),
        "b2_plan_io": (c.c_int, [P, c.POINTER(c.c_int64), c.POINTER(c.c_int),
                                 c.POINTER(c.c_int64)]),
        "b2_plan_info": (c.c_int, [P, c.POINTER(c.c_double), c.POINTER(c.c_double),
                                   c.POINTER(c.c_int), c.POINTER(c.c_int)]),
        "b2_forward": (c.c_int, [P, P, P, c.c_int, P]),
        "b2_forward_host": (c.c_int, [P, P, P, c.c_int]),
        "b2_bench": (c.c_int, [P, c.c_int, c.c_int, c.c_int, c.c_uint64,
                               c.POINTER(c.c_float), c.POINTER(c.c_float)]),
        "b2_bench_e2e": (c.c_int, [P, c.c_int, c.c_int, c.c_int, c.c_uint64,
                                   c.POINTER(c.c_float), c.POINTER(c.c_float)]),
        "b2_gen_input": (c.c_int, [P, P, c.c_int, c.c_uint64, P]),
        "b2_profile_ops": (c.c_int, [P, c.c_int, c.c_int, c.POINTER(c.c_float),
                                     c.POINTER(c.c_int), c.POINTER(c.c_int)]),
        "b2_read_tensor": (c.c_int, [P, c.c_int, c.c_int, P, c.c_size_t]),
        "b2_plan_memory": (c.c_int, [P, c.POINTER(c.c_uint64)]),
        "b2_plan_destroy": (None, [P]),
        "b2_last_error": (c.c_char_p, []),
        "b2_version": (c.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


EXPORTED = ("b2_plan_create", "b2_plan_io", "b2_plan_info", "b2_forward", "b2_forward_host",
            "b2_bench", "b2_bench_e2e", "b2_gen_input", "b2_profile_ops", "b2_read_tensor",
            "b2_plan_memory", "b2_plan_destroy",
            "b2_last_error", "b2_version")


def load_library(path: os.PathLike | None = None):
    """Load (once) the in-tree libb2.so; raise LaunchFailure if absent."""
    global _lib
    with _lib_lock:
        if _lib is None:
            # B2_LIB: alternate build of the same ABI (A/B timing tools only)
            p = Path(path) if path else Path(os.environ.get("B2_LIB", LIB_PATH))
            if not p.exists():
                raise errors.LaunchFailure(
                    f"libb2.so not built at {p}; run `python -m paper_2006_05096_b200.build`")
            _lib = _declare(ctypes.CDLL(str(p)))
        return _lib


def _raise(rc: int, during: str):
    msg = load_library().b2_last_error().decode(errors="replace")
    text = f"{during}: {msg}"
    if rc in (B2_ERR_FORMAT, B2_ERR_UNSUPPORTED):
        raise errors.PlanFormatError(text, status=rc)
    if rc == B2_ERR_ARG:
        raise errors.InvalidRequest(text, status=rc)
    if during == "create" or rc == B2_ERR_NODEVICE:
        raise errors.LaunchFailure(text, status=rc)
    raise errors.CellFailure(text, status=rc)


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


class Plan:
    """A b200-plan resident on the current CUDA device."""

    def __init__(self, blob: bytes, dtype: int = DT_FROM_PLAN):
        lib = load_library()
        self._lib = lib
        self._h = ctypes.c_void_p()
        self._blob = blob
        rc = lib.b2_plan_create(blob, len(blob), dtype, ctypes.byref(self._h))
        if rc != B2_OK:
            _raise(rc, "create")
        i, k, o = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64()
        lib.b2_plan_io(self._h, ctypes.byref(i), ctypes.byref(k), ctypes.byref(o))
        self.in_elems, self.in_kind, self.out_elems = i.value, k.value, o.value
        f, w, n, d = ctypes.c_double(), ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
        lib.b2_plan_info(self._h, ctypes.byref(f), ctypes.byref(w), ctypes.byref(n),
                         ctypes.byref(d))
        self.flops_per_sample = f.value
        self.weight_bytes = w.value
        self.launches_per_forward = n.value
        self.dtype = d.value
        self.lock = threading.Lock()

    @property
    def in_dtype(self):
        return np.int64 if self.in_kind == IN_TOKENS else np.float32

    def close(self):
        if self._h:
            self._lib.b2_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- execution -----------------------------------------------------------
    def predict(self, x: np.ndarray) -> np.ndarray:
        """Host batch in, host fp32 outputs out (H2D + graph + D2H)."""
        x = np.ascontiguousarray(x, dtype=self.in_dtype)
        if x.ndim != 2 or x.shape[1] != self.in_elems or x.shape[0] < 1:
            raise errors.InvalidRequest(
                f"expected a non-empty [batch, {self.in_elems}] input, got {x.shape}")
        out = np.empty((x.shape[0], self.out_elems), dtype=np.float32)
        with self.lock:
            rc = self._lib.b2_forward_host(self._h, x.ctypes.data, out.ctypes.data, x.shape[0])
        if rc != B2_OK:
            _raise(rc, "forward")
        return out

    def forward_device(self, d_in: int, d_out: int, batch: int, stream: int = 0):
        """Device pointers (e.g. torch tensor .data_ptr()); enqueued, not synced."""
        rc = self._lib.b2_forward(self._h, ctypes.c_void_p(d_in), ctypes.c_void_p(d_out), batch,
                                  ctypes.c_void_p(stream) if stream else None)
        if rc != B2_OK:
            _raise(rc, "forward")

    def gen_input(self, d_in: int, batch: int, seed: int, stream: int = 0):
        rc = self._lib.b2_gen_input(self._h, ctypes.c_void_p(d_in), batch, seed,
                                    ctypes.c_void_p(stream) if stream else None)
        if rc != B2_OK:
            _raise(rc, "gen_input")

    def bench(self, batch: int, n: int, warmup: int = 10, seed: int = 0,
              e2e: bool = False) -> tuple[np.ndarray, np.ndarray]:
        """(latencies_ms[n], completions_ms[n]) from CUDA events."""
        lat = np.zeros(n, dtype=np.float32)
        comp = np.zeros(n, dtype=np.float32)
        fn = self._lib.b2_bench_e2e if e2e else self._lib.b2_bench
        with self.lock:
            rc = fn(self._h, batch, warmup, n, seed, _fptr(lat), _fptr(comp))
        if rc != B2_OK:
            _raise(rc, "bench")
        return lat, comp

    def read_tensor(self, batch: int, tensor: int, elems: int, kind: int,
                    rows=None) -> np.ndarray:
        """Activation `tensor` of the last forward at `batch`, as float64 (or
        int32 ids) — the verification hook used by the layerwise parity tests.
        None when the executor fused the tensor into its consumer (never
        materialised, e.g. the stem output under the fused stem/max-pool).
        ``rows``: keep only these samples (converted after the slice, so a
        batch-256 activation is never widened to float64 whole)."""
        if kind == 1:
            buf = np.empty(batch * elems, dtype=np.int32)
        elif self.dtype == DT_BF16:
            buf = np.empty(batch * elems, dtype=np.uint16)
        else:
            buf = np.empty(batch * elems, dtype=np.float32)
        rc = self._lib.b2_read_tensor(self._h, batch, tensor, buf.ctypes.data, buf.nbytes)
        if rc == B2_ERR_FUSED:
            return None
        if rc != B2_OK:
            _raise(rc, "read_tensor")
        if rows is not None:
            buf = buf.reshape(batch, elems)[list(rows)].reshape(-1)
        if buf.dtype == np.uint16:
            return (buf.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        return buf.astype(np.float64) if kind != 1 else buf

    def device_bytes(self) -> int:
        """Device memory held by the plan (b2_plan_memory)."""
        v = ctypes.c_uint64()
        rc = self._lib.b2_plan_memory(self._h, ctypes.byref(v))
        if rc != B2_OK:
            _raise(rc, "plan_memory")
        return int(v.value)

    def profile_ops(self, batch: int, iters: int = 5) -> list[tuple[int, float]]:
        cap = 4096
        ms = np.zeros(cap, dtype=np.float32)
        kinds = np.zeros(cap, dtype=np.int32)
        n = ctypes.c_int()
        with self.lock:
            rc = self._lib.b2_profile_ops(self._h, batch, iters, _fptr(ms), ctypes.byref(n),
                                          kinds.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
        if rc != B2_OK:
            _raise(rc, "profile_ops")
        return [(int(kinds[i]), float(ms[i])) for i in range(n.value)]


def version() -> str:
    return load_library().b2_version().decode()


__all__ = ["Plan", "load_library", "version", "EXPORTED", "DT_BF16", "DT_FP32", "DT_FROM_PLAN"]
