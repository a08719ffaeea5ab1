"""The ``b200-plan`` variant format: what the converter emits and libb2 executes.

A plan is a flat, topologically ordered list of fused ops over named
activation tensors, plus fp32 weights.  It is the on-disk format between the
converter plugins (the reference's ConverterPlugin boundary,
pkg/src/modelci/converter/plugins.py:32-68) and the executor (the reference's
MockServer, pkg/src/modelci/mockserve/server.py:94-127).  The byte layout is
mirrored in C++ by paper_2006_05096_b200/csrc/runtime.cu (b2_plan_create) and in numpy by
oracle/plan_ref.py.

Layout (little endian):

    header  "B2PL" u32 version u32 dtype(0 fp32, 1 bf16) u32 n_tensors
            u32 n_weights u32 n_ops u32 input_kind(0 dense f32, 1 token ids i64)
            u32 in_elems u32 out_elems u32 meta_len u32 reserved[2]      (48 B)
    tensors n_tensors x {u32 kind(0 activation, 1 int32 ids) u32 elems
                         i32 shape[4]}                                   (24 B)
    weights n_weights x {u64 offset u64 numel i32 shape[4]}               (32 B)
    ops     n_ops x {u32 kind, i32 p[31]}                                (128 B)
    meta    meta_len bytes of UTF-8 JSON (model name, flops/sample, ...)
    pad     to a 64 B boundary
    data    fp32 weights, each starting on a 64 B boundary
    crc     u32 zlib.crc32 of everything before it

Activations are stored channels-last (NHWC for images, [seq, hidden] for
sequences); ``elems`` is the per-sample element count.  Weights use the
layouts documented per op below.  Activation codes: 0 none, 1 relu, 2 relu6,
3 gelu (erf), 4 tanh.
"""

from __future__ import annotations

import json
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from .errors import PlanFormatError

MAGIC = b"B2PL"
VERSION = 1
DT_FP32, DT_BF16 = 0, 1
IN_DENSE, IN_TOKENS = 0, 1
T_ACT, T_IDS = 0, 1
ACT_NONE, ACT_RELU, ACT_RELU6, ACT_GELU, ACT_TANH = 0, 1, 2, 3, 4
NPARAM = 31

_HDR = struct.Struct("<4sIIIIIIIIIII")
_TEN = struct.Struct("<II4i")
_WGT = struct.Struct("<QQ4i")
_OP = struct.Struct("<I31i")

# -- op kinds and their parameter slots (p[i]) --------------------------------
# INPUT: fp32 sample laid out (C,H,W) -> NHWC activation with C zero-padded.
OP_INPUT = 1
P_IN_OUT, P_IN_C, P_IN_H, P_IN_W, P_IN_CPAD = range(5)
# TOKENS: int64 ids [seq] -> int32 ids tensor.  With has_mask the sample is
# [ids(seq), attention_mask(seq)] (int64, 1 = attend, 0 = padding) and the
# mask is packed into a key-validity bit tensor: (seq + 31) // 32 int32 words
# per sample, bit j % 32 of word j // 32 = key j valid.
OP_TOKENS = 2
P_TK_OUT, P_TK_SEQ, P_TK_VOCAB, P_TK_HASMASK, P_TK_MASK = range(5)
# CONV: out = act(conv(in, w) + bias + res); w [Cout, R, S, Cin] (OHWI)
OP_CONV = 3
(P_CV_IN, P_CV_OUT, P_CV_W, P_CV_B, P_CV_H, P_CV_W_, P_CV_CIN, P_CV_COUT, P_CV_R, P_CV_S,
 P_CV_STRIDE, P_CV_PAD, P_CV_OH, P_CV_OW, P_CV_ACT, P_CV_RES) = range(16)
# LINEAR: out[M,N] = act(A[M,K] W[N,K]^T + bias + res); M = batch*rows;
# A row r lives at in + r*a_stride (a_stride = K unless strided, e.g. pooler)
OP_LINEAR = 4
(P_LN_IN, P_LN_OUT, P_LN_W, P_LN_B, P_LN_K, P_LN_N, P_LN_ROWS, P_LN_ACT, P_LN_RES,
 P_LN_ASTRIDE) = range(10)
# DWCONV: depthwise RxR, w [C, R, R]
OP_DWCONV = 5
(P_DW_IN, P_DW_OUT, P_DW_W, P_DW_B, P_DW_H, P_DW_W_, P_DW_C, P_DW_STRIDE, P_DW_PAD,
 P_DW_OH, P_DW_OW, P_DW_ACT, P_DW_R) = range(13)
# MAXPOOL k x k
OP_MAXPOOL = 6
(P_MP_IN, P_MP_OUT, P_MP_H, P_MP_W, P_MP_C, P_MP_K, P_MP_STRIDE, P_MP_PAD, P_MP_OH,
 P_MP_OW) = range(10)
# AVGPOOL (global): [H,W,C] -> [C]
OP_AVGPOOL = 7
P_AP_IN, P_AP_OUT, P_AP_H, P_AP_W, P_AP_C = range(5)
# LAYERNORM over the last dim D of rows: out = LN(in + res) * gamma + beta
OP_LAYERNORM = 8
(P_LNM_IN, P_LNM_OUT, P_LNM_G, P_LNM_B, P_LNM_D, P_LNM_ROWS, P_LNM_EPS,
 P_LNM_RES) = range(8)
# EMBED: word[ids] + pos[0:seq] + type[0] then LayerNorm
OP_EMBED = 9
(P_EM_IDS, P_EM_OUT, P_EM_WORD, P_EM_POS, P_EM_TYPE, P_EM_G, P_EM_B, P_EM_D, P_EM_SEQ,
 P_EM_VOCAB, P_EM_EPS) = range(11)
# ATTENTION: qkv [seq, 3*H*Dh] (Q|K|V, head-major) -> out [seq, H*Dh];
# softmax(QK^T / sqrt(Dh) + bias) V with bias = 0 for valid keys and
# float32 min for padded keys (transformers' extended attention mask) when
# has_mask (the mask tensor is TOKENS' packed key bits)
OP_ATTENTION = 10
P_AT_QKV, P_AT_OUT, P_AT_HEADS, P_AT_DH, P_AT_SEQ, P_AT_HASMASK, P_AT_MASK = range(7)
# OUTPUT: concat per sample into the fp32 output: p0 = n, then (tensor, offset)
OP_OUTPUT = 11
# ACT: standalone activation over elems per sample
OP_ACT = 12
P_AC_IN, P_AC_OUT, P_AC_ELEMS, P_AC_ACT = range(4)

OP_NAMES = {OP_INPUT: "input", OP_TOKENS: "tokens", OP_CONV: "conv", OP_LINEAR: "linear",
            OP_DWCONV: "dwconv", OP_MAXPOOL: "maxpool", OP_AVGPOOL: "avgpool",
            OP_LAYERNORM: "layernorm", OP_EMBED: "embed", OP_ATTENTION: "attention",
            OP_OUTPUT: "output", OP_ACT: "act"}


def f32_bits(x: float) -> int:
    return struct.unpack("<i", struct.pack("<f", float(x)))[0]


def bits_f32(b: int) -> float:
    return struct.unpack("<f", struct.pack("<i", int(b)))[0]


@dataclass
class TensorDef:
    kind: int
    shape: tuple

    @property
    def elems(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n


@dataclass
class Op:
    kind: int
    p: list

    def __getitem__(self, i):
        return self.p[i]

    @property
    def name(self) -> str:
        return OP_NAMES.get(self.kind, f"op{self.kind}")


@dataclass
class Plan:
    dtype: int
    input_kind: int
    in_elems: int
    out_elems: int
    tensors: list = field(default_factory=list)
    weights: list = field(default_factory=list)   # numpy fp32 arrays
    ops: list = field(default_factory=list)
    meta: dict = field(default_factory=dict)


class PlanBuilder:
    """Emitters append tensors/weights/ops; ``build()`` serialises."""

    def __init__(self, name: str):
        self.tensors: list[TensorDef] = []
        self.weights: list[np.ndarray] = []
        self.ops: list[Op] = []
        self.meta = {"model": name}
        self.input_kind = IN_DENSE
        self.in_elems = 0
        self.out_elems = 0

    def tensor(self, *shape, kind=T_ACT) -> int:
        self.tensors.append(TensorDef(kind, tuple(int(s) for s in shape)))
        return len(self.tensors) - 1

    def weight(self, arr) -> int:
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.float32))
        self.weights.append(a)
        return len(self.weights) - 1

    def op(self, kind: int, **slots) -> Op:
        p = [0] * NPARAM
        for k, v in slots.items():
            p[int(k[1:])] = int(v)
        o = Op(kind, p)
        self.ops.append(o)
        return o

    def op_p(self, kind: int, params) -> Op:
        p = [0] * NPARAM
        for i, v in enumerate(params):
            p[i] = int(v)
        o = Op(kind, p)
        self.ops.append(o)
        return o

    def shape(self, t: int) -> tuple:
        return self.tensors[t].shape

    def build(self, dtype: int = DT_BF16) -> bytes:
        return encode(Plan(dtype=dtype, input_kind=self.input_kind, in_elems=self.in_elems,
                           out_elems=self.out_elems, tensors=self.tensors,
                           weights=self.weights, ops=self.ops, meta=self.meta))


def _align(n: int, a: int = 64) -> int:
    return (n + a - 1) // a * a


def encode(plan: Plan) -> bytes:
    meta = json.dumps(plan.meta, sort_keys=True, separators=(",", ":")).encode()
    out = bytearray(_HDR.pack(MAGIC, VERSION, plan.dtype, len(plan.tensors), len(plan.weights),
                              len(plan.ops), plan.input_kind, plan.in_elems, plan.out_elems,
                              len(meta), 0, 0))
    for t in plan.tensors:
        shp = list(t.shape) + [0] * (4 - len(t.shape))
        out += _TEN.pack(t.kind, t.elems, *shp)
    offset = 0
    for w in plan.weights:
        shp = list(w.shape) + [0] * (4 - w.ndim)
        if w.ndim > 4:
            raise PlanFormatError("weights have at most 4 dims")
        out += _WGT.pack(offset, w.size, *shp)
        offset = _align(offset + 4 * w.size)
    for o in plan.ops:
        out += _OP.pack(o.kind, *o.p)
    out += meta
    out += b"\0" * (_align(len(out)) - len(out))
    data = bytearray(offset)
    off = 0
    for w in plan.weights:
        raw = w.astype("<f4", copy=False).tobytes()
        data[off:off + len(raw)] = raw
        off = _align(off + len(raw))
    out += data
    return bytes(out) + struct.pack("<I", zlib.crc32(out))


def decode(blob: bytes, verify_crc: bool = True) -> Plan:
    """Parse a plan.  ``verify_crc=False`` skips the whole-blob CRC for callers
    that hand the bytes to ``b2_plan_create`` next (it verifies them again)."""
    if len(blob) < _HDR.size + 4:
        raise PlanFormatError("truncated plan")
    (magic, version, dtype, nt, nw, no, in_kind, in_elems, out_elems, meta_len, _r0,
     _r1) = _HDR.unpack_from(blob, 0)
    if magic != MAGIC:
        raise PlanFormatError("bad magic, not a b200-plan")
    if version != VERSION:
        raise PlanFormatError(f"unsupported plan version {version}")
    if verify_crc and zlib.crc32(memoryview(blob)[:-4]) != struct.unpack("<I", blob[-4:])[0]:
        raise PlanFormatError("CRC mismatch, plan corrupted")
    pos = _HDR.size
    need = pos + nt * _TEN.size + nw * _WGT.size + no * _OP.size + meta_len
    if need > len(blob) - 4:
        raise PlanFormatError("truncated plan tables")
    tensors = []
    for _ in range(nt):
        kind, elems, *shp = _TEN.unpack_from(blob, pos)
        pos += _TEN.size
        shape = tuple(s for s in shp if s > 0)
        td = TensorDef(kind, shape)
        if td.elems != elems:
            raise PlanFormatError("tensor element count mismatch")
        tensors.append(td)
    wdesc = []
    for _ in range(nw):
        off, numel, *shp = _WGT.unpack_from(blob, pos)
        pos += _WGT.size
        wdesc.append((off, numel, tuple(s for s in shp if s > 0)))
    ops = []
    for _ in range(no):
        kind, *p = _OP.unpack_from(blob, pos)
        pos += _OP.size
        ops.append(Op(kind, list(p)))
    for o in ops:
        if o.kind == OP_OUTPUT:
            for j in range(o.p[0]):
                t, off = o.p[1 + 2 * j], o.p[2 + 2 * j]
                if not (0 <= t < nt) or off < 0 or off + tensors[t].elems > out_elems:
                    raise PlanFormatError("OUTPUT op writes outside the output row")
    meta = json.loads(blob[pos:pos + meta_len].decode()) if meta_len else {}
    pos = _align(pos + meta_len)
    weights = []
    for off, numel, shape in wdesc:
        start = pos + off
        if start + 4 * numel > len(blob) - 4:
            raise PlanFormatError("weight data out of range")
        arr = np.frombuffer(blob, dtype="<f4", count=numel, offset=start)
        weights.append(arr.reshape(shape) if shape else arr)
    return Plan(dtype=dtype, input_kind=in_kind, in_elems=in_elems, out_elems=out_elems,
                tensors=tensors, weights=weights, ops=ops, meta=meta)


def with_dtype(blob: bytes, dtype: int) -> bytes:
    """Same plan, different execution dtype (header field + CRC rewritten)."""
    body = bytearray(blob[:-4])
    struct.pack_into("<I", body, 8, dtype)
    return bytes(body) + struct.pack("<I", zlib.crc32(body))


def flops_per_sample(plan: Plan) -> int:
    """Algorithmic multiply-add FLOPs (2 per MAC) of the contraction ops."""
    total = 0
    true_c = {o[P_IN_OUT]: o[P_IN_C] for o in plan.ops if o.kind == OP_INPUT}
    for o in plan.ops:
        if o.kind == OP_CONV:
            cin = min(o[P_CV_CIN], true_c.get(o[P_CV_IN], o[P_CV_CIN]))   # stem: 3 of 8
            total += 2 * o[P_CV_OH] * o[P_CV_OW] * o[P_CV_COUT] * o[P_CV_R] * o[P_CV_S] * cin
        elif o.kind == OP_LINEAR:
            total += 2 * o[P_LN_ROWS] * o[P_LN_N] * o[P_LN_K]
        elif o.kind == OP_DWCONV:
            total += 2 * o[P_DW_OH] * o[P_DW_OW] * o[P_DW_C] * o[P_DW_R] * o[P_DW_R]
        elif o.kind == OP_ATTENTION:
            s, h, d = o[P_AT_SEQ], o[P_AT_HEADS], o[P_AT_DH]
            total += 2 * 2 * h * s * s * d
    return total
