"""CPU oracle for the executor's forward: numpy restatement of every b200-plan op.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never by the product path
(paper_2006_05096_b200/ must fail loudly without libb2.so instead of falling
back here).

What it restates.  The reference executor, MockServer.predict
(pkg/src/modelci/mockserve/server.py:117-127), returns zeros after a sleep and
computes nothing, so there is no reference forward to follow line by line.
The forward semantics are the ones the converter defines (zoo.py docstring,
plan.py op table), and this oracle follows them op by op in
float64 (or float32).  It is pinned two ways (tests/test_oracle.py):

* toy graphs (C1): against oracle/toyref.c, an independent C fp64 restatement
  of the toy op semantics over the reference's toy-binary layout
  (toyformat.py:117-149), and against tests/golden/mlp_golden.json;
* torchvision ResNet-50 / MobileNetV2 / VGG-16 and transformers BertModel
  (third-party modules absent from /root/reference; versions torchvision
  0.26.0, transformers 5.5.0 as installed in this image): against the modules'
  own fp64 CPU forward at small batch (tests/test_oracle.py, CPU only).

Weights are the plan's fp32 values (BN already folded by the converter).
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_05096_b200 import plan as P  # noqa: E402

try:
    from scipy.special import erf as _erf
except ImportError:  # pragma: no cover
    _erf = np.vectorize(math.erf)


def _act(x, code):
    if code == P.ACT_NONE:
        return x
    if code == P.ACT_RELU:
        return np.maximum(x, 0)
    if code == P.ACT_RELU6:
        return np.clip(x, 0, 6)
    if code == P.ACT_GELU:
        return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))
    if code == P.ACT_TANH:
        return np.tanh(x)
    raise ValueError(f"unknown activation {code}")


def _pad_hw(x, pad, value=0.0):
    if pad == 0:
        return x
    return np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)), constant_values=value)


def conv2d_nhwc(x, w, bias, stride, pad):
    """x [B,H,W,C], w [Cout,R,S,C] -> [B,OH,OW,Cout] via im2col + GEMM."""
    B, H, W, C = x.shape
    cout, R, S, _ = w.shape
    xp = _pad_hw(x, pad)
    OH = (H + 2 * pad - R) // stride + 1
    OW = (W + 2 * pad - S) // stride + 1
    sb, sh, sw, sc = xp.strides
    cols = np.lib.stride_tricks.as_strided(
        xp, shape=(B, OH, OW, R, S, C), strides=(sb, sh * stride, sw * stride, sh, sw, sc))
    out = cols.reshape(B * OH * OW, R * S * C) @ w.reshape(cout, R * S * C).T
    if bias is not None:
        out = out + bias
    return out.reshape(B, OH, OW, cout)


def dwconv_nhwc(x, w, bias, stride, pad):
    B, H, W, C = x.shape
    R = w.shape[1]
    xp = _pad_hw(x, pad)
    OH = (H + 2 * pad - R) // stride + 1
    OW = (W + 2 * pad - R) // stride + 1
    out = np.zeros((B, OH, OW, C), dtype=x.dtype)
    for r in range(R):
        for s in range(R):
            out += xp[:, r:r + stride * OH:stride, s:s + stride * OW:stride, :] * w[:, r, s]
    if bias is not None:
        out += bias
    return out


def maxpool_nhwc(x, k, stride, pad):
    B, H, W, C = x.shape
    xp = _pad_hw(x, pad, -np.inf)
    OH = (H + 2 * pad - k) // stride + 1
    OW = (W + 2 * pad - k) // stride + 1
    out = np.full((B, OH, OW, C), -np.inf, dtype=x.dtype)
    for r in range(k):
        for s in range(k):
            np.maximum(out, xp[:, r:r + stride * OH:stride, s:s + stride * OW:stride, :], out=out)
    return out


def layernorm(x, g, b, eps):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def attention(qkv, heads, dh, keymask=None):
    """qkv [B,S,3*H*Dh] -> [B,S,H*Dh]; softmax(QK^T/sqrt(Dh) + bias) V with
    bias = float32-min on padded keys (``keymask`` [B,S] bool, True = attend;
    transformers' extended attention mask: modeling_bert's
    get_extended_attention_mask, (1 - mask) * finfo.min), 0 elsewhere."""
    B, S, _ = qkv.shape
    q, k, v = np.split(qkv.reshape(B, S, 3, heads, dh), 3, axis=2)
    q, k, v = (t[:, :, 0].transpose(0, 2, 1, 3) for t in (q, k, v))   # [B,H,S,Dh]
    sc = q @ k.transpose(0, 1, 3, 2) / math.sqrt(dh)
    if keymask is not None:
        bias = np.where(np.asarray(keymask, bool), 0.0, float(np.finfo(np.float32).min))
        sc = sc + bias[:, None, None, :]
    sc = sc - sc.max(-1, keepdims=True)
    p = np.exp(sc)
    p /= p.sum(-1, keepdims=True)
    return (p @ v).transpose(0, 2, 1, 3).reshape(B, S, heads * dh)


def pack_keymask(valid):
    """[B,S] bool -> [B,(S+31)//32] int32 words, bit j%32 of word j//32 = key
    j valid (the TOKENS op's mask tensor, kernels.cu tokens_kernel)."""
    valid = np.asarray(valid, bool)
    B, S = valid.shape
    nw = (S + 31) // 32
    bits = np.zeros((B, nw * 32), bool)
    bits[:, :S] = valid
    w = (bits.reshape(B, nw, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(-1)
    return w.astype(np.uint32).view(np.int32).astype(np.int64)


def unpack_keymask(words, S):
    w = np.asarray(words, dtype=np.int64).reshape(len(words), -1).astype(np.uint32)
    bits = (w[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(len(w), -1)[:, :S].astype(bool)


def round_bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32 (the kernels'
    __float2bfloat16_rn)."""
    a = np.array(x, dtype=np.float32, copy=True)
    u = a.view(np.uint32)
    u += np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    u &= np.uint32(0xFFFF0000)
    return a


def bf16_weight_ids(plan) -> set:
    """Weights the bf16 executor stores as bf16 (contraction weights and
    embedding tables); biases and LayerNorm affine stay fp32."""
    ids = set()
    for o in plan.ops:
        if o.kind in (P.OP_CONV, P.OP_LINEAR, P.OP_DWCONV):
            ids.add(o[2])
        elif o.kind == P.OP_EMBED:
            ids |= {o[P.P_EM_WORD], o[P.P_EM_POS], o[P.P_EM_TYPE]}
    return ids


class _Bf16Store(dict):
    """Activation store that rounds every floating tensor to bf16 on write —
    the rounding points of the bf16 executor (each op reads bf16, computes in
    fp32, writes bf16)."""

    def __setitem__(self, k, v):
        if v.dtype.kind == "f":
            v = round_bf16(v).astype(np.float64)
        super().__setitem__(k, v)


def run_op(plan, o, T, W, B, x, out, dtype=np.float64):
    """Execute one plan op on the host tensors ``T`` (dict tensor -> array)."""
    def shaped(t):
        return T[t].reshape((B,) + plan.tensors[t].shape)

    def wt(i):
        return None if i < 0 else W[i]

    k = o.kind
    if k == P.OP_INPUT:
        C, H, Wd, Cp = o[P.P_IN_C], o[P.P_IN_H], o[P.P_IN_W], o[P.P_IN_CPAD]
        img = np.asarray(x, dtype=dtype).reshape(B, C, H, Wd).transpose(0, 2, 3, 1)
        buf = np.zeros((B, H, Wd, Cp), dtype=dtype)
        buf[..., :C] = img
        T[o[P.P_IN_OUT]] = buf
    elif k == P.OP_TOKENS:
        S = o[P.P_TK_SEQ]
        xi = np.asarray(x, dtype=np.int64).reshape(B, -1)
        T[o[P.P_TK_OUT]] = xi[:, :S]
        if o[P.P_TK_HASMASK]:
            T[o[P.P_TK_MASK]] = pack_keymask(xi[:, S:2 * S] != 0)
    elif k == P.OP_CONV:
        y = conv2d_nhwc(shaped(o[P.P_CV_IN]), W[o[P.P_CV_W]], wt(o[P.P_CV_B]),
                        o[P.P_CV_STRIDE], o[P.P_CV_PAD])
        if o[P.P_CV_RES] >= 0:
            y = y + shaped(o[P.P_CV_RES])
        T[o[P.P_CV_OUT]] = _act(y, o[P.P_CV_ACT])
    elif k == P.OP_LINEAR:
        K, N, rows, astride = o[P.P_LN_K], o[P.P_LN_N], o[P.P_LN_ROWS], o[P.P_LN_ASTRIDE]
        flat = T[o[P.P_LN_IN]].reshape(B, -1)
        idx = np.arange(rows)[:, None] * astride + np.arange(K)[None, :]
        a = flat[:, idx]                                     # [B, rows, K]
        y = a @ W[o[P.P_LN_W]].T
        if o[P.P_LN_B] >= 0:
            y = y + W[o[P.P_LN_B]]
        if o[P.P_LN_RES] >= 0:
            y = y + T[o[P.P_LN_RES]].reshape(B, rows, N)
        T[o[P.P_LN_OUT]] = _act(y, o[P.P_LN_ACT])
    elif k == P.OP_DWCONV:
        y = dwconv_nhwc(shaped(o[P.P_DW_IN]), W[o[P.P_DW_W]], wt(o[P.P_DW_B]),
                        o[P.P_DW_STRIDE], o[P.P_DW_PAD])
        T[o[P.P_DW_OUT]] = _act(y, o[P.P_DW_ACT])
    elif k == P.OP_MAXPOOL:
        T[o[P.P_MP_OUT]] = maxpool_nhwc(shaped(o[P.P_MP_IN]), o[P.P_MP_K],
                                        o[P.P_MP_STRIDE], o[P.P_MP_PAD])
    elif k == P.OP_AVGPOOL:
        T[o[P.P_AP_OUT]] = shaped(o[P.P_AP_IN]).mean(axis=(1, 2))
    elif k == P.OP_LAYERNORM:
        D, rows = o[P.P_LNM_D], o[P.P_LNM_ROWS]
        v = T[o[P.P_LNM_IN]].reshape(B, rows, D)
        if o[P.P_LNM_RES] >= 0:
            v = v + T[o[P.P_LNM_RES]].reshape(B, rows, D)
        T[o[P.P_LNM_OUT]] = layernorm(v, W[o[P.P_LNM_G]], W[o[P.P_LNM_B]],
                                      P.bits_f32(o[P.P_LNM_EPS]))
    elif k == P.OP_EMBED:
        ids = T[o[P.P_EM_IDS]]
        e = W[o[P.P_EM_WORD]][ids] + W[o[P.P_EM_POS]][None, :ids.shape[1]] + \
            W[o[P.P_EM_TYPE]][None, None, :]
        T[o[P.P_EM_OUT]] = layernorm(e, W[o[P.P_EM_G]], W[o[P.P_EM_B]],
                                     P.bits_f32(o[P.P_EM_EPS]))
    elif k == P.OP_ATTENTION:
        S, H, Dh = o[P.P_AT_SEQ], o[P.P_AT_HEADS], o[P.P_AT_DH]
        km = unpack_keymask(T[o[P.P_AT_MASK]], S) if o[P.P_AT_HASMASK] else None
        T[o[P.P_AT_OUT]] = attention(T[o[P.P_AT_QKV]].reshape(B, S, 3 * H * Dh), H, Dh, km)
    elif k == P.OP_ACT:
        T[o[P.P_AC_OUT]] = _act(T[o[P.P_AC_IN]], o[P.P_AC_ACT])
    elif k == P.OP_OUTPUT:
        for j in range(o[0]):
            t, off = o[1 + 2 * j], o[2 + 2 * j]
            v = T[t].reshape(B, -1)
            out[:, off:off + v.shape[1]] = v
    else:
        raise ValueError(f"oracle: unknown op kind {k}")


def forward(plan, x, dtype=np.float64, emulate_bf16: bool = False):
    """Run a decoded plan (plan.decode) on a host batch.

    ``x``: dense inputs [B, in_elems] (float) or token ids [B, seq] (int).
    Returns the fp output [B, out_elems] in ``dtype``.  ``emulate_bf16``
    reproduces the bf16 executor's rounding points (bf16 weights and
    activations, fp32 biases/affines, wide accumulation) so bf16 kernels can be
    checked against their own arithmetic rather than against fp32.
    """
    if isinstance(plan, (bytes, bytearray)):
        plan = P.decode(plan)
    if emulate_bf16:
        dtype = np.float64
        keep = bf16_weight_ids(plan)
        W = [round_bf16(w).astype(dtype) if i in keep else w.astype(dtype)
             for i, w in enumerate(plan.weights)]
    else:
        W = [w.astype(dtype) for w in plan.weights]
    B = x.shape[0]
    T: dict[int, np.ndarray] = _Bf16Store() if emulate_bf16 else {}

    out = np.zeros((B, plan.out_elems), dtype=dtype)
    for o in plan.ops:
        run_op(plan, o, T, W, B, x, out, dtype)
        for key, val in list(T.items()):   # keep the working precision
            if val.dtype.kind == "f" and val.dtype != dtype:
                T[key] = val.astype(dtype)
    return out


def make_inputs(plan, batch: int, seed: int = 0):
    """Host-side seeded inputs for parity runs: N(0,1) fp32 images/vectors, or
    uniform token ids in [0, vocab)."""
    if isinstance(plan, (bytes, bytearray)):
        plan = P.decode(plan)
    rng = np.random.default_rng(seed)
    if plan.input_kind == P.IN_TOKENS:
        tk = next(o for o in plan.ops if o.kind == P.OP_TOKENS)
        S = tk[P.P_TK_SEQ]
        ids = rng.integers(0, tk[P.P_TK_VOCAB], size=(batch, S), dtype=np.int64)
        if tk[P.P_TK_HASMASK]:   # attention_mask = 1 (the profiling payload)
            return np.concatenate([ids, np.ones((batch, S), np.int64)], 1)
        return ids
    return rng.standard_normal((batch, plan.in_elems), dtype=np.float32)


def normwise_err(got, ref) -> float:
    """max|got-ref| / max|ref| — the tolerance metric of SURVEY.md §8c."""
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref)) /
                 max(np.max(np.abs(ref)), 1e-30))


def op_io(o):
    """(input tensor ids, output tensor id) of an op (OUTPUT: no output)."""
    k = o.kind
    if k in (P.OP_INPUT, P.OP_TOKENS):
        return [], o[0]
    if k == P.OP_ATTENTION and o[P.P_AT_HASMASK]:
        return [o[P.P_AT_QKV], o[P.P_AT_MASK]], o[P.P_AT_OUT]
    if k == P.OP_CONV:
        return [o[P.P_CV_IN]] + ([o[P.P_CV_RES]] if o[P.P_CV_RES] >= 0 else []), o[P.P_CV_OUT]
    if k == P.OP_LINEAR:
        return [o[P.P_LN_IN]] + ([o[P.P_LN_RES]] if o[P.P_LN_RES] >= 0 else []), o[P.P_LN_OUT]
    if k == P.OP_LAYERNORM:
        return [o[P.P_LNM_IN]] + ([o[P.P_LNM_RES]] if o[P.P_LNM_RES] >= 0 else []), o[1]
    if k == P.OP_OUTPUT:
        return [o[1 + 2 * j] for j in range(o[0])], None
    return [o[0]], o[1]


# Layerwise teacher-forced bound for bf16 kernels (tests): one round-to-nearest
# of the op output is <= u = 2^-8 = 3.91e-3 normwise; +15% for fp32
# accumulation order and near-tie elements.  An fp32 kernel: 1e-5.
BF16_LAYERWISE_TOL = 4.5e-3


def layerwise_errors(plan, read_tensor, x, emulate_bf16: bool, roundings=None):
    """Teacher-forced per-op parity.

    Every op is recomputed on the host from the executor's OWN input tensors
    (``read_tensor(t) -> float64/int array`` after a device forward on ``x``)
    and compared with the executor's output tensor.  Unlike an end-to-end
    comparison this does not amplify rounding through a deep network, so the
    bound is one rounding of the op's own output.  Returns [(op_index, name,
    normwise_err)].

    The reference value of each op is its EXACT (float64) result on the
    executor's bf16 inputs and bf16 weights, not rounded to bf16: a correct
    bf16 kernel then differs from it by one round-to-nearest of its output
    (bf16 keeps 8 significant bits: <= 2^-8 of the element's binade, so
    <= u = 2^-8 = 3.91e-3 normwise) plus its fp32 accumulation error.
    Tensors the executor never materialises are teacher-forced from the
    oracle: rounded to bf16 where the kernel holds them as bf16 on chip (the
    stem's output before the fused max-pool), exact where the kernel folds
    them into an fp32 accumulator (a projection shortcut consumed only as
    the residual of the block's last conv: its K blocks are appended to that
    conv's GEMM, so it is never rounded).

    ``roundings`` (a dict, optional) receives, per op index, how many bf16
    roundings separate the exact value from the kernel's output: 1 for most
    ops; 2 for attention (P = softmax(QK^T) is rounded to bf16 before PV) and
    for ops fed by a tensor the kernel rounds on chip (kernel and oracle round
    the same fp32/exact value and can land one ulp apart at near-ties).  A
    test's bound is BF16_LAYERWISE_TOL x roundings.  Per-sample ops only, so ``x`` and ``read_tensor`` may
    be restricted to a subset of the batch rows (the full-size parity tests
    check rows 0, B/2-1 and B-1 of a batch-256 forward).
    """
    if isinstance(plan, (bytes, bytearray)):
        plan = P.decode(plan)
    B = x.shape[0]
    if emulate_bf16:
        keep = bf16_weight_ids(plan)
        W = [round_bf16(w).astype(np.float64) if i in keep else w.astype(np.float64)
             for i, w in enumerate(plan.weights)]
    else:
        W = [w.astype(np.float64) for w in plan.weights]
    out = np.zeros((B, plan.out_elems))
    res = []
    oracle_t = {}   # oracle values of tensors the executor fused away (never materialised)
    consumers: dict = {}
    for o in plan.ops:
        if o.kind == P.OP_CONV:
            consumers.setdefault(o[P.P_CV_IN], []).append("in")
            if o[P.P_CV_RES] >= 0:
                consumers.setdefault(o[P.P_CV_RES], []).append("res")
        elif o.kind == P.OP_LINEAR:
            consumers.setdefault(o[P.P_LN_IN], []).append("in")
            if o[P.P_LN_RES] >= 0:
                consumers.setdefault(o[P.P_LN_RES], []).append("res")
        else:
            for t in op_io(o)[0]:
                consumers.setdefault(t, []).append("in")
    for i, o in enumerate(plan.ops):
        ins, dst = op_io(o)
        if dst is None:
            continue
        T = {}     # exact: the op's output is compared before any bf16 rounding
        for t in ins:
            v = read_tensor(t)
            if v is None:          # fused intermediate: teacher-force from the oracle chain
                v = oracle_t[t]
            if plan.tensors[t].kind == P.T_IDS:
                dict.__setitem__(T, t, np.asarray(v, dtype=np.int64).reshape(B, -1))
            else:
                dict.__setitem__(T, t, np.asarray(v, dtype=np.float64))
        if roundings is not None:
            fed = any(t in oracle_t and emulate_bf16 and not
                      (consumers.get(t) and all(c == "res" for c in consumers[t])) for t in ins)
            roundings[i] = 2 if (o.kind == P.OP_ATTENTION or fed) else 1
        run_op(plan, o, T, W, B, x, out, np.float64)
        ref = np.asarray(T[dst], dtype=np.float64).reshape(B, -1)
        got = read_tensor(dst)
        if got is None:
            folded = consumers.get(dst) and all(c == "res" for c in consumers[dst])
            oracle_t[dst] = round_bf16(ref).astype(np.float64) \
                if emulate_bf16 and not folded else ref
            continue
        got = np.asarray(got, dtype=np.float64).reshape(B, -1)
        res.append((i, o.name, normwise_err(got, ref)))
    return res


def layerwise_check(plan, read_tensor, x, emulate_bf16: bool):
    """layerwise_errors with each op's bound: [(op, name, err, bound)] and the
    ops over it.  bf16: BF16_LAYERWISE_TOL x the op's bf16 roundings; fp32:
    1e-5."""
    rnd: dict = {}
    res = layerwise_errors(plan, read_tensor, x, emulate_bf16, roundings=rnd)
    out = [(i, n, e, (BF16_LAYERWISE_TOL * rnd.get(i, 1)) if emulate_bf16 else 1e-5)
           for i, n, e in res]
    return out, [r for r in out if not r[2] <= r[3]]
