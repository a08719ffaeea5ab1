"""Per-shape conv parity on the GPU: single-conv plans through every tcgen05
conv path (banded implicit GEMM with resident or streamed weights and 1..4 M
tiles per band, the TMA-im2col GEMM, the space-to-depth stem) checked
layerwise against the numpy oracle (plan_ref.conv2d_nhwc on the bf16-rounded
operands, fp64 accumulation).  Tolerance: plan_ref.BF16_LAYERWISE_TOL
(4.5e-3 normwise = one bf16 rounding of the op output, u = 2^-8, + 15%; the
same bound as tests/test_gpu.py's layerwise gate).

Batch sizes are chosen so both the small-batch (one M tile per band) and the
large-batch (multi-tile bands) configurations run for each shape.
"""
import numpy as np
import pytest

import plan_ref
from paper_2006_05096_b200 import plan as P
from paper_2006_05096_b200 import runtime as R

pytestmark = pytest.mark.gpu

TOL = plan_ref.BF16_LAYERWISE_TOL


@pytest.fixture(autouse=True)
def developer_knobs(monkeypatch):
    """These tests pin kernel variants through the B2_* selection knobs,
    which libb2 honours only with B2_DEV=1."""
    monkeypatch.setenv("B2_DEV", "1")


def conv_plan(H, W, C, N, k, stride, act=1, seed=0):
    pad = k // 2
    OH = (H + 2 * pad - k) // stride + 1
    OW = (W + 2 * pad - k) // stride + 1
    b = P.PlanBuilder("conv")
    Cp = max(8, C)
    x = b.tensor(H, W, Cp)
    b.in_elems = C * H * W
    b.op_p(P.OP_INPUT, [x, C, H, W, Cp])
    rng = np.random.default_rng(seed)
    y = b.tensor(OH, OW, N)
    w = rng.standard_normal((N, k, k, Cp)) * (1.0 / np.sqrt(k * k * C))
    w[..., C:] = 0.0
    bias = rng.standard_normal(N) * 0.1
    b.op_p(P.OP_CONV, [x, y, b.weight(w), b.weight(bias), H, W, Cp, N, k, k, stride, pad,
                       OH, OW, act, -1])
    b.out_elems = b.tensors[y].elems
    b.op_p(P.OP_OUTPUT, [1, y, 0])
    return b.build(P.DT_FP32)


def check(blob, batch, seed=3):
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, batch, seed)
    plan = R.Plan(blob, P.DT_BF16)
    try:
        out = plan.predict(x)
        assert np.isfinite(out).all()
        rt = lambda t: plan.read_tensor(batch, t, pl.tensors[t].elems, pl.tensors[t].kind)
        errs, bad = plan_ref.layerwise_check(pl, rt, x, True)
        assert not bad, bad
    finally:
        plan.close()


@pytest.mark.parametrize("H,W,C,N,batch", [
    (56, 56, 64, 64, 1),      # layer1 3x3, small batch (1 tile per band)
    (56, 56, 64, 64, 16),     # layer1 3x3, multi-tile bands, resident weights
    (28, 28, 128, 128, 2),
    (28, 28, 128, 128, 24),   # layer2 3x3: two channel groups
    (14, 14, 256, 256, 12),   # layer3 3x3: BN = 256
    (7, 7, 512, 512, 32),     # layer4 3x3: two N tiles, streamed weights
    (112, 112, 64, 128, 2),   # VGG block 2
    (224, 224, 64, 64, 1),    # VGG block 1: a row spans two M tiles
    (20, 36, 64, 192, 5),     # ragged: N = 3 x 64, partial last band
])
def test_conv3x3(gpu_required, monkeypatch, H, W, C, N, batch):
    monkeypatch.setenv("B2_BAND_MAX_N", "4096")   # every shape through the band kernel
    check(conv_plan(H, W, C, N, 3, 1), batch)
    monkeypatch.setenv("B2_BAND", "0")            # and through the im2col GEMM
    check(conv_plan(H, W, C, N, 3, 1), batch)


@pytest.mark.parametrize("batch", [1, 2, 16])
def test_stem_s2d(gpu_required, batch):
    """7x7/2 stem on 3 channels: the space-to-depth band path (16-ch, 32B swizzle)."""
    check(conv_plan(224, 224, 3, 64, 7, 2), batch)


@pytest.mark.parametrize("N,act,batch", [(32, 2, 1), (32, 2, 8), (64, 1, 3), (32, 0, 2)])
def test_stem_s2d_3x3(gpu_required, monkeypatch, N, act, batch):
    """3x3/2 stem (MobileNetV2: 3 -> 32, ReLU6): space-to-depth band path with
    2 x 4 taps and a half-empty 64-wide tile, then the s2d GEMM path."""
    check(conv_plan(224, 224, 3, N, 3, 2, act=act), batch)
    monkeypatch.setenv("B2_BAND", "0")
    check(conv_plan(224, 224, 3, N, 3, 2, act=act), batch)


@pytest.mark.parametrize("k,stride,H,C,N", [(3, 2, 28, 128, 128), (1, 2, 28, 256, 512),
                                             (5, 1, 14, 64, 64)])
def test_other_convs(gpu_required, k, stride, H, C, N):
    """Strided / 5x5 convs: band path for stride 1 k x k, im2col GEMM otherwise."""
    check(conv_plan(H, H, C, N, k, stride), 4)


def stem_pool_plan(seed=0):
    """ResNet stem: 7x7/2 conv (3 -> 64, ReLU) then 3x3/2 max-pool."""
    b = P.PlanBuilder("stem_pool")
    x = b.tensor(224, 224, 8)
    b.in_elems = 3 * 224 * 224
    b.op_p(P.OP_INPUT, [x, 3, 224, 224, 8])
    rng = np.random.default_rng(seed)
    y = b.tensor(112, 112, 64)
    w = rng.standard_normal((64, 7, 7, 8)) * (1.0 / np.sqrt(147))
    w[..., 3:] = 0.0
    b.op_p(P.OP_CONV, [x, y, b.weight(w), b.weight(rng.standard_normal(64) * 0.1), 224, 224, 8,
                       64, 7, 7, 2, 3, 112, 112, 1, -1])
    z = b.tensor(56, 56, 64)
    b.op_p(P.OP_MAXPOOL, [y, z, 112, 112, 64, 3, 2, 1, 56, 56])
    b.out_elems = b.tensors[z].elems
    b.op_p(P.OP_OUTPUT, [1, z, 0])
    return b.build(P.DT_FP32)


@pytest.mark.parametrize("batch", [1, 3, 16])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_stem_maxpool(gpu_required, monkeypatch, batch, fused):
    """Stem + max-pool: fused (stem_pool_kernel; the stem output is never
    materialised, so the pool is checked against the oracle's own stem) and
    unfused.  Batch 3 and 16 put unit ranges across image boundaries and start
    ranges mid-image (the recomputed halo row)."""
    monkeypatch.setenv("B2_POOL_FUSION", fused)
    blob = stem_pool_plan()
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, batch, 5)
    plan = R.Plan(blob, P.DT_BF16)
    try:
        out = plan.predict(x)
        assert np.isfinite(out).all()
        rt = lambda t: plan.read_tensor(batch, t, pl.tensors[t].elems, pl.tensors[t].kind)
        assert (rt(pl.ops[1][1]) is None) == (fused == "1")
        errs, bad = plan_ref.layerwise_check(pl, rt, x, True)
        assert errs and not bad, errs
    finally:
        plan.close()


def linear_plan(K, N, res, seed=0):
    """One LINEAR (+ optional residual from a second LINEAR), ReLU."""
    b = P.PlanBuilder("lin")
    x = b.tensor(K)
    b.in_elems = K
    b.op_p(P.OP_INPUT, [x, K, 1, 1, K])
    rng = np.random.default_rng(seed)
    r = -1
    if res:
        r = b.tensor(N)
        b.op_p(P.OP_LINEAR, [x, r, b.weight(rng.standard_normal((N, K)) / np.sqrt(K)),
                             b.weight(rng.standard_normal(N) * 0.1), K, N, 1, 0, -1, K])
    y = b.tensor(N)
    b.op_p(P.OP_LINEAR, [x, y, b.weight(rng.standard_normal((N, K)) / np.sqrt(K)),
                         b.weight(rng.standard_normal(N) * 0.1), K, N, 1, 1, r, K])
    b.out_elems = b.tensors[y].elems
    b.op_p(P.OP_OUTPUT, [1, y, 0])
    return b.build(P.DT_FP32)


@pytest.mark.parametrize("M,K,N,res", [
    (4173, 256, 1024, True),    # CTA-pair GEMM, residual fold, ragged M (pair tail)
    (8192, 1024, 256, False),
    (6000, 512, 192, False),    # N not a multiple of the tile: BN = 128, ragged N
    (50176, 64, 256, True),
    (5000, 16, 96, False),      # K <= 32: narrow A boxes (16-wide, 32B swizzle)
    (3000, 24, 144, True),      #   24 -> 32-wide box, 8 zero-filled columns, residual fold
    (7000, 32, 16, False),      #   32-wide (64B swizzle), BN = 32 for N = 16
])
@pytest.mark.parametrize("pair", ["1", "0"])
def test_gemm_shapes(gpu_required, monkeypatch, M, K, N, res, pair):
    """Row-parallel GEMMs through the CTA-pair (cta_group::2) kernel and the
    single-CTA kernel; M is the batch of a one-row-per-sample plan."""
    monkeypatch.setenv("B2_PAIR", pair)
    check(linear_plan(K, N, res), M)


@pytest.mark.parametrize("H,C,N,k,stride,batch", [
    (7, 512, 512, 3, 1, 128),    # layer4 3x3 via im2col, CTA pair
    (14, 256, 256, 3, 1, 40),    # layer3 3x3
    (14, 512, 512, 3, 2, 96),    # strided 3x3 (im2col, pair)
    (14, 1024, 2048, 1, 2, 96),  # strided 1x1 downsample
])
def test_late_convs(gpu_required, H, C, N, k, stride, batch):
    check(conv_plan(H, H, C, N, k, stride), batch)


def shortcut_plan(H, C, Cm, N, stride, seed=0):
    """Bottleneck tail with a projection shortcut:
    t = relu(conv3x3/stride(x)); out = relu(conv1x1(t) + conv1x1/stride(x))."""
    b = P.PlanBuilder("shortcut")
    x = b.tensor(H, H, C)
    b.in_elems = C * H * H
    b.op_p(P.OP_INPUT, [x, C, H, H, C])
    rng = np.random.default_rng(seed)
    OH = (H + 2 - 3) // stride + 1
    t = b.tensor(OH, OH, Cm)
    b.op_p(P.OP_CONV, [x, t, b.weight(rng.standard_normal((Cm, 3, 3, C)) / np.sqrt(9 * C)),
                       b.weight(rng.standard_normal(Cm) * 0.1), H, H, C, Cm, 3, 3, stride, 1,
                       OH, OH, 1, -1])
    d = b.tensor(OH, OH, N)
    b.op_p(P.OP_CONV, [x, d, b.weight(rng.standard_normal((N, 1, 1, C)) / np.sqrt(C)),
                       b.weight(rng.standard_normal(N) * 0.1), H, H, C, N, 1, 1, stride, 0,
                       OH, OH, 0, -1])
    y = b.tensor(OH, OH, N)
    b.op_p(P.OP_CONV, [t, y, b.weight(rng.standard_normal((N, 1, 1, Cm)) / np.sqrt(Cm)),
                       b.weight(rng.standard_normal(N) * 0.1), OH, OH, Cm, N, 1, 1, 1, 0,
                       OH, OH, 1, d])
    b.out_elems = b.tensors[y].elems
    b.op_p(P.OP_OUTPUT, [1, y, 0])
    return b.build(P.DT_FP32)


@pytest.mark.parametrize("H,C,Cm,N,stride,batch", [
    (56, 64, 64, 256, 1, 6),      # ResNet layer1 block 0
    (56, 256, 128, 512, 2, 4),    # layer2 block 0 (strided shortcut via im2col TMA)
    (14, 1024, 512, 2048, 2, 8),  # layer4 block 0
    (56, 256, 128, 512, 2, 8),    # M >= 4096: the CTA-pair GEMM with the folded shortcut
    (28, 512, 256, 1024, 2, 24),  # layer3 block 0, pair
    (14, 1024, 512, 2048, 2, 96), # layer4 block 0, pair
])
@pytest.mark.parametrize("fold", ["1", "0"])
def test_shortcut_fold(gpu_required, monkeypatch, H, C, Cm, N, stride, batch, fold):
    """Projection shortcut folded into the block's last 1x1 conv (its output is
    never materialised; read_tensor reports it fused) vs run as its own conv."""
    monkeypatch.setenv("B2_DS_FOLD", fold)
    blob = shortcut_plan(H, C, Cm, N, stride)
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, batch, 9)
    plan = R.Plan(blob, P.DT_BF16)
    try:
        out = plan.predict(x)
        assert np.isfinite(out).all()
        rt = lambda t: plan.read_tensor(batch, t, pl.tensors[t].elems, pl.tensors[t].kind)
        assert (rt(pl.ops[2][1]) is None) == (fold == "1")
        errs, bad = plan_ref.layerwise_check(pl, rt, x, True)
        assert errs and not bad, errs
    finally:
        plan.close()


def chain_plan(H, C, Cm, N1, N2, shortcut, seed=0):
    """Block tail + next block's first conv:
    t = relu(conv1x1(x, C->Cm)); O = relu(conv1x1(t, Cm->N1) + R);
    T1 = relu(conv1x1(O, N1->N2)); R = x (identity, C == N1) or a 1x1
    projection of x (shortcut=1) / strided by 2 (shortcut=2, t from a 3x3/2)."""
    b = P.PlanBuilder("chain")
    x = b.tensor(H, H, C)
    b.in_elems = C * H * H
    b.op_p(P.OP_INPUT, [x, C, H, H, C])
    rng = np.random.default_rng(seed)
    st = 2 if shortcut == 2 else 1
    OH = H // st
    k = 3 if shortcut == 2 else 1
    t = b.tensor(OH, OH, Cm)
    b.op_p(P.OP_CONV, [x, t, b.weight(rng.standard_normal((Cm, k, k, C)) / np.sqrt(k * k * C)),
                       b.weight(rng.standard_normal(Cm) * 0.1), H, H, C, Cm, k, k, st, k // 2,
                       OH, OH, 1, -1])
    if shortcut:
        r = b.tensor(OH, OH, N1)
        b.op_p(P.OP_CONV, [x, r, b.weight(rng.standard_normal((N1, 1, 1, C)) / np.sqrt(C)),
                           b.weight(rng.standard_normal(N1) * 0.1), H, H, C, N1, 1, 1, st, 0,
                           OH, OH, 0, -1])
    else:
        r = x
    o = b.tensor(OH, OH, N1)
    b.op_p(P.OP_CONV, [t, o, b.weight(rng.standard_normal((N1, 1, 1, Cm)) / np.sqrt(Cm)),
                       b.weight(rng.standard_normal(N1) * 0.1), OH, OH, Cm, N1, 1, 1, 1, 0,
                       OH, OH, 1, r])
    t1 = b.tensor(OH, OH, N2)
    b.op_p(P.OP_CONV, [o, t1, b.weight(rng.standard_normal((N2, 1, 1, N1)) / np.sqrt(N1)),
                       b.weight(rng.standard_normal(N2) * 0.1), OH, OH, N1, N2, 1, 1, 1, 0,
                       OH, OH, 1, -1])
    b.out_elems = b.tensors[o].elems + b.tensors[t1].elems
    b.op_p(P.OP_OUTPUT, [2, o, 0, t1, b.tensors[o].elems])
    return b.build(P.DT_FP32)


@pytest.mark.parametrize("H,C,Cm,N1,N2,shortcut,batch", [
    (56, 256, 64, 256, 64, 0, 3),      # layer1 blocks 1-2: identity residual, 2 O chunks
    (56, 64, 64, 256, 64, 1, 2),       # layer1 block 0: projection shortcut (stride 1)
    (28, 512, 128, 512, 128, 0, 5),    # layer2: 4 O chunks, N2 = 128
    (28, 256, 128, 512, 128, 2, 4),    # layer2 block 0: strided shortcut (im2col)
    (14, 1024, 256, 1024, 256, 0, 9),  # layer3: 8 O chunks, N2 = 256
    (9, 128, 64, 128, 192, 0, 7),      # one O chunk, N2 = 192, ragged M
])
@pytest.mark.parametrize("chain", ["1", "0"])
def test_chain(gpu_required, monkeypatch, H, C, Cm, N1, N2, shortcut, batch, chain):
    """Chained block tail + next conv1 (chain_tc.cu) against the oracle, both
    layerwise and end to end on the two outputs; and the unchained path."""
    if shortcut == 0 and C != N1:
        pytest.skip("identity residual needs C == N1")
    monkeypatch.setenv("B2_CHAIN", chain)
    check(chain_plan(H, C, Cm, N1, N2, shortcut), batch)


@pytest.mark.parametrize("H,batch", [(224, 1), (224, 3), (30, 5), (14, 40)])
def test_band8_image_conv(gpu_required, H, batch):
    """3x3/s1 conv on a 3-channel image padded to 8 (VGG conv1_1): the CGW = 8
    band variant, paired taps per UMMA step over overlapping core matrices."""
    check(conv_plan(H, H, 3, 64, 3, 1), batch)


@pytest.mark.parametrize("M,K,N,res", [
    (300, 2048, 512, False),   # 6 tiles, 32 K blocks: split 8
    (200, 1024, 512, True),    # split + residual added in the finalize pass
    (64, 4096, 1024, True),
    (2, 2048, 1000, False),    # ResNet fc at batch 2: ragged last N tile (1000 = 3 x 256 + 232)
])
@pytest.mark.parametrize("split", ["1", "0"])
def test_split_k(gpu_required, monkeypatch, M, K, N, res, split):
    """Small-batch split-K (partials red.add'ed into an fp32 workspace, then a
    finalize pass adds bias / residual / activation) against the oracle."""
    monkeypatch.setenv("B2_SPLIT", split)
    monkeypatch.setenv("B2_PAIR", "0")
    check(linear_plan(K, N, res), M)


@pytest.mark.parametrize("batch", [1, 4])
def test_split_k_conv(gpu_required, batch):
    """layer4 3x3 (K = 4608) at small batch: im2col A under split-K."""
    check(conv_plan(7, 7, 512, 512, 3, 1), batch)


def check_fp32(blob, batch, seed=3):
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, batch, seed)
    plan = R.Plan(blob, P.DT_FP32)
    try:
        out = plan.predict(x)
        assert np.isfinite(out).all()
        rt = lambda t: plan.read_tensor(batch, t, pl.tensors[t].elems, pl.tensors[t].kind)
        errs = plan_ref.layerwise_errors(pl, rt, x, False)
        bad = [e for e in errs if not e[2] <= 1e-5]
        assert not bad, bad
    finally:
        plan.close()


@pytest.mark.parametrize("kind,args,batch", [
    ("linear", (1024, 256, True), 300),        # plain GEMM + residual, ragged M
    ("linear", (768, 3072, False), 64),
    ("linear", (2048, 1000, False), 5),        # ragged N tile
    ("conv", (14, 14, 256, 256, 3, 1), 6),     # im2col A (3x3), 72 K blocks
    ("conv", (28, 28, 128, 256, 3, 2), 3),     # strided im2col
    ("conv", (56, 56, 64, 64, 1, 1), 2),
])
@pytest.mark.parametrize("tf32", ["1", "0"])
def test_fp32_3xtf32(gpu_required, monkeypatch, kind, args, batch, tf32):
    """fp32 plans: 3xTF32 tcgen05 GEMM (hi/lo split, chunked TMEM partial sums)
    vs the CUDA-core FFMA path, layerwise within 1e-5 of fp64."""
    monkeypatch.setenv("B2_TF32", tf32)
    blob = linear_plan(*args) if kind == "linear" else conv_plan(*args)
    check_fp32(blob, batch)


def dw_plan(H, W, C, stride, act, seed=0):
    """One depthwise 3x3 conv (pad 1) on an [H, W, C] input."""
    OH = (H + 2 - 3) // stride + 1
    OW = (W + 2 - 3) // stride + 1
    b = P.PlanBuilder("dw")
    x = b.tensor(H, W, C)
    b.in_elems = C * H * W
    b.op_p(P.OP_INPUT, [x, C, H, W, C])
    rng = np.random.default_rng(seed)
    y = b.tensor(OH, OW, C)
    w = rng.standard_normal((C, 3, 3)) / 3.0
    bias = rng.standard_normal(C) * 0.1
    b.op_p(P.OP_DWCONV, [x, y, b.weight(w), b.weight(bias), H, W, C, stride, 1, OH, OW, act, 3])
    b.out_elems = b.tensors[y].elems
    b.op_p(P.OP_OUTPUT, [1, y, 0])
    return b.build(P.DT_FP32)


@pytest.mark.parametrize("H,W,C,stride,act", [
    (5, 5, 8, 1, 2), (13, 17, 24, 1, 1), (7, 7, 40, 1, 0), (9, 31, 16, 1, 2),
    (13, 13, 24, 2, 2), (8, 15, 8, 2, 1), (112, 112, 32, 1, 2), (56, 56, 144, 2, 2),
])
@pytest.mark.parametrize("owt", ["0", "1", "2", "4", "8"])
def test_dwconv_strip_edges(gpu_required, monkeypatch, H, W, C, stride, act, owt):
    """Depthwise 3x3: the row-strip kernel at every strip width (ragged last
    strips, rows narrower than one strip, image-edge zero fill) and the flat
    kernel (B2_DW_OWT=1), bf16 layerwise and fp32 against the fp64 oracle."""
    if owt != "0":
        monkeypatch.setenv("B2_DW_OWT", owt)
        monkeypatch.setenv("B2_DW_OWT2", owt)
    blob = dw_plan(H, W, C, stride, act)
    check(blob, 3)
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, 3, 4)
    plan = R.Plan(blob, P.DT_FP32)
    try:
        assert plan_ref.normwise_err(plan.predict(x), plan_ref.forward(blob, x)) <= 1e-5
    finally:
        plan.close()


@pytest.mark.parametrize("H,W,batch", [
    (56, 56, 48),    # ResNet layer1 3x3: 336 bands, CTA pairs
    (56, 56, 23),    # odd band count: the last pair's peer has no band
    (224, 224, 3),   # VGG block 1: two column segments per row
    (30, 44, 40),    # ragged: partial last band, W not a multiple of the pitch
])
@pytest.mark.parametrize("pair", ["1", "0"])
def test_band_pair(gpu_required, monkeypatch, H, W, batch, pair):
    """N = 64 3x3 convs on the CTA-pair band kernel (M = 256 UMMAs over two
    bands, each CTA holding half of the resident weights) and the single-CTA one."""
    monkeypatch.setenv("B2_BAND_PAIR", pair)
    check(conv_plan(H, W, 64, 64, 3, 1), batch)


def conv_pool2_plan(H, W, C, N, seed=0):
    """3x3/1 conv (ReLU) then a 2x2/2 max-pool: VGG's block ends."""
    b = P.PlanBuilder("conv_pool2")
    x = b.tensor(H, W, C)
    b.in_elems = C * H * W
    b.op_p(P.OP_INPUT, [x, C, H, W, C])
    rng = np.random.default_rng(seed)
    y = b.tensor(H, W, N)
    w = rng.standard_normal((N, 3, 3, C)) * (1.0 / np.sqrt(9 * C))
    b.op_p(P.OP_CONV, [x, y, b.weight(w), b.weight(rng.standard_normal(N) * 0.1), H, W, C, N,
                       3, 3, 1, 1, H, W, 1, -1])
    z = b.tensor(H // 2, W // 2, N)
    b.op_p(P.OP_MAXPOOL, [y, z, H, W, N, 2, 2, 0, H // 2, W // 2])
    b.out_elems = b.tensors[z].elems
    b.op_p(P.OP_OUTPUT, [1, z, 0])
    return b.build(P.DT_FP32)


@pytest.mark.parametrize("H,W,C,N,batch", [
    (224, 224, 64, 128, 2),    # two column segments per row
    (112, 112, 64, 128, 3),
    (112, 112, 128, 128, 2),   # VGG conv2_2 + pool2
    (100, 120, 64, 128, 3),    # ragged band tail, W below one pitch
    (224, 224, 64, 64, 2),     # N = 64 (VGG conv1_2 + pool1): one-row bands, rows paired
    (112, 112, 64, 64, 3),     #   across consecutive units of a CTA
])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_band_maxpool2(gpu_required, monkeypatch, H, W, C, N, batch, fused):
    """Band conv with the 2x2/2 max-pool fused into its epilogue (the conv
    output is never materialised) and unfused."""
    monkeypatch.setenv("B2_POOL_FUSION", fused)
    blob = conv_pool2_plan(H, W, C, N)
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, batch, 5)
    plan = R.Plan(blob, P.DT_BF16)
    try:
        out = plan.predict(x)
        assert np.isfinite(out).all()
        rt = lambda t: plan.read_tensor(batch, t, pl.tensors[t].elems, pl.tensors[t].kind)
        assert (rt(pl.ops[1][1]) is None) == (fused == "1")
        errs, bad = plan_ref.layerwise_check(pl, rt, x, True)
        assert errs and not bad, errs
    finally:
        plan.close()
