"""b200-plan format: round trip, corruption, dtype rewrite, toy lowering errors."""
import numpy as np
import pytest

from paper_2006_05096_b200 import plan as P
from paper_2006_05096_b200 import zoo
from paper_2006_05096_b200.errors import PlanFormatError, ToyFormatError


def test_round_trip_mlp():
    blob = zoo.build_plan("mlp", P.DT_BF16)
    pl = P.decode(blob)
    assert pl.dtype == P.DT_BF16 and pl.in_elems == 784 and pl.out_elems == 10
    assert [o.kind for o in pl.ops] == [P.OP_INPUT, P.OP_LINEAR, P.OP_LINEAR, P.OP_OUTPUT]
    assert pl.ops[1][P.P_LN_ACT] == P.ACT_RELU          # relu fused into the first linear
    assert pl.meta["flops_per_sample"] == 406528         # BASELINE.md FLOP count
    assert P.decode(P.encode(pl)) .ops[1].p == pl.ops[1].p


def test_dtype_rewrite_keeps_crc():
    blob = zoo.build_plan("mlp", P.DT_BF16)
    f32 = P.with_dtype(blob, P.DT_FP32)
    assert P.decode(f32).dtype == P.DT_FP32 and len(f32) == len(blob)


def test_corruption_detected():
    blob = bytearray(zoo.build_plan("mlp"))
    with pytest.raises(PlanFormatError, match="magic"):
        P.decode(b"XXXX" + bytes(blob[4:]))
    blob[100] ^= 1
    with pytest.raises(PlanFormatError, match="CRC"):
        P.decode(bytes(blob))
    with pytest.raises(PlanFormatError):
        P.decode(b"B2PL")


def test_toy_semantics_errors():
    bad_chain = {"layers": [{"op": "linear", "in_dim": 2, "out_dim": 3, "weights": [0.0] * 6},
                            {"op": "linear", "in_dim": 4, "out_dim": 1, "weights": [0.0] * 4}]}
    with pytest.raises(ToyFormatError, match="chain"):
        zoo.emit_toy(bad_chain)
    bad_count = {"layers": [{"op": "linear", "in_dim": 2, "out_dim": 3, "weights": [0.0] * 5}]}
    with pytest.raises(ToyFormatError):
        zoo.emit_toy(bad_count)
    unknown = {"layers": [{"op": "conv", "in_dim": 2, "out_dim": 2, "weights": []}]}
    with pytest.raises(ToyFormatError, match="semantics"):
        zoo.emit_toy(unknown)


def test_norm_and_gelu_lowering():
    g = {"layers": [{"op": "linear", "in_dim": 8, "out_dim": 8, "weights": [0.1] * 64},
                    {"op": "norm", "in_dim": 8, "out_dim": 8, "weights": [1.0] * 8 + [0.0] * 8},
                    {"op": "gelu", "in_dim": 8, "out_dim": 8, "weights": []}]}
    pl = P.decode(zoo.emit_toy(g).build())
    assert [o.kind for o in pl.ops] == [P.OP_INPUT, P.OP_LINEAR, P.OP_LAYERNORM, P.OP_ACT,
                                        P.OP_OUTPUT]


@pytest.mark.parametrize("name,flops", [("resnet50", 8178368512), ("mobilenet_v2", 601548544),
                                        ("bert", 22348431360), ("vgg16", 30940528640),
                                        ("mlp", 406528)])
def test_flops_count_true_channels(name, flops):
    """Algorithmic FLOPs use the model's true channels (the 3-channel stem is
    padded to 8 in the plan; the padding is not work) — the roofline numerator
    (SURVEY.md §8(d)); libb2's b2_plan_info applies the same rule."""
    pl = P.decode(zoo.build_plan(name, P.DT_BF16, seed=0))
    assert P.flops_per_sample(pl) == pl.meta["flops_per_sample"] == flops
