"""Pinning the CPU oracle (oracle/plan_ref.py) before trusting it:

* C1 MLP: against oracle/toyref.c (independent C fp64 restatement over the
  reference's toy-binary bytes) and tests/golden/mlp_golden.json;
* ResNet-50 / MobileNetV2 / VGG-16 / BERT-base: against the torchvision / transformers
  modules' own fp64 CPU forward (third-party, not in /root/reference; parity
  of the converter's BN folding, OHWI layouts, QKV fusion and flatten order).
* the device input generator's CPU restatement (oracle/gen_ref.py) sanity.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import gen_ref
import plan_ref
import toyref
from paper_2006_05096_b200 import plan as P
from paper_2006_05096_b200 import toyformat, zoo

# 2 * MACs of torchvision vgg16 at 224x224 (13 convs + 3 linears; 30.941 GFLOP)
VGG16_FLOPS = 30940528640
GOLD = json.loads((Path(__file__).parent / "golden" / "mlp_golden.json").read_text())


def test_mlp_oracle_matches_c_restatement_and_golden():
    g = zoo.make_mlp_graph(GOLD["seed"])
    blob = toyformat.encode_binary(g)
    assert hashlib.sha256(blob).hexdigest() == GOLD["toy_binary_sha256"]
    x = np.random.default_rng(GOLD["x_seed"]).standard_normal((4, 784))
    c_out = toyref.forward(blob, x)
    np.testing.assert_allclose(c_out, np.array(GOLD["logits"]), rtol=0, atol=1e-12)
    py_out = plan_ref.forward(zoo.emit_toy(g).build(P.DT_FP32), x)
    # plan weights are fp32: agreement to fp32 rounding of the weights
    assert plan_ref.normwise_err(py_out, c_out) < 1e-6


def test_toyref_rejects_corruption():
    blob = bytearray(toyformat.encode_binary(zoo.make_mlp_graph(0)))
    blob[20] ^= 1
    with pytest.raises(ValueError, match="CRC"):
        toyref.forward(bytes(blob), np.zeros((1, 784)))


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2", "vgg16", "bert"])
def test_oracle_matches_framework_forward(name):
    import torch
    torch.set_num_threads(8)
    model = zoo.make_torch_model(name, 0)
    pl = P.decode(zoo.emit_torch(name, model).build(P.DT_FP32))
    x = plan_ref.make_inputs(pl, 1, 3)
    out = plan_ref.forward(pl, x)
    md = model.double()
    with torch.no_grad():
        if name == "bert":
            r = md(input_ids=torch.from_numpy(x[:, :128]),
                   attention_mask=torch.from_numpy(x[:, 128:]))
            ref = torch.cat([r.last_hidden_state.reshape(1, -1), r.pooler_output], 1).numpy()
        else:
            ref = md(torch.from_numpy(x.astype(np.float64)).reshape(1, 3, 224, 224)).numpy()
    # only the plan's fp32 weight storage separates the two
    assert plan_ref.normwise_err(out, ref) < 2e-5
    assert pl.meta["flops_per_sample"] == {"resnet50": 8178368512, "mobilenet_v2": 601548544,
                                           "vgg16": VGG16_FLOPS, "bert": 22348431360}[name]


def padded_bert_inputs(pl, lengths, seed=7):
    """Token ids + attention_mask for a padded batch: sample i attends to its
    first lengths[i] tokens (the rest are [PAD] = 0, as a tokenizer pads)."""
    S = 128
    x = plan_ref.make_inputs(pl, len(lengths), seed)
    for i, n in enumerate(lengths):
        x[i, n:S] = 0
        x[i, S:] = 0
        x[i, S:S + n] = 1
    return x


def test_oracle_bert_padded_batch_matches_transformers():
    """QK^T -> mask -> softmax -> PV: a padded batch (lengths 128, 77, 5)
    through the oracle equals transformers' BertModel with attention_mask,
    padded query rows included."""
    import torch
    torch.set_num_threads(8)
    model = zoo.make_torch_model("bert", 0)
    pl = P.decode(zoo.emit_torch("bert", model).build(P.DT_FP32))
    x = padded_bert_inputs(pl, [128, 77, 5])
    out = plan_ref.forward(pl, x)
    with torch.no_grad():
        r = model.double()(input_ids=torch.from_numpy(x[:, :128]),
                           attention_mask=torch.from_numpy(x[:, 128:]))
    ref = torch.cat([r.last_hidden_state.reshape(3, -1), r.pooler_output], 1).numpy()
    assert plan_ref.normwise_err(out, ref) < 2e-5
    # the mask matters: without it the short samples change completely
    nomask = x.copy()
    nomask[:, 128:] = 1
    assert plan_ref.normwise_err(plan_ref.forward(pl, nomask)[2], ref[2]) > 0.1


def test_keymask_pack_roundtrip():
    rng = np.random.default_rng(0)
    m = rng.random((5, 128)) < 0.5
    w = plan_ref.pack_keymask(m)
    assert w.shape == (5, 4) and np.array_equal(plan_ref.unpack_keymask(w, 128), m)
    assert plan_ref.pack_keymask(np.ones((1, 128), bool)).tolist() == [[-1, -1, -1, -1]]


def test_bf16_emulation_is_round_to_nearest_even():
    x = np.array([1.0, 1.00390625, 1.01171875, -3.14159, 65504.0], dtype=np.float32)
    r = plan_ref.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.015625   # ties to even
    assert abs(r[3] - np.float32(-3.140625)) < 1e-7


def test_gen_ref_distribution():
    z = gen_ref.normal(200000, 5)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    t = gen_ref.tokens(100000, 30522, 5)
    assert t.min() >= 0 and t.max() < 30522
