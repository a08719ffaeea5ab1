"""BERT attention mask on the GPU (QK^T -> mask -> softmax -> PV): padded
batches through the tcgen05 attention kernel (bf16) and the SIMT kernel
(fp32 plans) against the oracle, which is pinned to transformers'
BertModel(attention_mask=...) in tests/test_oracle.py."""
import numpy as np
import pytest

import plan_ref
from paper_2006_05096_b200 import plan as P
from paper_2006_05096_b200 import runtime as R
from paper_2006_05096_b200 import zoo

pytestmark = pytest.mark.gpu


def padded(pl, lengths, seed=7):
    x = plan_ref.make_inputs(pl, len(lengths), seed)
    for i, n in enumerate(lengths):
        x[i, n:128] = 0
        x[i, 128:] = 0
        x[i, 128:128 + n] = 1
    return x


@pytest.fixture(scope="module")
def bert_blob():
    return zoo.build_plan("bert", P.DT_BF16, seed=0)


@pytest.mark.parametrize("dtype", [P.DT_FP32, P.DT_BF16])
def test_padded_batch_end_to_end(gpu_required, bert_blob, dtype):
    blob = P.with_dtype(bert_blob, dtype)
    pl = P.decode(blob)
    x = padded(pl, [128, 77, 5, 1, 128, 33])
    ref = plan_ref.forward(pl, x)
    plan = R.Plan(blob, dtype)
    try:
        y = plan.predict(x)
        rt = lambda t: plan.read_tensor(len(x), t, pl.tensors[t].elems, pl.tensors[t].kind)
        _, bad = plan_ref.layerwise_check(pl, rt, x, dtype == P.DT_BF16)
    finally:
        plan.close()
    err = plan_ref.normwise_err(y, ref)
    assert err <= (1e-4 if dtype == P.DT_FP32 else 2e-2), err
    assert not bad, bad[:5]
    # masking works: a short sample's valid positions and pooled output do not
    # depend on what its padded positions hold
    x2 = x.copy()
    x2[2, 5:128] = 1234
    plan = R.Plan(blob, dtype)
    try:
        y2 = plan.predict(x2)
    finally:
        plan.close()
    keep = np.r_[0:5 * 768, 128 * 768:129 * 768]
    assert plan_ref.normwise_err(y2[2, keep], y[2, keep]) <= (1e-5 if dtype == P.DT_FP32
                                                             else 1e-2)
    assert plan_ref.normwise_err(y2[2], y[2]) > 0.01      # the padded rows themselves changed


def test_mask_words_match_oracle_and_full_mask_is_unmasked(gpu_required, bert_blob):
    pl = P.decode(bert_blob)
    x = padded(pl, [128, 64, 31, 1])
    plan = R.Plan(bert_blob, P.DT_BF16)
    try:
        plan.predict(x)
        tk = next(o for o in pl.ops if o.kind == P.OP_TOKENS)
        words = plan.read_tensor(4, tk[P.P_TK_MASK], 4, P.T_IDS)
        assert np.array_equal(np.asarray(words).reshape(4, 4),
                              plan_ref.pack_keymask(x[:, 128:] != 0))
        # all-ones mask == the same ids with the mask half ignored by an unmasked plan
        full = plan_ref.make_inputs(pl, 8, 3)
        y_mask = plan.predict(full)
    finally:
        plan.close()
    unmasked = zoo.emit_bert(zoo.make_torch_model("bert", 0), mask=False).build(P.DT_BF16)
    plan = R.Plan(unmasked, P.DT_BF16)
    try:
        y_plain = plan.predict(full[:, :128])
    finally:
        plan.close()
    assert np.array_equal(y_mask, y_plain)
