"""Model emitters: framework graphs -> ``b200-plan`` ops (the converter's core).

The reference's converter only re-encodes toy graphs
(pkg/src/modelci/converter/plugins.py:141-167); the north star needs real
networks, so this module lowers

* toy graphs (C1 MLP)            -> INPUT, LINEAR(+bias,+fused act), LAYERNORM, ACT
* torchvision ResNet-50 / MobileNetV2 / VGG-16 (C2, C4)
                                  -> INPUT, CONV(+folded BN,+act,+residual), DWCONV,
                                     MAXPOOL, AVGPOOL, LINEAR
* transformers BertModel (C3)    -> TOKENS, EMBED(+LN), LINEAR(QKV fused), ATTENTION,
                                     LINEAR(+residual), LAYERNORM, LINEAR(+gelu), pooler

BatchNorm is folded into the preceding conv in float64 (w' = w*g/sqrt(v+e),
b' = beta - mean*g/sqrt(v+e)) and stored as fp32.  Convolution weights are
re-laid out OIHW -> OHWI to match the NHWC activations; VGG's first classifier
weight is permuted from (C,H,W) to (H,W,C) flatten order.

Toy op semantics (undefined by the reference, defined here):
``linear`` weights are row-major [out][in] optionally followed by out biases;
``relu``/``gelu`` are elementwise (in == out, no weights); ``norm`` is a
LayerNorm over the feature dim with optional gamma+beta, eps 1e-5.
"""

from __future__ import annotations

import math

import numpy as np

from . import plan as P
from .errors import ToyFormatError

IMAGE_MODELS = ("resnet50", "mobilenet_v2", "vgg16")
ALL_MODELS = ("mlp",) + IMAGE_MODELS + ("bert",)

# -- toy graphs -----------------------------------------------------------------


def make_mlp_graph(seed: int = 0, dims=(784, 256, 10)) -> dict:
    """C1: linear 784->256 (+bias), relu, linear 256->10 (+bias); nn.Linear's
    default U(-1/sqrt(in), 1/sqrt(in)) init drawn from a seeded numpy RNG."""
    rng = np.random.default_rng(seed)
    layers = []
    for i, (din, dout) in enumerate(zip(dims[:-1], dims[1:])):
        bound = 1.0 / math.sqrt(din)
        w = rng.uniform(-bound, bound, size=(dout, din))
        b = rng.uniform(-bound, bound, size=(dout,))
        layers.append({"op": "linear", "in_dim": din, "out_dim": dout,
                       "weights": w.ravel().tolist() + b.tolist()})
        if i < len(dims) - 2:
            layers.append({"op": "relu", "in_dim": dout, "out_dim": dout, "weights": []})
    return {"layers": layers}


_TOY_ACTS = {"relu": P.ACT_RELU, "gelu": P.ACT_GELU}


def emit_toy(graph: dict, name: str = "toy") -> P.PlanBuilder:
    layers = graph["layers"]
    for i in range(1, len(layers)):
        if layers[i]["in_dim"] != layers[i - 1]["out_dim"]:
            raise ToyFormatError(f"layer {i}: in_dim {layers[i]['in_dim']} does not chain "
                                 f"from out_dim {layers[i - 1]['out_dim']}")
    b = P.PlanBuilder(name)
    d0 = layers[0]["in_dim"]
    x = b.tensor(d0)
    b.in_elems = d0
    b.op_p(P.OP_INPUT, [x, d0, 1, 1, d0])
    flops = 0
    i = 0
    while i < len(layers):
        layer = layers[i]
        op, din, dout, ws = layer["op"], layer["in_dim"], layer["out_dim"], layer["weights"]
        if op == "linear":
            if len(ws) not in (din * dout, din * dout + dout):
                raise ToyFormatError(f"layer {i}: linear needs {din * dout} or "
                                     f"{din * dout + dout} weights, got {len(ws)}")
            w = np.asarray(ws[:din * dout], dtype=np.float64).reshape(dout, din)
            bias = -1
            if len(ws) > din * dout:
                bias = b.weight(np.asarray(ws[din * dout:], dtype=np.float64))
            act = P.ACT_NONE
            if i + 1 < len(layers) and layers[i + 1]["op"] in _TOY_ACTS:
                act = _TOY_ACTS[layers[i + 1]["op"]]
                i += 1
            y = b.tensor(dout)
            b.op_p(P.OP_LINEAR, [x, y, b.weight(w), bias, din, dout, 1, act, -1, din])
            flops += 2 * din * dout
            x = y
        elif op in _TOY_ACTS:
            if din != dout or ws:
                raise ToyFormatError(f"layer {i}: {op} needs in_dim == out_dim and no weights")
            y = b.tensor(dout)
            b.op_p(P.OP_ACT, [x, y, dout, _TOY_ACTS[op]])
            x = y
        elif op == "norm":
            if din != dout or len(ws) not in (0, 2 * dout):
                raise ToyFormatError(f"layer {i}: norm needs in_dim == out_dim and 0 or "
                                     f"{2 * dout} weights")
            g = np.asarray(ws[:dout] if ws else np.ones(dout))
            be = np.asarray(ws[dout:] if ws else np.zeros(dout))
            y = b.tensor(dout)
            b.op_p(P.OP_LAYERNORM, [x, y, b.weight(g), b.weight(be), dout, 1,
                                    P.f32_bits(1e-5), -1])
            x = y
        else:
            raise ToyFormatError(f"layer {i}: op '{op}' has no executable semantics")
        i += 1
    dout = layers[-1]["out_dim"]
    b.out_elems = dout
    b.op_p(P.OP_OUTPUT, [1, x, 0])
    b.meta["flops_per_sample"] = flops
    return b


# -- torchvision CNNs --------------------------------------------------------------


def _fold(conv, bn):
    """(weight OHWI fp64, bias fp64) with BN folded in."""
    w = conv.weight.detach().double().numpy()
    bias = conv.bias.detach().double().numpy() if conv.bias is not None else \
        np.zeros(w.shape[0])
    if bn is not None:
        g = bn.weight.detach().double().numpy()
        beta = bn.bias.detach().double().numpy()
        mean = bn.running_mean.detach().double().numpy()
        var = bn.running_var.detach().double().numpy()
        scale = g / np.sqrt(var + bn.eps)
        w = w * scale[:, None, None, None]
        bias = (bias - mean) * scale + beta
    return w, bias


class _CnnEmitter:
    def __init__(self, name: str, c_in: int = 3, hw: int = 224, c_pad: int = 8):
        self.b = P.PlanBuilder(name)
        self.flops = 0
        x = self.b.tensor(hw, hw, c_pad)
        self.b.in_elems = c_in * hw * hw
        self.b.op_p(P.OP_INPUT, [x, c_in, hw, hw, c_pad])
        self.x = x
        self.true_c = c_in

    def conv(self, x, conv, bn, act, res=-1):
        H, W, C = self.b.shape(x)
        w, bias = _fold(conv, bn)
        cout, cin_w, R, S = w.shape
        groups = conv.groups
        stride, pad = conv.stride[0], conv.padding[0]
        OH = (H + 2 * pad - R) // stride + 1
        OW = (W + 2 * pad - S) // stride + 1
        y = self.b.tensor(OH, OW, cout)
        if groups == 1:
            if cin_w != C:   # zero-padded input channels (stem)
                wp = np.zeros((cout, C, R, S))
                wp[:, :cin_w] = w
                w = wp
            self.b.op_p(P.OP_CONV, [x, y, self.b.weight(w.transpose(0, 2, 3, 1)),
                                    self.b.weight(bias), H, W, C, cout, R, S, stride, pad,
                                    OH, OW, act, res])
            self.flops += 2 * OH * OW * cout * R * S * cin_w
        else:
            if not (groups == C == cout and cin_w == 1 and R == S):
                raise ValueError("only depthwise grouped convs are supported")
            self.b.op_p(P.OP_DWCONV, [x, y, self.b.weight(w[:, 0]), self.b.weight(bias), H, W,
                                      C, stride, pad, OH, OW, act, R])
            self.flops += 2 * OH * OW * C * R * S
        return y

    def maxpool(self, x, k, stride, pad):
        H, W, C = self.b.shape(x)
        OH = (H + 2 * pad - k) // stride + 1
        OW = (W + 2 * pad - k) // stride + 1
        y = self.b.tensor(OH, OW, C)
        self.b.op_p(P.OP_MAXPOOL, [x, y, H, W, C, k, stride, pad, OH, OW])
        return y

    def avgpool(self, x):
        H, W, C = self.b.shape(x)
        y = self.b.tensor(C)
        self.b.op_p(P.OP_AVGPOOL, [x, y, H, W, C])
        return y

    def linear(self, x, lin, act=P.ACT_NONE, weight=None):
        w = (weight if weight is not None else lin.weight.detach().double().numpy())
        n, k = w.shape
        y = self.b.tensor(n)
        bias = self.b.weight(lin.bias.detach().double().numpy()) if lin.bias is not None else -1
        self.b.op_p(P.OP_LINEAR, [x, y, self.b.weight(w), bias, k, n, 1, act, -1, k])
        self.flops += 2 * n * k
        return y

    def finish(self, y):
        self.b.out_elems = self.b.tensors[y].elems
        self.b.op_p(P.OP_OUTPUT, [1, y, 0])
        self.b.meta["flops_per_sample"] = self.flops
        return self.b


def _act_of(m) -> int:
    import torch.nn as nn
    if isinstance(m, nn.ReLU6):
        return P.ACT_RELU6
    if isinstance(m, nn.ReLU):
        return P.ACT_RELU
    raise ValueError(f"unsupported activation {type(m).__name__}")


def emit_resnet(model, name="resnet50") -> P.PlanBuilder:
    e = _CnnEmitter(name)
    x = e.conv(e.x, model.conv1, model.bn1, P.ACT_RELU)
    x = e.maxpool(x, model.maxpool.kernel_size, model.maxpool.stride, model.maxpool.padding)
    for layer in (model.layer1, model.layer2, model.layer3, model.layer4):
        for blk in layer:
            if blk.downsample is not None:
                ident = e.conv(x, blk.downsample[0], blk.downsample[1], P.ACT_NONE)
            else:
                ident = x
            h = e.conv(x, blk.conv1, blk.bn1, P.ACT_RELU)
            h = e.conv(h, blk.conv2, blk.bn2, P.ACT_RELU)
            x = e.conv(h, blk.conv3, blk.bn3, P.ACT_RELU, res=ident)
    x = e.avgpool(x)
    return e.finish(e.linear(x, model.fc))


def _emit_conv_norm_act(e, x, seq):
    mods = list(seq.children())
    act = _act_of(mods[2]) if len(mods) > 2 else P.ACT_NONE
    return e.conv(x, mods[0], mods[1], act)


def emit_mobilenet_v2(model, name="mobilenet_v2") -> P.PlanBuilder:
    import torch.nn as nn
    from torchvision.models.mobilenetv2 import InvertedResidual
    e = _CnnEmitter(name)
    x = e.x
    for m in model.features:
        if isinstance(m, InvertedResidual):
            inp = x
            mods = list(m.conv.children())
            h = x
            j = 0
            while j < len(mods):
                mod = mods[j]
                if isinstance(mod, nn.Conv2d):      # 1x1 project + BN (+ residual)
                    h = e.conv(h, mod, mods[j + 1], P.ACT_NONE,
                               res=inp if m.use_res_connect else -1)
                    j += 2
                else:                               # Conv2dNormActivation
                    h = _emit_conv_norm_act(e, h, mod)
                    j += 1
            x = h
        else:
            x = _emit_conv_norm_act(e, x, m)
    x = e.avgpool(x)
    lin = [c for c in model.classifier if isinstance(c, nn.Linear)][0]
    return e.finish(e.linear(x, lin))


def emit_vgg(model, name="vgg16") -> P.PlanBuilder:
    import torch.nn as nn
    e = _CnnEmitter(name)
    x = e.x
    feats = list(model.features)
    j = 0
    while j < len(feats):
        m = feats[j]
        if isinstance(m, nn.Conv2d):
            act = P.ACT_NONE
            if j + 1 < len(feats) and isinstance(feats[j + 1], nn.ReLU):
                act = P.ACT_RELU
                j += 1
            x = e.conv(x, m, None, act)
        elif isinstance(m, nn.MaxPool2d):
            x = e.maxpool(x, m.kernel_size, m.stride, m.padding)
        j += 1
    H, W, C = e.b.shape(x)
    if (H, W) != (7, 7):
        raise ValueError("VGG emitter expects a 7x7 feature map (224x224 input)")
    cls = list(model.classifier)
    lins = [(i, c) for i, c in enumerate(cls) if isinstance(c, nn.Linear)]
    # flatten: NHWC storage means (H,W,C) order; permute torch's (C,H,W) columns
    w0 = lins[0][1].weight.detach().double().numpy()
    w0 = w0.reshape(w0.shape[0], C, H, W).transpose(0, 2, 3, 1).reshape(w0.shape[0], -1)
    flat = x  # [7,7,512] is already the per-sample flat vector in (H,W,C) order
    y = flat
    for n, (i, lin) in enumerate(lins):
        act = P.ACT_RELU if i + 1 < len(cls) and isinstance(cls[i + 1], nn.ReLU) else P.ACT_NONE
        y = e.linear(y, lin, act, weight=w0 if n == 0 else None)
    return e.finish(y)


# -- BERT ---------------------------------------------------------------------------


def emit_bert(model, seq: int = 128, name="bert", mask: bool = True) -> P.PlanBuilder:
    """BertModel -> plan.  ``mask``: the sample is [input_ids, attention_mask]
    (padded batches, transformers semantics); the profiling payload sets the
    mask to ones (attention_mask=1)."""
    cfg = model.config
    D, H = cfg.hidden_size, cfg.num_attention_heads
    Dh = D // H
    eps = cfg.layer_norm_eps
    b = P.PlanBuilder(name)
    b.input_kind = P.IN_TOKENS
    b.in_elems = 2 * seq if mask else seq
    flops = 0

    def lin(x, module, rows, act=P.ACT_NONE, res=-1, weight=None, bias=None, astride=None):
        nonlocal flops
        w = weight if weight is not None else module.weight.detach().double().numpy()
        bb = bias if bias is not None else module.bias.detach().double().numpy()
        n, k = w.shape
        y = b.tensor(rows, n) if rows > 1 else b.tensor(n)
        b.op_p(P.OP_LINEAR, [x, y, b.weight(w), b.weight(bb), k, n, rows, act, res,
                             astride if astride is not None else k])
        flops += 2 * rows * n * k
        return y

    def layernorm(x, ln, res=-1):
        y = b.tensor(seq, D)
        b.op_p(P.OP_LAYERNORM, [x, y, b.weight(ln.weight.detach().double().numpy()),
                                b.weight(ln.bias.detach().double().numpy()), D, seq,
                                P.f32_bits(ln.eps), res])
        return y

    ids = b.tensor(seq, kind=P.T_IDS)
    mbits = b.tensor((seq + 31) // 32, kind=P.T_IDS) if mask else 0
    b.op_p(P.OP_TOKENS, [ids, seq, cfg.vocab_size, int(mask), mbits])
    emb = model.embeddings
    x = b.tensor(seq, D)
    b.op_p(P.OP_EMBED, [ids, x, b.weight(emb.word_embeddings.weight.detach().numpy()),
                        b.weight(emb.position_embeddings.weight.detach().numpy()[:seq]),
                        b.weight(emb.token_type_embeddings.weight.detach().numpy()[0]),
                        b.weight(emb.LayerNorm.weight.detach().numpy()),
                        b.weight(emb.LayerNorm.bias.detach().numpy()), D, seq, cfg.vocab_size,
                        P.f32_bits(emb.LayerNorm.eps)])
    for layer in model.encoder.layer:
        sa = layer.attention.self
        wqkv = np.concatenate([m.weight.detach().double().numpy()
                               for m in (sa.query, sa.key, sa.value)], 0)
        bqkv = np.concatenate([m.bias.detach().double().numpy()
                               for m in (sa.query, sa.key, sa.value)], 0)
        qkv = lin(x, None, seq, weight=wqkv, bias=bqkv)
        ctx = b.tensor(seq, D)
        b.op_p(P.OP_ATTENTION, [qkv, ctx, H, Dh, seq, int(mask), mbits])
        flops += 4 * H * seq * seq * Dh
        ao = layer.attention.output
        a = lin(ctx, ao.dense, seq, res=x)
        x1 = layernorm(a, ao.LayerNorm)
        hmid = lin(x1, layer.intermediate.dense, seq, act=P.ACT_GELU)
        o = lin(hmid, layer.output.dense, seq, res=x1)
        x = layernorm(o, layer.output.LayerNorm)
    pooled = lin(x, model.pooler.dense, 1, act=P.ACT_TANH, astride=seq * D)
    b.out_elems = seq * D + D
    b.op_p(P.OP_OUTPUT, [2, x, 0, pooled, seq * D])
    b.meta["flops_per_sample"] = flops
    b.meta["seq"] = seq
    b.meta["attention_mask"] = bool(mask)
    return b


# -- seeded synthetic models ---------------------------------------------------------


def make_torch_model(name: str, seed: int = 0, calibrate: bool = True):
    """Random-init model under torch.manual_seed(seed); BN running stats are
    calibrated with one seeded train-mode pass (momentum=None) so folded BN is
    non-trivial and logits stay O(1) (SURVEY.md §7 'Calibrate BN')."""
    import torch
    torch.manual_seed(seed)
    if name == "bert":
        from transformers import BertConfig, BertModel
        m = BertModel(BertConfig(), add_pooling_layer=True)
        return m.eval()
    import torchvision.models as tvm
    m = getattr(tvm, name)(weights=None)
    bns = [mod for mod in m.modules() if isinstance(mod, torch.nn.BatchNorm2d)]
    if calibrate and bns:
        for bn in bns:
            bn.momentum = None
            bn.reset_running_stats()
        g = torch.Generator().manual_seed(seed + 1)
        x = torch.randn(8, 3, 224, 224, generator=g)
        m.train()
        with torch.no_grad():
            m(x)
    return m.eval()


def emit_torch(name: str, model) -> P.PlanBuilder:
    if name == "resnet50" or name.startswith("resnet"):
        return emit_resnet(model, name)
    if name == "mobilenet_v2":
        return emit_mobilenet_v2(model, name)
    if name.startswith("vgg"):
        return emit_vgg(model, name)
    if name == "bert":
        return emit_bert(model)
    raise ValueError(f"no emitter for '{name}'")


def build_plan(name: str, dtype: int = P.DT_BF16, seed: int = 0) -> bytes:
    """Seeded synthetic model -> plan bytes (bench / tests entry point)."""
    if name == "mlp":
        return emit_toy(make_mlp_graph(seed), "mlp").build(dtype)
    return emit_torch(name, make_torch_model(name, seed)).build(dtype)
