"""The benchmark configurations of BASELINE.json as ModelSpecs over reference node kinds.

The reference has no EV-FlowNet / E2Depth / ResNet-18 definitions
(SURVEY.md section 0), so each config model is spelled with the reference's
own node kinds (graph.py:66-76) exactly as SURVEY.md appendix A.4 fixes
them; the same spec + seeded WeightManifest feed both the oracle and the
GPU engine.

* C1 ``evflownet``  4x256x256 count+timestamp input, 58 nodes, 3,535,128 params
* C2 ``unet_e2depth`` build_unet(levels=4, base=32) on 5x264x352 voxels
* C3 ``resnet18`` 2x180x240 count input, BN folded, fc as linear, 67 nodes
* recurrent: ``recurrent_unet`` -- an E2Depth-style UNet whose encoder
  stages are ConvLSTM cells (the paper's Table I networks), built from
  the reference kinds conv / sigmoid / tanh / mul / add / concat / sparsify plus this package's
  ``delay`` node for h_{t-1} and c_{t-1} (graph.py NODE_KINDS)
"""

from __future__ import annotations

from .graph import ModelSpec, NodeSpec
from .models import UNetConfig, build_unet
from .tensors import TileShape, conv_output_hw


class _B:
    def __init__(self, tp):
        self.tp, self.nodes = tp, []

    def n(self, nid, kind, inputs, **attrs):
        self.nodes.append(NodeSpec(nid, kind, list(inputs), attrs))
        return nid

    def sconv(self, nid, src, out_ch, k, stride=1, pad=None):
        sp = self.n(f"{nid}_sp", "sparsify", [src], tp=self.tp)
        return self.n(nid, "conv", [sp], out_channels=out_ch, kernel=[k, k], stride=stride,
                      padding=k // 2 if pad is None else pad)


def evflownet_spec(tp: float = 0.0, tile=TileShape(6, 6)) -> ModelSpec:
    """C1: 4 stride-2 encoders, 2 residual blocks, 4 bilinear decoders with
    per-level flow heads."""
    b = _B(tp)
    src, skips = "input", []
    for i in range(4):
        src = b.n(f"enc{i}_act", "relu", [b.sconv(f"enc{i}", src, 32 * 2 ** i, 3, stride=2)])
        skips.append(src)
    for r in range(2):
        a = b.n(f"res{r}a_act", "relu", [b.sconv(f"res{r}a", src, 256, 3)])
        s = b.n(f"res{r}_add", "add", [b.sconv(f"res{r}b", a, 256, 3), src])
        src = b.n(f"res{r}_act", "relu", [s])
    pred = None
    for i, ch in enumerate((128, 64, 32, 16)):
        parts = [src, skips[3 - i]] + ([pred] if pred else [])
        cat = b.n(f"dec{i}_cat", "concat", parts)
        up = b.n(f"dec{i}_up", "upsample", [cat], factor=2, mode="bilinear")
        src = b.n(f"dec{i}_act", "relu", [b.sconv(f"dec{i}", up, ch, 3)])
        pred = b.n(f"pred{i}_act", "tanh", [b.sconv(f"pred{i}", src, 2, 1)])
    return ModelSpec("evflownet-256", (4, 256, 256), b.nodes, pred, tile=tile)


def resnet18_spec(tp: float = 0.0, n_classes: int = 101, tile=TileShape(6, 6)) -> ModelSpec:
    """C3: ResNet-18 on 2x180x240 count histograms (N-Caltech101 shape)."""
    b = _B(tp)
    x = b.n("stem_act", "relu", [b.sconv("stem", "input", 64, 7, stride=2, pad=3)])
    x = b.n("stem_pool", "maxpool", [x], window=[3, 3], stride=2)
    ch_in = 64
    for si, ch in enumerate((64, 128, 256, 512)):
        for bi in range(2):
            st = 2 if (si > 0 and bi == 0) else 1
            p = f"s{si}b{bi}"
            y = b.n(f"{p}a_act", "relu", [b.sconv(f"{p}a", x, ch, 3, stride=st)])
            y = b.sconv(f"{p}b", y, ch, 3)
            sc = x if (st == 1 and ch_in == ch) else b.sconv(f"{p}_sc", x, ch, 1, stride=st, pad=0)
            x = b.n(f"{p}_act", "relu", [b.n(f"{p}_add", "add", [y, sc])])
            ch_in = ch
    fc = b.n("fc", "linear", [x], out_features=n_classes)
    return ModelSpec("resnet18-ncaltech", (2, 180, 240), b.nodes, fc, tile=tile)


def unet_e2depth_spec(tp: float = 0.0) -> ModelSpec:
    """C2: build_unet(levels=4, base 32) on a 5-bin voxel grid zero-padded to 264x352."""
    return build_unet(UNetConfig(levels=4, base_channels=32, in_shape=(5, 264, 352), tp=tp))


def convlstm_cell(b: _B, p: str, x: str, hidden: int, shape, k: int = 3) -> str:
    """ConvLSTM cell over node `x` (C_x, H, W) with `hidden` channels; returns the id of h_t.

    z = [x, h_{t-1}];  i, f, o = sigmoid(conv(z)),  g = tanh(conv(z));
    c_t = f * c_{t-1} + i * g;  h_t = o * tanh(c_t)
    (inc_mul carries the product increments, increment_ops.py:241-254; h_{t-1}, c_{t-1} are delay nodes)."""
    _, h, w = shape
    hp = b.n(f"{p}_hprev", "delay", [], source=f"{p}_h", shape=[hidden, h, w])
    cp = b.n(f"{p}_cprev", "delay", [], source=f"{p}_c", shape=[hidden, h, w])
    z = b.n(f"{p}_z", "sparsify", [b.n(f"{p}_cat", "concat", [x, hp])], tp=b.tp)
    gate = {}
    for g, act in (("i", "sigmoid"), ("f", "sigmoid"), ("o", "sigmoid"), ("g", "tanh")):
        conv = b.n(f"{p}_{g}conv", "conv", [z], out_channels=hidden, kernel=[k, k], stride=1, padding=k // 2)
        gate[g] = b.n(f"{p}_{g}", act, [conv])
    c = b.n(f"{p}_c", "add", [b.n(f"{p}_fc", "mul", [gate["f"], cp]), b.n(f"{p}_ig", "mul", [gate["i"], gate["g"]])])
    return b.n(f"{p}_h", "mul", [gate["o"], b.n(f"{p}_tc", "tanh", [c])])


def recurrent_unet_spec(levels: int = 3, base: int = 16, in_shape=(5, 264, 352), tp: float = 0.0,
                        tile=TileShape(6, 6)) -> ModelSpec:
    """E2Depth-style recurrent UNet: 5x5 head, `levels` stride-2 encoder convs each followed by a
    ConvLSTM, two residual blocks, bilinear decoders over [x, skip] and a 1x1 sigmoid prediction."""
    b = _B(tp)
    c, h, w = in_shape
    x = b.n("head_act", "relu", [b.sconv("head", "input", base, 5)])
    skips = []
    for i in range(levels):
        co = base * 2 ** (i + 1)
        h, w = conv_output_hw(h, w, 3, 3, 2, 1)
        y = b.n(f"enc{i}_act", "relu", [b.sconv(f"enc{i}", x, co, 3, stride=2)])
        x = convlstm_cell(b, f"enc{i}_lstm", y, co, (co, h, w))
        skips.append((x, co))
    ch = base * 2 ** levels
    for r in range(2):
        a = b.n(f"res{r}a_act", "relu", [b.sconv(f"res{r}a", x, ch, 3)])
        x = b.n(f"res{r}_act", "relu", [b.n(f"res{r}_add", "add", [b.sconv(f"res{r}b", a, ch, 3), x])])
    for i in reversed(range(levels)):
        co = base * 2 ** i
        up = b.n(f"dec{i}_up", "upsample", [b.n(f"dec{i}_cat", "concat", [x, skips[i][0]])], factor=2, mode="bilinear")
        x = b.n(f"dec{i}_act", "relu", [b.sconv(f"dec{i}", up, co, 5 if i == 0 else 3)])
    pred = b.n("pred_act", "sigmoid", [b.sconv("pred", x, 1, 1)])
    return ModelSpec(f"recurrent-unet-l{levels}-b{base}", tuple(in_shape), b.nodes, pred, tile=tile)


CONFIGS = {"evflownet": evflownet_spec, "resnet18": resnet18_spec, "unet_e2depth": unet_e2depth_spec,
           "recurrent_unet": recurrent_unet_spec}
