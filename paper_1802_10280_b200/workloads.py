"""Layer tables of the paper's workloads (Table 3) and BASELINE configs.

Shapes are the standard Caffe definitions the paper's SkimCaffe models use;
SURVEY §8(c) readings R#15/R#16 pin the variants against Table 3:
  * AlexNet with groups=2 on conv2/4/5 gives 724.4M MACs / 60.95M weights
    (Table 3: 724M / 61M).
  * ResNet-50 v1 (stride on the first 1x1 of a downsampling block) gives
    3.858G MACs / 25.50M weights (Table 3: 3.9G / 25.5M).
  * GoogLeNet (no aux classifiers) gives 57 conv layers / 19 sparse / 6.99M
    weights; its MAC total (1.58G) does NOT match Table 3's 1.43G — reading
    R#17, left unpinned.
"Sparse" layers (R#15): AlexNet conv2-5; GoogLeNet conv2/3x3 + the 3x3/5x5 of
the nine inception modules; ResNet-50 the 16 bottleneck 3x3 convolutions.
Per-layer sparsities are never printed by the paper (R#14): 80% is ASSUMED.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List


@dataclass(frozen=True)
class Layer:
    name: str
    C: int          # total input channels
    H: int
    W: int
    M: int          # output channels
    K: int          # square filter
    stride: int = 1
    pad: int = 0
    groups: int = 1
    sparse: bool = False
    kind: str = "conv"  # "conv" or "fc"

    @property
    def E(self) -> int:
        return (self.H + 2 * self.pad - self.K) // self.stride + 1

    @property
    def F(self) -> int:
        return (self.W + 2 * self.pad - self.K) // self.stride + 1

    @property
    def weights(self) -> int:
        return self.M * (self.C // self.groups) * self.K * self.K

    @property
    def macs(self) -> int:
        return self.weights * self.E * self.F


def _fc(name, cin, cout):
    return Layer(name, cin, 1, 1, cout, 1, kind="fc")


# ------------------------------------------------------------------ AlexNet
def alexnet_full() -> List[Layer]:
    return [
        Layer("conv1", 3, 227, 227, 96, 11, 4, 0, 1),
        Layer("conv2", 96, 27, 27, 256, 5, 1, 2, 2, sparse=True),
        Layer("conv3", 256, 13, 13, 384, 3, 1, 1, 1, sparse=True),
        Layer("conv4", 384, 13, 13, 384, 3, 1, 1, 2, sparse=True),
        Layer("conv5", 384, 13, 13, 256, 3, 1, 1, 2, sparse=True),
        _fc("fc6", 256 * 6 * 6, 4096), _fc("fc7", 4096, 4096), _fc("fc8", 4096, 1000),
    ]


# ------------------------------------------------------------------ GoogLeNet
_INCEPTION = [  # name, size, in, 1x1, 3x3red, 3x3, 5x5red, 5x5, pool_proj
    ("inception_3a", 28, 192, 64, 96, 128, 16, 32, 32),
    ("inception_3b", 28, 256, 128, 128, 192, 32, 96, 64),
    ("inception_4a", 14, 480, 192, 96, 208, 16, 48, 64),
    ("inception_4b", 14, 512, 160, 112, 224, 24, 64, 64),
    ("inception_4c", 14, 512, 128, 128, 256, 24, 64, 64),
    ("inception_4d", 14, 512, 112, 144, 288, 32, 64, 64),
    ("inception_4e", 14, 528, 256, 160, 320, 32, 128, 128),
    ("inception_5a", 7, 832, 256, 160, 320, 32, 128, 128),
    ("inception_5b", 7, 832, 384, 192, 384, 48, 128, 128),
]


def googlenet_full() -> List[Layer]:
    L = [
        Layer("conv1/7x7_s2", 3, 224, 224, 64, 7, 2, 3),
        Layer("conv2/3x3_reduce", 64, 56, 56, 64, 1),
        Layer("conv2/3x3", 64, 56, 56, 192, 3, 1, 1, sparse=True),
    ]
    for name, s, cin, c1, r3, c3, r5, c5, pp in _INCEPTION:
        L += [
            Layer(name + "/1x1", cin, s, s, c1, 1),
            Layer(name + "/3x3_reduce", cin, s, s, r3, 1),
            Layer(name + "/3x3", r3, s, s, c3, 3, 1, 1, sparse=True),
            Layer(name + "/5x5_reduce", cin, s, s, r5, 1),
            Layer(name + "/5x5", r5, s, s, c5, 5, 1, 2, sparse=True),
            Layer(name + "/pool_proj", cin, s, s, pp, 1),
        ]
    L.append(_fc("loss3/classifier", 1024, 1000))
    return L


# ------------------------------------------------------------------ ResNet-50 v1
def resnet50_full(v15: bool = False) -> List[Layer]:
    """ResNet-50 v1 (Caffe; stride on the first 1x1) or, with v15=True, v1.5
    (stride on the 3x3 of each downsampling block; NEXT-3 stride-2 workload)."""
    L = [Layer("conv1", 3, 224, 224, 64, 7, 2, 3)]
    stages = [("res2", 3, 64, 256, 56, 1), ("res3", 4, 128, 512, 28, 2),
              ("res4", 6, 256, 1024, 14, 2), ("res5", 3, 512, 2048, 7, 2)]
    cin, size = 64, 56
    for name, blocks, mid, out, osize, first_stride in stages:
        for b in range(blocks):
            bn = "%s%s" % (name, "abcdef"[b])
            s = first_stride if b == 0 else 1
            isz = size if b == 0 else osize
            if b == 0:
                L.append(Layer(bn + "_branch1", cin, isz, isz, out, 1, s, 0))
            if v15:  # 1x1 at the input size, stride-2 3x3 (isz -> osize)
                L.append(Layer(bn + "_branch2a", cin if b == 0 else out, isz, isz, mid, 1, 1, 0))
                L.append(Layer(bn + "_branch2b", mid, isz, isz, mid, 3, s, 1, sparse=True))
            else:
                L.append(Layer(bn + "_branch2a", cin if b == 0 else out, isz, isz, mid, 1, s, 0))
                L.append(Layer(bn + "_branch2b", mid, osize, osize, mid, 3, 1, 1, sparse=True))
            L.append(Layer(bn + "_branch2c", mid, osize, osize, out, 1, 1, 0))
        cin, size = out, osize
    L.append(_fc("fc1000", 2048, 1000))
    return L


def _sparse(l: Layer) -> Layer:
    """The same layer marked as pruned (workloads that benchmark a normally-dense layer group)."""
    return Layer(l.name, l.C, l.H, l.W, l.M, l.K, l.stride, l.pad, l.groups, sparse=True, kind=l.kind)


def conv_layers(layers: List[Layer]) -> List[Layer]:
    return [l for l in layers if l.kind == "conv"]


# ------------------------------------------------------------------ BASELINE configs
TINY = Layer("tiny", 16, 14, 14, 32, 3, 1, 1, 1, sparse=True)


@dataclass(frozen=True)
class Workload:
    name: str
    net: str
    layers: List[Layer] = field(default_factory=list)
    batch: int = 128
    sparsity_permille: int = 800  # ASSUMED 80% (reading R#14)


def workload(name: str) -> Workload:
    """The five BASELINE.json configs."""
    if name == "tiny":
        return Workload("tiny", "tiny", [TINY], batch=1)
    if name == "alexnet":
        return Workload("alexnet", "alexnet", [l for l in alexnet_full() if l.sparse])
    if name == "googlenet":
        return Workload("googlenet", "googlenet", [l for l in googlenet_full() if l.sparse])
    if name == "googlenet_1x1":  # R#19: the 37 1x1 layers benchmarked as their own pruned group
        return Workload("googlenet_1x1", "googlenet",
                        [_sparse(l) for l in googlenet_full() if l.kind == "conv" and l.K == 1])
    if name == "resnet50":
        return Workload("resnet50", "resnet50", [l for l in resnet50_full() if l.sparse])
    if name == "alexnet_convs":  # NEXT-2 whole conv stack: conv1 dense (unpruned) + conv2-5 sparse
        return Workload("alexnet_convs", "alexnet", conv_layers(alexnet_full()))
    if name == "resnet50_convs":  # NEXT-2 whole conv stack: 53 convs, the 16 3x3 sparse, the rest dense
        return Workload("resnet50_convs", "resnet50", conv_layers(resnet50_full()))
    if name == "alexnet_conv1":  # NEXT-3: the 11x11 / stride-4 first layer on the sparse path (80%, R#14)
        return Workload("alexnet_conv1", "alexnet", [_sparse(alexnet_full()[0])])
    if name == "resnet50_v15":  # NEXT-3: three of the 16 sparse 3x3 layers have stride 2
        return Workload("resnet50_v15", "resnet50_v15", [l for l in resnet50_full(v15=True) if l.sparse])
    raise KeyError(name)


SWEEP_DENSITIES_PERMILLE = [50, 100, 150, 200, 300, 400, 500, 600, 700, 800, 900, 1000]


def sweep_layer() -> Layer:
    """C5: AlexNet conv3 shape, density sweep (BASELINE configs[4])."""
    return [l for l in alexnet_full() if l.name == "conv3"][0]
