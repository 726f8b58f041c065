"""Layer descriptors and the five BASELINE.json workloads.

`LayerDesc` mirrors dpgrad::LayerDescriptor (reference layers.hpp:69-194): the same kinds in the
same enum order (layers.hpp:19-30), the same factory arguments and defaults, and the same
parameter order (weight then bias; table) as build_model (layers.hpp:926-973). It packs into the
C struct `dpg_layer_desc` of include/dpg.h.

The model definitions are the ones pinned in SURVEY.md §8(d).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

LINEAR, EMBEDDING, CONV2D, LAYER_NORM, GROUP_NORM, RELU, FLATTEN = range(7)
KIND_NAMES = ["linear", "embedding", "conv2d", "layer_norm", "group_norm", "relu", "flatten"]


class CLayerDesc(ctypes.Structure):
    """dpg_layer_desc (include/dpg.h) == dpgo_layer (oracle/dpg_oracle.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("has_bias", ctypes.c_int32),
        ("in_features", ctypes.c_int64),
        ("out_features", ctypes.c_int64),
        ("vocab_size", ctypes.c_int64),
        ("embedding_dim", ctypes.c_int64),
        ("in_channels", ctypes.c_int64),
        ("out_channels", ctypes.c_int64),
        ("kernel_h", ctypes.c_int64),
        ("kernel_w", ctypes.c_int64),
        ("stride", ctypes.c_int64),
        ("padding", ctypes.c_int64),
        ("norm_size", ctypes.c_int64),
        ("groups", ctypes.c_int64),
        ("eps", ctypes.c_double),
    ]


@dataclass(frozen=True)
class LayerDesc:
    kind: int
    has_bias: bool = True
    in_features: int = 0
    out_features: int = 0
    vocab_size: int = 0
    embedding_dim: int = 0
    in_channels: int = 0
    out_channels: int = 0
    kernel_h: int = 0
    kernel_w: int = 0
    stride: int = 1
    padding: int = 0
    norm_size: int = 0   # layer_norm: normalized numel (1-D shape); group_norm: channels
    groups: int = 0
    eps: float = 1e-5

    # factories: LayerDescriptor::linear / embedding / conv2d / relu / flatten (layers.hpp:96-163)
    @staticmethod
    def linear(i: int, o: int, bias: bool = True) -> "LayerDesc":
        if i <= 0 or o <= 0:
            raise ValueError("linear: feature counts must be positive")
        return LayerDesc(LINEAR, bias, in_features=i, out_features=o)

    @staticmethod
    def embedding(vocab: int, dim: int) -> "LayerDesc":
        if vocab <= 0 or dim <= 0:
            raise ValueError("embedding: extents must be positive")
        return LayerDesc(EMBEDDING, False, vocab_size=vocab, embedding_dim=dim)

    @staticmethod
    def conv2d(ic: int, oc: int, kh: int, kw: int, stride: int = 1, padding: int = 0,
               bias: bool = True) -> "LayerDesc":
        if min(ic, oc, kh, kw, stride) <= 0:
            raise ValueError("conv2d: channel, kernel, and stride extents must be positive")
        return LayerDesc(CONV2D, bias, in_channels=ic, out_channels=oc, kernel_h=kh, kernel_w=kw,
                         stride=stride, padding=padding)

    @staticmethod
    def layer_norm(m: int, eps: float = 1e-5) -> "LayerDesc":
        # LayerDescriptor::layer_norm(Shape{m}, eps) (layers.hpp:128-138), 1-D normalized shape
        if m <= 0:
            raise ValueError("layer_norm: normalized shape must be non-empty")
        if eps <= 0:
            raise ValueError("layer_norm: eps must be positive")
        return LayerDesc(LAYER_NORM, False, norm_size=m, eps=eps)

    @staticmethod
    def group_norm(groups: int, channels: int, eps: float = 1e-5) -> "LayerDesc":
        # LayerDescriptor::group_norm (layers.hpp:140-150)
        if groups <= 0 or channels <= 0 or channels % groups:
            raise ValueError("group_norm: groups must be positive and divide channels")
        if eps <= 0:
            raise ValueError("group_norm: eps must be positive")
        return LayerDesc(GROUP_NORM, False, norm_size=channels, groups=groups, eps=eps)

    @staticmethod
    def relu() -> "LayerDesc":
        return LayerDesc(RELU, False)

    @staticmethod
    def flatten() -> "LayerDesc":
        return LayerDesc(FLATTEN, False)

    def param_shapes(self) -> List[Tuple[str, Tuple[int, ...]]]:
        if self.kind == LINEAR:
            s = [("weight", (self.out_features, self.in_features))]
            if self.has_bias:
                s.append(("bias", (self.out_features,)))
            return s
        if self.kind == EMBEDDING:
            return [("table", (self.vocab_size, self.embedding_dim))]
        if self.kind == CONV2D:
            s = [("weight", (self.out_channels, self.in_channels, self.kernel_h, self.kernel_w))]
            if self.has_bias:
                s.append(("bias", (self.out_channels,)))
            return s
        if self.kind in (LAYER_NORM, GROUP_NORM):  # build_model: gamma = 1, beta = 0
            return [("gamma", (self.norm_size,)), ("beta", (self.norm_size,))]
        return []

    def to_c(self) -> CLayerDesc:
        return CLayerDesc(self.kind, int(self.has_bias), self.in_features, self.out_features,
                          self.vocab_size, self.embedding_dim, self.in_channels, self.out_channels,
                          self.kernel_h, self.kernel_w, self.stride, self.padding, self.norm_size,
                          self.groups, self.eps)


def c_layers(layers: Sequence[LayerDesc]):
    arr = (CLayerDesc * len(layers))()
    for i, l in enumerate(layers):
        arr[i] = l.to_c()
    return arr


def params_meta(layers: Sequence[LayerDesc]):
    """[(layer index, slot, name, shape, numel, offset)] in (l, k) order."""
    out, off = [], 0
    for li, l in enumerate(layers):
        for k, (name, shape) in enumerate(l.param_shapes()):
            n = 1
            for e in shape:
                n *= e
            out.append((li, k, name, shape, n, off))
            off += n
    return out


def param_count(layers: Sequence[LayerDesc]) -> int:
    return sum(m[4] for m in params_meta(layers))


@dataclass(frozen=True)
class Workload:
    name: str
    layers: Tuple[LayerDesc, ...]
    in_shape: Tuple[int, ...]          # per-sample input shape
    batch: int
    classes: int
    tokens: int = 0                    # embedding models: vocab for synthetic ids
    description: str = ""
    extra: dict = field(default_factory=dict)


L = LayerDesc

MNIST_LAYERS = (L.conv2d(1, 16, 8, 8, 2, 0), L.relu(), L.conv2d(16, 32, 4, 4, 2, 0), L.relu(),
                L.flatten(), L.linear(512, 32), L.relu(), L.linear(32, 10))
CIFAR_LAYERS = (L.conv2d(3, 32, 3, 3, 2, 1), L.relu(), L.conv2d(32, 64, 3, 3, 2, 1), L.relu(),
                L.conv2d(64, 64, 3, 3, 2, 1), L.relu(), L.conv2d(64, 128, 3, 3, 2, 1), L.relu(),
                L.flatten(), L.linear(512, 10))
EMBED_LAYERS = (L.embedding(10000, 128), L.flatten(), L.linear(32768, 2))

WORKLOADS = {
    "mnist_b64": Workload("mnist_b64", MNIST_LAYERS, (1, 28, 28), 64, 10,
                          description="MNIST 2-conv + 2-linear CNN, one DP-SGD step, batch 64"),
    "cifar_b512": Workload("cifar_b512", CIFAR_LAYERS, (3, 32, 32), 512, 10,
                           description="CIFAR-10 4-layer CNN, batch 512, full DP-SGD step"),
    "embed_b512": Workload("embed_b512", EMBED_LAYERS, (256,), 512, 2, tokens=10000,
                           description="Embedding 10000x128 + Linear, T=256, batch 512"),
    "cifar_b4096": Workload("cifar_b4096", CIFAR_LAYERS, (3, 32, 32), 4096, 10,
                            description="CIFAR-10 CNN, batch 4096, sharded by sample"),
}
# cfg2 is a single-layer harness, not a model: per_sample_rule_linear on A,B [256, 64, 512]
LINEAR_T64 = dict(b=256, t=64, d=512, r=512)

assert param_count(MNIST_LAYERS) == 26010
assert param_count(CIFAR_LAYERS) == 135306
assert param_count(EMBED_LAYERS) == 1345538
