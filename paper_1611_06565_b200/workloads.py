"""Seeded synthetic workloads (BASELINE.json `configs`) -- inputs only.

This module holds no arithmetic of the method: it only describes layer
shapes and draws the seeded inputs that both the CUDA path and the oracle are
fed (by the tests and bench.py).  Recipe (reading #12):
one ``torch.Generator('cpu').manual_seed(seed)`` per config, x drawn first,
then g, both fp32, in the distributions BASELINE.json names.  The paper's
workloads (ImageNet 2-D images, C3D video volumes)
are not available here; these shapes stand in for them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Tuple

import torch


@dataclass(frozen=True)
class LayerConfig:
    name: str
    N: int
    batch: int
    C: int
    K: int
    dims: Tuple[int, ...]
    r: int
    pad: int
    m: int
    xdist: str          # "uniform" | "normal" | "relu_normal"
    gdist: str          # "uniform" | "he"  (N(0, 2/(C r^N)))
    desc: str = ""

    @property
    def out_dims(self):
        return tuple(d + 2 * self.pad - self.r + 1 for d in self.dims)

    @property
    def padding(self):
        return (self.pad,) * self.N

    @property
    def alpha(self):
        return self.m + self.r - 1

    def direct_flops(self, batch=None) -> int:
        """Direct-convolution-equivalent flops 2 B K C prod(out) r^N (BASELINE metric)."""
        b = self.batch if batch is None else batch
        return 2 * b * self.K * self.C * math.prod(self.out_dims) * self.r ** self.N

    def winograd_gemm_flops(self, batch=None) -> int:
        """Algorithmic flops of stage a3: 2 alpha^N T C K."""
        b = self.batch if batch is None else batch
        T = b * math.prod(-(-o // self.m) for o in self.out_dims)
        return 2 * self.alpha ** self.N * T * self.C * self.K

    def tiles(self, batch=None) -> int:
        b = self.batch if batch is None else batch
        return b * math.prod(-(-o // self.m) for o in self.out_dims)

    def with_batch(self, b):
        return replace(self, batch=b)


CONFIGS = {
    "c1": LayerConfig("c1", 2, 1, 4, 4, (8, 8), 3, 0, 2, "uniform", "uniform",
                      "2D 8x8, 4->4, F(2x2,3x3), valid"),
    "c2": LayerConfig("c2", 2, 32, 128, 128, (56, 56), 3, 1, 4, "normal", "he",
                      "2D VGG-style 56x56, 32x128->128, F(4x4,3x3)"),
    "c3": LayerConfig("c3", 3, 16, 64, 128, (16, 56, 56), 3, 1, 2, "normal", "he",
                      "3D video 16x56x56, 16x64->128, F(2^3,3^3)"),
    "c4": LayerConfig("c4", 3, 32, 256, 256, (8, 28, 28), 3, 1, 4, "relu_normal", "he",
                      "3D volumetric 8x28x28, 32x256->256, F(4^3,3^3)"),
    "c5": LayerConfig("c5", 4, 8, 32, 32, (8, 8, 16, 16), 3, 1, 2, "normal", "he",
                      "4D 8x8x16x16, 8x32->32, F(2^4,3^4)"),
}

# Shrunken parity cases: same N, m, r, padding and distributions; ragged
# spatial extents (partial edge tiles), T spanning several 128-row GEMM
# blocks with a partial last block, C / K not multiples of the tile widths.
SMALL = {
    "c1": CONFIGS["c1"],
    "c2": LayerConfig("c2s", 2, 3, 24, 40, (29, 23), 3, 1, 4, "normal", "he"),
    "c3": LayerConfig("c3s", 3, 2, 16, 48, (5, 13, 11), 3, 1, 2, "normal", "he"),
    "c4": LayerConfig("c4s", 3, 6, 40, 72, (6, 13, 10), 3, 1, 4, "relu_normal", "he"),
    "c5": LayerConfig("c5s", 4, 4, 8, 12, (3, 4, 5, 6), 3, 1, 2, "normal", "he"),
}


def make_inputs(cfg: LayerConfig, seed: int = 0, batch: int = None):
    """(x [B][C][dims], g [K][C][r^N]) as CPU float32 tensors, x drawn first."""
    B = cfg.batch if batch is None else batch
    gen = torch.Generator("cpu").manual_seed(seed)
    xs = (B, cfg.C) + tuple(cfg.dims)
    if cfg.xdist == "uniform":
        x = torch.rand(xs, generator=gen, dtype=torch.float32) * 2 - 1
    elif cfg.xdist == "normal":
        x = torch.randn(xs, generator=gen, dtype=torch.float32)
    elif cfg.xdist == "relu_normal":
        x = torch.randn(xs, generator=gen, dtype=torch.float32).clamp_min_(0)
    else:
        raise ValueError(cfg.xdist)
    gs = (cfg.K, cfg.C) + (cfg.r,) * cfg.N
    if cfg.gdist == "uniform":
        g = torch.rand(gs, generator=gen, dtype=torch.float32) * 2 - 1
    elif cfg.gdist == "he":
        g = torch.randn(gs, generator=gen, dtype=torch.float32) * math.sqrt(2.0 / (cfg.C * cfg.r ** cfg.N))
    else:
        raise ValueError(cfg.gdist)
    return x.contiguous(), g.contiguous()


def tolerance(cfg: LayerConfig):
    """(relL2, max-abs / max|y|) bounds of BASELINE.json north_star."""
    return (2e-6, 1e-4) if cfg.m == 2 else (1e-5, 1e-3)


# ---------------------------------------------------------------- paper nets
# The paper's own 2-D measurements (DESIGN.md reading
# #16): Figure 4 propagates 224x224 images through three convolution layers of
# 32 channels and 32 kernels of size 4x4, at batch 1, 20 and
# 200, reported in megavoxels per second; Figure 3 is one 4x4 layer on a
# 1024x1024 image.  Unstated and read here: valid convolution
# (no padding), C = K = 32 for every layer including Figure 3's, x ~ N(0, 1),
# g ~ N(0, 2 / (C r^2)).  Transforms: F(5, 4) (Table 1 (c), D = 8, the paper's
# choice for 4x4 kernels) and F(3, 4) (D = 6).
@dataclass(frozen=True)
class NetConfig:
    name: str
    layers: Tuple[LayerConfig, ...]
    batches: Tuple[int, ...]
    desc: str = ""

    @property
    def in_voxels(self) -> int:
        """Input voxels of one sample (the MVox/s numerator, reading #16)."""
        return math.prod(self.layers[0].dims)

    def direct_flops(self, batch: int) -> int:
        return sum(l.direct_flops(batch) for l in self.layers)


def _chain(name, dims, depth, C, r, m, batches, desc):
    layers = []
    for i in range(depth):
        layers.append(LayerConfig("%s_l%d" % (name, i + 1), len(dims), batches[0], C, C, tuple(dims), r, 0, m,
                                  "normal", "he"))
        dims = [d - r + 1 for d in dims]
    return NetConfig(name, tuple(layers), tuple(batches), desc)


NETS = {
    "fig4_f54": _chain("fig4_f54", [224, 224], 3, 32, 4, 5, (1, 20, 200),
                       "Figure 4: 224x224 through 3 layers 32->32, 4x4 kernels, F(5x5,4x4) (D=8)"),
    "fig4_f34": _chain("fig4_f34", [224, 224], 3, 32, 4, 3, (1, 20, 200),
                       "Figure 4: 224x224 through 3 layers 32->32, 4x4 kernels, F(3x3,4x4) (D=6)"),
    "fig3_f54": _chain("fig3_f54", [1024, 1024], 1, 32, 4, 5, (1,),
                       "Figure 3: one 4x4 layer on a 1024x1024 image, 32->32, F(5x5,4x4) (D=8)"),
}


def make_net_inputs(net: NetConfig, seed: int = 0, batch: int = 1):
    """(x [B][C][dims], [g_1 .. g_L]) as CPU float32 tensors: x first, then
    each layer's kernels in order, from one seeded generator."""
    gen = torch.Generator("cpu").manual_seed(seed)
    l0 = net.layers[0]
    x = torch.randn((batch, l0.C) + tuple(l0.dims), generator=gen, dtype=torch.float32)
    gs = []
    for l in net.layers:
        gs.append((torch.randn((l.K, l.C) + (l.r,) * l.N, generator=gen, dtype=torch.float32)
                   * math.sqrt(2.0 / (l.C * l.r ** l.N))).contiguous())
    return x.contiguous(), gs
