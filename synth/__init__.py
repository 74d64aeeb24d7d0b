"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds NONE of the method's arithmetic: it only draws random numbers with the
shapes and value distributions of the paper's workload (CIFAR-10-shaped
images; "pixel/255"; init N(0, 0.01^2), zero biases).
Both sides receive exactly the same fp32 values (the oracle widens them to
fp64), so any difference is the path's own arithmetic.

Recipe:
  images  : uint8 i.i.d. uniform {0..255} / 255, shape [B,3,H,W], PCG64(1000 + step)
  labels  : uniform {0..9}, int32, same generator
  weights : N(0, 0.01^2) fp32 per conv layer (KCRS) and FC ([O, F] NCHW flatten), PCG64(seed)
  biases  : zero unless bias_std > 0 (tests exercise the bias path)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PAPER_NETS = {  # conv1:conv2 kernel counts of the four §5.2 architectures
    "50:500": (50, 500),
    "150:800": (150, 800),
    "300:1000": (300, 1000),
    "500:1500": (500, 1500),
}


@dataclass
class NetSpec:
    """A §5.2-shaped network: conv(5x5)+bias+ReLU+pool per layer, then FC + softmax."""
    in_c: int = 3
    in_hw: int = 32
    kernels: tuple = (500, 1500)
    k: int = 5
    classes: int = 10
    relu: bool = True
    pool: bool = True
    name: str = "paper-500:1500"

    def shapes(self):
        """Per conv layer: (C_in, H_in, K, H_out_conv, H_out_pool)."""
        out = []
        c, h = self.in_c, self.in_hw
        for K in self.kernels:
            ho = h - self.k + 1
            hp = ho // 2 if self.pool else ho
            out.append((c, h, K, ho, hp))
            c, h = K, hp
        return out

    @property
    def fc_in(self):
        c, _, K, _, hp = self.shapes()[-1]
        return K * hp * hp

    def layers(self):
        return [{"relu": self.relu, "pool": self.pool} for _ in self.kernels]


def paper_net(name="500:1500", in_hw=32):
    k1, k2 = PAPER_NETS[name]
    return NetSpec(kernels=(k1, k2), in_hw=in_hw, name=f"paper-{name}")


def tiny_net():
    """BASELINE config 0: 1 conv layer, 8 kernels on 32x32x3."""
    return NetSpec(kernels=(8,), name="tiny-8")


def scaled_net():
    """BASELINE config 4: 224x224x3 input, 512/2048 kernels."""
    return NetSpec(kernels=(512, 2048), in_hw=224, name="scaled-512:2048")


def images(B, C=3, H=32, W=32, step=0):
    g = np.random.Generator(np.random.PCG64(1000 + step))
    px = g.integers(0, 256, size=(B, C, H, W), dtype=np.int64)
    y = g.integers(0, 10, size=(B,), dtype=np.int64).astype(np.int32)
    return (px.astype(np.float32) / np.float32(255.0)), y


def params(net: NetSpec, seed=42, std=0.01, bias_std=0.0):
    """fp32 parameters, NCHW/KCRS conventions: w{i} [K,C,k,k], b{i} [K], wfc [O,F], bfc [O]."""
    g = np.random.Generator(np.random.PCG64(seed))
    p = {}
    for i, (c, _, K, _, _) in enumerate(net.shapes()):
        p[f"w{i}"] = (g.standard_normal((K, c, net.k, net.k)) * std).astype(np.float32)
        p[f"b{i}"] = (g.standard_normal(K) * bias_std).astype(np.float32) if bias_std > 0 \
            else np.zeros(K, np.float32)
    p["wfc"] = (g.standard_normal((net.classes, net.fc_in)) * std).astype(np.float32)
    p["bfc"] = (g.standard_normal(net.classes) * bias_std).astype(np.float32) if bias_std > 0 \
        else np.zeros(net.classes, np.float32)
    return p


def normal(shape, seed, std=1.0, dtype=np.float32):
    g = np.random.Generator(np.random.PCG64(seed))
    return (g.standard_normal(shape) * std).astype(dtype)


def uniform(shape, seed, lo=0.0, hi=1.0, dtype=np.float32):
    g = np.random.Generator(np.random.PCG64(seed))
    return g.uniform(lo, hi, size=shape).astype(dtype)
