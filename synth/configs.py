"""Workload shapes of BASELINE.json configs 1-5 ("Concrete
synthetic inputs").  The paper prints no architectures; these are the survey's
synthetic choices shaped like its CIFAR / ImageNet use.

A layer is a plain dict:
  kind: 'conv' | 'convT' | 'dense';  c_in, c_out, k, s, d, g;
  padding_mode: 'circular' | 'zeros';  H: input spatial size of the layer's
  forward call (for 'convT', the SMALL input size; the output is H*s).
"""
from __future__ import annotations

from typing import Dict, List


def _L(c_in, c_out, H, k=3, s=1, d=1, g=1, kind="conv", mode="circular"):
    return dict(kind=kind, c_in=c_in, c_out=c_out, k=k, s=s, d=d, g=g,
                padding_mode=mode, H=H)


def cfg1() -> List[Dict]:
    """Config 1: one 3x3 orthogonal conv 16->16, stride 1, x (2,16,8,8)."""
    return [_L(16, 16, 8)]


def cfg2() -> List[Dict]:
    """Config 2 "CIFAR-AOC-12": stem 3->64 @32; 2x 64 @32; down 64->128 s2;
    2x 128 @16; down 128->256 s2; 2x 256 @8; down 256->512 s2; 2x 512 @4.
    All 3x3 circular, chained, batch 256."""
    L = [_L(3, 64, 32), _L(64, 64, 32), _L(64, 64, 32),
         _L(64, 128, 32, s=2), _L(128, 128, 16), _L(128, 128, 16),
         _L(128, 256, 16, s=2), _L(256, 256, 8), _L(256, 256, 8),
         _L(256, 512, 8, s=2), _L(512, 512, 4), _L(512, 512, 4)]
    return L


def cfg3() -> List[Dict]:
    """Config 3 "ImageNet AOC-ResNet34-shape": stem RKO 4x4 s4 3->64 (224->56);
    widths 64/128/256/512 at 56/28/14/7 with 6/8/12/6 3x3 convs, the first conv
    of stages 2-4 is 3x3 s2 c->2c.  33 layers, batch 256."""
    L = [_L(3, 64, 224, k=4, s=4)]
    L += [_L(64, 64, 56) for _ in range(6)]
    H = 56
    for c, n in ((128, 8), (256, 12), (512, 6)):
        L.append(_L(c // 2, c, H, s=2))
        H //= 2
        L += [_L(c, c, H) for _ in range(n - 1)]
    return L


def cfg4() -> List[Dict]:
    """Config 4 "1024-ch paths @56": (a) g=32; (b) d=2; (c) s=2 (56->28);
    (d) transposed s=2 (small 56 -> big 112); (e) transposed g=32 d=2 s=1.
    Each layer is fed independently (not chained)."""
    return [_L(1024, 1024, 56, g=32), _L(1024, 1024, 56, d=2),
            _L(1024, 1024, 56, s=2), _L(1024, 1024, 56, s=2, kind="convT"),
            _L(1024, 1024, 56, g=32, d=2, kind="convT")]


def cfg5(n: int) -> List[Dict]:
    """Config 5: 64 dense n x n matrices (OrthoLinear weights)."""
    return [_L(n, n, 0, k=1, kind="dense") for _ in range(64)]


CONFIGS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4}
BATCH = {1: 2, 2: 256, 3: 256, 4: 256}
CHAIN = {1: True, 2: True, 3: True, 4: False}
NAMES = {1: "config 1: one 3x3 16->16 circular layer",
         2: "config 2: CIFAR-AOC-12 (12 orthogonal 3x3 convs 64-512 ch, 3 stride-2), 32x32",
         3: "config 3: ImageNet AOC-ResNet34-shape (33 orthogonal convs, RKO 4x4 s4 stem), 224x224",
         4: "config 4: 1024-ch paths at 56x56 (g32, d2, s2, transposed s2, transposed g32 d2)"}
