"""Seeded generators (SURVEY.md §8(d) "Values and seeds").

* parameter matrix (m x n): Q0 + 0.1 * G / sqrt(max(m, n)), Q0 the sign-fixed
  QR factor of a seeded Gaussian (near-orthogonal default, reading R21);
  ``stress=True`` gives G / sqrt(n) (Gaussian stress set, run with T = 30);
* power-iteration start vectors: seeded unit Gaussians;
* activations N(0, 1); bias N(0, 0.01) for parity tests.

Seeds are ``np.random.SeedSequence([cfg, layer, group, matrix, role])``.
Everything is drawn in float64 and rounded once to float32 (RNE); consumers
that need the exact values the GPU sees use the float32 arrays.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

ROLE_ID = {"Q": 1, "U": 2, "R": 3, "W": 4, "v": 5, "x": 6, "b": 7, "K": 8}


def rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) for k in key])))


def param_matrix(m: int, n: int, key: Sequence[int], stress: bool = False) -> np.ndarray:
    """float32 m x n parameter matrix for seed key (cfg, layer, group, matrix, role)."""
    if m == 0 or n == 0:
        return np.zeros((m, n), np.float32)
    r = rng(*key)
    G = r.standard_normal((m, n))
    if stress:
        return (G / np.sqrt(n)).astype(np.float32)
    A = r.standard_normal((max(m, n), min(m, n)))
    Q, Rr = np.linalg.qr(A)
    Q = Q * np.sign(np.diag(Rr))[None, :]          # sign fix -> unique factor
    Q0 = Q if m >= n else Q.T
    return (Q0 + 0.1 * G / np.sqrt(max(m, n))).astype(np.float32)


def param_matrix_torch(m: int, n: int, key: Sequence[int], torch, device, stress: bool = False):
    """Same recipe as param_matrix with the Gaussian drawn by a seeded torch
    generator and the QR on `device` (large dense-sweep matrices only; not
    bit-identical to the NumPy draw)."""
    seed = int(np.random.SeedSequence([int(k) for k in key]).generate_state(1)[0])
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    G = torch.randn((m, n), generator=g, device=device, dtype=torch.float64)
    if stress:
        return (G / np.sqrt(n)).float()
    A = torch.randn((max(m, n), min(m, n)), generator=g, device=device, dtype=torch.float64)
    Q, R = torch.linalg.qr(A)
    Q = Q * torch.sign(torch.diagonal(R))[None, :]
    Q0 = Q if m >= n else Q.T
    return (Q0 + 0.1 * G / np.sqrt(max(m, n))).float()


def unit_vector(n: int, key: Sequence[int]) -> np.ndarray:
    if n == 0:
        return np.zeros(0, np.float32)
    v = rng(*key).standard_normal(n)
    return (v / np.linalg.norm(v)).astype(np.float32)


def activations(shape, key: Sequence[int]) -> np.ndarray:
    """N(0,1) float32 array of the given shape (NCHW or NHWC is the caller's)."""
    return rng(*key).standard_normal(shape).astype(np.float32)


def bias(n: int, key: Sequence[int]) -> np.ndarray:
    return (0.01 * rng(*key).standard_normal(n)).astype(np.float32)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 -> bfloat16 (RNE) and back to float32 (input casting only)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)
