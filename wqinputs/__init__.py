"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests,
smoke() and bench.py.

This module holds NONE of the method's arithmetic (no B-spline evaluation, no
quadrature, no weights, no coefficients): only knot vectors, Greville
abscissae (an input-construction convention, not part of WQ) and seeded
control nets, as recorded in DESIGN.md "Input recipe".  Geometry readings:
R9 (noise scaled by local Greville spacing) and R10 (quarter annulus).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def uniform_open_knots(p: int, n_el: int) -> np.ndarray:
    """[0]*(p+1) ++ [k/n_el, k=1..n_el-1] ++ [1]*(p+1), each k/n_el as double."""
    inner = [float(k) / float(n_el) for k in range(1, n_el)]
    return np.array([0.0] * (p + 1) + inner + [1.0] * (p + 1), dtype=np.float64)


def graded_open_knots(p: int, n_el: int, ratio: float = 1.08) -> np.ndarray:
    """Open knots on [0,1] with geometrically graded spans (NEXT f1 config)."""
    h = np.array([ratio ** k for k in range(n_el)], dtype=np.float64)
    x = np.concatenate([[0.0], np.cumsum(h)])
    x = x / x[-1]
    x[-1] = 1.0
    return np.concatenate([[0.0] * p, x, [1.0] * p]).astype(np.float64)


def greville(p: int, knots: np.ndarray) -> np.ndarray:
    """gamma_k = (xi_{k+1} + ... + xi_{k+p}) / p, summed left to right."""
    n = knots.size - p - 1
    g = np.empty(n)
    for k in range(n):
        s = 0.0
        for t in range(1, p + 1):
            s += float(knots[k + t])
        g[k] = s / p
    return g


def _local_spacing(g: np.ndarray) -> np.ndarray:
    """sigma(k) = min(gamma_k - gamma_{k-1}, gamma_{k+1} - gamma_k), one-sided at ends."""
    d = np.diff(g)
    s = np.empty_like(g)
    s[0] = d[0]
    s[-1] = d[-1]
    s[1:-1] = np.minimum(d[:-1], d[1:])
    return s


def _tensor(arrs):
    """Tensor grid of per-direction arrays, first direction fastest -> (N, d)."""
    mesh = np.meshgrid(*arrs, indexing="ij")
    return np.stack([m.reshape(-1, order="F") for m in mesh], axis=1)


def control_net(kind: str, p: int, knots, amp: float, seed: int = 0) -> np.ndarray:
    """Control points [N_DOF][d], row = linear index with k_1 fastest.

    kind = "grid":    Greville grid + amp * s_k * U(-1,1) noise (reading R9)
    kind = "annulus": Greville samples of the quarter annulus r in [1,2], extruded
                      z in [0,1] (reading R10), + amp * s_k * U(-1,1) noise
    kind = "affine:<a00,a01,...>": exact affine image of the Greville grid
    """
    d = len(knots)
    gs = [greville(p, k) for k in knots]
    G = _tensor(gs)
    if kind == "grid":
        P = G.copy()
    elif kind == "annulus":
        assert d in (2, 3)
        r = 1.0 + G[:, 0]
        th = 0.5 * math.pi * G[:, 1]
        cols = [r * np.cos(th), r * np.sin(th)]
        if d == 3:
            cols.append(G[:, 2])
        P = np.stack(cols, axis=1)
    elif kind.startswith("affine:"):
        a = np.array([float(v) for v in kind.split(":", 1)[1].split(",")]).reshape(d, d)
        P = G @ a.T
        return np.ascontiguousarray(P)
    else:
        raise ValueError(kind)
    if amp:
        sig = [_local_spacing(g) for g in gs]
        S = _tensor(sig).min(axis=1)
        rng = np.random.default_rng(seed)
        U = rng.uniform(-1.0, 1.0, size=(G.shape[0], d))
        P = P + amp * S[:, None] * U
    return np.ascontiguousarray(P, dtype=np.float64)


@dataclass
class Config:
    name: str
    d: int
    p: int
    n_el: int
    geometry: str
    amp: float
    matrices: tuple = ("stiffness", "mass")
    seed: int = 0
    knots_kind: str = "uniform"
    _cache: dict = field(default_factory=dict, repr=False)

    def knots(self):
        if self.knots_kind == "uniform":
            k = uniform_open_knots(self.p, self.n_el)
        else:
            k = graded_open_knots(self.p, self.n_el)
        return [k.copy() for _ in range(self.d)]

    def ctrl(self):
        key = "ctrl"
        if key not in self._cache:
            self._cache[key] = control_net(self.geometry, self.p, self.knots(), self.amp, self.seed)
        return self._cache[key]

    @property
    def n_dof(self):
        return (self.n_el + self.p) ** self.d

    def exact_nnz(self):
        n = self.n_el + self.p
        per = (2 * self.p + 1) * n - self.p * (self.p + 1)
        return per ** self.d


# BASELINE.json configs; C4 is a degree sweep.
def baseline_config(name: str, p: int | None = None) -> Config:
    if name == "C1":
        return Config("C1", 2, 3, 16, "grid", 0.1, ("stiffness", "mass"))
    if name == "C2":
        return Config("C2", 3, 3, 32, "grid", 0.1, ("stiffness", "mass"))
    if name == "C3":
        return Config("C3", 3, 6, 64, "annulus", 0.05, ("stiffness",))
    if name == "C4":
        return Config(f"C4p{p}", 3, int(p), 100, "grid", 0.1, ("stiffness",))
    if name == "C5":
        return Config("C5", 3, 4, 256, "annulus", 0.05, ("stiffness",))
    raise ValueError(name)


C4_DEGREES = (2, 3, 4, 6, 8, 10)
