"""Seeded synthetic stand-ins for the five BASELINE.json configs (c0..c4).

The reference's datasets (Spellman, GSE25219, ...) are not in this image, so
each config is generated from numpy PCG64 with seed 42 + config id, with the
shapes, sizes and value distributions BASELINE.json states.  Every
generator returns variable-major float64 arrays (variable v contiguous), the
layout of the reference's Dataset.values columns (analysis.hpp:16-22).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    call: str                 # "pairs" | "pairwise" | "cross"
    alpha: float
    c: float
    est: int                  # 0 = MIC_approx, 1 = MIC_e
    X: np.ndarray             # variables (pairwise/pairs) or the X set (cross)
    Y: np.ndarray | None = None
    xi: np.ndarray | None = None   # pair list for call == "pairs"
    yi: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.X.shape[1])

    @property
    def npairs(self) -> int:
        if self.call == "pairs":
            return int(self.xi.size)
        if self.call == "pairwise":
            p = self.X.shape[0]
            return p * (p - 1) // 2
        return int(self.X.shape[0] * self.Y.shape[0])


def _rng(cfg: int, seed: int | None) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(42 + cfg if seed is None else seed))


_FUNCS = [
    lambda x: 2.0 * x - 1.0,
    lambda x: 4.0 * (x - 0.5) ** 2,
    lambda x: np.sin(4.0 * np.pi * x),
    lambda x: 2.0 ** (10.0 * x) / 1024.0,
]


def config0(npairs: int = 256, n: int = 1000, seed: int | None = None) -> Workload:
    """256 independent pairs, n=1000: y = f(x) + N(0, s^2); f cycles over four
    functions plus an independent U[0,1) draw, s over {0, .1, .3, 1}."""
    g = _rng(0, seed)
    sig = [0.0, 0.1, 0.3, 1.0]
    X = np.empty((2 * npairs, n))
    for i in range(npairs):
        x = g.random(n)
        fi = i % 5
        base = g.random(n) if fi == 4 else _FUNCS[fi](x)
        y = base + g.normal(0.0, 1.0, n) * sig[i % 4]
        X[2 * i], X[2 * i + 1] = x, y
    xi = np.arange(0, 2 * npairs, 2, dtype=np.int32)
    return Workload("c0", "pairs", 0.6, 15.0, 0, X, xi=xi, yi=xi + 1,
                    meta=dict(npairs=npairs, n=n))


def config1(p: int = 4381, n: int = 23, seed: int | None = None) -> Workload:
    """4381 x 23 all-pairs (Spellman shape): 70% iid N(0,1); 30% +-L_m(t) +
    N(0, .3^2) over 20 shared latent courses (sine, period U[5,23], phase
    U[0,2pi), w.p. 0.8; else the ramp 2t/22 - 1)."""
    g = _rng(1, seed)
    t = np.arange(n, dtype=np.float64)
    lat = np.empty((20, n))
    for m in range(20):
        if g.random() < 0.8:
            lat[m] = np.sin(2 * np.pi * t / g.uniform(5, 23) + g.uniform(0, 2 * np.pi))
        else:
            lat[m] = 2 * t / max(n - 1, 1) - 1
    X = g.normal(0.0, 1.0, (p, n))
    driven = g.random(p) < 0.3
    ms = g.integers(0, 20, p)
    sign = np.where(g.random(p) < 0.5, -1.0, 1.0)
    noise = g.normal(0.0, 0.3, (p, n))
    X[driven] = sign[driven, None] * lat[ms[driven]] + noise[driven]
    return Workload("c1", "pairwise", 0.6, 15.0, 0, X, meta=dict(p=p, n=n))


def config2(p: int = 2000, n: int = 500, seed: int | None = None) -> Workload:
    """2000 x 500 Poisson counts as float64; lambda log-uniform [0.1, 50]; half
    the variables coupled to a shared latent through lambda * exp(0.8 z)."""
    g = _rng(2, seed)
    lam = np.exp(g.uniform(np.log(0.1), np.log(50.0), p))
    z = g.normal(0.0, 1.0, n)
    coupled = np.arange(p) % 2 == 0
    rate = np.repeat(lam[:, None], n, axis=1)
    rate[coupled] *= np.exp(0.8 * z)[None, :]
    X = g.poisson(rate).astype(np.float64)
    return Workload("c2", "pairwise", 0.6, 15.0, 1, X, meta=dict(p=p, n=n))


def config3(p: int = 1000, n: int = 1340, seed: int | None = None) -> Workload:
    """1000 x 1340 Gaussian, rank-10 structure X = L F + E; a random 5% of the
    variables through exp / cube / tanh (monotone: M is rank-invariant)."""
    g = _rng(3, seed)
    L = g.normal(0.0, 1.0, (p, 10))
    F = g.normal(0.0, 1.0, (10, n))
    X = L @ F + g.normal(0.0, 1.0, (p, n))
    pick = g.choice(p, max(1, p // 20), replace=False)
    for k, v in enumerate(pick):
        X[v] = [np.exp, lambda a: a ** 3, np.tanh][k % 3](X[v] / 4.0)
    return Workload("c3", "pairwise", 0.6, 15.0, 0, X, meta=dict(p=p, n=n, transformed=pick.tolist()))


def config4(px: int = 64, py: int = 64, n: int = 10000, seed: int | None = None) -> Workload:
    """64 x 64 cross, n=10000, alpha=.75 (B=1000): shared u ~ U[0,1);
    X_i = u + N(0,.01^2); Y_j = f_{j mod 4}(u) + N(0, s_j^2), s_j in {.05,.5};
    a random 6 of the Y_j replaced by independent U[0,1) (~10% of pairs)."""
    g = _rng(4, seed)
    u = g.random(n)
    X = u[None, :] + g.normal(0.0, 0.01, (px, n))
    Y = np.empty((py, n))
    for j in range(py):
        Y[j] = _FUNCS[j % 4](u) + g.normal(0.0, [0.05, 0.5][j % 2], n)
    for j in g.choice(py, min(py, max(1, round(0.1 * py))), replace=False):
        Y[j] = g.random(n)
    return Workload("c4", "cross", 0.75, 15.0, 1, X, Y=Y, meta=dict(px=px, py=py, n=n))


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def make(cfg: int, **kw) -> Workload:
    return CONFIGS[cfg](**kw)
