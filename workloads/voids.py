"""Seeded void (spherical / circular hole) sampling -- reading R12 of DESIGN.md.

Per candidate draw: centre c ~ U[lo, hi]^d, then radius r ~ U[r_min, r_max];
accept iff ||c - c_j|| > r + r_j for every accepted void j; stop when `count`
voids are accepted.  RNG: numpy.random.default_rng(seed) (PCG64).
No method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np


def sample_voids(count: int, r_min: float, r_max: float, seed: int, dim: int = 3,
                 lo: float = 0.15, hi: float = 0.85, max_draws: int = 1_000_000):
    """Return (centres [count,dim] float64, radii [count] float64, draws int)."""
    rng = np.random.default_rng(seed)
    centres = np.zeros((count, dim))
    radii = np.zeros(count)
    k = 0
    draws = 0
    while k < count:
        if draws >= max_draws:
            raise RuntimeError("void sampling did not converge")
        c = rng.uniform(lo, hi, dim)
        r = rng.uniform(r_min, r_max)
        draws += 1
        if k:
            d = np.sqrt(((centres[:k] - c) ** 2).sum(axis=1))
            if np.any(d <= r + radii[:k]):
                continue
        centres[k] = c
        radii[k] = r
        k += 1
    return centres, radii, draws


def config_voids(cfg):
    """Voids of a workload config (see configs.py)."""
    g = cfg.geometry
    if g["kind"] == "explicit":
        return (np.asarray(g["centres"], dtype=np.float64).reshape(-1, cfg.dim),
                np.asarray(g["radii"], dtype=np.float64).reshape(-1))
    if g["kind"] == "none":
        return np.zeros((0, cfg.dim)), np.zeros(0)
    c, r, _ = sample_voids(g["count"], g["r_min"], g["r_max"], g["seed"], cfg.dim)
    return c, r
