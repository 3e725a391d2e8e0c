"""Exact classification against spherical voids (oracle).  TEST INFRASTRUCTURE ONLY.

PAPER.md:55: the indicator alpha(x) is 1 in Omega_phys and epsilon in
Omega_fict.  Here Omega_fict is the union of the open balls ||x - c_j|| < r_j
(reading R14: a point exactly on a sphere is physical).

A box is
  'fict' iff it lies inside one open ball  (its farthest point is inside),
  'phys' iff it misses every open ball    (its nearest point is at distance >= r),
  'cut'  otherwise.
(Voids are pairwise separated, ||c_i - c_j|| > r_i + r_j, so a connected box
inside the union lies inside a single ball.)
"""
from __future__ import annotations

import numpy as np

PHYS, FICT, CUT = 0, 1, 2


def point_is_fictitious(pts, centres, radii):
    pts = np.atleast_2d(pts)
    if len(radii) == 0:
        return np.zeros(len(pts), dtype=bool)
    d2 = ((pts[:, None, :] - centres[None, :, :]) ** 2).sum(axis=2)
    return np.any(d2 < radii[None, :] ** 2, axis=1)


def classify_box(lo, hi, centres, radii):
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    if len(radii) == 0:
        return PHYS
    far2 = np.maximum((lo - centres) ** 2, (hi - centres) ** 2).sum(axis=1)
    if np.any(far2 < radii ** 2):
        return FICT
    near = np.maximum(np.maximum(lo - centres, centres - hi), 0.0)
    near2 = (near ** 2).sum(axis=1)
    if np.all(near2 >= radii ** 2):
        return PHYS
    return CUT


def classify_cells(dim, n, centres, radii):
    """Kind of every cell, cell index c = (cz*n + cy)*n + cx (x fastest)."""
    h = 1.0 / n
    ncell = n ** dim
    idx = np.array(cell_coords(np.arange(ncell), dim, n), dtype=np.float64).T  # [ncell, dim]
    lo = idx * h
    hi = lo + h
    inside_one = np.zeros(ncell, dtype=bool)
    misses_all = np.ones(ncell, dtype=bool)
    for c, r in zip(centres, radii):
        far2 = np.maximum((lo - c) ** 2, (hi - c) ** 2).sum(axis=1)
        inside_one |= far2 < r * r
        near = np.maximum(np.maximum(lo - c, c - hi), 0.0)
        misses_all &= (near ** 2).sum(axis=1) >= r * r
    kinds = np.full(ncell, CUT, dtype=np.uint8)
    kinds[misses_all] = PHYS
    kinds[inside_one] = FICT
    return kinds


def cell_coords(c, dim, n):
    out = []
    for _ in range(dim):
        out.append(c % n)
        c //= n
    return tuple(out)
