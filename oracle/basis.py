"""Integrated-Legendre hierarchical basis (oracle).  TEST INFRASTRUCTURE ONLY.

PAPER.md:34 / :62: p-FEM mesh with "high-order integrated Legendre shape
functions that are hierarchical in nature, i.e. the set of basis functions of
order p contains all basis functions from order 1 up to p".  The paper does not
print the normalisation; reading R-B1 (SPEC.md:72 D-B1):
    N_0 = (1 - xi)/2,  N_1 = (1 + xi)/2,
    N_k = (P_k - P_{k-2}) / sqrt(2 (2k - 1))      for k >= 2  (degree k),
so  dN_k/dxi = sqrt((2k-1)/2) P_{k-1}  and  int N_j' N_k' = delta_jk (j,k >= 2).

Element modes are tuples (k_x, k_y[, k_z]) of 1D mode indices.  Tensor space:
all (p+1)^d tuples.  Trunk space (Table 1): vertex modes, and
modes whose internal (k>=2) degrees sum to <= p.  Mode order (level tag,
P:207 "arithmetic p-sequence"): tensor -> max of the 1D orders (nodal = 1);
trunk -> 1 for vertex modes, else the sum of internal degrees.

Local ordering convention (documented in include/fcm_mg.h, implemented here
independently): modes sorted by (order, S, deg_x, deg_y, deg_z, off) with
S = sum_{a internal} 2^a, deg_a = k_a if internal else 0,
off = sum_{a nodal} k_a 2^a; element DOF index = rank * n_f + component.
"""
from __future__ import annotations

import functools

import numpy as np
from numpy.polynomial import legendre as npleg


@functools.lru_cache(maxsize=None)
def gauss(npts: int):
    """Gauss-Legendre rule on [-1, 1] (library primitive)."""
    return npleg.leggauss(npts)


def _mode_coeffs(k: int) -> np.ndarray:
    """Legendre-series coefficients of 1D mode k (R-B1)."""
    c = np.zeros(max(k + 1, 2))
    if k == 0:
        # (1 - xi)/2 = P0/2 - P1/2
        c[0], c[1] = 0.5, -0.5
    elif k == 1:
        c[0], c[1] = 0.5, 0.5
    else:
        c[k] = 1.0
        c[k - 2] = -1.0
        c /= np.sqrt(2.0 * (2 * k - 1))
    return c


def modes_1d(p: int, xi):
    """Values and derivatives of 1D modes 0..p at points xi: arrays [p+1, len(xi)]."""
    xi = np.atleast_1d(np.asarray(xi, dtype=np.float64))
    v = np.zeros((p + 1, xi.size))
    d = np.zeros((p + 1, xi.size))
    for k in range(p + 1):
        c = _mode_coeffs(k)
        v[k] = npleg.legval(xi, c)
        d[k] = npleg.legval(xi, npleg.legder(c))
    return v, d


def order_1d(k: int) -> int:
    return 1 if k < 2 else k


def mode_order(mode, space: str) -> int:
    internal = [k for k in mode if k >= 2]
    if space == "tensor":
        return max(order_1d(k) for k in mode)
    if not internal:
        return 1
    return int(sum(internal))


def _sort_key(mode, space):
    S = sum(1 << a for a, k in enumerate(mode) if k >= 2)
    degs = [k if k >= 2 else 0 for k in mode] + [0] * (3 - len(mode))
    off = sum(k << a for a, k in enumerate(mode) if k < 2)
    return (mode_order(mode, space), S, degs[0], degs[1], degs[2], off)


def element_modes(dim: int, p: int, space: str = "tensor"):
    """Element mode tuples in the hierarchical local order (see module doc)."""
    import itertools
    modes = []
    for m in itertools.product(range(p + 1), repeat=dim):
        m = tuple(reversed(m))  # (k_x, k_y, k_z)
        if space == "trunk":
            internal = [k for k in m if k >= 2]
            if internal and sum(internal) > p:
                continue
        modes.append(m)
    modes.sort(key=lambda m: _sort_key(m, space))
    return modes


def element_dof_count(dim, p, space, n_f, q=None):
    modes = element_modes(dim, p, space)
    if q is not None:
        modes = [m for m in modes if mode_order(m, space) <= q]
    return len(modes) * n_f


def eval_element(modes, pts_ref):
    """Values [nm, npts] and reference gradients [nm, npts, dim] of element modes
    at reference points pts_ref [npts, dim] (tensor products of 1D modes)."""
    pts_ref = np.atleast_2d(pts_ref)
    npts, dim = pts_ref.shape
    p = max(max(m) for m in modes)
    p = max(p, 1)
    V = []
    D = []
    for a in range(dim):
        v, d = modes_1d(p, pts_ref[:, a])
        V.append(v)
        D.append(d)
    nm = len(modes)
    val = np.ones((nm, npts))
    grad = np.ones((nm, npts, dim))
    for i, m in enumerate(modes):
        for a in range(dim):
            val[i] *= V[a][m[a]]
            for g in range(dim):
                grad[i, :, g] *= (D[a][m[a]] if g == a else V[a][m[a]])
    return val, grad
