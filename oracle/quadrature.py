"""Space-tree cut-cell quadrature, element matrices and loads (oracle).
TEST INFRASTRUCTURE ONLY.

Weak form, PAPER.md:56-60 (Eq. weakform), with strong Dirichlet (reading R7):
  a(u,v) = int (B v)^T alpha(x) C (B u) dOmega,
  b(v)   = int alpha(x) (N v)^T f dOmega + int (N v)^T g_N dGamma_N.
Poisson: K_ab = int alpha grad N_a . grad N_b ;  f = 1.
Elasticity (3D, isotropic, E, nu; C of P:60):
  K_(a,i),(b,j) = int alpha [ lam dN_a/dx_i dN_b/dx_j + mu dN_a/dx_j dN_b/dx_i
                              + mu delta_ij grad N_a . grad N_b ],
  lam = E nu/((1+nu)(1-2nu)), mu = E/(2(1+nu));  traction g_N = (1,0,0) on one
  box face (reading R8: not alpha-weighted, the face is physical).
Cut-cell integration ("octree scheme with a depth of 3"; reading R13):
  a cell is recursively bisected; only cut sub-boxes are subdivided, down to
  `depth` levels; every leaf gets a (p+1)^d Gauss rule; uncut leaves take the
  leaf's alpha, depth-`depth` cut leaves take alpha per Gauss point (SPEC D-I1).
Element DOF order: basis.element_modes rank * n_f + component.
"""
from __future__ import annotations

import numpy as np

from . import basis, geometry


def leaves(lo, hi, depth, centres, radii, level=0):
    """List of (lo, hi, kind) leaves of the integration space tree of box [lo, hi]."""
    kind = geometry.classify_box(lo, hi, centres, radii)
    if kind != geometry.CUT or level == depth:
        return [(np.array(lo, dtype=np.float64), np.array(hi, dtype=np.float64), kind)]
    dim = len(lo)
    mid = 0.5 * (np.asarray(lo) + np.asarray(hi))
    out = []
    for corner in range(1 << dim):
        clo = np.array([lo[a] if not (corner >> a) & 1 else mid[a] for a in range(dim)])
        chi = np.array([mid[a] if not (corner >> a) & 1 else hi[a] for a in range(dim)])
        out.extend(leaves(clo, chi, depth, centres, radii, level + 1))
    return out


def lame(E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return lam, mu


def _leaf_points(lo, hi, cell_lo, h, npts1d, dim):
    """Gauss points of a leaf: reference coords [-1,1]^d of the cell, physical coords,
    and weights including the Jacobian of the physical cell."""
    xg, wg = basis.gauss(npts1d)
    grids = []
    wts = []
    for a in range(dim):
        # map [-1,1] -> [lo_a, hi_a] (physical)
        xa = 0.5 * (lo[a] + hi[a]) + 0.5 * (hi[a] - lo[a]) * xg
        grids.append(xa)
        wts.append(wg * 0.5 * (hi[a] - lo[a]))
    mesh = np.meshgrid(*grids, indexing="ij")
    wmesh = np.meshgrid(*wts, indexing="ij")
    phys = np.stack([m.ravel() for m in mesh], axis=1)
    w = np.ones(phys.shape[0])
    for wm in wmesh:
        w = w * wm.ravel()
    ref = 2.0 * (phys - cell_lo) / h - 1.0
    return ref, phys, w


def element_matrices(cfg, cell_idx, centres, radii, modes=None):
    """Element stiffness K [m, m] and body load f [m] of one cell by space-tree
    quadrature (module doc).  Returns (K, f)."""
    dim, n, p = cfg.dim, cfg.n, cfg.p
    h = 1.0 / n
    if modes is None:
        modes = basis.element_modes(dim, p, cfg.space)
    n_f = cfg.n_f
    nm = len(modes)
    cell_lo = np.array(cell_idx, dtype=np.float64) * h
    lv = leaves(cell_lo, cell_lo + h, cfg.depth, centres, radii)
    K = np.zeros((nm * n_f, nm * n_f))
    f = np.zeros(nm * n_f)
    if cfg.physics == "elasticity":
        lam, mu = lame(cfg.E, cfg.nu)
    # all leaves' Gauss points at once (the sum over leaves is the same integral)
    refs, ws, alphas = [], [], []
    for lo, hi, kind in lv:
        ref, phys, w = _leaf_points(lo, hi, cell_lo, h, p + 1, dim)
        if kind == geometry.PHYS:
            alpha = np.ones(len(w))
        elif kind == geometry.FICT:
            alpha = np.full(len(w), cfg.alpha)
        else:
            alpha = np.where(geometry.point_is_fictitious(phys, centres, radii), cfg.alpha, 1.0)
        refs.append(ref)
        ws.append(w)
        alphas.append(alpha)
    ref, w, alpha = np.concatenate(refs), np.concatenate(ws), np.concatenate(alphas)
    if True:
        val, gref = basis.eval_element(modes, ref)
        G = gref * (2.0 / h)                     # physical gradients [nm, npts, dim]
        wa = w * alpha
        if cfg.physics == "poisson":
            Gf = G.reshape(nm, -1)                # sum over (point, direction)
            K += (Gf * np.repeat(wa, dim)[None, :]) @ Gf.T
            f += val @ wa                         # f = 1, alpha-weighted
        else:
            KK = K.reshape(nm, n_f, nm, n_f)
            dot = np.einsum("aqd,bqd,q->ab", G, G, wa)
            for i in range(n_f):
                for j in range(n_f):
                    KK[:, i, :, j] += (lam * np.einsum("aq,bq,q->ab", G[:, :, i], G[:, :, j], wa)
                                       + mu * np.einsum("aq,bq,q->ab", G[:, :, j], G[:, :, i], wa))
                KK[:, i, :, i] += mu * dot
            # body force 0
    return K, f


def traction_load(cfg, cell_idx, face, modes=None, g=(1.0, 0.0, 0.0)):
    """int_{face} N . g dGamma over one cell face `face` = 2*axis + side (side 1 = upper).
    (p+1)^(d-1) Gauss points on the face (exact for the polynomial integrand)."""
    dim, n, p = cfg.dim, cfg.n, cfg.p
    h = 1.0 / n
    if modes is None:
        modes = basis.element_modes(dim, p, cfg.space)
    n_f = cfg.n_f
    axis, side = face // 2, face % 2
    xg, wg = basis.gauss(p + 1)
    others = [a for a in range(dim) if a != axis]
    mesh = np.meshgrid(*([xg] * (dim - 1)), indexing="ij")
    wmesh = np.meshgrid(*([wg] * (dim - 1)), indexing="ij")
    npts = mesh[0].size
    ref = np.zeros((npts, dim))
    ref[:, axis] = 1.0 if side else -1.0
    w = np.ones(npts) * (0.5 * h) ** (dim - 1)
    for k, a in enumerate(others):
        ref[:, a] = mesh[k].ravel()
        w = w * wmesh[k].ravel()
    val, _ = basis.eval_element(modes, ref)
    f = np.zeros(len(modes) * n_f)
    for c in range(n_f):
        f[c::n_f] += g[c] * (val @ w)
    return f
