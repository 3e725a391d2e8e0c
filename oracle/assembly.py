"""Global assembly (oracle).  TEST INFRASTRUCTURE ONLY.

A = sum_c P_c^T K_c P_c over all cells (uncut phys: K_ref, uncut fict:
alpha*K_ref, cut: individual K_c), Dirichlet rows/columns eliminated (R7).
Two plain forms of the same definition:
  csr_matrix(...)     scipy COO -> CSR (duplicates summed)   [O6]
  ebe_apply(...)      y = sum_c P_c^T K_c (P_c x)            [O13, no global matrix]
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def element_matrix_of(prob, c):
    """K_c of cell c (full m x m)."""
    kind = prob.kinds[c]
    if kind == 2:
        return prob.cut_K[prob.cut_index[c]]
    return prob.K_ref * (prob.cfg.alpha if kind == 1 else 1.0)


def csr_matrix(prob):
    cd = prob.dof.cell_dofs
    ncell, m = cd.shape
    rows = np.repeat(cd, m, axis=1)                  # [ncell, m*m] row index a
    cols = np.tile(cd, (1, m))                       # col index b
    scale = np.where(prob.kinds == 1, prob.cfg.alpha, 1.0)
    vals = scale[:, None] * prob.K_ref.reshape(1, m * m)
    cut = np.nonzero(prob.kinds == 2)[0]
    if len(cut):
        vals = vals.copy()
        vals[cut] = prob.cut_K[prob.cut_index[cut]].reshape(len(cut), m * m)
    ok = (rows >= 0) & (cols >= 0)
    A = sp.coo_matrix((vals[ok], (rows[ok], cols[ok])), shape=(prob.dof.ndof, prob.dof.ndof))
    return A.tocsr()


def ebe_apply(prob, x, q=None):
    """y = A_q x in the full (fine) numbering with zeros outside level q: x is a full
    vector (entries outside level q are ignored); K_c leading m_q block."""
    cd = prob.dof.cell_dofs
    m = cd.shape[1] if q is None else prob.dof.level_m(q)
    cd = cd[:, :m]
    nd = prob.dof.ndof
    xe = np.append(np.asarray(x, dtype=np.float64), 0.0)
    if q is not None:
        mask = np.append(prob.dof.dof_order <= q, False)
        xe = xe * mask
    X = xe[cd]                                       # -1 -> appended zero
    K = prob.K_ref[:m, :m]
    scale = np.where(prob.kinds == 1, prob.cfg.alpha, 1.0)
    Y = (X @ K.T) * scale[:, None]
    cut = np.nonzero(prob.kinds == 2)[0]
    if len(cut):
        Kc = prob.cut_K[prob.cut_index[cut]][:, :m, :m]
        Y[cut] = np.einsum("cab,cb->ca", Kc, X[cut])
    ok = cd >= 0
    y = np.bincount(cd[ok], weights=Y[ok], minlength=nd)
    if q is not None:
        y = y * mask[:-1]
    return y
