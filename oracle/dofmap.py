"""Global DOF numbering, Dirichlet elimination and p-levels (oracle).
TEST INFRASTRUCTURE ONLY.

PAPER.md:100 "direct association of the topological components -- nodes,
edges, faces and solids -- with the degrees of freedom": a 1D mode k of a cell
is nodal (k in {0,1}: the vertex at cell index + k) or internal (k >= 2: the cell
interval).  A d-dim element mode therefore lives on the entity spanned by its
internal axes, at the position given by its nodal offsets.

Canonical DOF key (the interface convention of include/fcm_mg.h, computed here
independently): per axis X_a = 2*pos_a for a nodal axis (pos = vertex index),
2*cell_a + 1 for an internal axis; deg_a = k_a if internal else 0;
  key = ((((X_z*(2n+1) + X_y)*(2n+1) + X_x)*(p+1) + deg_z)*(p+1) + deg_y)*(p+1) + deg_x)*n_f + comp.
The oracle numbers the free DOFs in ascending key order.

Dirichlet (reading R7): every DOF of an entity lying on a Dirichlet box face
(nodal axis a at position 0 or n) is eliminated (u = 0 strongly).
Levels (Eq. restrictionoperation): level q keeps the DOFs whose mode
order is <= q; R = [I 0] is index selection, R^T zero extension.
"""
from __future__ import annotations

import numpy as np

from . import basis


class DofMap:
    def __init__(self, cfg):
        self.cfg = cfg
        dim, n, p, n_f = cfg.dim, cfg.n, cfg.p, cfg.n_f
        self.modes = basis.element_modes(dim, p, cfg.space)
        self.mode_orders = np.array([basis.mode_order(m, cfg.space) for m in self.modes])
        nm = len(self.modes)
        self.m = nm * n_f
        ncell = n ** dim
        cells = np.arange(ncell)
        cc = []
        t = cells.copy()
        for _ in range(dim):
            cc.append(t % n)
            t = t // n
        keys = np.zeros((ncell, nm, n_f), dtype=np.int64)
        dirich = np.zeros((ncell, nm), dtype=bool)
        mask = cfg.dirichlet_mask
        for i, mode in enumerate(self.modes):
            X = []
            degs = []
            for a in range(dim):
                k = mode[a]
                if k < 2:
                    pos = cc[a] + k
                    X.append(2 * pos)
                    degs.append(0)
                    if (mask >> (2 * a)) & 1:
                        dirich[:, i] |= pos == 0
                    if (mask >> (2 * a + 1)) & 1:
                        dirich[:, i] |= pos == n
                else:
                    X.append(2 * cc[a] + 1)
                    degs.append(k)
            while len(X) < 3:
                X.append(np.zeros(ncell, dtype=np.int64))
                degs.append(0)
            base = ((X[2] * (2 * n + 1) + X[1]) * (2 * n + 1) + X[0])
            base = ((base * (p + 1) + degs[2]) * (p + 1) + degs[1]) * (p + 1) + degs[0]
            for c in range(n_f):
                keys[:, i, c] = base * n_f + c
        keys = keys.reshape(ncell, nm * n_f)
        dmask = np.repeat(dirich, n_f, axis=1)
        free_keys = np.unique(keys[~dmask])
        self.keys = free_keys                                   # [ndof] ascending
        gl = np.searchsorted(free_keys, keys)
        gl[dmask] = -1
        self.cell_dofs = gl                                     # [ncell, m], -1 = Dirichlet
        self.ndof = len(free_keys)
        order_local = np.repeat(self.mode_orders, n_f)
        dof_order = np.zeros(self.ndof, dtype=np.int64)
        ok = gl >= 0
        dof_order[gl[ok]] = np.broadcast_to(order_local, gl.shape)[ok]
        self.dof_order = dof_order
        self.local_order = order_local

    def level_dofs(self, q):
        """Sorted global indices of level q (mode order <= q)."""
        return np.nonzero(self.dof_order <= q)[0]

    def level_m(self, q):
        return int((self.local_order <= q).sum())
