"""Build a whole finite-cell problem from a workloads.Config (oracle).
TEST INFRASTRUCTURE ONLY.

Steps: voids -> cell classification (geometry) ->
element matrices by space-tree quadrature (K_ref = the uncut physical cell,
alpha*K_ref for uncut fictitious cells, individual K_c for cut cells) -> load
vector -> DOF map with Dirichlet elimination -> (optionally) global CSR.
"""
from __future__ import annotations

import numpy as np

from . import assembly, basis, geometry, quadrature
from .dofmap import DofMap


class Problem:
    def __init__(self, cfg, centres=None, radii=None, build_csr=True, cut_cells_only=None):
        from workloads import config_voids
        self.cfg = cfg
        if centres is None:
            centres, radii = config_voids(cfg)
        self.centres = np.asarray(centres, dtype=np.float64).reshape(-1, cfg.dim)
        self.radii = np.asarray(radii, dtype=np.float64).reshape(-1)
        dim, n = cfg.dim, cfg.n
        self.modes = basis.element_modes(dim, cfg.p, cfg.space)
        self.kinds = geometry.classify_cells(dim, n, self.centres, self.radii)
        # reference element: one uncut physical cell (cell 0's shape; h-dependent only)
        self.K_ref, self.f_ref = quadrature.element_matrices(
            cfg, (0,) * dim, np.zeros((0, dim)), np.zeros(0), self.modes)
        self.cut_cells = np.nonzero(self.kinds == geometry.CUT)[0]
        self.cut_index = np.full(n ** dim, -1, dtype=np.int64)
        self.cut_index[self.cut_cells] = np.arange(len(self.cut_cells))
        m = self.K_ref.shape[0]
        todo = self.cut_cells if cut_cells_only is None else np.asarray(cut_cells_only)
        self.cut_K = np.zeros((len(self.cut_cells), m, m))
        self.cut_f = np.zeros((len(self.cut_cells), m))
        for c in todo:
            K, f = quadrature.element_matrices(cfg, geometry.cell_coords(int(c), dim, n),
                                               self.centres, self.radii, self.modes)
            self.cut_K[self.cut_index[c]] = K
            self.cut_f[self.cut_index[c]] = f
        self.dof = DofMap(cfg)
        self.b = self._load()
        self.A = assembly.csr_matrix(self) if build_csr else None

    def element_load(self, c):
        kind = self.kinds[c]
        if kind == geometry.CUT:
            return self.cut_f[self.cut_index[c]]
        return self.f_ref * (self.cfg.alpha if kind == geometry.FICT else 1.0)

    def _load(self):
        cfg = self.cfg
        cd = self.dof.cell_dofs
        ncell, m = cd.shape
        F = np.where((self.kinds == geometry.FICT)[:, None], cfg.alpha, 1.0) * self.f_ref[None, :]
        if len(self.cut_cells):
            F[self.cut_cells] = self.cut_f
        if cfg.traction_face >= 0:
            axis, side = cfg.traction_face // 2, cfg.traction_face % 2
            ft = quadrature.traction_load(cfg, (0,) * cfg.dim, cfg.traction_face, self.modes)
            coord = (np.arange(ncell) // (cfg.n ** axis)) % cfg.n
            on = coord == (cfg.n - 1 if side else 0)
            F[on] += ft[None, :]
        ok = cd >= 0
        return np.bincount(cd[ok], weights=F[ok], minlength=self.dof.ndof)

    def apply(self, x, q=None):
        if self.A is not None and q is None:
            return self.A @ x
        return assembly.ebe_apply(self, x, q)
