"""The paper's 2D Poisson test problem of Section 4.1, psi = 0 (oracle).
TEST INFRASTRUCTURE ONLY -- it exists to pin the oracle's multigrid against the iteration
counts the paper prints (Table tab:testcaseA), not to run on the GPU.

PAPER.md:378-383 (Sec. 4.1, "Poisson problem on a square domain"):
  * unit square; psi = 0 is the mesh-fitting case, so the domain is the grid
    [0,1]^2 with n x n cells and no fictitious part;
  * manufactured solution  u_bar = cos(a x') sin(a y') / (2 kappa a^2),  a = 3 pi / 2,
    x', y' measured from the centre of the domain;
  * -kappa Laplace(u) = s with s = cos(a x') sin(a y'), kappa = 10;
  * u = u_bar on all four edges by the PENALTY method, beta = 1e4:
        a(u, v) + beta int_Gamma u v dGamma = int s v dOmega + beta int_Gamma u_bar v dGamma;
  * elementwise / patchwise AS, V(5,5), CG preconditioned by the p-multigrid,
    relative residual below 1e-9.
No Dirichlet DOF is eliminated (the penalty term carries the boundary condition).  The
element stiffness of a cell is kappa * K_ref (quadrature in quadrature.element_matrices);
the boundary mass and both load terms use a (p+4)-point Gauss rule per edge / cell, exact
for the polynomial parts and converged far below 1e-9 for the trigonometric ones.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import basis, quadrature
from .dofmap import DofMap

KAPPA = 10.0
BETA = 1e4
A_FREQ = 1.5 * math.pi


def u_bar(x, y, kappa=KAPPA):
    """Manufactured solution, coordinates relative to the domain centre (0.5, 0.5)."""
    return np.cos(A_FREQ * (x - 0.5)) * np.sin(A_FREQ * (y - 0.5)) / (2.0 * kappa * A_FREQ ** 2)


def source(x, y):
    """s = -kappa Laplace(u_bar) = cos(a x') sin(a y')."""
    return np.cos(A_FREQ * (x - 0.5)) * np.sin(A_FREQ * (y - 0.5))


class SquareProblem:
    """Duck-types oracle.problem.Problem for mg.Hierarchy: .cfg, .dof, .A (CSR), .b."""

    def __init__(self, n, p, block="element", kappa=KAPPA, beta=BETA):
        from workloads import small_config
        # dirichlet=0: no face eliminated (penalty BC); direct coarse solve (small system)
        cfg = small_config(2, n, p, coarse="direct", dirichlet=0, block=block)
        self.cfg = cfg
        self.dof = DofMap(cfg)
        modes = self.dof.modes
        h = 1.0 / n
        K_ref, _ = quadrature.element_matrices(cfg, (0, 0), np.zeros((0, 2)), np.zeros(0), modes)
        cd = self.dof.cell_dofs
        m = cd.shape[1]
        nq = p + 4
        xg, wg = basis.gauss(nq)
        # volume rule on the reference cell
        ref_v = np.stack(np.meshgrid(xg, xg, indexing="ij"), -1).reshape(-1, 2)
        w_v = np.outer(wg, wg).ravel() * (0.5 * h) ** 2
        val_v, _ = basis.eval_element(modes, ref_v)
        rows, cols, vals = [], [], []
        b = np.zeros(self.dof.ndof)
        for c in range(n * n):
            cc = np.array([c % n, c // n])
            g = cd[c]
            Ke = kappa * K_ref                              # a(u,v) = int kappa grad u . grad v
            X = (cc + 0.5 * (ref_v + 1.0)) * h
            fe = val_v @ (w_v * source(X[:, 0], X[:, 1]))   # int s v
            for axis in range(2):
                for side in range(2):
                    if cc[axis] != (n - 1 if side else 0):
                        continue
                    ref_e = np.zeros((nq, 2))
                    ref_e[:, axis] = 1.0 if side else -1.0
                    ref_e[:, 1 - axis] = xg
                    w_e = wg * 0.5 * h
                    v_e, _ = basis.eval_element(modes, ref_e)
                    Xe = (cc + 0.5 * (ref_e + 1.0)) * h
                    Ke = Ke + beta * (v_e * w_e) @ v_e.T    # beta int_Gamma u v
                    fe = fe + beta * (v_e @ (w_e * u_bar(Xe[:, 0], Xe[:, 1], kappa)))
            rows.append(np.repeat(g, m))
            cols.append(np.tile(g, m))
            vals.append(Ke.ravel())
            np.add.at(b, g, fe)
        nd = self.dof.ndof
        self.A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(nd, nd)).tocsr()
        self.b = b

    def nodal_error(self, x):
        """max |u_h - u_bar| over the grid vertices (vertex DOFs carry nodal values)."""
        n = self.cfg.n
        keys = self.dof.keys
        p1 = self.cfg.p + 1
        per = p1 ** 3 * self.cfg.n_f
        ent = keys // per
        deg = keys % per
        X = ent % (2 * n + 1)
        Y = (ent // (2 * n + 1)) % (2 * n + 1)
        vert = (X % 2 == 0) & (Y % 2 == 0) & (deg == 0)
        xv, yv = X[vert] / (2.0 * n), Y[vert] / (2.0 * n)
        return float(np.max(np.abs(x[vert] - u_bar(xv, yv))))
