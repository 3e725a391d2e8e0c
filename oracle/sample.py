"""Row samples of the level operator, the load and one additive-Schwarz update at sizes the
oracle cannot assemble (the full BASELINE workloads; SURVEY.md §8(c) "sampled outputs the oracle
can compute one by one").  TEST INFRASTRUCTURE ONLY.

Everything is a per-row restatement of the definitions the rest of the oracle uses globally:
  * operator row (levels P:118): (A_q x)_i = sum over the cells c
    whose level-q element DOFs contain i of K_c[a_i(c), :m_q] x_c, K_c = K_ref (uncut physical),
    alpha K_ref (uncut fictitious), the space-tree quadrature matrix (cut), computed lazily
    (module quadrature) for the cells a sample touches;
  * load row: b_i = sum over the cells c containing i of f_c[a_i(c)] (Problem._load);
  * Schwarz row (Eq. AdditiveSchwarz): (omega sum_B P_B A_B^{-1} P_B^T r)_i over the
    blocks B that contain i, A_B = the assembled level-q matrix restricted to B's DOFs, i.e.
    sum over the cells c touching B of K_c's entries between B's DOFs (mg.Level assembles the
    same sub-blocks from the global CSR matrix); blocks P:259 / R11: the level-q DOFs of one
    cell (elementwise) or of the 2^d cells around a grid vertex (patchwise, closure rule R19).
The per-row forms are pinned against mg.Level / assembly on small grids
(tests/test_oracle_sample.py)."""
from __future__ import annotations

import itertools

import numpy as np
import scipy.linalg as sla

from . import basis, geometry, quadrature
from .dofmap import DofMap


class LazyCells:
    """Cell kinds, DOF map and reference matrices of a workload; cut-cell matrices on demand."""

    def __init__(self, cfg, centres=None, radii=None):
        from workloads import config_voids
        self.cfg = cfg
        if centres is None:
            centres, radii = config_voids(cfg)
        self.centres = np.asarray(centres, dtype=np.float64).reshape(-1, cfg.dim)
        self.radii = np.asarray(radii, dtype=np.float64).reshape(-1)
        self.modes = basis.element_modes(cfg.dim, cfg.p, cfg.space)
        self.kinds = geometry.classify_cells(cfg.dim, cfg.n, self.centres, self.radii)
        self.K_ref, self.f_ref = quadrature.element_matrices(
            cfg, (0,) * cfg.dim, np.zeros((0, cfg.dim)), np.zeros(0), self.modes)
        self.dof = DofMap(cfg)
        self._cut = {}

    def _cut_mats(self, c):
        if c not in self._cut:
            self._cut[c] = quadrature.element_matrices(
                self.cfg, geometry.cell_coords(int(c), self.cfg.dim, self.cfg.n), self.centres, self.radii,
                self.modes)
        return self._cut[c]

    def K(self, c):
        k = self.kinds[c]
        if k == geometry.CUT:
            return self._cut_mats(c)[0]
        return self.K_ref * (self.cfg.alpha if k == geometry.FICT else 1.0)

    def f(self, c):
        k = self.kinds[c]
        if k == geometry.CUT:
            return self._cut_mats(c)[1]
        return self.f_ref * (self.cfg.alpha if k == geometry.FICT else 1.0)

    def cells_of(self, i, q=None):
        """Cells whose (level-q) element DOFs contain DOF i, with the local index of i
        (an inverse of cell_dofs: the flattened entries sorted by DOF, built once)."""
        if not hasattr(self, "_inc_order"):
            flat = self.dof.cell_dofs.ravel()
            self._inc_order = np.argsort(flat, kind="stable")
            self._inc_sorted = flat[self._inc_order]
        m = self.dof.m if q is None else self.dof.level_m(q)
        lo, hi = np.searchsorted(self._inc_sorted, [i, i + 1])
        e = self._inc_order[lo:hi]
        mm = self.dof.cell_dofs.shape[1]
        return [(int(k // mm), int(k % mm)) for k in e if k % mm < m]

    def cell_grid(self, c):
        return geometry.cell_coords(int(c), self.cfg.dim, self.cfg.n)

    def cell_index(self, coords):
        n = self.cfg.n
        c = 0
        for a in reversed(range(self.cfg.dim)):
            if not 0 <= coords[a] < n:
                return -1
            c = c * n + coords[a]
        return c


def operator_row(L: LazyCells, x, i, q):
    """(A_q x)_i; x in the oracle's full numbering (entries outside level q ignored)."""
    m = L.dof.level_m(q)
    mask = L.dof.dof_order <= q
    s = 0.0
    for c, a in L.cells_of(i, q):
        idx = L.dof.cell_dofs[c, :m]
        ok = (idx >= 0) & np.where(idx >= 0, mask[np.maximum(idx, 0)], False)
        s += float(L.K(c)[a, :m][ok] @ x[idx[ok]])
    return s


def load_row(L: LazyCells, i):
    """b_i (body load; configs without traction)."""
    assert L.cfg.traction_face < 0
    return float(sum(L.f(c)[a] for c, a in L.cells_of(i)))


def block_dofs(L: LazyCells, anchor, q, block):
    """Sorted level-q DOFs of one Schwarz block: elementwise -> anchor = cell coords, the free
    level-q DOFs of that cell; patchwise -> anchor = vertex coords, the union over the 2^d
    cells around the vertex (those inside the grid)."""
    d = L.cfg.dim
    m = L.dof.level_m(q)
    if block == "element":
        cells = [L.cell_index(anchor)]
    else:
        cells = [L.cell_index([anchor[a] - 1 + ((k >> a) & 1) for a in range(d)]) for k in range(1 << d)]
    ids = [L.dof.cell_dofs[c, :m] for c in cells if c >= 0]
    g = np.unique(np.concatenate(ids))
    return g[g >= 0]


def block_matrix(L: LazyCells, B, q):
    """A_B: the assembled level-q matrix restricted to the DOFs B (sum over every cell that
    holds a DOF of B of its element matrix entries between B's DOFs)."""
    m = L.dof.level_m(q)
    pos = {int(g): k for k, g in enumerate(B)}
    cells = sorted({c for g in B for c, _ in L.cells_of(int(g), q)})
    A = np.zeros((len(B), len(B)))
    for c in cells:
        idx = L.dof.cell_dofs[c, :m]
        loc = [(a, pos[int(g)]) for a, g in enumerate(idx) if g >= 0 and int(g) in pos]
        if not loc:
            continue
        aa = np.array([t[0] for t in loc])
        bb = np.array([t[1] for t in loc])
        A[np.ix_(bb, bb)] += L.K(c)[np.ix_(aa, aa)]
    return A


def blocks_containing(L: LazyCells, i, q, block):
    """Anchors (cell coords or vertex coords) of the blocks whose DOF set contains i."""
    d = L.cfg.dim
    out = set()
    for c, _ in L.cells_of(i, q):
        cc = L.cell_grid(c)
        if block == "element":
            out.add(tuple(cc))
            continue
        # i lies in patch v iff some cell around v holds i, i.e. v is a vertex of a cell of i
        for off in itertools.product(range(2), repeat=d):
            v = tuple(cc[a] + off[a] for a in range(d))
            if all(0 <= v[a] <= L.cfg.n for a in range(d)):
                out.add(v)
    res = []
    for v in sorted(out):
        B = block_dofs(L, v, q, block)
        if np.any(B == i):
            res.append(v)
    return res


class PerturbedCells:
    """LazyCells whose CUT-cell matrices carry a seeded symmetric entrywise relative perturbation
    K_ab (1 + delta E_ab), E_ab ~ N(0,1) (reading R18: the sensitivity of an ill-conditioned block
    to setup data that agrees only to the generator-parity level L0, not an evaluation order)."""

    def __init__(self, L: LazyCells, delta, seed=0):
        self._L, self.delta, self.seed = L, delta, seed

    def __getattr__(self, name):
        return getattr(self._L, name)

    def K(self, c):
        K = self._L.K(c)
        if self._L.kinds[c] != geometry.CUT:
            return K
        E = np.random.default_rng([self.seed, int(c)]).standard_normal(K.shape)
        E = 0.5 * (E + E.T)
        return K * (1.0 + self.delta * E)


def schwarz_row(L: LazyCells, r, i, q, block, omega, inv="lu", perturb=0.0):
    """(omega sum_B P_B A_B^{-1} P_B^T r)_i; A_B^{-1} applied by dense LU (inv="lu") or
    Cholesky (inv="chol") -- two backward-stable evaluations (reading R18); perturb > 0 evaluates
    it on PerturbedCells(L, perturb) (the setup-sensitivity leg of R18)."""
    if perturb > 0.0:
        L = PerturbedCells(L, perturb)
    s = 0.0
    for v in blocks_containing(L, i, q, block):
        B = block_dofs(L, v, q, block)
        A = block_matrix(L, B, q)
        rb = r[B]
        if inv == "lu":
            y = sla.lu_solve(sla.lu_factor(A), rb)
        else:
            y = sla.cho_solve(sla.cho_factor(A), rb)
        s += y[int(np.nonzero(B == i)[0][0])]
    return omega * s
