"""Pins of the multi-level hp oracle (oracle/mlhp.py): the basis construction (reading R25) against
properties the mathematics fixes, and the hp-multigrid against the paper's printed plate counts
(Sec. 4.2 Table perPlateRef)."""
import itertools
import json
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import basis  # noqa: E402
from oracle.mlhp import MlhpHierarchy, MlhpProblem  # noqa: E402
from workloads import hp_plate, small_config  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")


def _mixed(dim=2, n=3, p=2, k=2, **kw):
    """A mesh with several refinement depths side by side: one void cut by the grid."""
    kw.setdefault("dirichlet", 0)
    void = ([[0.45] * dim], [0.28]) if dim == 2 else ([[0.3] * dim], [0.15])
    return small_config(dim, n, p, voids=void, kmax=k, **kw)


def _leaf_points(P, leaf, npts):
    j, idx = leaf
    h = P.mesh.h(j)
    lo = np.array(idx, dtype=np.float64) * h
    xg, wg = basis.gauss(npts)
    pts, w = [], []
    for c in itertools.product(range(npts), repeat=P.cfg.dim):
        pts.append([lo[a] + 0.5 * h * (xg[c[a]] + 1) for a in range(P.cfg.dim)])
        w.append(np.prod([0.5 * h * wg[c[a]] for a in range(P.cfg.dim)]))
    return np.array(pts), np.array(w)


def _mass(P):
    M = np.zeros((P.ndof, P.ndof))
    for leaf, d in zip(P.mesh.leaves, P.leaf_dofs):
        funcs = P.leaf_functions(leaf)
        pts, w = _leaf_points(P, leaf, P.cfg.p + 1)
        V, _ = P.eval_functions(funcs, pts)
        M[np.ix_(d, d)] += (V * w) @ V.T
    return M


def _u(P, coef, pts):
    """u_h(x) = sum_i coef_i N_i(x) (scalar problem), each point evaluated in the leaf containing it."""
    out = np.zeros(len(pts))
    for t, x in enumerate(pts):
        for leaf, d in zip(P.mesh.leaves, P.leaf_dofs):
            j, idx = leaf
            h = P.mesh.h(j)
            lo = np.array(idx) * h
            if np.all(x >= lo - 1e-14) and np.all(x <= lo + h + 1e-14):
                V, _ = P.eval_functions(P.leaf_functions(leaf), x[None, :])
                out[t] = coef[d] @ V[:, 0]
                break
    return out


def test_activation_hand_count():
    """n = 2, p = 1, only base element (0,0) refined once, no Dirichlet: base vertices 9 - 1 (the
    corner (0,0) touches only the refined element), level-1 vertices of the overlay that are not on
    the overlay boundary x = 1/2 or y = 1/2: (0,0), (1/4,0), (0,1/4), (1/4,1/4) -> 12 DOFs (R25)."""
    cfg = small_config(2, 2, 1, kmax=1, dirichlet=0)
    P = MlhpProblem(cfg, refine=lambda j, idx: idx == (0, 0))
    assert P.ndof == 12
    base = sorted(k[1:3] for k, c in P.keys if k[0] == 0)
    assert (0, 0) not in base and len(base) == 8
    lvl1 = sorted(k[1:3] for k, c in P.keys if k[0] == 1)
    assert lvl1 == [(0, 0), (0, 2), (2, 0), (2, 2)]


@pytest.mark.parametrize("dim,n,p,k", [(2, 3, 2, 2), (2, 3, 3, 1), (3, 3, 2, 1)])
def test_linear_independence(dim, n, p, k):
    """The global mass matrix of the multi-level basis is SPD (R25 independence)."""
    P = MlhpProblem(_mixed(dim, n, p, k))
    assert len({l[0] for l in P.mesh.leaves}) == k + 1, "several depths side by side"
    ev = np.linalg.eigvalsh(_mass(P))
    assert ev[0] > 1e-12 * ev[-1], (ev[0], ev[-1])


def test_c0_traces():
    """Every function of the basis is continuous across every leaf interface, hanging ones
    included (R25 compatibility): u_h for random coefficients agrees from both sides."""
    P = MlhpProblem(_mixed(2, 3, 2, 2))
    rng = np.random.default_rng(5)
    coef = rng.standard_normal(P.ndof)
    checked = 0
    for leaf in P.mesh.leaves[::3]:
        j, idx = leaf
        h = P.mesh.h(j)
        lo = np.array(idx) * h
        for axis in range(2):
            for t in (0.17, 0.5, 0.83):
                x = lo.copy()
                x[axis] = lo[axis] + h            # the leaf's upper face along `axis`
                x[1 - axis] = lo[1 - axis] + t * h
                if x[axis] >= 1.0 - 1e-12:
                    continue
                inside = P.eval_functions(P.leaf_functions(leaf), x[None, :])[0][:, 0] @ coef[P.leaf_dofs[P.mesh.leaves.index(leaf)]]
                nb = x.copy()
                nb[axis] += 1e-9 * h
                other = _u(P, coef, nb[None, :])[0]
                assert abs(inside - other) <= 1e-6 * max(1.0, abs(inside)), (leaf, axis, t, inside, other)
                checked += 1
    assert checked > 20


@pytest.mark.parametrize("dim,n,p,k", [(2, 3, 2, 2), (2, 2, 3, 2)])
def test_polynomial_reproduction(dim, n, p, k):
    """The L2 projection onto the multi-level space reproduces every x^a y^b with a, b <= p
    exactly (the base space Q_p is contained in the hp space)."""
    P = MlhpProblem(_mixed(dim, n, p, k))
    M = _mass(P)
    rng = np.random.default_rng(3)
    test_pts = rng.random((40, dim))
    for a, b in [(0, 0), (1, 0), (p, 1), (p, p)]:
        poly = lambda X: X[:, 0] ** a * X[:, 1] ** b  # noqa: E731
        F = np.zeros(P.ndof)
        for leaf, d in zip(P.mesh.leaves, P.leaf_dofs):
            pts, w = _leaf_points(P, leaf, p + 2)
            V, _ = P.eval_functions(P.leaf_functions(leaf), pts)
            F[d] += V @ (w * poly(pts))
        c = np.linalg.solve(M, F)
        err = np.max(np.abs(_u(P, c, test_pts) - poly(test_pts)))
        assert err < 1e-9, (a, b, err)


@pytest.mark.parametrize("physics", ["poisson", "elasticity"])
def test_uniform_refinement_equals_fine_grid(physics):
    """Refining EVERY base element to depth k gives exactly the space of the uniform n 2^k grid:
    same DOF count, and (same cut-cell quadrature points) the same discrete energy b^T A^-1 b
    as the uniform-grid oracle (oracle/problem.py) -- basis-independent."""
    from oracle.problem import Problem
    void = ([[0.43, 0.52]], [0.27])
    kw = {} if physics == "poisson" else {"dirichlet": 0b0001, "traction_face": 1}
    cfg = small_config(2, 3, 2, physics=physics, voids=void, kmax=1, refine="all", **kw)
    if physics == "poisson":
        cfg = cfg.replace(dirichlet=0b0101)
    P = MlhpProblem(cfg)
    U = Problem(cfg.replace(n=6, kmax=0))
    assert P.ndof == U.dof.ndof
    e_hp = P.b @ np.linalg.solve(P.A.toarray(), P.b)
    e_un = U.b @ np.linalg.solve(U.A.toarray(), U.b)
    assert abs(e_hp - e_un) <= 1e-10 * abs(e_un), (e_hp, e_un)


def test_hp_level_sequence():
    """P:207 / Fig. hpmultigrid: p reduced first in the overlays, then the refinement depth;
    p = 3, k = 2 -> (3,2), (2,2), (1,2), (1,1), (1,0); the level DOF sets are nested."""
    P = MlhpProblem(_mixed(2, 3, 3, 2))
    seq = P.level_sequence()
    assert seq == [(3, 2), (2, 2), (1, 2), (1, 1), (1, 0)]
    sets = [set(P.level_dofs(*l).tolist()) for l in seq]
    assert len(sets[0]) == P.ndof
    for a, b in zip(sets, sets[1:]):
        assert b < a


def test_blocks_overlap_bound():
    """Elementwise blocks are per base element (R26): every DOF lies in at most 2^d of them;
    patchwise blocks at most 3^d; omega * lambda_max(M^-1 A) < 2 with the paper's omega."""
    P = MlhpProblem(_mixed(2, 3, 2, 2))
    for blk, bound in (("element", 4), ("patch", 9)):
        H = MlhpHierarchy(P, block=blk)
        lv = H.levels[0]
        cnt = np.bincount(np.concatenate(lv.blocks), minlength=lv.n)
        assert cnt.max() <= bound
        A = lv.A.toarray()
        Minv = np.zeros_like(A)
        for b, inv in zip(lv.blocks, lv.inv):
            Minv[np.ix_(b, b)] += inv
        lam = np.max(np.real(np.linalg.eigvals(Minv @ A)))
        assert H.omega * lam < 2.0, (blk, lam)


def test_vcycle_one_level_reduces_to_direct():
    """k = 0, p = 1: one level -> the V-cycle is the direct coarse solve."""
    P = MlhpProblem(small_config(2, 4, 1, kmax=0, dirichlet=0b0001))
    H = MlhpHierarchy(P)
    assert len(H.levels) == 1
    x = H.vcycle(P.b)
    assert np.allclose(P.A @ x, P.b, rtol=1e-12, atol=1e-14)


def test_plate_paper_counts():
    """PAPER.md:735-804 (Table perPlateRef, p = 2, CG with the hp-multigrid preconditioner, V(5,5)):
      * elementwise AS smoother, k = 0: 12 (h = 1/8), 9 (h = 1/16) -- reproduced exactly;
      * elementwise counts grow with the refinement depth;
      * patchwise AS smoother: 6-7 for every depth ("independent of the refinement depth"),
        here within +-2 and spread <= 1 over k = 0..2.
    Geometry reading R28 (hp_plate), tolerance 1e-9 (the paper's Sec. 4 tolerance)."""
    gold = json.load(open(GOLDEN))["plate_cg_mg_p2"]
    for n in (8, 16):
        el, pa = [], []
        for k in range(3):
            P = MlhpProblem(hp_plate(n, k))
            el.append(MlhpHierarchy(P, block="element").fcg(P.b, rtol=1e-9)[1])
            pa.append(MlhpHierarchy(P, block="patch").fcg(P.b, rtol=1e-9)[1])
        g_el = gold["element"][str(n)]
        g_pa = gold["patch"][str(n)]
        assert el[0] == g_el[0], (n, el, g_el)
        assert el[2] > 2 * el[0], (n, el)
        assert max(pa) - min(pa) <= 1, (n, pa)
        assert all(abs(a - g) <= 2 for a, g in zip(pa, g_pa)), (n, pa, g_pa)


def test_fully_refined_base_drops_empty_coarse_level():
    """Every base element cut (n = 2, one large void) and refined: no base vertex is active (R25),
    so (1,0) is empty and dropped; the V-cycle still solves (coarsest level (1,1) direct)."""
    cfg = small_config(2, 2, 2, voids=([[0.5, 0.5]], [0.3]), kmax=1, dirichlet=0b0101)
    P = MlhpProblem(cfg)
    assert len(P.level_dofs(1, 0)) == 0
    assert P.level_sequence() == [(2, 1), (1, 1)]
    x, it, hist = MlhpHierarchy(P).fcg(P.b)
    assert hist[-1] < cfg.rtol


@pytest.mark.parametrize("block", ["element", "patch"])
def test_k0_hp_hierarchy_equals_uniform_oracle(block):
    """k = 0 (no refinement): the hp oracle is the uniform p-multigrid -- same DOF set, same blocks
    (base element = cell; base-vertex patch = the closure patch, R19/R26), same V-cycle, so the
    stand-alone MG histories and FCG iterates coincide to rounding."""
    from oracle.mg import Hierarchy
    from oracle.problem import Problem
    cfg = small_config(2, 5, 3, voids=([[0.47, 0.52]], [0.26]), kmax=0, block=block, coarse="direct",
                       dirichlet=0b0101)
    P = MlhpProblem(cfg)
    U = Problem(cfg)
    assert P.ndof == U.dof.ndof
    perm = np.zeros(P.ndof, dtype=np.int64)   # hp DOF -> uniform DOF via the entity keys
    n = cfg.n
    p = cfg.p
    for i, (k, c) in enumerate(P.keys):
        X, dg = k[1:3], k[3:5]
        # the uniform key convention of dofmap.py (X_z = deg_z = 0 in 2D)
        key = ((((X[1] * (2 * n + 1) + X[0]) * (p + 1) + 0) * (p + 1) + dg[1]) * (p + 1) + dg[0]) * cfg.n_f + c
        perm[i] = np.searchsorted(U.dof.keys, key)
        assert U.dof.keys[perm[i]] == key
    assert len(np.unique(perm)) == P.ndof
    Hh, Hu = MlhpHierarchy(P), Hierarchy(U)
    _, ih, hh = Hh.mg_solve(P.b, rtol=1e-10, maxit=60)
    _, iu, hu = Hu.mg_solve(U.b, rtol=1e-10, maxit=60)
    assert ih == iu and np.allclose(hh, hu, rtol=1e-8, atol=1e-14)
    xh, _, _ = Hh.fcg(P.b)
    xu, _, _ = Hu.fcg(U.b)
    assert np.allclose(xh, xu[perm], rtol=0, atol=1e-9 * np.abs(xu).max())
