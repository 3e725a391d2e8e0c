"""Pins of oracle/assembly.py and oracle/mg.py (no GPU): SPD, binary transfers,
Schwarz bounds and special cases, V-cycle special cases, direct-solve agreement,
manufactured-solution convergence, and the paper's iteration counts (method level)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import assembly, basis, quadrature
from oracle.dofmap import DofMap
from oracle.mg import Hierarchy, Level, fcg, pcg
from oracle.problem import Problem
from workloads import get_config, small_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.fixture(scope="module")
def cfg1():
    return Problem(get_config("cfg1"))


@pytest.fixture(scope="module")
def small3d():
    return Problem(small_config(3, 5, 3, voids=2, seed=7))


def test_spd_and_symmetry(cfg1, small3d):
    # P5
    for P in (cfg1, small3d):
        A = P.A
        assert abs(A - A.T).max() <= 1e-14 * abs(A).max()
        np.linalg.cholesky(A.toarray())
    ev = np.linalg.eigvalsh(cfg1.A.toarray())
    assert ev[0] > 0


def test_ebe_equals_csr(small3d):
    P = small3d
    x = np.random.default_rng(0).standard_normal(P.dof.ndof)
    y1 = P.A @ x
    y2 = assembly.ebe_apply(P, x)
    assert np.linalg.norm(y1 - y2) <= 1e-14 * np.linalg.norm(y1)
    for q in range(1, P.cfg.p + 1):
        I = P.dof.level_dofs(q)
        xq = np.zeros(P.dof.ndof)
        xq[I] = x[I]
        yq = assembly.ebe_apply(P, xq, q)
        ref = P.A[I][:, I] @ x[I]
        assert np.linalg.norm(yq[I] - ref) <= 1e-14 * np.linalg.norm(ref)


def test_binary_transfers(small3d):
    # P6 / P:118: A_{q-1} = R A_q R^T with an explicit 0/1 R; R R^T = I; adjointness
    H = Hierarchy(small3d, coarse="direct")
    rng = np.random.default_rng(1)
    for q in range(small3d.cfg.p, 1, -1):
        nq, nc = H.levels[q].n, H.levels[q - 1].n
        R = np.zeros((nc, nq))
        R[np.arange(nc), H.sel[q]] = 1.0
        Aq = H.levels[q].A.toarray()
        Ac = H.levels[q - 1].A.toarray()
        assert np.array_equal(R @ Aq @ R.T, Ac)
        assert np.array_equal(R @ R.T, np.eye(nc))
        v, w = rng.standard_normal(nq), rng.standard_normal(nc)
        assert abs((R @ v) @ w - v @ (R.T @ w)) < 1e-13


def _lam_max(lv):
    A = lv.A.toarray()
    M = np.stack([lv.schwarz(e) for e in np.eye(lv.n)], 1)
    assert np.abs(M - M.T).max() < 1e-12 * np.abs(M).max()
    lam = np.linalg.eigvals(M @ A).real
    assert lam.min() > 0
    return lam.max()


def test_schwarz_bounds_and_overlap(cfg1, small3d):
    # the paper's omega keeps rho(I - omega M^-1 A) < 1, i.e. omega*lambda_max < 2.
    # (Reading R17: the quoted bound lambda_max <= 2^d is not attained exactly --
    # measured 5.1 in 2D / 9.4-10 in 3D elementwise; the A-orthogonal colouring bound 3^d holds.)
    for P in (cfg1, small3d):
        d = P.cfg.dim
        H = Hierarchy(P, coarse="direct")
        lv = H.levels[P.cfg.p]
        lam = _lam_max(lv)
        assert lam <= 3 ** d and H.omega * lam < 2.0
        assert H.omega == GOLD["omega"][f"{d}d_element"]
        cnt = np.bincount(np.concatenate(lv.blocks), minlength=lv.n)
        assert cnt.max() <= GOLD["n_max_cartesian"][str(d)] and cnt.min() >= 1
    Pp = Problem(small_config(3, 4, 2, voids=2, seed=7))
    Hp = Hierarchy(Pp, block="patch", coarse="direct")
    lam = _lam_max(Hp.levels[2])
    assert Hp.omega == GOLD["omega"]["3d_patch"] and Hp.omega * lam < 2.0
    Hp = Hierarchy(cfg1, block="patch", coarse="direct")
    lv = Hp.levels[3]
    cnt = np.bincount(np.concatenate(lv.blocks), minlength=lv.n)
    assert cnt.max() <= 3 ** 2 and cnt.min() >= 1
    assert Hp.omega == GOLD["omega"]["2d_patch"]


def test_schwarz_single_block_exact(cfg1):
    # one block covering every DOF with omega = 1 is the exact solve
    H = Hierarchy(cfg1, coarse="direct")
    lv = H.levels[3]
    lv.blocks = [np.arange(lv.n)]
    lv.inv = [np.linalg.inv(lv.A.toarray())]
    b = cfg1.b
    x = lv.schwarz(b)
    assert np.linalg.norm(lv.A @ x - b) <= 1e-8 * np.linalg.norm(b)


def test_schwarz_block_order_independent(small3d):
    # the result does not depend on the block order beyond rounding
    H = Hierarchy(small3d, coarse="direct")
    lv = H.levels[3]
    r = np.random.default_rng(2).standard_normal(lv.n)
    z1 = lv.schwarz(r)
    perm = np.random.default_rng(3).permutation(len(lv.blocks))
    lv.blocks = [lv.blocks[i] for i in perm]
    lv.inv = [lv.inv[i] for i in perm]
    z2 = lv.schwarz(r)
    assert np.linalg.norm(z1 - z2) <= 1e-12 * np.linalg.norm(z1)


def test_vcycle_special_cases(small3d):
    P = small3d
    rng = np.random.default_rng(4)
    # one level (p = 1): V = A0^{-1}
    P1 = Problem(P.cfg.replace(p=1), P.centres, P.radii)
    H1 = Hierarchy(P1, coarse="direct")
    b = rng.standard_normal(P1.dof.ndof)
    assert np.linalg.norm(P1.A @ H1.vcycle(b) - b) <= 1e-9 * np.linalg.norm(b)
    # n_s = 0: V = R^T A0^{-1} R (composed over the levels)
    H0 = Hierarchy(P, coarse="direct", n_pre=0, n_post=0)
    r = rng.standard_normal(P.dof.ndof)
    z = H0.vcycle(r)
    i1 = P.dof.level_dofs(1)
    ref = np.zeros(P.dof.ndof)
    ref[i1] = np.linalg.solve(P.A[i1][:, i1].toarray(), r[i1])
    assert np.linalg.norm(z - ref) <= 1e-10 * np.linalg.norm(ref)
    # linearity and symmetry with the direct coarse solve, required by CG
    H = Hierarchy(P, coarse="direct")
    r1, r2 = rng.standard_normal(P.dof.ndof), rng.standard_normal(P.dof.ndof)
    v1, v2 = H.vcycle(r1), H.vcycle(r2)
    v12 = H.vcycle(2.0 * r1 - 3.0 * r2)
    assert np.linalg.norm(v12 - (2 * v1 - 3 * v2)) <= 1e-12 * np.linalg.norm(v12)
    assert abs(v1 @ r2 - r1 @ v2) <= 1e-10 * abs(v1 @ r2)


def test_standalone_mg_contracts(cfg1):
    # multigrid as a solver x += V(b - A x); every contraction number rho_i < 1
    # (a sign error in the coarse correction or a wrong omega makes it diverge).  The loop is
    # retyped here and must agree with Hierarchy.mg_solve step by step.
    H = Hierarchy(cfg1)
    A, b = cfg1.A, cfg1.b
    x = np.zeros_like(b)
    res = [np.linalg.norm(b)]
    for _ in range(12):
        x = x + H.vcycle(b - A @ x)
        res.append(np.linalg.norm(b - A @ x))
    rho = np.array(res[1:]) / np.array(res[:-1])
    assert rho.max() < 0.9
    xm, it, hist = H.mg_solve(b, rtol=0.0, maxit=12)
    assert it == 12 and np.allclose(np.array(hist), np.array(res) / res[0], rtol=1e-9)
    assert np.linalg.norm(xm - x) <= 1e-12 * np.linalg.norm(x)


def test_standalone_mg_single_level_is_exact():
    # one level with a direct coarse solve: V = A^{-1}, so the stand-alone solver
    # reaches the solution in one cycle (closed form: rho_1 = 0 up to rounding)
    from workloads import small_config
    P = Problem(small_config(3, 4, 1, voids=1, seed=3, coarse="direct"))
    H = Hierarchy(P)
    x, it, hist = H.mg_solve(P.b, rtol=1e-12, maxit=5)
    assert it == 1 and hist[1] < 1e-12
    xd = np.linalg.solve(P.A.toarray(), P.b)
    assert np.linalg.norm(x - xd) <= 1e-11 * np.linalg.norm(xd)


def test_coarse_cg_matches_direct(small3d):
    # inner AS-CG and direct coarse solve agree to 1e-10
    Hd = Hierarchy(small3d, coarse="direct")
    Hc = Hierarchy(small3d, coarse="as_pcg")
    Hj = Hierarchy(small3d, coarse="jacobi_pcg")
    r = small3d.b[small3d.dof.level_dofs(1)]
    xd = Hd.coarse_solve(r)
    for H in (Hc, Hj):
        x = H.coarse_solve(r)
        assert np.linalg.norm(x - xd) <= 1e-10 * np.linalg.norm(xd)
    assert Hc.coarse_iters[-1] < Hj.coarse_iters[-1]


def test_fcg_matches_direct_solve(cfg1):
    # P9: FCG + V-cycle solution vs the dense direct solution, consistent with rtol 1e-10
    H = Hierarchy(cfg1)
    x, it, hist = H.fcg(cfg1.b)
    xs = spla.spsolve(cfg1.A.tocsc(), cfg1.b)
    assert hist[-1] < 1e-10 and it < 30
    assert np.linalg.norm(cfg1.b - cfg1.A @ x) < 1e-10 * np.linalg.norm(cfg1.b) * 1.01
    A = cfg1.A
    # energy-norm error bounded by the residual: ||e||_A <= ||r|| / sqrt(lambda_min)
    assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)
    x0, it0, _ = fcg(lambda v: A @ v, np.zeros(cfg1.dof.ndof), H.vcycle, 1e-10, 10)
    assert it0 == 0 and not np.any(x0)


def _manufactured_energy_error(dim, n, p):
    """u = prod sin(pi x_i), f = d pi^2 prod sin(pi x_i) on the void-free unit box, u = 0
    on the boundary; returns the energy error sqrt(a(u,u) - b.x) (Galerkin orthogonality)."""
    cfg = small_config(dim, n, p, coarse="direct")
    dm = DofMap(cfg)
    modes = dm.modes
    P = Problem(cfg)
    h = 1.0 / n
    xg, wg = basis.gauss(p + 3)
    mesh = np.meshgrid(*([xg] * dim), indexing="ij")
    wm = np.meshgrid(*([wg] * dim), indexing="ij")
    ref = np.stack([m.ravel() for m in mesh], 1)
    w = np.prod(np.stack([m.ravel() for m in wm], 1), axis=1) * (h / 2) ** dim
    val, _ = basis.eval_element(modes, ref)
    b = np.zeros(dm.ndof)
    for c in range(n ** dim):
        cc = [(c // n ** a) % n for a in range(dim)]
        xp = (np.array(cc) + 0.5 * (ref + 1)) * h
        f = dim * math.pi ** 2 * np.prod(np.sin(math.pi * xp), axis=1)
        fe = val @ (w * f)
        ok = dm.cell_dofs[c] >= 0
        np.add.at(b, dm.cell_dofs[c][ok], fe[ok])
    H = Hierarchy(P)
    x, it, _ = H.fcg(b, rtol=1e-13)
    aa = dim * math.pi ** 2 / 2 ** dim
    return math.sqrt(max(aa - b @ x, 0.0))


@pytest.mark.parametrize("dim,p", [(2, 1), (2, 2), (2, 3), (3, 2)])
def test_manufactured_solution_rate(dim, p):
    # P10: energy error ratio ~ 2^p when h is halved (+-15%)
    n0 = 4 if dim == 2 else 2
    e1 = _manufactured_energy_error(dim, n0, p)
    e2 = _manufactured_energy_error(dim, 2 * n0, p)
    assert 2 ** p * 0.85 <= e1 / e2 <= 2 ** p * 1.15 * (1.2 if p == 3 else 1.0)


@pytest.mark.parametrize("n", [8, 16])
def test_paper_iteration_counts_2d_elementwise(n):
    # P11 (method level, loose): PAPER.md:493-496 CG + p-MG, elementwise AS (5,5), psi = 0,
    # tol 1e-9: 7-9 iterations.  Our square uses strong u = 0 and f = 1 instead of the
    # paper's penalty BC and manufactured source, so +-2 iterations.
    tab = GOLD["cg_mg_psi0_elementwise"]
    col = {8: 0, 16: 1}[n]
    for p in (2, 3, 4, 5):
        P = Problem(small_config(2, n, p, coarse="direct"))
        H = Hierarchy(P)
        assert H.omega == GOLD["omega"]["2d_element"]
        _, it, _ = H.fcg(P.b, rtol=1e-9)
        assert abs(it - tab[str(p)][col]) <= 2, (p, it)


# ---- the paper's own test problem (Sec. 4.1, psi = 0): penalty BC + manufactured source ----
def _square(n, p, block="element", **kw):
    from oracle.paper_square import SquareProblem
    return SquareProblem(n, p, block, **kw)


def test_square_problem_harness():
    # the harness itself, pinned without the multigrid: with a stiff penalty
    # the discrete solution converges spectrally to the manufactured u_bar at the vertices
    # (a wrong source sign, kappa or penalty term would leave an O(1) error); with the paper's
    # beta = 1e4 the boundary penalty error ~ kappa |du/dn| / beta ~ 1e-5 dominates.
    errs = []
    for p in (2, 3, 5):
        P = _square(8, p, beta=1e8)
        x = spla.spsolve(P.A.tocsc(), P.b)
        errs.append(P.nodal_error(x))
    assert errs[0] < 5e-6 and errs[1] < errs[0] / 5 and errs[2] < 5e-9, errs
    P = _square(8, 3)
    x = spla.spsolve(P.A.tocsc(), P.b)
    assert 1e-6 < P.nodal_error(x) < 3e-5
    # SPD with the penalty
    assert abs(P.A - P.A.T).max() < 1e-12 * abs(P.A).max()


@pytest.mark.parametrize("n", [8, 16])
def test_paper_square_elementwise_cg_counts_exact(n):
    # P11: CG + p-MG (V(5,5), elementwise AS, omega = 1/3), psi = 0, tol 1e-9: the oracle on
    # the paper's own problem reproduces every printed count exactly.
    tab = GOLD["cg_mg_psi0_elementwise"]
    col = {8: 0, 16: 1}[n]
    got = []
    for p in (2, 3, 4, 5):
        H = Hierarchy(_square(n, p))
        assert H.omega == GOLD["omega"]["2d_element"]
        _, it, _ = H.fcg(H.prob.b, rtol=GOLD["square_problem"]["tol"])
        got.append(it)
    assert got == [tab[str(p)][col] for p in (2, 3, 4, 5)], got


def test_paper_square_elementwise_mg_solver_counts():
    # multigrid as a stand-alone solver, h = 1/8: printed 12/10/17/14
    tab = GOLD["mg_solver_psi0_elementwise"]
    for p in (2, 3, 4, 5):
        H = Hierarchy(_square(8, p))
        _, it, hist = H.mg_solve(H.prob.b, rtol=1e-9, maxit=100)
        assert abs(it - tab[str(p)][0]) <= 1, (p, it)
        rho = np.array(hist[1:]) / np.array(hist[:-1])
        assert rho.max() < 0.5


def test_paper_square_patchwise_counts():
    # Reading R19.  Table 1 fixes the patch block as every DOF whose
    # support intersects the 2^d cells around a vertex, m = (2p+1)^d ("closure").  With those
    # blocks the oracle needs 3 CG iterations where the paper prints 5-6: a
    # superset of the blocks the printed counts imply.  The same patch machinery with the
    # "interior" membership predicate (support inside the patch, m = (2p-1)^d) reproduces the
    # printed CG counts to +-1 -- pinning the vertex enumeration, boundary clipping and
    # assembled sub-blocks -- and the closure blocks can only be stronger (never more iterations).
    tab = GOLD["cg_mg_psi0_patchwise"]
    for p in (2, 3, 4, 5):
        P = _square(8, p, "patch")
        Hi = Hierarchy(P, patch_rule="interior")
        assert Hi.omega == GOLD["omega"]["2d_patch"]
        _, it_i, _ = Hi.fcg(P.b, rtol=1e-9)
        assert abs(it_i - tab[str(p)][0]) <= 1, (p, it_i)
        Hc = Hierarchy(P)
        _, it_c, _ = Hc.fcg(P.b, rtol=1e-9)
        assert it_c <= it_i <= tab[str(p)][0] + 1
        sizes_c = {len(b) for b in Hc.levels[p].blocks}
        sizes_i = {len(b) for b in Hi.levels[p].blocks}
        assert max(sizes_c) == (2 * p + 1) ** 2 and (2 * p - 1) ** 2 in sizes_i
        for bi, bc in zip(Hi.levels[p].blocks, Hc.levels[p].blocks):   # same vertex order
            assert set(bi) <= set(bc)


def _patch_by_keys(dof, v, q, n, d):
    """Independent enumeration of a closure patch block from the DOF keys alone: the free
    level-q DOFs whose entity (key coordinates X = 2*vertex or 2*cell+1 per axis) lies in the
    closed box of the 2^d cells around vertex v (clipped to the grid)."""
    p = dof.cfg.p
    per = (p + 1) ** 3 * dof.cfg.n_f
    ent = dof.keys // per
    X = [ent % (2 * n + 1), (ent // (2 * n + 1)) % (2 * n + 1), ent // (2 * n + 1) ** 2]
    vc = [(v // (n + 1) ** a) % (n + 1) for a in range(d)]
    ok = dof.dof_order <= q
    for a in range(d):
        lo, hi = max(vc[a] - 1, 0), min(vc[a] + 1, n)
        ok &= (X[a] >= 2 * lo) & (X[a] <= 2 * hi)
    return np.nonzero(ok)[0]


@pytest.mark.parametrize("dim,n,p", [(2, 4, 3), (3, 3, 2), (3, 3, 4)])
def test_patch_membership_matches_key_enumeration(dim, n, p):
    # every vertex (interior, face, edge, corner; strong Dirichlet on all faces) on every
    # level: the oracle's patch block == the key-box enumeration; interior vertices have
    # Table 1's (2q+1)^d free DOFs when no Dirichlet entity is inside the box
    P = Problem(small_config(dim, n, p, coarse="direct", block="patch"))
    H = Hierarchy(P)
    for q in range(2, p + 1):
        lv = H.levels[q]
        blocks = {tuple(sorted(lv.idx[b])) for b in lv.blocks}
        ref = set()
        for v in range((n + 1) ** dim):
            g = _patch_by_keys(P.dof, v, q, n, dim)
            if len(g):
                ref.add(tuple(sorted(g)))
            vc = [(v // (n + 1) ** a) % (n + 1) for a in range(dim)]
            if all(2 <= c <= n - 2 for c in vc):
                assert len(g) == (2 * q + 1) ** dim
        assert blocks == ref, q
        assert max(len(b) for b in lv.blocks) <= (2 * q + 1) ** dim


# ---- h-coarsening below p = 1 (PAPER.md:227 Remark; reading R21) ---------------------------
def _p1_levels(n, dim=3, voids=None, **kw):
    from oracle.mg import GeometricLevels
    cfg = small_config(dim, n, 1, voids=voids, coarse="direct", **kw)
    P = Problem(cfg)
    H = Hierarchy(P, coarse="as_pcg")
    lv = H.levels[1]
    G = GeometricLevels(cfg, lv.A, P.dof.keys[lv.idx], lv.blocks, lv.inv, 2.0 / 15.0 if dim == 3 else 1.0 / 3.0,
                        5, 5)
    return cfg, P, G


@pytest.mark.parametrize("dim", [2, 3])
def test_gmg_prolongation_reproduces_multilinear_functions(dim):
    # standard (bi/tri)linear interpolation: P maps any multilinear function sampled on the
    # coarse vertices to the same function on the fine vertices (no Dirichlet elimination here)
    _, _, G = _p1_levels(8, dim, dirichlet=0)
    rng = np.random.default_rng(3)
    c = rng.standard_normal(1 << dim)
    def f(pos, n):
        x = pos[:, :dim] / n
        out = np.zeros(len(pos))
        for m in range(1 << dim):
            t = np.ones(len(pos))
            for a in range(dim):
                if (m >> a) & 1:
                    t = t * x[:, a]
            out += c[m] * t
        return out
    fc = f(G.pos[1], G.n[1])
    ff = f(G.pos[0], G.n[0])
    assert np.abs(G.P[0] @ fc - ff).max() < 1e-13
    # each fine vertex's weights sum to 1 (partition of unity)
    assert np.allclose(np.asarray(G.P[0].sum(axis=1)).ravel(), 1.0, atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_gmg_galerkin_equals_rediscretisation(dim):
    # on a void-free box the Galerkin operator P^T A_h P of nested (bi/tri)linear spaces is the
    # operator rediscretised on the coarse grid (independent assembly by the oracle's Problem)
    cfg, P, G = _p1_levels(8, dim)
    coarse = Problem(small_config(dim, 4, 1, coarse="direct"))
    assert np.array_equal(G.pos[1][:, :dim] * 2, np.stack(
        [((coarse.dof.keys // 8) // (9 ** a)) % 9 for a in range(dim)], 1))
    assert abs(G.A[1] - coarse.A).max() < 1e-13 * abs(coarse.A).max()


def test_gmg_vcycle_symmetric_and_pcg_exact():
    cfg, P, G = _p1_levels(8, 3, voids=2, seed=4)
    rng = np.random.default_rng(5)
    r1, r2 = rng.standard_normal((2, G.A[0].shape[0]))
    assert abs(r2 @ G.vcycle(r1) - r1 @ G.vcycle(r2)) < 1e-10 * abs(r1 @ G.vcycle(r1))
    x, it = pcg(lambda v: G.A[0] @ v, r1, G.vcycle, 1e-12, 100, rel_to="r0")
    xs = spla.spsolve(G.A[0].tocsc(), r1)
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs) and it <= 15


def test_gmg_coarse_iterations_h_independent():
    # the geometric V-cycle makes the p=1 solve's iteration count nearly h-independent
    # (CG + elementwise AS alone grows like 1/h)
    its = []
    for n in (8, 16):
        P = Problem(small_config(3, n, 2, coarse="gmg_pcg"))
        H = Hierarchy(P)
        I1 = P.dof.level_dofs(1)
        H.coarse_solve(P.b[I1])
        its.append(H.coarse_iters[-1])
    assert its[1] <= its[0] + 2 and its[1] <= 10, its
