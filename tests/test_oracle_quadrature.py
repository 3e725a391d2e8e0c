"""Pins of oracle/quadrature.py and oracle/geometry.py (no GPU): closed-form
Kronecker element matrices, alpha-consistency, volumes, loads, elasticity energies."""
import math

import numpy as np
import pytest

from oracle import basis, geometry, quadrature
from oracle.problem import Problem
from workloads import get_config, small_config


def _K1M1(p):
    """1D reference stiffness / mass on [-1,1], written out from the closed forms (P1),
    independent of the quadrature code."""
    K = np.zeros((p + 1, p + 1))
    K[:2, :2] = [[0.5, -0.5], [-0.5, 0.5]]
    K[2:, 2:] = np.eye(p - 1)
    M = np.zeros((p + 1, p + 1))
    M[0, 0] = M[1, 1] = 2 / 3
    M[0, 1] = M[1, 0] = 1 / 3
    if p >= 2:
        M[0, 2] = M[2, 0] = M[1, 2] = M[2, 1] = -1 / math.sqrt(6)
    if p >= 3:
        M[0, 3] = M[3, 0] = 1 / (3 * math.sqrt(10))
        M[1, 3] = M[3, 1] = -1 / (3 * math.sqrt(10))
    for k in range(2, p + 1):
        M[k, k] = 2 / ((2 * k + 1) * (2 * k - 3))
        if k + 2 <= p:
            M[k, k + 2] = M[k + 2, k] = -1 / ((2 * k + 1) * math.sqrt((2 * k - 1) * (2 * k + 3)))
    return K, M


def _kron_Kref(dim, p, h, modes):
    # P2: 2D K_ref = K(x)M + M(x)K ; 3D K_ref = (h/2)(K(x)M(x)M + M(x)K(x)M + M(x)M(x)K)
    K, M = _K1M1(p)
    nm = len(modes)
    out = np.zeros((nm, nm))
    for i, a in enumerate(modes):
        for j, b in enumerate(modes):
            s = 0.0
            for g in range(dim):
                t = 1.0
                for ax in range(dim):
                    t *= (K if ax == g else M)[a[ax], b[ax]]
                s += t
            out[i, j] = s * (h / 2) ** (dim - 2)
    return out


@pytest.mark.parametrize("dim,p", [(2, 1), (2, 3), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_Kref_kronecker_closed_form(dim, p):
    cfg = small_config(dim, 4, p)
    modes = basis.element_modes(dim, p)
    K, f = quadrature.element_matrices(cfg, (1,) * dim, np.zeros((0, dim)), np.zeros(0), modes)
    ref = _kron_Kref(dim, p, 1.0 / 4, modes)
    assert np.abs(K - ref).max() <= 1e-14 * np.abs(ref).max()
    # exactly one zero eigenvalue (constants) for scalar Poisson (P2)
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 1
    # body load f = 1: product of 1D mode integrals (int N0 = int N1 = 1, int N2 = -2/sqrt6, else 0)
    I1 = np.zeros(p + 1)
    I1[:2] = 1.0
    if p >= 2:
        I1[2] = -2 / math.sqrt(6)
    fref = np.array([np.prod([I1[k] for k in m]) for m in modes]) * (0.5 / 4) ** dim
    assert np.allclose(f, fref, atol=1e-16)


@pytest.mark.parametrize("p,nnz", [(1, 40), (2, 641), (3, 2208), (4, 3889)])
def test_Kref_sparsity_3d(p, nnz):
    # SURVEY §8(c) P2 counts of structurally nonzero K_ref entries in 3D
    modes = basis.element_modes(3, p)
    ref = _kron_Kref(3, p, 1.0, modes)
    assert int((np.abs(ref) > 1e-14).sum()) == nnz


@pytest.mark.parametrize("cfg", [get_config("cfg1"), small_config(3, 6, 2, voids=3, seed=1)],
                         ids=["cfg1", "3d"])
def test_alpha_one_consistency(cfg):
    # P3: with alpha = 1 every cut-cell matrix equals K_ref (Gauss rules exact on the leaves);
    # with alpha = eps everywhere inside the voids it is between eps*K_ref and K_ref
    P1 = Problem(cfg.replace(alpha=1.0), build_csr=False)
    assert len(P1.cut_cells) > 0
    err = np.abs(P1.cut_K - P1.K_ref[None]).max()
    assert err <= 1e-13 * np.abs(P1.K_ref).max()
    assert np.allclose(P1.cut_f, P1.f_ref[None], atol=1e-15)


def _alpha_volume(cfg, centres, radii):
    """int alpha over [0,1]^d by the space-tree rule (sum of cell load partition of unity)."""
    P = Problem(cfg, centres, radii, build_csr=False)
    vert = [i for i, m in enumerate(P.modes) if max(m) < 2]
    tot = 0.0
    for c in range(cfg.n ** cfg.dim):
        tot += P.element_load(c)[vert].sum()
    return tot


def test_volume_converges_with_depth():
    # P4: sum of vertex loads (partition of unity, f = 1) = int alpha; -> |phys| + eps|fict|
    c = np.array([[0.43, 0.52, 0.47]])
    r = np.array([0.31])
    exact = 1.0 - (1 - 1e-8) * 4 / 3 * math.pi * r[0] ** 3
    errs = []
    for depth in (0, 1, 2, 3):
        cfg = small_config(3, 4, 1, voids=(c, r), depth=depth, dirichlet=0)
        errs.append(abs(_alpha_volume(cfg, c, r) - exact))
    vvoid = 4 / 3 * math.pi * r[0] ** 3
    # a dropped leaf, a wrong leaf weight or a missing alpha is an O(vvoid) error
    assert max(errs[1:]) < 5e-3 * vvoid
    assert errs[3] < errs[0]


def test_classification_exact():
    c = np.array([[0.5, 0.5, 0.5]])
    r = np.array([0.25])
    assert geometry.classify_box([0.45] * 3, [0.55] * 3, c, r) == geometry.FICT
    assert geometry.classify_box([0.0] * 3, [0.1] * 3, c, r) == geometry.PHYS
    assert geometry.classify_box([0.7, 0.45, 0.45], [0.8, 0.55, 0.55], c, r) == geometry.CUT
    # a box touching the sphere from outside at one point is physical (R14 tie-break)
    assert geometry.classify_box([0.75, 0.4, 0.4], [0.9, 0.6, 0.6], c, r) == geometry.PHYS
    assert not geometry.point_is_fictitious([[0.75, 0.5, 0.5]], c, r)[0]


def test_config_geometry_statistics():
    # SURVEY §8 "Seeded geometry statistics": cfg1 28 cut / 32 fict; cfg2 1039 cut / 266 fict
    from workloads import config_voids
    for name, cut, fict in (("cfg1", 28, 32), ("cfg2", 1039, 266)):
        cfg = get_config(name)
        c, r = config_voids(cfg)
        k = geometry.classify_cells(cfg.dim, cfg.n, c, r)
        assert (k == geometry.CUT).sum() == cut and (k == geometry.FICT).sum() == fict


def _lin_field(modes, h, fn):
    """Element vector of a vector field linear in x (vertex DOFs only), n_f = 3."""
    u = np.zeros(len(modes) * 3)
    for i, m in enumerate(modes):
        if max(m) < 2:
            x = np.array(m, dtype=float) * h
            u[3 * i:3 * i + 3] = fn(x)
    return u


def test_elasticity_energies():
    # lam/mu placement pins: pure dilatation u = x has energy density 9lam + 6mu,
    # simple shear u = (y,0,0) has mu; 6 rigid-body zero modes
    cfg = small_config(3, 2, 2, physics="elasticity", E=2.0, nu=0.25)
    modes = basis.element_modes(3, 2)
    h = 0.5
    K, f = quadrature.element_matrices(cfg, (0, 0, 0), np.zeros((0, 3)), np.zeros(0), modes)
    lam, mu = quadrature.lame(2.0, 0.25)
    u = _lin_field(modes, h, lambda x: x)
    assert u @ K @ u == pytest.approx((9 * lam + 6 * mu) * h ** 3, rel=1e-13)
    u = _lin_field(modes, h, lambda x: np.array([x[1], 0, 0]))
    assert u @ K @ u == pytest.approx(mu * h ** 3, rel=1e-13)
    u = _lin_field(modes, h, lambda x: np.array([0, x[0], 0]))
    v = _lin_field(modes, h, lambda x: np.array([x[1], 0, 0]))
    # u + v is the rotation-free pure shear: energy 4*mu*(1/2)^2*... check bilinearity
    assert (u + v) @ K @ (u + v) == pytest.approx(4 * mu * h ** 3, rel=1e-13)
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 6
    assert np.abs(K - K.T).max() < 1e-15 * np.abs(K).max()
    assert np.all(f == 0)


def test_traction_load():
    # int_{x=1} N . (1,0,0): vertex x-loads on the face sum to the face area, y/z loads vanish
    cfg = small_config(3, 4, 3, space="trunk", physics="elasticity")
    P = Problem(cfg, build_csr=False)
    vert = [i for i, m in enumerate(P.modes) if max(m) < 2]
    tot = np.zeros(3)
    for c in range(cfg.n ** 3):
        fl = P.element_load(c)
    # assembled vector: sum over free vertex DOFs of component 0
    keys = P.dof.keys
    comp = keys % 3
    md = (keys // 3)
    degs = md % (4 ** 3)
    is_vertex = degs == 0
    for k in range(3):
        tot[k] = P.b[is_vertex & (comp == k)].sum()
    assert tot[0] == pytest.approx(1.0, rel=1e-13)
    assert abs(tot[1]) < 1e-15 and abs(tot[2]) < 1e-15
