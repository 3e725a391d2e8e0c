"""Pins of oracle/basis.py and oracle/dofmap.py against closed forms and the paper's
Table 1 (no GPU).  Each pin states what a plausible mistake it would catch."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import basis
from oracle.dofmap import DofMap
from workloads import get_config, small_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_nodal_and_vanishing_modes():
    # nodal Kronecker property at the endpoints; internal modes vanish
    v, _ = basis.modes_1d(5, [-1.0, 1.0])
    assert np.allclose(v[:, 0], [1, 0, 0, 0, 0, 0], atol=1e-15)
    assert np.allclose(v[:, 1], [0, 1, 0, 0, 0, 0], atol=1e-15)
    v, _ = basis.modes_1d(1, [0.0])
    assert np.allclose(v[:, 0], [0.5, 0.5])


def _gram(p, deriv):
    x, w = np.polynomial.legendre.leggauss(20)
    v, d = basis.modes_1d(p, x)
    f = d if deriv else v
    return (f * w) @ f.T


@pytest.mark.parametrize("p", [1, 2, 3, 6])
def test_1d_stiffness_closed_form(p):
    # P1: K = [[1/2,-1/2],[-1/2,1/2]] (+) I_{p-1}  (normalisation R-B1 / S:72)
    K = _gram(p, True)
    ref = np.zeros((p + 1, p + 1))
    ref[:2, :2] = [[0.5, -0.5], [-0.5, 0.5]]
    ref[2:, 2:] = np.eye(p - 1)
    assert np.allclose(K, ref, atol=5e-14)


@pytest.mark.parametrize("p", [2, 3, 5, 7])
def test_1d_mass_closed_form(p):
    # P1 closed forms of the integrated-Legendre mass matrix
    M = _gram(p, False)
    ref = np.zeros((p + 1, p + 1))
    ref[0, 0] = ref[1, 1] = 2 / 3
    ref[0, 1] = ref[1, 0] = 1 / 3
    ref[0, 2] = ref[2, 0] = ref[1, 2] = ref[2, 1] = -1 / math.sqrt(6)
    if p >= 3:
        ref[0, 3] = ref[3, 0] = 1 / (3 * math.sqrt(10))
        ref[1, 3] = ref[3, 1] = -1 / (3 * math.sqrt(10))
    for k in range(2, p + 1):
        ref[k, k] = 2 / ((2 * k + 1) * (2 * k - 3))
        if k + 2 <= p:
            ref[k, k + 2] = ref[k + 2, k] = -1 / ((2 * k + 1) * math.sqrt((2 * k - 1) * (2 * k + 3)))
    assert np.allclose(M, ref, atol=5e-14)


def test_derivatives_match_finite_differences():
    x = np.linspace(-0.9, 0.9, 7)
    eps = 1e-6
    _, d = basis.modes_1d(5, x)
    vp, _ = basis.modes_1d(5, x + eps)
    vm, _ = basis.modes_1d(5, x - eps)
    assert np.allclose(d, (vp - vm) / (2 * eps), atol=1e-8)


@pytest.mark.parametrize("dim,space", [(2, "tensor"), (3, "tensor"), (2, "trunk"), (3, "trunk")])
def test_hierarchical_prefix(dim, space):
    # P:34 "the set of basis functions of order p contains all basis functions from order 1 up to p";
    # the level-q modes are a prefix of the order-p list (so level matrices are leading blocks)
    for p in range(1, 6):
        full = basis.element_modes(dim, p, space)
        for q in range(1, p + 1):
            sub = basis.element_modes(dim, q, space)
            assert full[:len(sub)] == sub
            assert all(basis.mode_order(m, space) <= q for m in sub)
            assert all(basis.mode_order(m, space) > q for m in full[len(sub):])


def test_mode_counts():
    # S:33, S:53-55 (2D): tensor (p+1)^2; trunk 4 + 4(p-1) + (p-2)(p-3)/2
    for p in range(1, 8):
        assert len(basis.element_modes(2, p, "tensor")) == (p + 1) ** 2
        assert len(basis.element_modes(2, p, "trunk")) == 4 + 4 * (p - 1) + ((p - 2) * (p - 3) // 2 if p >= 3 else 0)
        assert len(basis.element_modes(3, p, "tensor")) == (p + 1) ** 3
    assert len(basis.element_modes(2, 2, "trunk")) == 8
    assert len(basis.element_modes(2, 4, "trunk")) == 17


def _table1(space, n, p, n_f):
    t = GOLD["table1_mmax"]
    if space == "tensor":
        return eval(t["tensor"])
    if p < 4:
        return eval(t["trunk_p_lt_4"])
    if p <= 5:
        return eval(t["trunk_4_le_p_le_5"])
    return eval(t["trunk_p_ge_6_printed"]) / 6.0   # reading G1


def _patch_size(space, p, n_f):
    # number of DOFs supported on the 2x2x2 cells around an interior vertex (n = 2 patch)
    cfg = small_config(3, 4, p, space=space, dirichlet=0,
                       physics="elasticity" if n_f == 3 else "poisson", traction_face=-1)
    dm = DofMap(cfg)
    cells = [(cz * 4 + cy) * 4 + cx for cz in (1, 2) for cy in (1, 2) for cx in (1, 2)]
    return len(np.unique(dm.cell_dofs[cells]))


@pytest.mark.parametrize("space", ["tensor", "trunk"])
def test_table1_block_sizes(space):
    # P:316-320 Table 1: maximum AS block size m_max, n = 1 elementwise, n = 2 patchwise
    for p in range(1, 8):
        m_el = len(basis.element_modes(3, p, space))
        assert m_el == _table1(space, 1, p, 1)
        assert 3 * m_el == _table1(space, 1, p, 3)
    for p in range(1, 5):
        assert _patch_size(space, p, 1) == _table1(space, 2, p, 1)
    assert _patch_size(space, 2, 3) == _table1(space, 2, 2, 3)


def test_dof_counts_configs():
    # BASELINE.json configs: cfg1 "~2.4k DOFs", cfg2 "~275k DOFs"; full grids (R9)
    d1 = DofMap(get_config("cfg1"))
    assert d1.ndof == (3 * 16 - 1) ** 2  # 2209 free of (3*16+1)^2 = 2401
    d2 = DofMap(get_config("cfg2"))
    assert d2.ndof == (2 * 32 - 1) ** 3  # 250,047 free of 65^3 = 274,625


def test_trunk_elasticity_count_formula():
    # cfg4: trunk p=3, n_f=3: n_f[(n+1)^3 + 3 n (n+1)^2 (p-1)] total ("~5.7M" at n=64, R10)
    def total(n):
        return 3 * ((n + 1) ** 3 + 3 * n * (n + 1) ** 2 * 2)

    def free(n):  # x = 0 face clamped: drop nodal x position 0
        # vertices n(n+1)^2; x-edges n(n+1)^2; y-, z-edges n*n*(n+1) each; 2 modes per edge
        return 3 * (n * (n + 1) ** 2 + (n * (n + 1) ** 2 + 2 * n * n * (n + 1)) * 2)
    for n in (2, 3):
        cfg = small_config(3, n, 3, space="trunk", physics="elasticity", dirichlet=0, traction_face=-1)
        assert DofMap(cfg).ndof == total(n)
        cfg = small_config(3, n, 3, space="trunk", physics="elasticity")
        assert DofMap(cfg).ndof == free(n)
    assert total(64) == 5_691_075
    assert free(64) == 5_628_480


def test_dofmap_sharing_and_keys():
    # conformity: a vertex DOF is shared by 2^d cells, an interior-mode DOF by 1
    cfg = small_config(3, 3, 3, dirichlet=0)
    dm = DofMap(cfg)
    counts = np.bincount(dm.cell_dofs.ravel(), minlength=dm.ndof)
    modes = dm.modes
    # DOF of the centre vertex (1,1,1)... every interior vertex appears in 8 cells
    assert counts.max() == 8
    interior = [i for i, m in enumerate(modes) if min(m) >= 2]
    assert np.all(counts[dm.cell_dofs[:, interior].ravel()] == 1)
    assert np.all(np.diff(dm.keys) > 0)
