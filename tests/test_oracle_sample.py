"""Pins of oracle/sample.py (per-row operator / load / Schwarz samples used at full workload
size) against the oracle's global forms on small grids: assembly (CSR A, load b) and mg.Level's
assembled Schwarz blocks, elementwise and patchwise (R11, R19), scalar and elasticity."""
import numpy as np
import pytest

from oracle.mg import Hierarchy
from oracle.problem import Problem
from oracle.sample import LazyCells, load_row, operator_row, schwarz_row
from workloads import small_config

CASES = [
    dict(dim=3, n=5, p=2, voids=2, seed=5),
    dict(dim=3, n=4, p=3, voids=1, seed=7, block="patch"),
    dict(dim=2, n=6, p=3, voids=1, seed=3, block="patch"),
    dict(dim=3, n=4, p=2, space="trunk", physics="elasticity", voids=1, seed=6),
]


@pytest.mark.parametrize("args", CASES)
def test_rows_match_global_oracle(args):
    cfg = small_config(**args)
    P = Problem(cfg)
    H = Hierarchy(P)
    L = LazyCells(cfg)
    assert np.array_equal(L.dof.keys, P.dof.keys) and np.array_equal(L.kinds, P.kinds)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(P.dof.ndof)
    rows = rng.choice(P.dof.ndof, size=12, replace=False)
    for q in range(1, cfg.p + 1):
        I = P.dof.level_dofs(q)
        xq = np.zeros_like(x)
        xq[I] = x[I]
        ref = P.A[I][:, I] @ x[I]
        full = np.zeros_like(x)
        full[I] = ref
        for i in rows:
            if P.dof.dof_order[i] <= q:
                assert abs(operator_row(L, xq, int(i), q) - full[i]) <= 1e-12 * np.abs(P.A).dot(np.abs(xq)).max()
    if cfg.traction_face < 0:
        for i in rows:
            assert abs(load_row(L, int(i)) - P.b[i]) <= 1e-13 * np.abs(P.b).max()
    for q in range(2, cfg.p + 1):
        lv = H.levels[q]
        r = rng.standard_normal(lv.n)
        ref = lv.omega * lv.schwarz(r)
        rfull = np.zeros(P.dof.ndof)
        rfull[lv.idx] = r
        pos = np.full(P.dof.ndof, -1)
        pos[lv.idx] = np.arange(lv.n)
        for i in rows[:5]:
            if pos[i] < 0:
                continue
            v = schwarz_row(L, rfull, int(i), q, H.block, lv.omega)
            assert abs(v - ref[pos[i]]) <= 1e-10 * np.abs(ref).max(), (q, i, v, ref[pos[i]])
