"""Native multi-level hp generator (gen_hp.cpp, host code of libfcm_mg.so) against the oracle
(oracle/mlhp.py): DOF sets (keys), level prefixes, load vector, leaf matrices (assembled), at
1e-13 -- the generator's parity level L0 for the hp path.  CPU only (no GPU needed)."""
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from hp_common import HP_CASES, hp_config, key_perm  # noqa: E402


@pytest.mark.parametrize("name", sorted(HP_CASES))
def test_hp_generator_matches_oracle(name):
    from oracle.mlhp import MlhpProblem
    from paper_2010_00881_b200.fcm import HpDisc
    cfg = hp_config(name)
    D = HpDisc(cfg)
    P = MlhpProblem(cfg)
    assert D.ndof == P.ndof
    perm = key_perm(P, D.keys())
    # levels: same sequence, same sizes, and every level is a PREFIX of the library's numbering
    seq = P.level_sequence()
    assert list(zip(D.level_q.tolist(), D.level_k.tolist())) == seq
    for l, (q, kc) in enumerate(seq):
        lv = set(P.level_dofs(q, kc).tolist())
        assert D.level_n[l] == len(lv)
        assert set(perm[:D.level_n[l]].tolist()) == lv
    b = D.load()
    assert np.linalg.norm(b - P.b[perm]) <= 1e-13 * np.linalg.norm(P.b)
    ptr, dofs, K, info = D.leaves()
    assert D.nleaves == len(P.mesh.leaves)
    rows, cols, vals, o = [], [], [], 0
    for L in range(D.nleaves):
        d = dofs[ptr[L]:ptr[L + 1]]
        assert np.all(np.diff(d) > 0), "leaf DOFs ascending (level prefixes)"
        g = perm[d]
        m = len(g)
        Ke = K[o:o + m * m].reshape(m, m)
        assert np.allclose(Ke, Ke.T, rtol=0, atol=1e-14 * max(1.0, np.abs(Ke).max()))
        rows.append(np.repeat(g, m))
        cols.append(np.tile(g, m))
        vals.append(Ke.ravel())
        o += m * m
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(P.ndof, P.ndof)).tocsr()
    assert abs(A - P.A).max() <= 1e-13 * abs(P.A).max()


def test_hp_generator_rejects_bad_spec():
    from paper_2010_00881_b200._lib import FcmError
    from paper_2010_00881_b200.fcm import HpDisc
    from workloads import small_config
    with pytest.raises(FcmError):
        HpDisc(small_config(2, 4, 2, kmax=9))


def test_hp_abi_rejects_null_handles():
    """The multi-level hp and low-rank entry points check their arguments before touching the
    device (CPU-safe): NULL handles / buffers give FCM_EINVAL and a message."""
    import ctypes as C
    from paper_2010_00881_b200 import _lib
    L = _lib.lib()
    i64, i32, f = C.c_int64(), C.c_int32(), C.c_float()
    assert L.fcm_hp_setup(None, None, None) == -1
    assert L.fcm_hp_apply(None, 0, None, None) == -1
    assert L.fcm_hp_smooth(None, 0, None, None) == -1
    assert L.fcm_hp_vcycle(None, None, None) == -1
    assert L.fcm_hp_pcg_solve(None, None, None, 1e-10, 10, C.byref(i32), None) == -1
    assert L.fcm_hp_mg_solve(None, None, None, 1e-10, 10, C.byref(i32), None) == -1
    assert L.fcm_hp_time_smooth(None, 0, None, None, 5, C.byref(f)) == -1
    assert L.fcm_hp_export_blocks(None, 0, C.byref(i64), C.byref(i64), C.byref(i64), None, None, None) == -1
    assert L.fcm_hp_stats(None, None, None, None) == -1
    assert L.fcm_mg_lowrank_info(None, 2, C.byref(i64), C.byref(i64)) == -1
    assert L.fcm_hp_disc_info(None, None, None, None, None, None) == -1
    assert b"NULL" in L.fcm_last_error() or len(L.fcm_last_error()) > 0
