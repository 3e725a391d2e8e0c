"""L0 of the parity ladder: the product's workload generator (C++ in
libfcm_mg.so, no GPU needed) against the oracle's quadrature, plus the C-ABI export check."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import geometry
from oracle.problem import Problem
from paper_2010_00881_b200 import _lib
from paper_2010_00881_b200.fcm import generate
from workloads import config_voids, get_config, small_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "fcm_mg.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(fcm_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name


CASES = [
    ("cfg1", get_config("cfg1")),
    ("3d_p2_voids", small_config(3, 6, 2, voids=3, seed=1)),
    ("3d_p3_voids", small_config(3, 5, 3, voids=2, seed=4)),
    ("3d_p4", small_config(3, 4, 4, voids=2, seed=5)),
    ("3d_trunk_elast", small_config(3, 4, 3, space="trunk", physics="elasticity", voids=2, seed=6)),
    ("2d_p5_depth4", small_config(2, 6, 5, voids=2, seed=3, depth=4)),
]


@pytest.mark.parametrize("name,cfg", CASES, ids=[c[0] for c in CASES])
def test_generator_matches_oracle(name, cfg):
    c, r = config_voids(cfg)
    P = Problem(cfg, c, r, build_csr=False)
    G = generate(cfg, c, r)
    assert np.array_equal(G.kind, P.kinds)
    assert np.array_equal(G.cut_cells, P.cut_cells)
    scale = np.abs(P.K_ref).max()
    assert np.abs(G.K_ref - P.K_ref).max() <= 1e-13 * scale
    assert np.allclose(G.f_ref, P.f_ref, rtol=0, atol=1e-15 * max(1e-300, np.abs(P.f_ref).max()) + 1e-300) \
        or np.abs(G.f_ref - P.f_ref).max() <= 1e-14 * np.abs(P.f_ref).max()
    if len(P.cut_cells):
        err = np.sqrt(((G.cut_K - P.cut_K) ** 2).sum(axis=(1, 2)))
        nrm = np.sqrt((P.cut_K ** 2).sum(axis=(1, 2)))
        assert (err / nrm).max() <= 1e-12
        if cfg.physics == "poisson":
            ferr = np.abs(G.cut_f - P.cut_f).max(axis=1) / np.abs(P.cut_f).max(axis=1)
            assert ferr.max() <= 1e-12
    if cfg.traction_face >= 0:
        from oracle import quadrature
        ft = quadrature.traction_load(cfg, (0,) * cfg.dim, cfg.traction_face, P.modes)
        assert np.abs(G.f_traction - ft).max() <= 1e-14 * np.abs(ft).max()


def test_generator_cfg2_sample():
    # config 2 at full size: classification of every cell, element matrices of sampled cut cells
    cfg = get_config("cfg2")
    c, r = config_voids(cfg)
    G = generate(cfg, c, r)
    kinds = geometry.classify_cells(3, cfg.n, c, r)
    assert np.array_equal(G.kind, kinds)
    assert (G.kind == 2).sum() == 1039 and (G.kind == 1).sum() == 266
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(G.cut_cells, 12, replace=False))
    P = Problem(cfg, c, r, build_csr=False, cut_cells_only=sample)
    for cell in sample:
        i = np.searchsorted(G.cut_cells, cell)
        Kg, Ko = G.cut_K[i], P.cut_K[P.cut_index[cell]]
        assert np.linalg.norm(Kg - Ko) <= 1e-12 * np.linalg.norm(Ko)
