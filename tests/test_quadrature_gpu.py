"""L0 on the device: fcm_gen_cut_matrices_device (the GPU space-tree quadrature)
against the oracle's quadrature (oracle/quadrature.py) and against the host generator, per cut
cell, <= 1e-12 relative Frobenius (the two sides sum the same leaf integrals in different
orders; the box classification is bit-identical by construction)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.problem import Problem  # noqa: E402
from workloads import config_voids, get_config, small_config  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [
    ("cfg1", get_config("cfg1")),
    ("3d_p2_voids", small_config(3, 6, 2, voids=3, seed=1)),
    ("3d_p3_voids", small_config(3, 5, 3, voids=2, seed=4)),
    ("3d_p4", small_config(3, 4, 4, voids=2, seed=5)),
    ("2d_p5_depth4", small_config(2, 6, 5, voids=2, seed=3, depth=4)),
    ("3d_p2_depth1", small_config(3, 5, 2, voids=2, seed=2, depth=1)),
]


def _rel_per_cell(A, B):
    err = np.sqrt(((A - B) ** 2).reshape(len(A), -1).sum(axis=1))
    nrm = np.sqrt((B ** 2).reshape(len(B), -1).sum(axis=1))
    return (err / nrm).max()


@pytest.mark.parametrize("name,cfg", CASES, ids=[c[0] for c in CASES])
def test_device_quadrature_matches_oracle(name, cfg):
    from paper_2010_00881_b200.fcm import generate
    c, r = config_voids(cfg)
    P = Problem(cfg, c, r, build_csr=False)
    G = generate(cfg, c, r, device=True)
    assert np.array_equal(G.cut_cells, P.cut_cells) and len(G.cut_cells) > 0
    assert _rel_per_cell(G.cut_K, P.cut_K) <= 1e-12
    assert _rel_per_cell(G.cut_f, P.cut_f) <= 1e-12
    assert np.array_equal(G.cut_K, np.swapaxes(G.cut_K, 1, 2))   # exactly symmetric


@pytest.mark.parametrize("cfg_name,count", [("cfg2", 200), ("cfg3", 96), ("cfg5", 200)])
def test_device_quadrature_matches_host_generator_full_size(cfg_name, count):
    # the BASELINE configs' own geometry (seeded voids, cell size, p): a sample of cut cells,
    # device vs the host C++ generator
    from paper_2010_00881_b200.fcm import classify, generate
    cfg = get_config(cfg_name)
    c, r = config_voids(cfg)
    kind, _ = classify(cfg, c, r)
    cut = np.nonzero(kind == 2)[0]
    rng = np.random.default_rng(1)
    sample = np.sort(rng.choice(cut, min(count, len(cut)), replace=False)).astype(np.int64)
    Gd = generate(cfg, c, r, cut_cells=sample, kind=kind, device=True)
    Gh = generate(cfg, c, r, cut_cells=sample, kind=kind, device=False)
    assert _rel_per_cell(Gd.cut_K, Gh.cut_K) <= 1e-12
    assert _rel_per_cell(Gd.cut_f, Gh.cut_f) <= 1e-12
