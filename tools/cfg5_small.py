"""cfg5's void recipe (1000 seeded voids, r in [0.01, 0.03], seed 5) on a coarser grid, GPU vs
CPU oracle on IDENTICAL element matrices (the product generator's, fed to both): FCG residual
histories, elementwise vs patchwise Schwarz.  Is the slow FCG convergence of config 5 the
method or the implementation?  Usage: tools/cfg5_small.py n [maxit]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import assembly  # noqa: E402
from oracle.mg import Hierarchy  # noqa: E402
from oracle.problem import Problem  # noqa: E402
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import config_voids, get_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = {"n": n}
for block in ("element", "patch"):
    cfg = get_config("cfg5").replace(n=n, block=block, name=f"cfg5_n{n}_{block}")
    c, r = config_voids(cfg)
    G = generate(cfg, c, r)
    P = Problem(cfg, c, r, build_csr=False, cut_cells_only=[])
    assert np.array_equal(P.cut_cells, G.cut_cells)
    P.cut_K, P.cut_f = G.cut_K, G.cut_f
    P.A = assembly.csr_matrix(P)
    P.b = P._load()
    S = Solver(cfg, P.K_ref, P.kinds, P.cut_cells, P.cut_K)
    pos = np.searchsorted(P.dof.keys, S.dof_keys())
    b = torch.from_numpy(np.ascontiguousarray(P.b[pos])).cuda()
    x, it, hist = S.pcg_solve(b, maxit=maxit)
    t0 = time.time()
    H = Hierarchy(P)
    xo, ito, ho = H.fcg(P.b, maxit=maxit)
    out[block] = {"ndof": int(P.dof.ndof), "n_cut": int(len(G.cut_cells)), "gpu_iters": it,
                  "oracle_iters": ito, "gpu_hist": [float(v) for v in hist],
                  "oracle_hist": [float(v) for v in ho], "oracle_s": time.time() - t0,
                  "coarse_iters_oracle_mean": float(np.mean(H.coarse_iters)) if H.coarse_iters else 0}
    print(json.dumps({block: {k: v for k, v in out[block].items() if "hist" not in k}}), flush=True)
print(json.dumps(out))
