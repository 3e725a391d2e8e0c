"""A small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
elementwise 3D p=2 with the tiled coarse kernel, patchwise 3D p=3 (k_patch_smooth streaming +
fast-diagonalisation warps, batched Gauss-Jordan setup) and the grid-wide coarse kernel."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import small_config  # noqa: E402

cases = [small_config(3, 6, 2, voids=3, seed=1), small_config(3, 4, 3, voids=1, seed=7, block="patch")]
for cfg in cases:
    G = generate(cfg)
    S = Solver.from_problem(cfg, G)
    b = S.load(G)
    x, it, hist = S.pcg_solve(b)
    torch.cuda.synchronize()
    print(cfg.name, "FCG iterations", it, "relres", hist[-1], S.coarse_info()[0], flush=True)
os.environ["FCM_COARSE_TILED"] = "0"
cfg = cases[0]
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
x, it, hist = S.pcg_solve(b)
torch.cuda.synchronize()
print(cfg.name, "grid-wide coarse: FCG iterations", it, S.coarse_info()[0], flush=True)
