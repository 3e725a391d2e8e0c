"""FCM_PATCH_PROF=1: when do the streaming and the fast-diagonalisation warps of k_patch_smooth
finish inside one launch (cfg3, each patch level, fused / streaming-only / FD-only)."""
import os
import sys

import torch

os.environ["FCM_PATCH_PROF"] = "1"
sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
del G
for q in range(2, cfg.p + 1):
    r = b[: S.ndofs(q)].clone()
    x = torch.zeros_like(r)
    for k in (0, 1, 2):
        for _ in range(3):
            S.smooth_part(r, x, q, k)
        torch.cuda.synchronize()
