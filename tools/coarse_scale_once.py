"""One coarse solve of the config-5 geometry at p = 1 (ncu target for the grid-wide kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg5")).replace(p=1, coarse_maxit=int(os.environ.get("MAXIT", "20")))
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
x, it = S.coarse_solve(b)
torch.cuda.synchronize()
print("iters", it)
