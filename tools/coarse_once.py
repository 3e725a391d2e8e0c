"""Run the cfg2 coarse solve a few times (target for ncu captures of the coarse kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
S = Solver.from_problem(cfg, G, coarse=os.environ.get("COARSE", "as_pcg"))
b = S.load(G)
r = b[: S.ndofs(1)].clone()
for _ in range(int(os.environ.get("REPS", "3"))):
    x, it = S.coarse_solve(r)
torch.cuda.synchronize()
print("iters", it)
