"""Coarse-level cost at config-5 scale without the p=3 quadrature: the config-5 geometry at
p = 1 (the coarse level alone: 16.6M DOFs), one coarse solve of the load vector, timed."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg5")).replace(p=1)
t = time.time(); G = generate(cfg); print(f"generator {time.time() - t:.1f}s cut {len(G.cut_cells)}", flush=True)
t = time.time(); S = Solver.from_problem(cfg, G); b = S.load(G); torch.cuda.synchronize()
print(f"setup {time.time() - t:.1f}s ndofs {S.ndofs(1)} kernel {S.coarse_info()}", flush=True)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    x, it = S.coarse_solve(b)
    torch.cuda.synchronize()
    dt = time.time() - t
    print(f"coarse solve: {it} iterations, {dt*1e3:.1f} ms, {dt/max(it,1)*1e6:.1f} us/iter", flush=True)
