import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfcm_mg_dry.so")
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config("cfg2")
G = generate(cfg)
for nb in (148, 296, 74):
    os.environ["FCM_COARSE_BLOCKS"] = str(nb)
    S = Solver.from_problem(cfg, G, coarse_maxit=200000 + 96)  # dry run: skip cell ops, stop by maxit
    r = S.load(G)[: S.ndofs(1)].clone()
    for _ in range(2): S.coarse_solve(r)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); x, it = S.coarse_solve(r); e1.record(); e1.synchronize()
    print(f"dry skeleton blocks={nb}: {e0.elapsed_time(e1):.3f} ms, {it} iters, {e0.elapsed_time(e1) / it * 1e3:.2f} us/iter")
