"""Slope of the V-cycle time in the number of smoothing sweeps (CUDA-event timed through the
C ABI): isolates the cost of one fine-level sweep (residual + smoother) from the coarse solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
for ns in (0, 1, 5):
    S = Solver.from_problem(cfg, G, n_pre=ns, n_post=ns)
    b = S.load(G)
    for _ in range(3):
        z = S.vcycle(b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        z = S.vcycle(b)
    e1.record(); e1.synchronize()
    print(f"V({ns},{ns}): {e0.elapsed_time(e1) / n * 1e3:.1f} us per V-cycle", flush=True)
    S.close()
