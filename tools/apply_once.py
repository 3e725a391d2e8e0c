"""cfg2 operator apply and smoother through the C ABI (target for ncu captures of the cell kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
x = torch.zeros_like(b)
for _ in range(int(os.environ.get("REPS", "3"))):
    y = S.apply(b)
    S.smooth(b, x, cfg.p)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
n = 50
e0.record()
for _ in range(n):
    y = S.apply(b)
e1.record(); e1.synchronize()
t_a = e0.elapsed_time(e1) / n
e0.record()
for _ in range(n):
    S.smooth(b, x, cfg.p)
e1.record(); e1.synchronize()
t_s = e0.elapsed_time(e1) / n
print(f"apply {t_a*1e3:.1f} us, smooth {t_s*1e3:.1f} us (incl. launch + fill)")
