"""Time single operator applies / smoother applies of cfg2 through the C ABI (CUDA events)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = sys.argv[1]
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
for q in range(cfg.p, 0, -1):
    x = torch.randn(S.ndofs(q), dtype=torch.float64, device="cuda")
    y = S.apply(x, q)
    for name, fn in (("apply", lambda: S.apply(x, q)), ("smooth", lambda: S.smooth(x, y, q))):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        n = 200
        e0.record()
        for _ in range(n): fn()
        e1.record(); e1.synchronize()
        print(f"{os.path.basename(_lib.LIB_PATH)} q={q} {name}: {e0.elapsed_time(e1) / n * 1e3:.2f} us per call", flush=True)
