"""A/B timing of V(5,5) on cfg2 for environment-switched kernel variants (same process,
alternating, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
variants = [v.split("=") for v in sys.argv[1:]] or [["FCM_CELL_PARAM", "1"], ["FCM_CELL_PARAM", "0"]]
res = {}
for rep in range(3):
    for k, v in variants:
        os.environ[k] = v
        S = Solver.from_problem(cfg, G)
        b = S.load(G)
        for _ in range(3):
            z = S.vcycle(b)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            z = S.vcycle(b)
        e1.record(); e1.synchronize()
        res.setdefault(f"{k}={v}", []).append(e0.elapsed_time(e1) / 20 * 1e3)
        S.close()
        del os.environ[k]
for k, t in res.items():
    print(f"{k}: V(5,5) {min(t):.1f} us (runs {', '.join(f'{x:.0f}' for x in t)})")
