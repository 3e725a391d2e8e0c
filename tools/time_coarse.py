"""Per-iteration cost of the cooperative coarse PCG on cfg2 (AS vs Jacobi), CUDA-event timed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
for coarse in ("as_pcg", "jacobi_pcg"):
    for nb in (148, 296):
        os.environ["FCM_COARSE_BLOCKS"] = str(nb)
        S = Solver.from_problem(cfg, G, coarse=coarse)
        b = S.load(G)
        r = b[: S.ndofs(1)].clone()
        for _ in range(3): S.coarse_solve(r)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 10
        for _ in range(n): x, it = S.coarse_solve(r)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"{coarse} blocks={nb}: {ms:.3f} ms/solve, {it} iters, {ms / it * 1e3:.2f} us/iter")
        S.close()
