"""Per-iteration cost of the coarse p=1 PCG on a workload (tiled vs grid-wide kernel, AS vs
Jacobi), CUDA-event timed, plus the agreement of the two kernels' results."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(os.environ.get("CFG", "cfg2"))
G = generate(cfg)
res = {}
for coarse in ("as_pcg", "jacobi_pcg"):
    for tiled in ("1", "0"):
        os.environ["FCM_COARSE_TILED"] = tiled
        S = Solver.from_problem(cfg, G, coarse=coarse)
        b = S.load(G)
        r = b[: S.ndofs(1)].clone()
        for _ in range(3):
            x, it = S.coarse_solve(r)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n):
            x, it = S.coarse_solve(r)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        res[(coarse, tiled)] = x.clone()
        print(f"{coarse} tiled={tiled}: {ms:.3f} ms/solve, {it} iters, {ms / max(it, 1) * 1e3:.2f} us/iter",
              flush=True)
        S.close()
    a, b2 = res[(coarse, "1")], res[(coarse, "0")]
    print(f"  {coarse}: rel diff tiled vs grid = {float((a - b2).norm() / b2.norm()):.3e}")
