"""Time the two populations of each patch level's smoother alone and together (cfg3)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
del G


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for q in range(2, cfg.p + 1):
    r = b[: S.ndofs(q)].clone()
    x = torch.zeros_like(r)
    out[q] = {f"part{k}_ms": timed(lambda: S.smooth_part(r, x, q, k)) for k in (0, 1, 2)}
    out[q]["n_irr"], _ = S.block_counts(q)
    out[q]["apply_ms"] = timed(lambda: S.apply(r, q))
r1 = b[: S.ndofs(1)].clone()
out["coarse_ms"] = timed(lambda: S.coarse_solve(r1), 3)
out["coarse_info"] = S.coarse_info()
out["vcycle_ms"] = timed(lambda: S.vcycle(b), 3)
print(json.dumps(out))
