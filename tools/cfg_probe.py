"""Probe a BASELINE config on one GPU: generator, setup, memory, per-level sweep times,
V-cycle time, FCG solve (iterations, time, true residual).  Usage: tools/cfg_probe.py cfg3 [maxit]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = get_config(name)
out = {"config": name}
t0 = time.time()
G = generate(cfg)
out["generator_s"] = time.time() - t0
out["n_cut"] = int(len(G.cut_cells))
torch.cuda.synchronize()
t0 = time.time()
S = Solver.from_problem(cfg, G)
b = S.load(G)
torch.cuda.synchronize()
out["setup_s"] = time.time() - t0
free, tot = torch.cuda.mem_get_info()
out["mem_used_GB"] = (tot - free) / 1e9
out["ndofs"] = [S.ndofs(q) for q in range(1, cfg.p + 1)]
out["blocks"] = {q: S.block_counts(q) for q in range(1, cfg.p + 1)}
out["coarse"] = S.coarse_info()
del G
print(json.dumps(out), flush=True)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


lev = {}
for q in range(2, cfg.p + 1):
    r = b[: S.ndofs(q)].clone()
    x = torch.zeros_like(r)
    lev[q] = {"smooth_ms": timed(lambda: S.smooth(r, x, q)), "apply_ms": timed(lambda: S.apply(r, q))}
out["levels"] = lev
r1 = b[: S.ndofs(1)].clone()
out["coarse_ms"] = timed(lambda: S.coarse_solve(r1), reps=2)
out["coarse_iters"] = S.coarse_solve(r1)[1]
xc, _ = S.coarse_solve(r1)
out["coarse_true_relres"] = float(torch.linalg.norm(r1 - S.apply(xc, 1)) / torch.linalg.norm(r1))
out["vcycle_ms"] = timed(lambda: S.vcycle(b), reps=2)
print(json.dumps(out), flush=True)
torch.cuda.synchronize()
t0 = time.time()
x, it, hist = S.pcg_solve(b, maxit=maxit)
torch.cuda.synchronize()
out["fcg_s"] = time.time() - t0
out["fcg_iters"] = it
out["fcg_hist"] = [float(v) for v in hist]
out["fcg_true_relres"] = float(torch.linalg.norm(b - S.apply(x)) / torch.linalg.norm(b))
out["stats"] = S.stats()
print(json.dumps(out), flush=True)
