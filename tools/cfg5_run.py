"""Config 5 (256^3 cells, p = 3, 455M DOFs) on ONE B200: generator, setup, the level-3 operator
and smoother kernels (algorithmic bytes vs time -> HBM fraction), one coarse solve, one V-cycle,
and one full FCG solve, CUDA-event timed.  Prints one JSON line (copied to profiles/)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config

cfg = get_config(os.environ.get("CFG", "cfg5"))
if os.environ.get("COARSE"):
    cfg = cfg.replace(coarse=os.environ["COARSE"])
out = {"workload": cfg.name}
t = time.time(); G = generate(cfg); out["generator_s"] = time.time() - t
t = time.time(); S = Solver.from_problem(cfg, G); b = S.load(G); torch.cuda.synchronize()
out["setup_s"] = time.time() - t
out["free_dofs"] = S.ndofs()
out["cut_cells"] = int(len(G.cut_cells))
out["irregular_blocks"] = {q: S.irregular_blocks(q) for q in range(1, cfg.p + 1)}
m = S.level_m(cfg.p)
del G


def log(*a):
    print(*a, file=sys.stderr, flush=True)


log("setup done", out)
log("irregular", out["irregular_blocks"])


def ev_time(fn, reps):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps, r


N = S.ndofs()
ta, _ = ev_time(lambda: S.apply(b), 3)
x = torch.zeros_like(b)
ts, _ = ev_time(lambda: S.smooth(b, x, cfg.p), 3)
nirr = S.irregular_blocks(cfg.p)
ncut = out["cut_cells"]
# algorithmic bytes: 24 B per DOF (x read, y RMW) + individual matrices counted packed m(m+1)/2
bytes_apply = 24 * N + ncut * m * (m + 1) // 2 * 8   # packed
bytes_smooth = 24 * N + nirr * m * (m + 1) // 2 * 8
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.0) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
out["level_p_apply"] = {"ms": ta, "algo_bytes": bytes_apply, "GBps": bytes_apply / ta / 1e6, "frac": bytes_apply / ta / 1e6 / peak}
out["level_p_smooth"] = {"ms": ts, "algo_bytes": bytes_smooth, "GBps": bytes_smooth / ts / 1e6, "frac": bytes_smooth / ts / 1e6 / peak}
out["hbm_peak_GBps"] = peak
log("kernels", out["level_p_apply"], out["level_p_smooth"])
tc, (xc, itc) = ev_time(lambda: S.coarse_solve(b[: S.ndofs(1)].clone()), 1)
out["coarse_solve"] = {"ms": tc, "iterations": itc, "kernel": S.coarse_info()[0]}
log("coarse", out["coarse_solve"])
tv, _ = ev_time(lambda: S.vcycle(b), 1)
out["vcycle_ms"] = tv
log("vcycle ms", tv)
torch.cuda.synchronize(); t = time.time()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
xs, it, hist = S.pcg_solve(b, maxit=int(os.environ.get("MAXIT", "500")))
e1.record(); e1.synchronize()
tsolve = e0.elapsed_time(e1) / 1e3
out["fcg"] = {"iterations": it, "seconds": tsolve, "final_relres": float(hist[-1]),
              "dof_iterations_per_s": N * it / tsolve}
print(json.dumps(out), flush=True)
