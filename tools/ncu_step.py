"""One timed step (fcm_pcg_solve) of a config inside a cudaProfilerStart/Stop range, for
ncu --profile-from-start off (launch list / full capture of the hot-path kernels only)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
what = sys.argv[2] if len(sys.argv) > 2 else "solve"
if len(sys.argv) > 3:
    cfg = cfg.replace(coarse=sys.argv[3])
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
x, it, _ = S.pcg_solve(b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if what == "solve":
    x, it, _ = S.pcg_solve(b)
elif what == "irr":
    xs = torch.zeros_like(b)
    S.smooth_part(b, xs, cfg.p, 1)
elif what == "vcycle":
    S.vcycle(b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iters", it)
