"""One hot-path kernel of a config inside a cudaProfilerStart/Stop range, for
ncu --profile-from-start off: what in {fd, irr, both (patch smoother populations), apply, smooth}
on level q.  Run once outside the range first (warm-up, lazy module load)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1])
if os.environ.get("COARSE"):
    cfg = cfg.replace(coarse=os.environ["COARSE"])
what = sys.argv[2]
q = int(sys.argv[3])
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
del G
r = b[: S.ndofs(q)].clone()
x = torch.zeros_like(r)


def once():
    if what in ("fd", "irr", "both"):
        S.smooth_part(r, x, q, {"irr": 1, "fd": 2, "both": 0}[what])
    elif what == "apply":
        S.apply(r, q)
    elif what == "smooth":
        S.smooth(r, x, q)


once()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    once()
e1.record()
e1.synchronize()
print(f"{cfg.name} {what} q={q}: {e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
torch.cuda.profiler.start()
once()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
