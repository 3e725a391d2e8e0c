"""Time the level-q operator apply and smoother sweep of a config with the warp-specialised cell
kernel split by population (FCM_WS_PART: 1 streaming warps only, 2 MMA warps only, 0 both)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1])
q = int(sys.argv[2])
G = generate(cfg)
S = Solver.from_problem(cfg, G)
b = S.load(G)
del G
r = b[: S.ndofs(q)].clone()
x = torch.zeros_like(r)


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


out = {"cfg": cfg.name, "q": q}
for part in ("0", "1", "2"):
    os.environ["FCM_WS_PART"] = part
    out["apply_part" + part] = timed(lambda: S.apply(r, q))
    out["smooth_part" + part] = timed(lambda: S.smooth(r, x, q))
os.environ["FCM_WS_PART"] = "0"
print(json.dumps(out), flush=True)
