"""Time the level-q operator apply and smoother sweep of a config with the warp-specialised cell
kernel split by population (FCM_WS_PART: 1 streaming warps only, 2 MMA warps only, 0 both), for
each warp-split variant given (FCM_WS_VARIANT, read at setup)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_00881_b200.fcm import Solver, generate  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1])
qs = [int(v) for v in sys.argv[2].split(",")]
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else [""]   # "": the library's per-mode default
G = generate(cfg)


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


for v in variants:
    if v:
        os.environ["FCM_WS_VARIANT"] = v
    else:
        os.environ.pop("FCM_WS_VARIANT", None)
    S = Solver.from_problem(cfg, G)
    b = S.load(G)
    for q in qs:
        r = b[: S.ndofs(q)].clone()
        x = torch.zeros_like(r)
        out = {"cfg": cfg.name, "q": q, "variant": v}
        for part in ("0", "1", "2"):
            os.environ["FCM_WS_PART"] = part
            out["apply_part" + part] = round(timed(lambda: S.apply(r, q)), 3)
            out["smooth_part" + part] = round(timed(lambda: S.smooth(r, x, q)), 3)
        os.environ["FCM_WS_PART"] = "0"
        print(json.dumps(out), flush=True)
        del r, x
    S.close()
    del b, S
    torch.cuda.empty_cache()
