"""hp path probe: generator/setup time, FCG time-to-1e-10, and per-operation event timings on the
paper's perforated plate (Table perPlateRef's largest case: h = 1/64, k = 3, p = 2, patchwise)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import HpDisc, HpSolver  # noqa: E402
from workloads import hp_plate  # noqa: E402


def ev(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 3
    block = sys.argv[3] if len(sys.argv) > 3 else "patch"
    coarse = sys.argv[4] if len(sys.argv) > 4 else "direct"
    cfg = hp_plate(n, k, block=block, coarse=coarse)
    t0 = time.time()
    D = HpDisc(cfg)
    tg = time.time() - t0
    t0 = time.time()
    S = HpSolver(D)
    torch.cuda.synchronize()
    ts = time.time() - t0
    b = torch.from_numpy(D.load()).cuda()
    out = {"case": cfg.name, "ndof": D.ndof, "levels": D.level_n.tolist(), "leaves": D.nleaves,
           "generator_s": tg, "setup_s": ts}
    x, it, hist = S.pcg_solve(b)
    out["fcg_iters"] = it
    out["relres"] = float(hist[-1])
    out["solve_ms"] = ev(lambda: S.pcg_solve(b, x=x), 5)
    r = b.clone()
    out["vcycle_ms"] = ev(lambda: S.vcycle(r), 20)
    for l in range(D.nlevels):
        xl = torch.zeros(S.ndofs(l), dtype=torch.float64, device="cuda")
        rl = r[: S.ndofs(l)].clone()
        out[f"apply_ms_l{l}"] = ev(lambda: S.apply(rl, l), 20)
        try:
            out[f"smooth_ms_l{l}"] = ev(lambda: S.smooth(rl, xl, l), 20)
        except Exception:
            pass
    blocks, invs = S.export_blocks(0)
    out["l0_blocks"] = len(blocks)
    out["l0_inverse_bytes"] = int(sum(len(bb) ** 2 for bb in blocks) * 8)
    out["l0_block_max"] = int(max(len(bb) for bb in blocks))
    out["stats"] = S.stats()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
