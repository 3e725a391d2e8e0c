#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/time_coarse.py 2>&1 | tail -12
FCM_VERBOSE=1 FCM_TILED_PROF=1 timeout 300 python - <<'PY' 2>&1 | tail -8
import os, sys, torch
sys.path.insert(0, ".")
from paper_2010_00881_b200.fcm import Solver, generate
from workloads import get_config
cfg = get_config("cfg2"); G = generate(cfg)
S = Solver.from_problem(cfg, G); b = S.load(G); r = b[: S.ndofs(1)].clone()
for _ in range(3): x, it = S.coarse_solve(r)
print("iters", it)
PY
