#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for A in 0 1; do
  echo "FCM_TILED_ATOMIC=$A"
  FCM_TILED_ATOMIC=$A FCM_TILED_PROF=1 FCM_VERBOSE=1 REPS=1 timeout 300 python tools/coarse_once.py 2>&1 | grep "phases\|iters"
  FCM_TILED_ATOMIC=$A timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
done
