#!/bin/bash
# per-brick model features and measured phase times of the tiled coarse kernel (cost-model calibration)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for T in default 17,2,8 8,8,4 bisect; do
  if [ "$T" = default ]; then unset FCM_TILE; else export FCM_TILE=$T; fi
  FCM_TILED_DUMP=1 FCM_VERBOSE=1 FCM_TILED_PROF=1 REPS=1 timeout 300 python tools/coarse_once.py 2>&1 | grep "brick .* feat" > gpurun_out/calib_$T.txt
done
wc -l gpurun_out/calib_*.txt
