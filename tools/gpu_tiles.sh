#!/bin/bash
# per-block phase distribution of the tiled coarse kernel for several partitions
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for T in default ${TILES:-"bisect" "17,2,8"}; do
  echo "== FCM_TILE=$T"
  if [ "$T" = default ]; then unset FCM_TILE; else export FCM_TILE=$T; fi
  FCM_VERBOSE=1 FCM_TILED_PROF=1 REPS=1 timeout 300 python tools/coarse_once.py 2>&1 | grep -v "^\[fcm\] \(level\|setup\|cell\|mma\|block\)" | tail -6
done
unset FCM_TILE
