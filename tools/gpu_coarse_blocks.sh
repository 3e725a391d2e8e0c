#!/bin/bash
# grid-wide coarse kernel at config-5 scale (p = 1 geometry): CTAs per SM sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for B in ${BLOCKS:-default 148 296 444 592}; do
  echo "== FCM_COARSE_BLOCKS=$B"
  if [ "$B" = default ]; then unset FCM_COARSE_BLOCKS; else export FCM_COARSE_BLOCKS=$B; fi
  timeout 900 python tools/coarse_scale.py 2>&1 | tail -3
done
