#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for C in ${COARSES:-as_pcg jacobi_pcg}; do
FCM_VERBOSE=1 FCM_TILED_PROF=1 COARSE=$C REPS=${REPS:-3} timeout 300 python tools/coarse_once.py 2>&1 | tail -5
done
