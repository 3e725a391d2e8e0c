#!/bin/bash
# A/B of the tiled coarse kernel's constant-coefficient fast path, then parity and a bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for F in 0 1; do
  echo "FCM_TILED_FAST=$F"
  FCM_TILED_FAST=$F COARSES=as_pcg REPS=${REPS:-1} bash tools/gpu_prof_tiled.sh 2>&1 | grep -v "tiled coarse"
done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "coarse or vcycle or fcg or mg_solve" 2>&1 | tail -3
timeout 600 python bench.py 2>/dev/null | tail -1
