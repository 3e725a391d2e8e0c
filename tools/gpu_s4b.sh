#!/bin/bash
# Session-4: dynamic patch scheduling + rotated tiles -- parity subset, then cfg3 A/B of the smoother parts
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or lowrank or patch or deterministic or identical" > gpurun_out/s4b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4b_pytest.log
for v in "A FCM_PATCH_DYN=1" "B FCM_PATCH_DYN=0" "C FCM_TILE_SWZ=0" "D FCM_TILE_SWZ=0 FCM_PATCH_DYN=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s4b_parts_$tag.json 2> gpurun_out/s4b_parts_$tag.err; echo "parts $tag ($*) rc=$?"; cat gpurun_out/s4b_parts_$tag.json; echo
done
