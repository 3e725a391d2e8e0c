#!/bin/bash
# Session-4: low-rank execution (cost model / all separate / all fused) with the dynamic FD claims
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "M FCM_WB_KERNEL=0" "S FCM_WB_KERNEL=1" "U FCM_WB_KERNEL=2" "M2 FCM_WB_KERNEL=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s4f_parts_$tag.json 2> gpurun_out/s4f_parts_$tag.err; echo "parts $tag ($*) rc=$?"; cat gpurun_out/s4f_parts_$tag.json; echo
done
