#!/bin/bash
# Session-5: rolled FD passes with the level-4 low-rank patches in the separate k_patch_wb launch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FCM_WB_KERNEL=1 timeout 600 python tools/patch_prof.py cfg3 > gpurun_out/s5j_prof.out 2> gpurun_out/s5j_prof.err; echo "rc=$?"
grep "patch_prof. q=4 part=0" gpurun_out/s5j_prof.err | tail -1
for v in "A FCM_WB_KERNEL=1" "B FCM_WB_KERNEL=1 FCM_FD_ROLL=0" "C X=1" "D FCM_FD_ROLL=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s5j_parts_$tag.json 2> gpurun_out/s5j_parts_$tag.err; echo "parts $tag ($*) rc=$?"
  python - <<PY
import json
d=json.load(open('gpurun_out/s5j_parts_$tag.json'))
print('$tag', {q:[round(d[q]['part%d_ms'%k],2) for k in (0,1,2)] for q in ('2','3','4')}, 'vcycle', round(d['vcycle_ms'],1))
PY
done
