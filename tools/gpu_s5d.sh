#!/bin/bash
# Session-5: low-rank patches in the separate k_patch_wb launch (FCM_WB_KERNEL=1) vs fused, with the population end times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FCM_WB_KERNEL=1 timeout 600 python tools/patch_prof.py cfg3 > gpurun_out/s5d_prof.out 2> gpurun_out/s5d_prof.err; echo "rc=$?"
grep "patch_prof. q=4" gpurun_out/s5d_prof.err
for v in "A X=1" "B FCM_WB_KERNEL=1"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s5d_parts_$tag.json 2> gpurun_out/s5d_parts_$tag.err; echo "parts $tag ($*) rc=$?"
  python - <<PY
import json
d=json.load(open('gpurun_out/s5d_parts_$tag.json'))
print('$tag', {q:[round(d[q]['part%d_ms'%k],2) for k in (0,1,2)] for q in ('2','3','4')}, 'vcycle', round(d['vcycle_ms'],1))
PY
done
