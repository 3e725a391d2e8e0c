#!/bin/bash
# Session-4: same-box bench A/B (new defaults vs FCM_PATCH_DYN=0 FCM_TILE_SWZ=0 FCM_L2_EVICT_FIRST=0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "new1 X=1" "old1 FCM_PATCH_DYN=0 FCM_TILE_SWZ=0 FCM_L2_EVICT_FIRST=0" "new2 X=1" "old2 FCM_PATCH_DYN=0 FCM_TILE_SWZ=0 FCM_L2_EVICT_FIRST=0" "dynonly FCM_TILE_SWZ=0 FCM_L2_EVICT_FIRST=0" "swzonly FCM_PATCH_DYN=0 FCM_L2_EVICT_FIRST=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4d_bench_$tag.json 2> gpurun_out/s4d_bench_$tag.err; echo "bench $tag rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/s4d_bench_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', round(d['ms_per_step'],1), 'ms', d['value'], 'sweep', round(r['launch_ms'],3), 'frac', round(r['frac'],3), 'clk', d['clocks'])"
done
