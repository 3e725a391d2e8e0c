#!/bin/bash
# Session-5 A/B on one box: warp-role map (FCM_PATCH_WMAP=1: FD warps on one scheduler) and the
# one-copy FD build (libfcm_mg_exp.so, -DFCM_FD_ONECOPY).  Parity subset first, then parts + bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
EXP=$PWD/paper_2010_00881_b200/libfcm_mg_exp.so
FCM_PATCH_WMAP=1 timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or lowrank or patch or deterministic or identical" > gpurun_out/s5b_pytest_wmap.log 2>&1; echo "pytest wmap rc=$?"; tail -2 gpurun_out/s5b_pytest_wmap.log
FCM_LIB_PATH=$EXP timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or lowrank or patch or deterministic or identical" > gpurun_out/s5b_pytest_exp.log 2>&1; echo "pytest exp rc=$?"; tail -2 gpurun_out/s5b_pytest_exp.log
for v in "A X=1" "B FCM_PATCH_WMAP=1" "C FCM_LIB_PATH=$EXP" "D FCM_LIB_PATH=$EXP FCM_PATCH_WMAP=1" "A2 X=1"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s5b_parts_$tag.json 2> gpurun_out/s5b_parts_$tag.err; echo "parts $tag ($*) rc=$?"
  python - <<PY
import json
d=json.load(open('gpurun_out/s5b_parts_$tag.json'))
print('$tag', {q:[round(d[q]['part%d_ms'%k],2) for k in (0,1,2)] for q in ('2','3','4')}, 'vcycle', round(d['vcycle_ms'],1))
PY
done
for v in "A X=1" "B FCM_PATCH_WMAP=1" "C FCM_LIB_PATH=$EXP" "D FCM_LIB_PATH=$EXP FCM_PATCH_WMAP=1"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s5b_bench_$tag.json 2> gpurun_out/s5b_bench_$tag.err; echo "bench $tag rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/s5b_bench_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', round(d['ms_per_step'],1), 'ms', d['value'], 'sweep', round(r['launch_ms'],3), 'frac', round(r['frac'],3), 'clk', d['clocks'])"
done
