#!/bin/bash
# Session-5: per-level rolled FD passes (level 4 rolled + k_patch_wb, levels 3/2 unrolled) -- parity, parts A/B, bench A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or lowrank or patch or deterministic or identical" > gpurun_out/s5k_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s5k_pytest.log
FCM_FD_ROLL=1 timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "lowrank or patch" > gpurun_out/s5k_pytest_roll1.log 2>&1; echo "pytest roll=1 rc=$?"; tail -2 gpurun_out/s5k_pytest_roll1.log
for v in "A X=1" "B FCM_FD_ROLL=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s5k_parts_$tag.json 2> gpurun_out/s5k_parts_$tag.err; echo "parts $tag ($*) rc=$?"
  python - <<PY
import json
d=json.load(open('gpurun_out/s5k_parts_$tag.json'))
print('$tag', {q:[round(d[q]['part%d_ms'%k],2) for k in (0,1,2)] for q in ('2','3','4')}, 'vcycle', round(d['vcycle_ms'],1))
PY
done
for v in "A X=1" "B FCM_FD_ROLL=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s5k_bench_$tag.json 2> gpurun_out/s5k_bench_$tag.err; echo "bench $tag rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/s5k_bench_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', round(d['ms_per_step'],1), 'ms', d['value'], 'sweep', round(r['launch_ms'],3), 'frac', round(r['frac'],3), 'clk', d['clocks'])"
done
