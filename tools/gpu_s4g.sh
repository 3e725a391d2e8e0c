#!/bin/bash
# Session-4: XOR-swizzled tiles + LOP3 addressing + incremental producer -- parity subset, A/B, bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or lowrank or patch or deterministic or identical" > gpurun_out/s4g_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4g_pytest.log
for v in "A X=1" "C FCM_TILE_SWZ=0" "A2 X=1"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s4g_parts_$tag.json 2> gpurun_out/s4g_parts_$tag.err; echo "parts $tag ($*) rc=$?"; cat gpurun_out/s4g_parts_$tag.json; echo
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s4g_bench.json 2> gpurun_out/s4g_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/s4g_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['ms_per_step'],1), 'ms', d['value'], 'sweep', round(r['launch_ms'],3), 'frac', round(r['frac'],3), 'clk', d['clocks'])"
