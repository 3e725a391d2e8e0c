#!/bin/bash
# Session-4: L2 evict_first on the streamed patch inverses (A/B), then the default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or patch729 or identical" > gpurun_out/s4c_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4c_pytest.log
for v in "E FCM_L2_EVICT_FIRST=1" "F FCM_L2_EVICT_FIRST=0" "G FCM_L2_EVICT_FIRST=1"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/s4c_parts_$tag.json 2> gpurun_out/s4c_parts_$tag.err; echo "parts $tag ($*) rc=$?"; cat gpurun_out/s4c_parts_$tag.json; echo
done
timeout 900 python bench.py > gpurun_out/s4c_bench.json 2> gpurun_out/s4c_bench.err; echo bench rc=$?; head -c 1500 gpurun_out/s4c_bench.json; echo
