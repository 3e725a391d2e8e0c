#!/bin/bash
# Session-5: FD passes with all lines of a lane together -- parity subset, population end times, parts
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-s5f}
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 600 -k "variants or lowrank or patch or deterministic or identical" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 600 python tools/patch_prof.py cfg3 > gpurun_out/${T}_prof.out 2> gpurun_out/${T}_prof.err; echo "rc=$?"
grep "patch_prof. q=4" gpurun_out/${T}_prof.err | awk 'NR%3==0'
for v in "A X=1" "B FCM_FD_ROLL=0"; do
  set -- $v; tag=$1; shift
  env "$@" timeout 600 python tools/patch_parts.py cfg3 > gpurun_out/${T}_parts_$tag.json 2> gpurun_out/${T}_parts_$tag.err; echo "parts $tag ($*) rc=$?"
  python - <<PY
import json
d=json.load(open('gpurun_out/${T}_parts_$tag.json'))
print('$tag', {q:[round(d[q]['part%d_ms'%k],2) for k in (0,1,2)] for q in ('2','3','4')}, 'vcycle', round(d['vcycle_ms'],1))
PY
done
