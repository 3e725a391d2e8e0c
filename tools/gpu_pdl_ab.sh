#!/bin/bash
# programmatic dependent launch on / off (cfg2 and cfg1 bench)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for P in 0 1 0 1; do
  printf "FCM_PDL=%s " $P
  FCM_PDL=$P timeout 300 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'M', round(d['ms_per_step'],2), 'ms', d['config']['fcg_iterations'])"
  printf "  cfg1 "
  FCM_PDL=$P timeout 300 python bench.py --config cfg1 --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M', round(d['ms_per_step'],3), 'ms')"
done
