#!/bin/bash
# k_cell_mma blocks-per-SM sweep on the cfg2 bench (FCM_MMA_BPS x FCM_LIST_BPS)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for M in ${MS:-1 2 4}; do for L in ${LS:-2 4 8}; do
  printf "mma_bps=%s list_bps=%s " $M $L
  FCM_MMA_BPS=$M FCM_LIST_BPS=$L timeout 300 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'M', round(d['ms_per_step'],2), 'ms')"
done; done
