#!/bin/bash
# quick GPU check: parity tests + bench sweep over coarse block counts + launch list
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -3
for nb in ${NBS:-0 148}; do
  FCM_COARSE_BLOCKS=$nb timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nb=$nb', round(d['value']/1e6,2),'M DOF-it/s', round(d['ms_per_step'],2),'ms', 'coarse launch ms', round(d['roofline']['launch_ms'],3), 'kc', d['roofline']['coarse_iters_per_launch'], 'fcg', d['config']['fcg_iterations'])"
done
if [ -n "$LAUNCHES" ]; then
  timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 1500 --csv --log-file gpurun_out/$LAUNCHES.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
fi
