#!/bin/bash
# Full measurement pass: bench line, reference arm, ncu launch list and one full capture
# of the top kernel.  Outputs in gpurun_out/.
set -x
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 1500 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; echo list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_pcg -s 3 -c 1 -o gpurun_out/prof_top python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_top.log 2>&1; echo full rc=$?
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt
