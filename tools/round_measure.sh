#!/bin/bash
# Full measurement pass: GPU tests, bench line, reference arm, ncu launch list and one full
# capture of the top kernel.  Outputs in gpurun_out/ (copy the summaries to profiles/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
FCM_HOST_LOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 1500 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; echo list rc=$?
FCM_HOST_LOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_tiled -s 3 -c 1 -o gpurun_out/prof_top python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_top.log 2>&1; echo full rc=$?
FCM_HOST_LOOP=1 timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_cell_mma -s 40 -c 2 -o gpurun_out/prof_cell python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cell.log 2>&1; echo cell rc=$?
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt
timeout 300 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2>/dev/null; echo cfg1 rc=$?
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>/dev/null; echo cfg4 rc=$?
