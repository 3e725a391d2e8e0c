#!/bin/bash
# hp path: bench line, launch list of the solve kernels, one full ncu capture of the smoother
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py --config hp_plate > gpurun_out/s3n_bench_hp.json 2> gpurun_out/s3n_bench_hp.err; echo bench rc=$?; head -c 2500 gpurun_out/s3n_bench_hp.json
timeout 600 python bench.py --config hp_plate128 --no-cpu-baseline > gpurun_out/s3n_bench_hp128.json 2> gpurun_out/s3n_bench_hp128.err; echo bench128 rc=$?; head -c 600 gpurun_out/s3n_bench_hp128.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_hp_ --csv --log-file gpurun_out/s3n_hp_launches.csv -s 3000 -c 1500 python bench.py --config hp_plate --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s3n_ncu_list.log 2>&1; echo list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hp_smooth_sym -s 200 -c 3 -o gpurun_out/s3n_prof_hpsmooth python tools/hp_probe.py 64 3 patch direct > gpurun_out/s3n_ncu_full.log 2>&1; echo full rc=$?
