#!/bin/bash
# Session-3 full pass: GPU suite, smoke, default bench (cfg3), reference arm, hp bench, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -m gpu -q --timeout 900 > gpurun_out/s3r_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3r_pytest_gpu.log
cp gpurun_out/parity_tolerances.json gpurun_out/s3r_parity_tolerances.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3r_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s3r_smoke.log
timeout 900 python bench.py > gpurun_out/s3r_bench.json 2> gpurun_out/s3r_bench.err; echo bench rc=$?; head -c 1200 gpurun_out/s3r_bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/s3r_bench_ref.json 2> gpurun_out/s3r_bench_ref.err; echo ref rc=$?
timeout 600 python bench.py --config hp_plate > gpurun_out/s3r_bench_hp.json 2> gpurun_out/s3r_bench_hp.err; echo hp rc=$?; head -c 600 gpurun_out/s3r_bench_hp.json; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hp_smooth_sym -s 100 -c 2 -o gpurun_out/s3r_prof_hpsmooth python tools/hp_probe.py 64 3 patch direct > gpurun_out/s3r_ncu_hp.log 2>&1; echo hpncu rc=$?
