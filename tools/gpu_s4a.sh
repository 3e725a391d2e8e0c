#!/bin/bash
# Session-4 validation pass of HEAD: GPU suite, smoke, default bench (cfg3), reference arm
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s4a_gpu_info.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s4a_smoke.log
timeout 900 python bench.py > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err; echo bench rc=$?; head -c 1500 gpurun_out/s4a_bench.json; echo
timeout 1800 python -m pytest tests/ -m gpu -q --timeout 900 > gpurun_out/s4a_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4a_pytest_gpu.log
cp gpurun_out/parity_tolerances.json gpurun_out/s4a_parity_tolerances.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/s4a_bench_ref.json 2> gpurun_out/s4a_bench_ref.err; echo ref rc=$?
