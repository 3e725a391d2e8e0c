#!/bin/bash
# Session 3 first pass: GPU suite (incl. the full-size cfg3 test) and the default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.txt
timeout 1500 python -m pytest tests/ -m gpu -q -x --timeout 900 > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench rc=$?; cat gpurun_out/s3_bench.json | head -c 3000
