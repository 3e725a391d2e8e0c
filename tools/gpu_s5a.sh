#!/bin/bash
# Session-5: re-validation of HEAD (XOR-swizzled k_patch_smooth) -- full GPU suite, smoke, bench, reference arm,
# ncu launch list of one cfg3 step and one full capture of the level-4 k_patch_smooth launch.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -m gpu -q --timeout 1200 > gpurun_out/s5a_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5a_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5a_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/s5a_smoke.log
timeout 900 python bench.py > gpurun_out/s5a_bench.json 2> gpurun_out/s5a_bench.err; echo bench rc=$?; tail -c 1500 gpurun_out/s5a_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/s5a_bench_ref.json 2> gpurun_out/s5a_bench_ref.err; echo ref rc=$?
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/s5a_gpu_info.txt
