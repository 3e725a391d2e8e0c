#!/bin/bash
# quick GPU check: parity tests, coarse-kernel timing, short bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/time_coarse.py 2>&1 | tail -12
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_quick.err | tee gpurun_out/bench_quick.json
