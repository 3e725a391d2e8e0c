#!/bin/bash
# low-rank individual patches (patch_wb.cuh): patch parity cases, full-size cfg3 rows, bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q --timeout 600 -k "patch" > gpurun_out/s3u_patch.log 2>&1; echo "patch rc=$?"; grep -E "^E  |passed|failed" gpurun_out/s3u_patch.log | head -12
cp gpurun_out/parity_tolerances.json gpurun_out/s3u_tol.json
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s3u_bench.json 2> gpurun_out/s3u_bench.err; echo bench rc=$?; head -c 1500 gpurun_out/s3u_bench.json; tail -3 gpurun_out/s3u_bench.err
timeout 600 python -m pytest tests/test_full_size_gpu.py -m gpu -q > gpurun_out/s3u_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "^E  |passed|failed" gpurun_out/s3u_fullsize.log | head
