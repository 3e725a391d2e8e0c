#!/bin/bash
# GPU suite after the equilibrated patch inversion (full-size test first, then everything).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_full_size_gpu.py -m gpu -q > gpurun_out/s3b_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/s3b_fullsize.log
timeout 1500 python -m pytest tests/ -m gpu -q --timeout 900 --deselect tests/test_full_size_gpu.py > gpurun_out/s3b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s3b_pytest_gpu.log
