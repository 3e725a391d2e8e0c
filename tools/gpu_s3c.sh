#!/bin/bash
# hp path parity on the GPU + the full-size cfg3 test with the setup-sensitivity tolerance.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hp_gpu.py -m gpu -q -x --timeout 600 > gpurun_out/s3c_hp.log 2>&1; echo "hp rc=$?"; tail -30 gpurun_out/s3c_hp.log
timeout 600 python -m pytest tests/test_full_size_gpu.py -m gpu -q > gpurun_out/s3c_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/s3c_fullsize.log
cp gpurun_out/parity_tolerances.json gpurun_out/s3c_parity_tolerances.json 2>/dev/null
