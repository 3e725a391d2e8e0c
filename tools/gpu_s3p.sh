#!/bin/bash
# m = 96 / 60 (trunk elasticity, config 4) on the MMA + warp-specialised path: parity, cfg4 bench A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q --timeout 600 -k "trunk or elast" > gpurun_out/s3p_trunk.log 2>&1; echo "trunk rc=$?"; tail -2 gpurun_out/s3p_trunk.log
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s3p_cfg4.json 2> gpurun_out/s3p_cfg4.err; echo cfg4 rc=$?; head -c 800 gpurun_out/s3p_cfg4.json; echo
FCM_CELL_WS=0 timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s3p_cfg4_nows.json 2>/dev/null; echo nows rc=$?; head -c 400 gpurun_out/s3p_cfg4_nows.json; echo
FCM_CELL_MMA=0 timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s3p_cfg4_nomma.json 2>/dev/null; echo nomma rc=$?; head -c 400 gpurun_out/s3p_cfg4_nomma.json; echo
