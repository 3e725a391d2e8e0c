#!/bin/bash
# full GPU suite with the low-rank patches + cfg3 V-cycle launch list + ncu of k_patch_wb + bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -m gpu -q --timeout 900 > gpurun_out/s3v_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^E  |passed|failed" gpurun_out/s3v_pytest_gpu.log | tail -8
cp gpurun_out/parity_tolerances.json gpurun_out/s3v_parity_tolerances.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/s3v_cfg3_vcycle_launches.csv python tools/ncu_step.py cfg3 vcycle > gpurun_out/s3v_ncu_list.log 2>&1; echo list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_patch_wb -c 1 -o gpurun_out/s3v_prof_wb python tools/ncu_step.py cfg3 irr > gpurun_out/s3v_ncu_wb.log 2>&1; echo wbncu rc=$?
timeout 900 python bench.py > gpurun_out/s3v_bench.json 2> gpurun_out/s3v_bench.err; echo bench rc=$?; head -c 3000 gpurun_out/s3v_bench.json
