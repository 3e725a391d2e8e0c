#!/bin/bash
# Session-4: V-cycle launch list + ncu --set full of the level-4 k_patch_smooth (new kernel)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/ncu_step.py cfg3 vcycle > gpurun_out/s4e_plain1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/s4e_cfg3_vcycle_launches.csv python tools/ncu_step.py cfg3 vcycle > gpurun_out/s4e_ncu_list.log 2>&1; echo list rc=$?
timeout 600 python tools/ncu_parts.py cfg3 both 4 > gpurun_out/s4e_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_patch_smooth -c 1 -o gpurun_out/s4e_prof_patch python tools/ncu_parts.py cfg3 both 4 > gpurun_out/s4e_ncu_patch.log 2>&1; echo full rc=$?
