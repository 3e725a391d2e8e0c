set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=cfg5 COARSE=gmg_pcg MAXIT=400 timeout 1500 python tools/cfg5_run.py > gpurun_out/s2_cfg5_gmg.json 2> gpurun_out/s2_cfg5_gmg.err; echo "cfg5 rc=$?"; tail -12 gpurun_out/s2_cfg5_gmg.err; cat gpurun_out/s2_cfg5_gmg.json
timeout 600 python tools/ncu_step.py cfg3 vcycle > gpurun_out/s2_plain_vc.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_cfg3_vcycle_launches.csv python tools/ncu_step.py cfg3 vcycle > gpurun_out/s2_ncu_vc.log 2>&1; echo "ncu rc=$?"
