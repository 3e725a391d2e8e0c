cd "${GRAFT_REPO_ROOT:-/root/repo}"
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/s2m_gpu_info.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/s2m_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2m_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/s2m_bench.json 2> gpurun_out/s2m_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/s2m_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/s2m_bench_ref.json 2> gpurun_out/s2m_bench_ref.err; echo "ref rc=$?"; tail -1 gpurun_out/s2m_bench_ref.json
timeout 600 python tools/ncu_step.py cfg3 vcycle > gpurun_out/s2m_plain_vc.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2m_cfg3_vcycle_launches.csv python tools/ncu_step.py cfg3 vcycle > gpurun_out/s2m_ncu_vc.log 2>&1; echo "list rc=$?"
timeout 600 python tools/ncu_parts.py cfg3 both 4 > gpurun_out/s2m_plain_both4.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_patch_smooth -c 1 -o gpurun_out/s2m_patch4 python tools/ncu_parts.py cfg3 both 4 > gpurun_out/s2m_ncu_patch4.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/s2m_patch4.ncu-rep --page details --csv > gpurun_out/s2m_patch4_details.csv 2>/dev/null
ncu -i gpurun_out/s2m_patch4.ncu-rep --page raw --csv > gpurun_out/s2m_patch4_raw.csv 2>/dev/null
CFG=cfg5 COARSE=gmg_pcg MAXIT=600 timeout 1200 python tools/cfg5_run.py > gpurun_out/s2m_cfg5.json 2> gpurun_out/s2m_cfg5.err; echo "cfg5 rc=$?"; tail -3 gpurun_out/s2m_cfg5.err
du -sh gpurun_out
