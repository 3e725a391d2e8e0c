set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/s2_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/s2_pytest_gpu.log
timeout 600 python bench.py --config cfg2 --coarse gmg_pcg --no-cpu-baseline > gpurun_out/s2_bench_cfg2_gmg.log 2>&1; echo "cfg2 gmg exit $?"; tail -3 gpurun_out/s2_bench_cfg2_gmg.log
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/s2_bench_cfg2.log 2>&1; echo "cfg2 exit $?"; tail -3 gpurun_out/s2_bench_cfg2.log
timeout 900 python bench.py --config cfg3 --coarse gmg_pcg --no-cpu-baseline > gpurun_out/s2_bench_cfg3_gmg.log 2>&1; echo "cfg3 gmg exit $?"; tail -3 gpurun_out/s2_bench_cfg3_gmg.log
