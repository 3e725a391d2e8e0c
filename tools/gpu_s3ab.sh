#!/bin/bash
# session-3 final pass: GPU suite, smoke, default bench, reference arm, hp bench, V-cycle launch list,
# ncu --set full of the level-4 patch sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -m gpu -q --timeout 900 > gpurun_out/s3ab_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^E  |passed|failed" gpurun_out/s3ab_pytest_gpu.log | tail -6
cp gpurun_out/parity_tolerances.json gpurun_out/s3ab_parity_tolerances.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3ab_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s3ab_smoke.log
timeout 900 python bench.py > gpurun_out/s3ab_bench.json 2> gpurun_out/s3ab_bench.err; echo bench rc=$?; head -c 700 gpurun_out/s3ab_bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/s3ab_bench_ref.json 2> gpurun_out/s3ab_bench_ref.err; echo ref rc=$?
timeout 600 python bench.py --config hp_plate > gpurun_out/s3ab_bench_hp.json 2> gpurun_out/s3ab_bench_hp.err; echo hp rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/s3ab_vcycle.csv python tools/ncu_step.py cfg3 vcycle > /dev/null 2>&1; echo list=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_patch_smooth -c 1 -o gpurun_out/s3ab_prof_patch python tools/ncu_step.py cfg3 vcycle > gpurun_out/s3ab_ncu_full.log 2>&1; echo full=$?
