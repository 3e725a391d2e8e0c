#!/bin/bash
# Session-5 final pass (per-level rolled FD): full GPU suite, smoke, bench, reference arm, cfg3 V-cycle launch list, ncu --set full of
# the level-4 k_patch_smooth launch (each ncu only after the same command exited 0 without it)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/s5l_bench.json 2> gpurun_out/s5l_bench.err; echo bench rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/s5l_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['ms_per_step'],1), 'ms', d['value'], 'e2e', d['e2e']['value'], 'sweep', round(r['launch_ms'],3), 'frac', round(r['frac'],3), 'path', d['path_roofline']['frac_of_measured_6546GBs'], 'clk', d['clocks'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/s5l_bench_ref.json 2> gpurun_out/s5l_bench_ref.err; echo ref rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5l_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s5l_smoke.log
timeout 600 python tools/ncu_step.py cfg3 vcycle > gpurun_out/s5l_plain1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/s5l_cfg3_vcycle_launches.csv python tools/ncu_step.py cfg3 vcycle > gpurun_out/s5l_ncu_list.log 2>&1; echo list rc=$?
timeout 600 python tools/ncu_parts.py cfg3 both 4 > gpurun_out/s5l_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_patch_smooth -c 1 -o gpurun_out/s5l_prof_patch python tools/ncu_parts.py cfg3 both 4 > gpurun_out/s5l_ncu_patch.log 2>&1; echo full rc=$?
timeout 2400 python -m pytest tests/ -m gpu -q --timeout 1200 > gpurun_out/s5l_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5l_pytest_gpu.log
