cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2 3 4; do timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -q --timeout 120 -k "vcycle_identical_setup and 2d_p4" 2>&1 | tail -1; python -c "
import json; d=json.load(open('gpurun_out/parity_tolerances.json'))
print([round(e['rel_diff']*1e11,2) for e in d if e['case']=='2d_p4' and 'identical' in e['check']])"; done
FCM_DETERMINISTIC=1 timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -q --timeout 120 -k "vcycle_identical_setup and 2d_p4" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q --timeout 300 -k "deterministic" > gpurun_out/s2n_det.log 2>&1; echo "det rc=$?"; tail -5 gpurun_out/s2n_det.log
timeout 300 python tools/ws_parts.py cfg5 2,3 2>&1 | grep cfg
