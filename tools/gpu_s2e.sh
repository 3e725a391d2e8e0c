cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 600 -k "patch" > gpurun_out/s2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2e_pytest.log
for w in "fd 4" "fd 3" "fd 2" "irr 4" "both 4" "both 3" "both 2"; do timeout 300 python tools/ncu_parts.py cfg3 $w 2>&1 | tail -1; done
timeout 600 python tools/ws_parts.py cfg5 3 > gpurun_out/s2e_ws5.json 2>&1; echo "ws5 rc=$?"; tail -2 gpurun_out/s2e_ws5.json
timeout 600 python tools/ws_parts.py cfg5 2 > gpurun_out/s2e_ws5q2.json 2>&1; echo "ws5q2 rc=$?"; tail -2 gpurun_out/s2e_ws5q2.json
