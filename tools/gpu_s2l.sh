cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 120 -k "forced_slab" > gpurun_out/s2l_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -15 gpurun_out/s2l_pytest1.log
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 120 -k "ws_single_cta or fallback or 3d_p3_ragged or 3d_p4_elem or 3d_p2 or trunk or gmg" > gpurun_out/s2l_pytest2.log 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/s2l_pytest2.log
timeout 300 python tools/ws_parts.py cfg5 2,3 2>&1 | grep cfg
