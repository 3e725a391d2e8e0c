cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 600 -k "ws_single_cta or fallback or 3d_p3_ragged or 3d_p4_elem or cfg1 or trunk or apply" > gpurun_out/s2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2g_pytest.log
timeout 600 python tools/ws_parts.py cfg5 3 2>&1 | tail -1
timeout 600 python tools/ws_parts.py cfg5 2 2>&1 | tail -1
timeout 300 python tools/ncu_parts.py cfg3 apply 4 2>&1 | tail -1
