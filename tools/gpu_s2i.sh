cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 120 -k "ws_single_cta or fallback or 3d_p3_ragged or 3d_p4_elem or 3d_p2 or trunk" > gpurun_out/s2i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s2i_pytest.log
timeout 300 python tools/ws_parts.py cfg5 2 2>&1 | tail -1
timeout 300 python tools/ws_parts.py cfg5 3 2>&1 | tail -1
