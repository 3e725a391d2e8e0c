cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 120 -k "apply and (3d_p2 or 3d_p3_ragged or 3d_p4_elem)" > gpurun_out/s2h_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -3 gpurun_out/s2h_pytest1.log
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 120 -k "ws_single_cta or fallback or 3d_p3_ragged or 3d_p4_elem or 3d_p2 or trunk" > gpurun_out/s2h_pytest2.log 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/s2h_pytest2.log
timeout 300 python tools/ws_parts.py cfg5 2 2>&1 | tail -1
timeout 300 python tools/ws_parts.py cfg5 3 2>&1 | tail -1
export FCM_WS_PART=2
timeout 300 python tools/ncu_parts.py cfg5 apply 3 > gpurun_out/s2h_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_cell_ws -c 1 -o gpurun_out/s2h_ws_mma_q3 python tools/ncu_parts.py cfg5 apply 3 > gpurun_out/s2h_ncu.log 2>&1; echo "ncu rc=$?"
