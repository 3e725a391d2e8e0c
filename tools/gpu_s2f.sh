cd "${GRAFT_REPO_ROOT:-/root/repo}"
export FCM_WS_PART=2
timeout 600 python tools/ncu_parts.py cfg5 apply 2 > gpurun_out/s2f_plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_cell_ws -c 1 -o gpurun_out/s2f_ws_mma_q2 python tools/ncu_parts.py cfg5 apply 2 > gpurun_out/s2f_ncu.log 2>&1; echo "rc=$?"
cat gpurun_out/s2f_plain.log | tail -1
ls -la gpurun_out
