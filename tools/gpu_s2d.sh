cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -x -q --timeout 600 -k "ws_single_cta or fallback or 3d_p3_ragged or 3d_p4_elem or 3d_p2 or cfg1 or trunk" > gpurun_out/s2d_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/s2d_pytest.log
CFG=cfg5 COARSE=gmg_pcg MAXIT=20 timeout 900 python tools/cfg5_run.py > gpurun_out/s2d_cfg5.json 2> gpurun_out/s2d_cfg5.err; echo "cfg5 rc=$?"; tail -4 gpurun_out/s2d_cfg5.err
FCM_CELL_WS=0 CFG=cfg5 COARSE=gmg_pcg MAXIT=20 timeout 900 python tools/cfg5_run.py > gpurun_out/s2d_cfg5_nows.json 2> gpurun_out/s2d_cfg5_nows.err; echo "cfg5 nows rc=$?"; tail -4 gpurun_out/s2d_cfg5_nows.err
timeout 600 python tools/ncu_parts.py cfg3 fd 4 > gpurun_out/s2d_plain_fd4.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_patch_smooth -c 1 -o gpurun_out/s2d_fd4 python tools/ncu_parts.py cfg3 fd 4 > gpurun_out/s2d_ncu_fd4.log 2>&1; echo "fd4 rc=$?"
ls -la gpurun_out/
