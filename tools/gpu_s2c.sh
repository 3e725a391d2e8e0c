cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() {  # name cfg what q kernel-regex
  timeout 600 python tools/ncu_parts.py $2 $3 $4 > gpurun_out/s2_plain_$1.log 2>&1 && \
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$5 -c 1 -o gpurun_out/s2_$1 python tools/ncu_parts.py $2 $3 $4 > gpurun_out/s2_ncu_$1.log 2>&1
  echo "$1 rc=$?"; cat gpurun_out/s2_plain_$1.log | tail -2
}
run fd4 cfg3 fd 4 k_patch_smooth
run fd2 cfg3 fd 2 k_patch_smooth
run irr4 cfg3 irr 4 k_patch_smooth
run apply5 cfg5 apply 3 k_cell_mma
run smooth5 cfg5 smooth 3 k_cell_mma
