#!/bin/bash
# Session-5 diagnostic: end times of the two warp populations of k_patch_smooth (cfg3)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/patch_prof.py cfg3 > gpurun_out/s5c_prof.out 2> gpurun_out/s5c_prof.err; echo "rc=$?"
grep patch_prof gpurun_out/s5c_prof.err
