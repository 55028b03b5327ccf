#!/bin/bash
# check (smoke + gpu tests + bench) then, if the bench ran clean, the ncu profile.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash scripts/gpu_check.sh
if grep -q "bench rc=0" gpurun_out/bench.log; then bash scripts/gpu_prof.sh > /dev/null 2>&1; fi
echo done
