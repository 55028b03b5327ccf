#!/bin/bash
# round-1 closing check of HEAD: smoke, all GPU tests, bench, App. B timings, ncu launch list + K12 capture
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash scripts/gpu_check.sh > /dev/null 2>&1
XS_FULL=0 bash scripts/gpu_xsparse.sh > /dev/null 2>&1
bash scripts/gpu_prof.sh > /dev/null 2>&1
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/pytest_xs.log
tail -n 2 gpurun_out/bench.log | cut -c1-300
cut -c1-200 gpurun_out/xsparse.jsonl
