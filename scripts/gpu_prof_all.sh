#!/bin/bash
# profile refresh: K12 decode (b=1 bench shape) launch list + full capture, split path b=2/8 full captures
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py --steps 500 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
bash scripts/gpu_prof.sh > /dev/null 2>&1
bash scripts/gpu_prof_split.sh > /dev/null 2>&1
tail -2 gpurun_out/bench.log | cut -c1-300
ls gpurun_out/*.ncu-rep
