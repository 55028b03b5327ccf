#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python scripts/bench_sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?" >> gpurun_out/sweep.err
timeout 600 python scripts/bench_calib.py --oracle > gpurun_out/calib.json 2> gpurun_out/calib.err; echo "calib rc=$?" >> gpurun_out/calib.err
timeout 600 python bench.py --steps 500 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
bash scripts/gpu_prof_split.sh > /dev/null 2>&1
tail -n 1 gpurun_out/sweep.err gpurun_out/calib.err gpurun_out/bench.log
