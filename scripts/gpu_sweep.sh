#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python scripts/bench_sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?" >> gpurun_out/sweep.err
timeout 600 python scripts/bench_calib.py --oracle > gpurun_out/calib.json 2> gpurun_out/calib.err; echo "calib rc=$?" >> gpurun_out/calib.err
tail -1 gpurun_out/sweep.err gpurun_out/calib.err
