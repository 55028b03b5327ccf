#!/bin/bash
# end-of-round refresh: GPU tests, smoke, bench, sweep, calibration, ncu (K12 + split path + calibration)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash scripts/gpu_check.sh > /dev/null 2>&1
timeout 1500 python scripts/bench_sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?" >> gpurun_out/sweep.err
timeout 600 python scripts/bench_calib.py --oracle > gpurun_out/calib.json 2> gpurun_out/calib.err; echo "calib rc=$?" >> gpurun_out/calib.err
bash scripts/gpu_prof.sh > /dev/null 2>&1
bash scripts/gpu_prof_split.sh > /dev/null 2>&1
bash scripts/gpu_prof_calib.sh > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/sweep.err gpurun_out/calib.err
tail -n 2 gpurun_out/bench.log | cut -c1-200
