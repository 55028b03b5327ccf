#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python scripts/bench_calib.py --n 2000000000 --k 0.5 --reps 1"
timeout 300 $CMD > gpurun_out/calib_plain.log 2>&1 || { cat gpurun_out/calib_plain.log; exit 1; }
cat gpurun_out/calib_plain.log | tail -c 400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"calib_hist" -s 2 -c 2 \
   -o gpurun_out/calib_prof -f $CMD > gpurun_out/ncu_calib.log 2>&1
tail -2 gpurun_out/ncu_calib.log
