#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python scripts/prof_decode.py --steps 6"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k12_|k3_" -s 8 -c 2 \
   -o gpurun_out/${TAG}_k12 -f $CMD > gpurun_out/ncu_k12.log 2>&1
tail -3 gpurun_out/ncu_k12.log
