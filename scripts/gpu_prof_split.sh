#!/bin/bash
# ncu --set full of the split path (KA, KB) at b = 2 and b = 8 (Llama2-7B shape)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
for b in 2 8; do
  CMD="python scripts/prof_decode.py --model llama2-7b --batch $b --steps 6"
  timeout 300 $CMD > gpurun_out/prof_plain_b$b.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_plain_b$b.log; exit 1; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ka_gate_up|kb_down" -s 4 -c 2 \
     -o gpurun_out/${TAG}_split_b$b -f $CMD > gpurun_out/ncu_split_b$b.log 2>&1
  tail -2 gpurun_out/ncu_split_b$b.log
done
