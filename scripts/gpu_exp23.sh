#!/bin/bash
# per-CTA traces of the Llama2-13B TP8 / TP4 shards (b = 1): split path and K12
cd "${GRAFT_REPO_ROOT:-.}"
for m in 1728 3456; do
  timeout 120 python scripts/trace_decode.py --model llama2-13b --m $m > gpurun_out/e23_split_$m.txt 2>&1
  timeout 120 python scripts/trace_decode.py --model llama2-13b --m $m --opt path=1 > gpurun_out/e23_k12_$m.txt 2>&1
done
