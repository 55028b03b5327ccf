#!/bin/bash
# K12 b = 1: bytes in flight vs the loaded latency of the last tiles' chain (tile height x ring depth)
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/e16_inflight.jsonl; : > $out
for i in 1 2; do
for cfg in "" "--opt rows_per_tile=4" "--opt rows_per_tile=4 --opt max_stages=2" "--opt rows_per_tile=2" "--opt rows_per_tile=2 --opt max_stages=3" "--opt rows_per_tile=2 --opt max_stages=2"; do
  timeout 60 python scripts/time_decode.py --model mistral-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e16.err
done; done
