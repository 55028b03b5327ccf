#!/bin/bash
# small TP shards of Llama2-13B (d = 5120) at b = 1: split path (default) vs K12 and its knobs
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/exp22.jsonl; : > $out
for m in 1728 3456 6912 13824; do
for cfg in "" "--opt path=1" "--opt path=1 --opt rows_per_tile=2" "--opt path=1 --opt rows_per_tile=4" "--opt path=1 --opt min_tiles=1" "--opt path=1 --opt rows_per_tile=2 --opt min_tiles=1"; do
  timeout 60 python scripts/time_decode.py --model llama2-13b --m $m $cfg --tag "m=$m $cfg" >> $out 2>> gpurun_out/exp22.err
done; done
