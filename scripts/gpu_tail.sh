#!/bin/bash
# K12 b = 1 tail experiments: tail-tile geometry sweep + App. D ablation timings + a trace of the default.
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/tail.jsonl; : > $out
for cfg in "" "--opt tail_rows=2 --opt tail_tiles=1" "--opt tail_rows=2 --opt tail_tiles=2" "--opt tail_rows=3 --opt tail_tiles=1" "--opt tail_rows=3 --opt tail_tiles=2" "--opt tail_rows=3 --opt tail_tiles=4" "--opt tail_rows=4 --opt tail_tiles=2"; do
  timeout 120 python scripts/time_decode.py --model mistral-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/tail.err
done
for model in mistral-7b llama2-7b; do for k in 0.5 0.7 0.9; do for c in 0 1 2; do
  timeout 120 python scripts/time_decode.py --model $model --k $k --tag "compaction=$c" --opt compaction=$c >> gpurun_out/ablation.jsonl 2>> gpurun_out/tail.err
done; done; done
timeout 120 python scripts/trace_decode.py --model mistral-7b > gpurun_out/trace_default.txt 2>&1
timeout 120 python scripts/trace_decode.py --model mistral-7b --opt tail_rows=2 --opt tail_tiles=2 > gpurun_out/trace_tail.txt 2>&1
