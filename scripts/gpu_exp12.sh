#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/e12_paths.jsonl; : > $out
for model in llama2-7b mistral-7b; do for b in 2 3 4; do for path in 0 1; do
  timeout 60 python scripts/time_decode.py --model $model --batch $b --tag "path=$path" --opt path=$path >> $out 2>> gpurun_out/e12.err
done; done; done
for b in 2 3; do for nr in 2 4; do
  timeout 60 python scripts/time_decode.py --model llama2-7b --batch $b --tag "path=1 nr=$nr" --opt path=1 --opt rows_per_tile=$nr >> $out 2>> gpurun_out/e12.err
done; done
