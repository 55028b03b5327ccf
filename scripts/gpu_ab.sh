#!/bin/bash
# A/B of two library builds on the same box, interleaved: libcats.so vs libcats_ab.so
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/ab.jsonl; : > $out
for i in 1 2 3; do for lib in libcats.so libcats_ab.so; do
for spec in "llama2-13b 1728 1" "llama2-7b 11008 2" "llama2-7b 11008 8"; do
  set -- $spec
  timeout 60 python scripts/time_decode.py --model $1 --m $2 --batch $3 --lib $lib --tag $lib >> $out 2>> gpurun_out/ab.err
done; done; done
