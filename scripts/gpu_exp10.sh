#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -m gpu -q -k "tail_geometry" --timeout 600 -p no:cacheprovider > gpurun_out/e10_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e10_tests.log
out=gpurun_out/e10_pool.jsonl; : > $out
for i in 1 2; do
for cfg in "" "--opt ud_pool=1" "--opt ud_pool=1 --opt lazy_tail=0" "--opt ud_pool=1 --opt tail_rows=2 --opt tail_tiles=1"; do
  timeout 120 python scripts/time_decode.py --model mistral-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e10.err
  timeout 120 python scripts/time_decode.py --model llama2-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e10.err
done; done
timeout 120 python scripts/trace_decode.py --model mistral-7b --opt ud_pool=1 > gpurun_out/e10_trace.txt 2>&1
