#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -m gpu -q -k "tail_geometry" --timeout 300 -p no:cacheprovider > gpurun_out/e20_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e20_tests.log
grep -q "pytest rc=0" gpurun_out/e20_tests.log || exit 1
out=gpurun_out/e20.jsonl; : > $out
for i in 1 2; do
for cfg in "" "--opt gate_first_tail=1" "--opt gate_first_tail=1 --opt lazy_tail=16" "--opt gate_first_tail=1 --opt lazy_tail=32" "--opt gate_first_tail=1 --opt lazy_tail=64"; do
  timeout 60 python scripts/time_decode.py --model mistral-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e20.err
  timeout 60 python scripts/time_decode.py --model llama2-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e20.err
done; done
timeout 60 python scripts/trace_decode.py --model mistral-7b --opt gate_first_tail=1 --opt lazy_tail=32 > gpurun_out/e20_trace.txt 2>&1
