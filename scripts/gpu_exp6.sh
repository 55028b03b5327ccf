#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -m gpu -q -k "tail_geometry or calibration" --timeout 900 -p no:cacheprovider > gpurun_out/e6_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e6_tests.log
out=gpurun_out/e6_tail.jsonl; : > $out
for cfg in "" "--opt tail_rows=2 --opt tail_tiles=1 --opt tail_fused=1" "--opt tail_rows=2 --opt tail_tiles=2 --opt tail_fused=1" "--opt tail_rows=2 --opt tail_tiles=3 --opt tail_fused=1" "--opt tail_rows=2 --opt tail_tiles=1" ; do
  timeout 120 python scripts/time_decode.py --model mistral-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e6.err
  timeout 120 python scripts/time_decode.py --model llama2-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e6.err
done
timeout 120 python scripts/trace_decode.py --model mistral-7b --opt tail_rows=2 --opt tail_tiles=2 --opt tail_fused=1 > gpurun_out/e6_trace.txt 2>&1
