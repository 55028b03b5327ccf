#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 300 python scripts/sanitize_run.py --debug > gpurun_out/e11_debug.log 2>&1
echo "debug rc=$?" >> gpurun_out/e11_debug.log
grep -q "tp ok" gpurun_out/e11_debug.log || exit 1
timeout 900 python -m pytest tests -m gpu -q -k "tail_geometry" --timeout 300 -p no:cacheprovider > gpurun_out/e11_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e11_tests.log
out=gpurun_out/e11_pool.jsonl; : > $out
for i in 1 2; do
for cfg in "" "--opt ud_pool=1" "--opt convert_ctas=8" "--opt ud_pool=1 --opt convert_ctas=8" "--opt ud_pool=1 --opt convert_ctas=32"; do
  timeout 60 python scripts/time_decode.py --model mistral-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e11.err
  timeout 60 python scripts/time_decode.py --model llama2-7b --tag "$cfg" $cfg >> $out 2>> gpurun_out/e11.err
done; done
timeout 60 python scripts/trace_decode.py --model mistral-7b --opt ud_pool=1 --opt convert_ctas=8 > gpurun_out/e11_trace.txt 2>&1
