#!/bin/bash
# tile-claim experiment: reservation cut-off (CATS_LAZY_TAIL x grid tiles) across shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/lazy.jsonl
: > $out
timeout 300 python -m pytest tests -m gpu -x -q -k "parity and not slow" > gpurun_out/lazy_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/lazy_tests.log
for LT in 0 1 2 4; do
  export CATS_LAZY_TAIL=$LT
  timeout 120 python scripts/time_decode.py --model mistral-7b >> $out 2>&1
  timeout 120 python scripts/time_decode.py --model llama2-7b --k 0.9 >> $out 2>&1
  timeout 120 python scripts/time_decode.py --model llama2-13b --m 1728 >> $out 2>&1
  timeout 120 python scripts/time_decode.py --model llama2-13b --m 6912 >> $out 2>&1
done
unset CATS_LAZY_TAIL
CATS_TRACE=1 timeout 120 python scripts/trace_decode.py > gpurun_out/lazy_trace.log 2>&1
CATS_TRACE=1 timeout 120 python scripts/trace_decode.py --model llama2-13b --m 1728 >> gpurun_out/lazy_trace.log 2>&1
tail -3 gpurun_out/lazy_tests.log; cat $out
