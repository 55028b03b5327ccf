#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1800 python -m pytest tests -m gpu -q -k "not calibration and not xsparse" --timeout 900 -p no:cacheprovider > gpurun_out/e21_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e21_tests.log
grep -q "pytest rc=0" gpurun_out/e21_tests.log || exit 1
out=gpurun_out/e21.jsonl; : > $out
for i in 1 2; do
for spec in "llama2-13b 13824 1" "llama2-13b 1728 1" "llama2-7b 11008 2" "llama2-7b 11008 4" "llama2-7b 11008 8" "mistral-7b 14336 1"; do
  set -- $spec
  timeout 60 python scripts/time_decode.py --model $1 --m $2 --batch $3 >> $out 2>> gpurun_out/e21.err
done; done
timeout 60 python scripts/trace_decode.py --model llama2-13b --m 1728 > gpurun_out/e21_tp8.txt 2>&1
timeout 60 python scripts/trace_decode.py --model llama2-7b --batch 2 > gpurun_out/e21_b2.txt 2>&1
