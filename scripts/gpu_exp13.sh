#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests -m gpu -q -k "every_planned or tp_shard or mixed or deterministic or small or split" --timeout 900 -p no:cacheprovider > gpurun_out/e13_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e13_tests.log
out=gpurun_out/e13_shards.jsonl; : > $out
for msh in 13824 3456 1728; do timeout 60 python scripts/time_decode.py --model llama2-13b --m $msh >> $out 2>> gpurun_out/e13.err; done
for b in 2 8; do timeout 60 python scripts/time_decode.py --model llama2-7b --batch $b >> $out 2>> gpurun_out/e13.err; done
