#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python bench.py --steps 400 --warmup 20 > gpurun_out/e7_bench.log 2>&1
for model in mistral-7b llama2-7b; do timeout 120 python scripts/time_decode.py --model $model >> gpurun_out/e7_td.jsonl 2>> gpurun_out/e7.err; done
timeout 900 python scripts/sanitize_run.py > gpurun_out/e7_san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python scripts/sanitize_run.py > gpurun_out/e7_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/e7_memcheck.log
