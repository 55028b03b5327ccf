#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/traceb.log
for b in 2 8; do timeout 120 python scripts/trace_decode.py --model llama2-7b --batch $b >> gpurun_out/traceb.log 2>&1; done
for b in 2 4 8; do timeout 120 python scripts/time_decode.py --model llama2-7b --batch $b 2>/dev/null | grep '^{' >> gpurun_out/traceb.log; done
grep -v "^Exception\|Traceback\|File \|AttributeError" gpurun_out/traceb.log
