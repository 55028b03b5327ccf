#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python scripts/trace_decode.py --json gpurun_out/trace_b1.json > gpurun_out/trace.log 2>&1
timeout 300 python scripts/trace_decode.py --dense >> gpurun_out/trace.log 2>&1
timeout 300 python scripts/trace_decode.py --batch 8 >> gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
