#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1800 python scripts/bench_sweep.py --only N3,C3 > gpurun_out/r02_sweep_b.jsonl 2> gpurun_out/e8_sweep.err
timeout 900 python scripts/sanitize_run.py --debug > gpurun_out/r02_debug_checks.log 2>&1
echo "debug-checks rc=$?" >> gpurun_out/r02_debug_checks.log
timeout 120 python scripts/trace_decode.py --model llama2-7b --batch 8 > gpurun_out/e8_trace_b8.txt 2>&1
