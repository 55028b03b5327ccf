#!/bin/bash
# KA at b = 8 (Llama2-7B): traces at b = 4 / 8 and one ncu --set full capture of ka_gate_up
cd "${GRAFT_REPO_ROOT:-.}"
timeout 120 python scripts/trace_decode.py --model llama2-7b --batch 8 > gpurun_out/e24_trace_b8.txt 2>&1
timeout 120 python scripts/trace_decode.py --model llama2-7b --batch 4 > gpurun_out/e24_trace_b4.txt 2>&1
timeout 120 python scripts/prof_decode.py --model llama2-7b --batch 8 > gpurun_out/e24_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ka_gate_up -s 2 -c 1 -o gpurun_out/e24_ka_b8 python scripts/prof_decode.py --model llama2-7b --batch 8 > gpurun_out/e24_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/e24_ncu.log
