#!/bin/bash
# KA in column parts vs full-row jobs at b = 8 / 4 (Llama2-7B): traces of both builds, ncu of the new KA
cd "${GRAFT_REPO_ROOT:-.}"
for lib in libcats.so libcats_ab.so; do for b in 8 4; do
  timeout 120 python scripts/trace_decode.py --model llama2-7b --batch $b --lib $lib > gpurun_out/e25_${lib}_b$b.txt 2>&1
done; done
timeout 120 python scripts/prof_decode.py --model llama2-7b --batch 8 > gpurun_out/e25_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ka_gate_up -s 2 -c 1 -o gpurun_out/e25_ka_b8 python scripts/prof_decode.py --model llama2-7b --batch 8 > gpurun_out/e25_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/e25_ncu.log
