#!/bin/bash
# K12 after the accumulator change: parity subset, a bench line, then one ncu --set full capture of K12
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k12 or app_d or fused_path or small or deterministic or mixed or decode_host or gate_act or t0 or full_size" > gpurun_out/r2d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2d_tests.log
timeout 600 python bench.py --steps 2000 --warmup 50 > gpurun_out/r2d_bench.log 2>&1
timeout 120 python scripts/prof_decode.py > gpurun_out/r2d_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k12_cats_mlp -s 10 -c 1 -o gpurun_out/r2d_k12 python scripts/prof_decode.py > gpurun_out/r2d_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2d_ncu.log
