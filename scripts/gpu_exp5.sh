#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests -m gpu -q -k "calibration" --timeout 1200 -p no:cacheprovider > gpurun_out/e5_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e5_tests.log
timeout 600 python scripts/bench_calib.py --source gaussian --reps 3 > gpurun_out/e5_calib.json 2> gpurun_out/e5_calib.err
timeout 300 python scripts/bench_calib.py --source gaussian --dtype f32 --n 2000000000 --reps 3 > gpurun_out/e5_calib_f32.json 2>> gpurun_out/e5_calib.err
timeout 120 python scripts/trace_decode.py --model mistral-7b > gpurun_out/e5_trace.txt 2>&1
timeout 120 python scripts/trace_decode.py --model llama2-13b --m 1728 > gpurun_out/e5_trace_tp8.txt 2>&1
