#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 2400 python -m pytest tests -m "gpu and not slow" -q --timeout 900 -p no:cacheprovider > gpurun_out/e4_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e4_tests.log
timeout 600 python scripts/bench_calib.py --source gaussian --reps 3 > gpurun_out/e4_calib.json 2> gpurun_out/e4_calib.err
timeout 300 python scripts/bench_calib.py --source gaussian --dtype f32 --n 2000000000 --reps 3 > gpurun_out/e4_calib_f32.json 2>> gpurun_out/e4_calib.err
timeout 1200 python -m pytest tests -m "gpu and slow" -q --timeout 1200 -p no:cacheprovider > gpurun_out/e4_slow.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e4_slow.log
