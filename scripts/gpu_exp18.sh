#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests -m gpu -q -k "calibration" --timeout 1200 -p no:cacheprovider > gpurun_out/e18_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e18_tests.log
timeout 600 python scripts/bench_calib.py --source gaussian --reps 3 > gpurun_out/e18_calib.json 2> gpurun_out/e18.err
