#!/bin/bash
# calibration: GPU parity (incl. the full-size config 4) + config-4 timings on both input sources
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests -m gpu -q -k "calibration" --timeout 1200 -p no:cacheprovider > gpurun_out/calib_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/calib_tests.log
timeout 900 python scripts/bench_calib.py --source gate --oracle > gpurun_out/calib_gate.json 2> gpurun_out/calib_gate.err
timeout 600 python scripts/bench_calib.py --source gaussian > gpurun_out/calib_gauss.json 2> gpurun_out/calib_gauss.err
timeout 300 python scripts/bench_calib.py --source gaussian --dtype f32 --n 2000000000 > gpurun_out/calib_f32.json 2> gpurun_out/calib_f32.err
tail -2 gpurun_out/calib_tests.log; cat gpurun_out/calib_*.json
