#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -m gpu -q -k "extreme" --timeout 600 -p no:cacheprovider > gpurun_out/e14_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e14_tests.log
timeout 300 python scripts/time_tp_reduce.py > gpurun_out/r02_tp_reduce_emulated.jsonl 2> gpurun_out/e14.err
