#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1800 python -m pytest tests -m gpu -q -k "every_planned or tp_shard or fused_path" --timeout 900 -p no:cacheprovider > gpurun_out/e9_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e9_tests.log
timeout 1800 python scripts/bench_sweep.py --only N3,C3 > gpurun_out/r02_sweep_b.jsonl 2> gpurun_out/e9_sweep.err
