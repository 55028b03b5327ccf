#!/bin/bash
# GPU test pass on a gpurun box: the -m gpu suite (optionally a -k filter), then a short bench line.
#   scripts/gpu_tests.sh <tag> [pytest -k expression]
tag=${1:-t}; kexpr=${2:-}
cd "${GRAFT_REPO_ROOT:-.}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ -n "$kexpr" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -k "$kexpr" --timeout 900 -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${tag}_tests.log
timeout 600 python bench.py --steps 400 --warmup 20 > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
tail -3 gpurun_out/${tag}_tests.log
