#!/bin/bash
# App. B input-sparse projection: GPU parity + the full GPU suite, then graph-timed shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xsparse.py -x -q > gpurun_out/pytest_xs.log 2>&1; echo "xs rc=$?" >> gpurun_out/pytest_xs.log
if [ "${XS_FULL:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/pytest_gpu.log
fi
: > gpurun_out/xsparse.jsonl
for shape in ${XS_SHAPES:-"4096:6144" "4096:12288" "5120:5120" "4096:4096"}; do
  set -- ${shape/:/ }
  for b in ${XS_BATCHES:-1 2 4 8}; do
    for k in 0.5 0.7; do
      timeout 120 python scripts/time_xsparse.py --d-in $1 --d-out $2 --batch $b --k $k >> gpurun_out/xsparse.jsonl 2>> gpurun_out/xsparse.err
    done
  done
done
tail -n 3 gpurun_out/pytest_xs.log gpurun_out/pytest_gpu.log
cut -c1-260 gpurun_out/xsparse.jsonl
