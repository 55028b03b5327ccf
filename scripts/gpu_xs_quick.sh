#!/bin/bash
# XS (App. B): GPU parity, then default-config timings at every batch size for two shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_xsparse.py -x -q > gpurun_out/pytest_xs.log 2>&1; echo "xs rc=$?" >> gpurun_out/pytest_xs.log
: > gpurun_out/xs_quick.jsonl
for shape in ${XS_SHAPES:-"4096:12288" "4096:6144" "5120:5120" "4096:4096"}; do
  set -- ${shape/:/ }
  for b in 1 2 4 8; do
    timeout 60 python scripts/time_xsparse.py --d-in $1 --d-out $2 --batch $b --k 0.5 >> gpurun_out/xs_quick.jsonl 2>> gpurun_out/xs_quick.err
  done
done
tail -n 2 gpurun_out/pytest_xs.log
cut -c1-200 gpurun_out/xs_quick.jsonl
