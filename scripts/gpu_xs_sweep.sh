#!/bin/bash
# XS (App. B) configuration sweep at b >= 2: column slab x cluster size forced through CATS_XS_COLS / CATS_XS_R
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/xs_sweep.jsonl
for shape in "4096:12288" "4096:6144"; do
  set -- ${shape/:/ }
  for b in 2 4 8; do
    for cols in 64 128; do
      for r in 1 2 3 4 6 8; do
        CATS_XS_COLS=$cols CATS_XS_R=$r timeout 60 python scripts/time_xsparse.py --d-in $1 --d-out $2 --batch $b --k 0.5 --reps 30 --tag "c${cols}r${r}" >> gpurun_out/xs_sweep.jsonl 2>> gpurun_out/xs_sweep.err
      done
    done
  done
done
cut -c1-120 gpurun_out/xs_sweep.jsonl
