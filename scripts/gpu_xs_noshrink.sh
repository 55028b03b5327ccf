#!/bin/bash
# XS: clusters kept at the forced R even when not all are co-resident (CATS_XS_NOSHRINK=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/xs_noshrink.jsonl
for shape in "4096:12288" "4096:6144" "4096:4096"; do
  set -- ${shape/:/ }
  for b in 4 8; do
    for r in 3 4; do
      CATS_XS_NOSHRINK=1 CATS_XS_COLS=128 CATS_XS_R=$r timeout 60 python scripts/time_xsparse.py --d-in $1 --d-out $2 --batch $b --k 0.5 --tag ns_c128r$r >> gpurun_out/xs_noshrink.jsonl 2>> gpurun_out/xs_noshrink.err
    done
  done
done
cut -c1-150 gpurun_out/xs_noshrink.jsonl
tail -3 gpurun_out/xs_noshrink.err
