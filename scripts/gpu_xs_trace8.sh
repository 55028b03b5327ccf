#!/bin/bash
# XS at b = 4/8: per-CTA traces (prologue vs row stream) and forced 64-column slabs (depth-4 register ring)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/xs_trace8.log
for b in 4 8; do
  timeout 60 python scripts/trace_xsparse.py --d-in 4096 --d-out 12288 --batch $b >> gpurun_out/xs_trace8.log 2>&1
done
: > gpurun_out/xs_c64.jsonl
for b in 8; do
  for r in 2 4 8; do
    CATS_XS_COLS=64 CATS_XS_R=$r timeout 60 python scripts/time_xsparse.py --d-in 4096 --d-out 12288 --batch $b --k 0.5 --tag c64r$r >> gpurun_out/xs_c64.jsonl 2>> gpurun_out/xs_c64.err
  done
done
tail -n 40 gpurun_out/xs_trace8.log
cut -c1-200 gpurun_out/xs_c64.jsonl
