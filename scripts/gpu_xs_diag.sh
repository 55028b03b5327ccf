#!/bin/bash
# App. B kernel XS: cluster / column-width experiments at b = 1 and 8 (one JSON line each)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/xs_diag.jsonl
for cfg in "auto" "128:1" "128:2" "128:3" "128:6" "256:1" "256:3" "256:6" "64:3" "64:6"; do
  for b in 1 8; do
    if [ "$cfg" = auto ]; then
      timeout 120 python scripts/time_xsparse.py --batch $b --k 0.5 --tag auto >> gpurun_out/xs_diag.jsonl 2>> gpurun_out/xs_diag.err
    else
      CATS_XS_COLS=${cfg%%:*} CATS_XS_R=${cfg##*:} timeout 120 python scripts/time_xsparse.py --batch $b --k 0.5 --tag $cfg >> gpurun_out/xs_diag.jsonl 2>> gpurun_out/xs_diag.err
    fi
  done
done
cut -c1-400 gpurun_out/xs_diag.jsonl
