#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for b in 1 2 4 8; do
  echo "== batch $b" 
  timeout 300 python scripts/trace_decode.py --batch $b 2>&1 | grep -v "Exception\|Trace\|del\|Attrib" | grep -E "K12 per|jobs_done|exit|k12_visible|consumer wait|producer busy|gate jobs|ud jobs"
done
