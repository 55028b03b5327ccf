#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2 3; do
timeout 300 python scripts/trace_decode.py 2>&1 | grep -E "jobs_done|exit|k12_visible" 
done
