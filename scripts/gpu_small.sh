#!/bin/bash
# small-layer (TP shard) knobs: K12 grid sizing and eager ring fill
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "1 0" "2 0" "3 0" "1 1" "2 1" "3 1"; do
  set -- $cfg
  export CATS_K12_MIN_TILES=$1 CATS_K12_EAGER=$2
  for m in 1792 3584 7168 14336; do
    timeout 120 python scripts/time_decode.py --m $m --tag "mt$1e$2" 2>/dev/null | grep '^{' | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['tag'], r['model'], r['m'], r['us'])"
  done
  timeout 120 python scripts/time_decode.py --model llama2-13b --m 1728 --tag "mt$1e$2" 2>/dev/null | grep '^{' | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['tag'], r['model'], r['m'], r['us'])"
done
