#!/bin/bash
# K12 L2 prefetch of static tiles (CATS_K12_L2PF) across shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for pf in 0 4 8; do
  export CATS_K12_L2PF=$pf
  for cfg in "--model mistral-7b" "--model llama2-7b --k 0.9" "--model llama2-7b" "--model llama2-13b" "--model mistral-7b --m 1792"; do
    timeout 120 python scripts/time_decode.py $cfg --tag pf$pf 2>/dev/null | grep '^{' | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['tag'], r['model'], r['m'], 'k', r['k'], r['us'])"
  done
done
