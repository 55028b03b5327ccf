#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for LT in 8 16 1000; do
  export CATS_LAZY_TAIL=$LT
  for cfg in "--model mistral-7b" "--model llama2-7b --k 0.9" "--model llama2-13b --m 1728" "--model llama2-7b --batch 2" "--model llama2-7b --batch 8"; do
    timeout 120 python scripts/time_decode.py $cfg --tag lt$LT 2>/dev/null | grep '^{' | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['tag'], r['model'], r['m'], 'b', r['b'], 'k', r['k'], r['us'])"
  done
done
