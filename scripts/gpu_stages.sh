#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for st in 0 2; do
  export CATS_K12_STAGES=$st
  for cfg in "--model mistral-7b" "--model llama2-7b --k 0.9" "--model llama2-13b --m 1728" "--model llama2-13b"; do
    timeout 120 python scripts/time_decode.py $cfg --tag st$st 2>/dev/null | grep '^{' | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['tag'], r['model'], r['m'], r['k'], r['us'])"
  done
done
