#!/bin/bash
# quick evaluation: GPU parity tests, graph-timed shapes, one trace; args: tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tag=${1:-eval}
out=gpurun_out/$tag.jsonl
: > $out
timeout 400 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for cfg in "--model mistral-7b" "--model mistral-7b --dense" "--model llama2-7b --k 0.9" "--model llama2-7b --k 0.7" \
           "--model llama2-13b --m 1728" "--model llama2-13b --m 3456" "--model llama2-13b --m 6912" "--model llama2-13b" \
           "--model llama2-7b --batch 2" "--model llama2-7b --batch 4" "--model llama2-7b --batch 8"; do
  timeout 120 python scripts/time_decode.py $cfg 2>/dev/null | grep '^{' >> $out
done
CATS_TRACE=1 timeout 120 python scripts/trace_decode.py > gpurun_out/${tag}_trace.log 2>&1
CATS_TRACE=1 timeout 120 python scripts/trace_decode.py --model llama2-13b --m 1728 >> gpurun_out/${tag}_trace.log 2>&1
tail -2 gpurun_out/${tag}_tests.log
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    r = json.loads(l)
    print(f"{r['model']:11s} m={r['m']:6d} b={r['b']} k={r['k']} dense={int(r['dense'])} us={r['us']:8.3f} eff={r['eff_GBps']:7.1f}")
PY
