#!/bin/bash
# batch-path evaluation: tests for the split path, graph-timed b = 2..8, traces at b = 2, 8
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tag=${1:-evalb}
out=gpurun_out/$tag.jsonl
: > $out
timeout 400 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for b in 2 4 8; do
  for k in 0.5 0.9; do
    timeout 120 python scripts/time_decode.py --model llama2-7b --batch $b --k $k 2>/dev/null | grep '^{' >> $out
  done
done
timeout 120 python scripts/time_decode.py --model llama2-7b --batch 8 --dense 2>/dev/null | grep '^{' >> $out
: > gpurun_out/${tag}_trace.log
for b in 2 8; do
  timeout 120 python scripts/trace_decode.py --model llama2-7b --batch $b >> gpurun_out/${tag}_trace.log 2>&1
done
tail -2 gpurun_out/${tag}_tests.log
python - "$out" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    r = json.loads(l)
    print(f"{r['model']:11s} m={r['m']:6d} b={r['b']} k={r['k']} dense={int(r['dense'])} us={r['us']:8.3f} eff={r['eff_GBps']:7.1f} union={r['union']}")
PY
grep -v "^Exception\|Traceback\|File \|AttributeError" gpurun_out/${tag}_trace.log
