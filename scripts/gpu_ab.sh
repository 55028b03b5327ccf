#!/bin/bash
# A/B of two library builds on the same box, interleaved: libcats.so vs libcats_ab.so
# (SPECS: "model m batch" triples; TESTS: a pytest -k expression run afterwards against libcats.so)
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/ab.jsonl; : > $out
SPECS=${SPECS:-"mistral-7b 14336 1;llama2-7b 11008 1;llama2-7b 11008 4"}
TESTS=${TESTS:-"k12 or app_d or fused_path or small or deterministic or mixed or decode_host or gate_act or t0"}
for i in 1 2 3; do for lib in libcats.so libcats_ab.so; do
IFS=';'; for spec in $SPECS; do
  IFS=' '; set -- $spec
  timeout 60 python scripts/time_decode.py --model $1 --m $2 --batch $3 --lib $lib --tag $lib >> $out 2>> gpurun_out/ab.err
done; IFS=' '; done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$TESTS" > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_tests.log
