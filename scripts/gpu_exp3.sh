#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_tp.py -q --timeout 600 -p no:cacheprovider > gpurun_out/e3_tp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e3_tp.log
out=gpurun_out/e3_paths.jsonl; : > $out
for spec in "mistral-7b 14336" "mistral-7b 7168" "mistral-7b 3584" "mistral-7b 1792" "llama2-7b 11008" "llama2-7b 2752"; do
  set -- $spec
  for path in 0 2; do
    timeout 120 python scripts/time_decode.py --model $1 --m $2 --tag "path=$path" --opt path=$path >> $out 2>> gpurun_out/e3.err
  done
done
python scripts/prof_calib.py > gpurun_out/e3_profcalib_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:calib_hist_tma -c 1 -o gpurun_out/calib_prof python scripts/prof_calib.py > gpurun_out/e3_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/e3_ncu.log
