#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests -m gpu -q -k "calibration and not full_size" --timeout 600 -p no:cacheprovider > gpurun_out/e2_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/e2_tests.log
timeout 600 python scripts/bench_calib.py --source gaussian --reps 3 > gpurun_out/e2_calib.json 2> gpurun_out/e2_calib.err
out=gpurun_out/e2_shards.jsonl; : > $out
for msh in 13824 6912 3456 1728; do for path in 0 2; do
  timeout 120 python scripts/time_decode.py --model llama2-13b --m $msh --tag "path=$path" --opt path=$path >> $out 2>> gpurun_out/e2.err
done; done
for msh in 3456 1728; do for mt in 1 2 4; do
  timeout 120 python scripts/time_decode.py --model llama2-13b --m $msh --tag "min_tiles=$mt" --opt min_tiles=$mt >> $out 2>> gpurun_out/e2.err
done; done
timeout 300 python -m pytest tests -m gpu -q -k "tp_shard" --timeout 600 -p no:cacheprovider > gpurun_out/e2_tp.log 2>&1
