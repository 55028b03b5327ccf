#!/bin/bash
# round-2 evidence: full GPU suite (incl. slow), the BASELINE sweep, calibration config 4 (both sources),
# the App. D ablation grid, a bench line, the launch list and one ncu --set full capture of K12
cd "${GRAFT_REPO_ROOT:-.}"
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/s2_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2_tests.log
timeout 2400 python scripts/bench_sweep.py > gpurun_out/r02_sweep.jsonl 2> gpurun_out/s2_sweep.err
timeout 900 python scripts/bench_calib.py --source gate --oracle > gpurun_out/r02_calib_gate.json 2> gpurun_out/s2_calib.err
timeout 600 python scripts/bench_calib.py --source gaussian > gpurun_out/r02_calib_gauss.json 2>> gpurun_out/s2_calib.err
for model in mistral-7b llama2-7b; do for k in 0.5 0.7 0.9; do for c in 0 1 2; do
  timeout 120 python scripts/time_decode.py --model $model --k $k --tag "compaction=$c" --opt compaction=$c >> gpurun_out/r02_ablation.jsonl 2>> gpurun_out/s2.err
done; done; done
timeout 600 python bench.py --steps 400 --warmup 20 > gpurun_out/s2_bench.log 2>&1
python scripts/prof_decode.py > gpurun_out/s2_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python scripts/prof_decode.py > gpurun_out/s2_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k12_cats_mlp -s 10 -c 1 -o gpurun_out/r02_k12 python scripts/prof_decode.py > gpurun_out/s2_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s2_ncu_full.log
