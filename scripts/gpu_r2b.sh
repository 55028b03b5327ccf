#!/bin/bash
# evidence after the lean-K12 restore: the BASELINE sweep, the App. D ablation grid, a Mistral trace,
# a bench line and the launch list (one ncu command)
cd "${GRAFT_REPO_ROOT:-.}"
timeout 2400 python scripts/bench_sweep.py > gpurun_out/r2b_sweep.jsonl 2> gpurun_out/r2b_sweep.err
: > gpurun_out/r2b_ablation.jsonl
for model in mistral-7b llama2-7b; do for k in 0.5 0.7 0.9; do for c in 0 1 2; do
  timeout 120 python scripts/time_decode.py --model $model --k $k --tag "compaction=$c" --opt compaction=$c >> gpurun_out/r2b_ablation.jsonl 2>> gpurun_out/r2b.err
done; done; done
timeout 120 python scripts/trace_decode.py --model mistral-7b > gpurun_out/r2b_trace_mistral.txt 2>&1
timeout 600 python bench.py --steps 2000 --warmup 50 > gpurun_out/r2b_bench.log 2>&1
python scripts/prof_decode.py > gpurun_out/r2b_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv python scripts/prof_decode.py > gpurun_out/r2b_ncu_list.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2b_ncu_list.log
