#!/bin/bash
# round-2 closing evidence: tests, sweep, calibration, ablation, TP reduction, bench, ncu (launch list + 2 captures)
cd "${GRAFT_REPO_ROOT:-.}"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/fin_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fin_tests.log
timeout 600 python bench.py --steps 400 --warmup 20 > gpurun_out/fin_bench.log 2>&1
timeout 2400 python scripts/bench_sweep.py > gpurun_out/fin_sweep.jsonl 2> gpurun_out/fin_sweep.err
timeout 900 python scripts/bench_calib.py --source gate --oracle > gpurun_out/fin_calib_gate.json 2> gpurun_out/fin_calib.err
timeout 600 python scripts/bench_calib.py --source gaussian > gpurun_out/fin_calib_gauss.json 2>> gpurun_out/fin_calib.err
: > gpurun_out/fin_ablation.jsonl
for model in mistral-7b llama2-7b; do for k in 0.5 0.7 0.9; do for c in 0 1 2; do
  timeout 120 python scripts/time_decode.py --model $model --k $k --tag "compaction=$c" --opt compaction=$c >> gpurun_out/fin_ablation.jsonl 2>> gpurun_out/fin.err
done; done; done
timeout 300 python scripts/time_tp_reduce.py > gpurun_out/fin_tp.jsonl 2>> gpurun_out/fin.err
python scripts/prof_decode.py > gpurun_out/fin_prof_plain.log 2>&1 && \
python scripts/prof_calib.py > gpurun_out/fin_profcalib_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv python scripts/prof_decode.py > gpurun_out/fin_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k12_cats_mlp -s 10 -c 1 -o gpurun_out/fin_k12 python scripts/prof_decode.py > gpurun_out/fin_ncu_k12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:calib_hist_tma -c 1 -o gpurun_out/fin_calib python scripts/prof_calib.py > gpurun_out/fin_ncu_calib.log 2>&1
echo "ncu rc=$?" >> gpurun_out/fin_ncu_calib.log
