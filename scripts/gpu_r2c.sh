#!/bin/bash
# closing evidence (round 2): full GPU suite, smoke, the BASELINE sweep, the App. D ablation grid,
# calibration config 4, Mistral / Llama2-7B b = 8 traces, TP reduction timing, bench lines (both arms)
cd "${GRAFT_REPO_ROOT:-.}"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2c_smoke.log
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c_tests.log
timeout 2400 python scripts/bench_sweep.py > gpurun_out/r2c_sweep.jsonl 2> gpurun_out/r2c_sweep.err
: > gpurun_out/r2c_ablation.jsonl
for model in mistral-7b llama2-7b; do for k in 0.5 0.7 0.9; do for c in 0 1 2; do
  timeout 120 python scripts/time_decode.py --model $model --k $k --tag "compaction=$c" --opt compaction=$c >> gpurun_out/r2c_ablation.jsonl 2>> gpurun_out/r2c.err
done; done; done
timeout 900 python scripts/bench_calib.py --source gate --oracle > gpurun_out/r2c_calib_gate.json 2> gpurun_out/r2c_calib.err
timeout 600 python scripts/bench_calib.py --source gaussian > gpurun_out/r2c_calib_gauss.json 2>> gpurun_out/r2c_calib.err
timeout 120 python scripts/trace_decode.py --model mistral-7b > gpurun_out/r2c_trace_mistral.txt 2>&1
timeout 120 python scripts/trace_decode.py --model llama2-13b --batch 8 > gpurun_out/r2c_trace_13b_b8.txt 2>&1
timeout 300 python scripts/time_tp_reduce.py > gpurun_out/r2c_tp.jsonl 2>> gpurun_out/r2c.err
timeout 600 python bench.py --steps 2000 --warmup 50 > gpurun_out/r2c_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2c_ref.log 2>&1
