#!/bin/bash
# The gpurun batches of this repo, one named batch per call (at most one ncu command per batch):
#
#   gpurun --timeout 3600 -- 'bash scripts/gpu_batch.sh <batch> [args]'
#
#   validate      smoke(), every -m gpu test, a bench line of each arm (ours, --impl reference)
#   evidence      the closing evidence: validate + BASELINE sweep, App. D ablation grid, calibration
#                 config 4 (both input sources), traces (Mistral b = 1, Llama2-13B b = 8), TP reduction
#   calib         calibration parity (incl. config 4) and config-4 timings (bf16 both sources, fp32)
#   ab            libcats.so vs libcats_ab.so (another build, same box), interleaved; env SPECS =
#                 "model m batch;..." and TESTS = a pytest -k expression run against libcats.so afterwards
#   paths         K12 vs KA + KB (options.path) on Mistral / Llama2-7B layers and shards
#   ncu_k12       bench line, then ncu --set full of K12 (Mistral b = 1)
#   ncu_ka MODEL B   traces of KA + KB, then ncu --set full of KA at (MODEL, b = B)
#   ncu_calib     ncu --set full of the calibration full pass (2e9 bf16)
#   ncu_list      ncu launch list (gpu__time_duration.sum) of scripts/prof_decode.py
#
# Outputs land in gpurun_out/<batch>_*; profiles/ holds the committed summaries.
cd "${GRAFT_REPO_ROOT:-.}"
o=gpurun_out
batch=$1
shift

validate() {
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${batch}_smoke.log 2>&1
    echo "smoke rc=$?" >> $o/${batch}_smoke.log
    timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > $o/${batch}_tests.log 2>&1
    echo "pytest rc=$?" >> $o/${batch}_tests.log
    timeout 600 python bench.py --steps 2000 --warmup 50 > $o/${batch}_bench.log 2>&1
    echo "bench rc=$?" >> $o/${batch}_bench.log
    timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $o/${batch}_ref.log 2>&1
    echo "ref rc=$?" >> $o/${batch}_ref.log
}

calib() {
    timeout 900 python scripts/bench_calib.py --source gate --oracle > $o/${batch}_calib_gate.json 2> $o/${batch}_calib.err
    timeout 600 python scripts/bench_calib.py --source gaussian > $o/${batch}_calib_gauss.json 2>> $o/${batch}_calib.err
}

case "$batch" in
validate)
    validate ;;
evidence)
    validate
    timeout 2400 python scripts/bench_sweep.py > $o/${batch}_sweep.jsonl 2> $o/${batch}_sweep.err
    : > $o/${batch}_ablation.jsonl
    for model in mistral-7b llama2-7b; do for k in 0.5 0.7 0.9; do for c in 0 1 2; do
        timeout 120 python scripts/time_decode.py --model $model --k $k --tag "compaction=$c" --opt compaction=$c \
            >> $o/${batch}_ablation.jsonl 2>> $o/${batch}.err
    done; done; done
    calib
    timeout 120 python scripts/trace_decode.py --model mistral-7b > $o/${batch}_trace_mistral.txt 2>&1
    timeout 120 python scripts/trace_decode.py --model llama2-13b --batch 8 > $o/${batch}_trace_13b_b8.txt 2>&1
    timeout 300 python scripts/time_tp_reduce.py > $o/${batch}_tp.jsonl 2>> $o/${batch}.err ;;
calib)
    timeout 1500 python -m pytest tests -m gpu -q -k "calibration" --timeout 1200 -p no:cacheprovider > $o/${batch}_tests.log 2>&1
    echo "pytest rc=$?" >> $o/${batch}_tests.log
    calib
    timeout 300 python scripts/bench_calib.py --source gaussian --dtype f32 --n 2000000000 > $o/${batch}_calib_f32.json 2>> $o/${batch}_calib.err ;;
ab)
    out=$o/ab.jsonl; : > $out
    SPECS=${SPECS:-"mistral-7b 14336 1;llama2-7b 11008 1;llama2-7b 11008 4"}
    TESTS=${TESTS:-"k12 or app_d or fused_path or small or deterministic or mixed or decode_host or gate_act or t0"}
    for i in 1 2 3; do for lib in libcats.so libcats_ab.so; do
        IFS=';'; for spec in $SPECS; do
            IFS=' '; set -- $spec
            timeout 60 python scripts/time_decode.py --model $1 --m $2 --batch $3 --lib $lib --tag $lib >> $out 2>> $o/ab.err
        done; IFS=' '
    done; done
    timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$TESTS" > $o/ab_tests.log 2>&1
    echo "tests rc=$?" >> $o/ab_tests.log ;;
paths)
    out=$o/${batch}.jsonl; : > $out
    for spec in "mistral-7b 14336" "mistral-7b 7168" "mistral-7b 3584" "mistral-7b 1792" "llama2-7b 11008" "llama2-7b 2752"; do
        set -- $spec
        for path in 0 2; do
            timeout 120 python scripts/time_decode.py --model $1 --m $2 --tag "path=$path" --opt path=$path >> $out 2>> $o/${batch}.err
        done
    done ;;
ncu_k12)
    timeout 600 python bench.py --steps 2000 --warmup 50 > $o/${batch}_bench.log 2>&1
    timeout 120 python scripts/prof_decode.py > $o/${batch}_plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k12_cats_mlp -s 10 -c 1 \
        -o $o/${batch}_k12 python scripts/prof_decode.py > $o/${batch}_ncu.log 2>&1
    echo "ncu rc=$?" >> $o/${batch}_ncu.log ;;
ncu_ka)
    model=${1:-llama2-7b}; b=${2:-8}
    timeout 120 python scripts/trace_decode.py --model $model --batch $b > $o/${batch}_trace.txt 2>&1
    timeout 120 python scripts/prof_decode.py --model $model --batch $b > $o/${batch}_plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:ka_gate_up -s 2 -c 1 \
        -o $o/${batch}_ka python scripts/prof_decode.py --model $model --batch $b > $o/${batch}_ncu.log 2>&1
    echo "ncu rc=$?" >> $o/${batch}_ncu.log ;;
ncu_calib)
    timeout 300 python scripts/prof_calib.py > $o/${batch}_plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:calib_hist_tma -c 1 \
        -o $o/${batch}_calib python scripts/prof_calib.py > $o/${batch}_ncu.log 2>&1
    echo "ncu rc=$?" >> $o/${batch}_ncu.log ;;
ncu_list)
    timeout 120 python scripts/prof_decode.py > $o/${batch}_plain.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${batch}_launches.csv \
        python scripts/prof_decode.py > $o/${batch}_ncu.log 2>&1
    echo "ncu rc=$?" >> $o/${batch}_ncu.log ;;
*)
    echo "unknown batch '$batch' (see the header of scripts/gpu_batch.sh)"; exit 2 ;;
esac
