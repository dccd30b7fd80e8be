#!/usr/bin/env bash
# One gpurun call's worth of checks (each step under its own timeout so a hang
# cannot eat the call). Usage: scripts/gpu_round.sh TAG [steps...]
#   steps: tests-split tests-new tests-all small small-variants capacity bench ref ncu sanitize
set -u
export PYTHONUNBUFFERED=1
cd "$(dirname "$0")/.."
TAG=$1; shift
O=gpurun_out
mkdir -p $O
for step in "$@"; do
  case $step in
    tests-split)
      timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -q -p no:cacheprovider --timeout 300 -k "split" > $O/tests_split_$TAG.log 2>&1; echo "rc=$?" >> $O/tests_split_$TAG.log ;;
    tests-new)
      timeout 900 python -m pytest tests/test_gpu_pricer.py tests/test_gpu_kv_exchange.py tests/test_gpu_ipc.py -q -p no:cacheprovider --timeout 400 > $O/tests_new_$TAG.log 2>&1; echo "rc=$?" >> $O/tests_new_$TAG.log ;;
    tests-all)
      timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 > $O/gpu_tests_$TAG.log 2>&1; echo "rc=$?" >> $O/gpu_tests_$TAG.log ;;
    small)
      timeout 900 python scripts/small_call_bench.py --grids ${SMALL_GRIDS:-auto,split,static,dynamic} --no-host $O/small_call_$TAG.json > $O/small_call_$TAG.log 2>&1 ;;
    small-variants)
      for v in ${VARIANTS:-0 1 2 4}; do
        ADR_SPLIT_VARIANT=$v timeout 400 python scripts/small_call_bench.py --grids split --no-host --no-trt --no-floor \
          --shapes ${VSHAPES:-B4c512k8,B8c1024k8,B16c1024k8,B8c1024k32,B16c1024k32,B64c1024k8,B32c2048k8,B64c4096k8,B64c4096k32} > $O/small_variant${v}_$TAG.log 2>&1
      done ;;
    capacity)
      for c in C4 C5; do
        timeout 900 python bench.py --capacity --capacity-config $c --steps 10 --warmup 3 > $O/capacity_${c}_$TAG.json 2> $O/capacity_${c}_$TAG.err
      done ;;
    bench)
      timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err ;;
    ref)
      timeout 600 python bench.py --impl reference > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err ;;
    ncu)
      timeout 1500 bash scripts/profile_ncu.sh $TAG > $O/ncu_$TAG.log 2>&1 ;;
    timeline-small)
      for sh in ${TL_SHAPES:-B4c512k8 B8c1024k8 B4c512k32 B16c1024k32}; do
        for g in ${TL_GRIDS:-static split}; do
          timeout 300 python scripts/timeline.py $sh --grid=$g --graph >> $O/timeline_small_$TAG.txt 2>&1
        done
      done ;;
    bmax)
      for m in llama2-7b llama2-13b llama3-8b; do
        timeout 600 python -m paper_2503_20552_b200.cli bmax --model $m --out $O/bmax_${m}_$TAG.json >> $O/bmax_$TAG.log 2>&1
      done ;;
    calibrate)
      timeout 900 python scripts/calibrate_coloc.py $O/coloc_curves_$TAG.json > $O/calibrate_$TAG.log 2>&1 ;;
    closed-loop)
      timeout ${CL_TIMEOUT:-2400} python scripts/closed_loop.py $O/closed_loop_$TAG.json --curves ${CURVES:-$O/coloc_curves_$TAG.json} ${CL_CASES:-4P4D} > $O/closed_loop_$TAG.log 2>&1 ;;
    sanitize)
      timeout 2400 bash scripts/sanitize.sh > $O/sanitize_$TAG.log 2>&1 ;;
  esac
  echo "step $step done"
done
