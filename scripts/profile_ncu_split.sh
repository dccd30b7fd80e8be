#!/usr/bin/env bash
# ncu evidence for the split-pair kernel (small calls): one --set full capture per
# shape of scripts/small_call_bench.py's eager chain (graph off: ncu replays each
# launch in isolation anyway). Outputs: gpurun_out/prof_split_<shape>_<tag>.ncu-rep
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p "$OUT"
NCU=${NCU:-ncu}
for sh in ${SHAPES:-B8c1024k8 B32c4096k8}; do
  timeout -s KILL 600 $NCU --set full --clock-control none --import-source on \
    -k 'regex:decode_split_kernel' -s 20 -c 2 -o "$OUT/prof_split_${sh}_${TAG}" -f \
    python scripts/small_call_bench.py --grids auto --no-host --no-trt --no-floor --reps 2 \
    --shapes $sh > "$OUT/ncu_split_${sh}_${TAG}.log" 2>&1 || true
done
ls -la "$OUT" | grep prof_split
