#!/usr/bin/env bash
# ncu evidence for the bench workload (run on the GPU box via gpurun, 1 GPU).
#   1) launch list of our kernels with device times (cold-cache, serialised:
#      compare shares, not absolutes)
#   2) one --set full capture of the main decode-attention kernel
# Outputs land in gpurun_out/; summaries are copied to profiles/ by
# scripts/summarize_ncu.py.
set -euo pipefail
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p "$OUT"
NCU=${NCU:-ncu}
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:decode_attn|decode_merge|kv_append' --csv --log-file "$OUT/launches_${TAG}.csv" \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_bench_${TAG}.json" 2>&1 || true
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on \
  -k 'regex:decode_attn_kernel' -s 40 -c 2 -o "$OUT/prof_${TAG}" -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full_${TAG}.log" 2>&1 || true
ls -la "$OUT"
