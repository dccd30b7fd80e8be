#!/usr/bin/env bash
# compute-sanitizer over scripts/sanitize_driver.py (run on a GPU box via gpurun).
# Logs: gpurun_out/sanitize_<tool>.log ; summary: gpurun_out/sanitize_summary.txt
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
: > gpurun_out/sanitize_summary.txt
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no --padding 64"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  filter="--kernel-name regex=decode_attn|decode_split|kv_append|pack_qkv|unpack_qkv|scatter_out|kv_transfer|check_tables"
  # initcheck must see every kernel: with the filter, the writes of torch's own kernels
  # (the zero-filled workspace, the synthetic inputs) are untracked and read as uninitialised
  [ "$tool" = initcheck ] && filter=""
  timeout ${CS_TIMEOUT:-1800} "$CS" --tool "$tool" $extra $filter \
    --print-limit 200 python scripts/sanitize_driver.py > "gpurun_out/sanitize_${tool}.log" 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_driver:' gpurun_out/sanitize_${tool}.log | tr '\n' ' ')" \
    >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
