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
  # torch's own kernels are outside the --kernel-name filter, so their writes are not
  # tracked and every cudaMemcpy of their outputs would read as uninitialised
  [ "$tool" = initcheck ] && extra="--check-api-memory-access no"
  timeout ${CS_TIMEOUT:-1800} "$CS" --tool "$tool" $extra --kernel-name regex='decode_attn|decode_split|kv_append|pack_qkv|unpack_qkv|scatter_out|kv_transfer|check_tables' \
    --print-limit 200 python scripts/sanitize_driver.py > "gpurun_out/sanitize_${tool}.log" 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_driver:' gpurun_out/sanitize_${tool}.log | tr '\n' ' ')" \
    >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
