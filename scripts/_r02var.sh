set -u
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for v in 1 0 3 4 7 8 9 2; do
  ADR_DECODE_VARIANT=$v timeout 300 python scripts/library_compare.py --only none $O/var_${v}_$rep.json > $O/var_${v}_$rep.log 2>&1
done
done
