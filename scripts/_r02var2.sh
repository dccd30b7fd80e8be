set -u
O=gpurun_out; mkdir -p $O
SH=B16c16384k8q64,B8c32768k8q64,B32c8192k8q64,B16c32768k8q64,B4c32768k32,B8c16384k32,B16c16384k8,B8c32768k8
for rep in 1 2; do
for v in 1 2 9; do
  ADR_DECODE_VARIANT=$v timeout 400 python scripts/small_call_bench.py --grids dynamic --no-host --no-floor --no-trt --shapes $SH > $O/var2_${v}_$rep.txt 2>&1
done
done
