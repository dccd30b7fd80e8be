set -u
O=gpurun_out; mkdir -p $O
SH=B4c1024k8q64,B8c2048k8q64,B16c2048k8q64,B8c8192k8q64,B8c16384k8q64,B16c4096k8q64,B32c2048k8q64
timeout 600 python scripts/small_call_bench.py --grids dynamic --no-host --no-trt --no-floor --shapes $SH > $O/g8_streamk_r02q.txt 2>&1
for v in 0 1 5; do echo "variant $v" >> $O/g8_split_r02q.txt; ADR_SPLIT_VARIANT=$v timeout 600 python scripts/small_call_bench.py --grids split --no-host --no-trt --no-floor --shapes $SH >> $O/g8_split_r02q.txt 2>&1; done
SH4=B16c4096k8,B8c8192k8,B32c2048k8,B64c1024k8
for v in 0 5; do echo "variant $v" >> $O/g4_split_r02q.txt; ADR_SPLIT_VARIANT=$v timeout 600 python scripts/small_call_bench.py --grids split --no-host --no-trt --no-floor --shapes $SH4 >> $O/g4_split_r02q.txt 2>&1; done
