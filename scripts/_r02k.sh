set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -q -p no:cacheprovider --timeout 300 -k "split" > $O/tests_static_r02k.log 2>&1; echo "rc=$?" >> $O/tests_static_r02k.log
ADR_SPLIT_DYNAMIC=1 timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -q -p no:cacheprovider --timeout 300 -k "split" > $O/tests_dyn_r02k.log 2>&1; echo "rc=$?" >> $O/tests_dyn_r02k.log
SH=B16c1024k32,B64c2048k8,B32c4096k8,B64c4096k8,B16c4096k32,B16c32768k8q64,B64c4096k32
timeout 600 python scripts/small_call_bench.py --grids auto --no-host --no-trt --no-floor --shapes $SH > $O/dyn_auto_r02k.txt 2>&1
echo "static" >> $O/dyn_var_r02k.txt
ADR_SPLIT_DYNAMIC=0 timeout 600 python scripts/small_call_bench.py --grids split --no-host --no-trt --no-floor --shapes $SH >> $O/dyn_var_r02k.txt 2>&1
for c in 1 4 16; do echo "dynamic cost $c" >> $O/dyn_var_r02k.txt; ADR_SPLIT_DYNAMIC=1 ADR_SPLIT_DYN_COST=$c timeout 600 python scripts/small_call_bench.py --grids split --no-host --no-trt --no-floor --shapes $SH >> $O/dyn_var_r02k.txt 2>&1; done
