set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py tests/test_gpu_graphs.py tests/test_gpu_runtime.py -q -p no:cacheprovider --timeout 300 -x > $O/tests_handoff_r02m.log 2>&1; echo "rc=$?" >> $O/tests_handoff_r02m.log
SH=B64c2048k8,B32c4096k8,B64c4096k8,B16c4096k32,B16c32768k8q64,B64c4096k32
for r in 1 2; do timeout 600 python scripts/small_call_bench.py --grids auto --no-host --no-floor --shapes $SH >> $O/handoff_r02m.txt 2>&1; done
for sh in C5 C3; do timeout 300 python scripts/timeline.py $sh >> $O/timeline_handoff_r02m.txt 2>&1; done
