set -u
O=gpurun_out; mkdir -p $O
timeout 600 python scripts/library_compare.py --only trt $O/var3_lib.json > $O/var3_lib.log 2>&1
SH=B16c16384k8q64,B8c32768k8q64,B32c8192k8q64,B16c32768k8q64,B4c32768k32,B8c16384k32,B16c16384k8,B8c32768k8
timeout 400 python scripts/small_call_bench.py --grids auto,dynamic --no-host --no-floor --no-trt --shapes $SH > $O/var3_shapes.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_var3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 > $O/gpu_tests_var3.log 2>&1; echo "rc=$?" >> $O/gpu_tests_var3.log
timeout 900 python bench.py > $O/bench_var3.json 2> $O/bench_var3.err
