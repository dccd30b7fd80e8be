set -u
O=gpurun_out; mkdir -p $O
bash scripts/gpu_round.sh r02r tests-all
SH=B16c16384k8q64,B8c32768k8q64,B16c32768k8q64,B32c8192k8q64
timeout 900 python scripts/small_call_bench.py --grids auto,split --no-host --no-floor --shapes $SH > $O/g8_large_r02r.txt 2>&1
bash scripts/gpu_round.sh r02r bench
