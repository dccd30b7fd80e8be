set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_decoder.py -q -p no:cacheprovider > $O/tests_decoder_r02j.log 2>&1; echo "rc=$?" >> $O/tests_decoder_r02j.log
bash scripts/gpu_round.sh r02j capacity
SH=B4c512k8,B8c1024k8,B16c1024k8,B4c512k32,B8c1024k32
for k in 0 1 2 4 8; do echo "force_k $k" >> $O/forcek_r02j.txt; ADR_SPLIT_FORCE_K=$k timeout 300 python scripts/small_call_bench.py --grids split --no-host --no-trt --no-floor --shapes $SH >> $O/forcek_r02j.txt 2>&1; done
TOOLS=initcheck CS_TIMEOUT=1500 bash scripts/sanitize.sh > $O/sanitize_r02j.log 2>&1
CURVES=profiles/coloc_curves_r02i.json CL_TIMEOUT=3000 CL_CASES="4P4D" bash scripts/gpu_round.sh r02j closed-loop
