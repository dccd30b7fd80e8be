set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pricer.py tests/test_gpu_decoder.py -q -p no:cacheprovider --timeout 400 > $O/tests_pricer_r02n.log 2>&1; echo "rc=$?" >> $O/tests_pricer_r02n.log
bash scripts/gpu_round.sh r02n bench
CURVES=profiles/coloc_curves_r02i.json CL_TIMEOUT=3600 CL_CASES="4P4D" bash scripts/gpu_round.sh r02n closed-loop
