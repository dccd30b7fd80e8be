O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_pricer.py -q -p no:cacheprovider --timeout 400 > $O/tests_part_r02v.log 2>&1; echo "rc=$?" >> $O/tests_part_r02v.log
timeout 600 python scripts/exec_latency.py 72 > $O/exec_latency_prio_r02v.txt 2>&1
timeout 900 python scripts/exec_under_prefill.py 72 auto > $O/exec_under_prefill_prio_r02v.txt 2>&1
