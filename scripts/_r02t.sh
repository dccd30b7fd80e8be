O=gpurun_out
timeout 600 python scripts/exec_latency.py 72 > $O/exec_latency_r02t.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python scripts/exec_latency.py 72 > $O/exec_latency_conn32_r02t.txt 2>&1
