set -u
O=gpurun_out; mkdir -p $O
timeout 600 python scripts/exec_under_prefill.py 72 > $O/exec_under_prefill_r02p.txt 2>&1
timeout 1200 python scripts/closed_loop.py $O/cl_c5_default_r02p.json --curves profiles/coloc_curves_r02i.json --requests 120 C5-70B-4P4D-longctx-ob0.7 > $O/cl_c5_default_r02p.log 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 1200 python scripts/closed_loop.py $O/cl_c5_conn32_r02p.json --curves profiles/coloc_curves_r02i.json --requests 120 C5-70B-4P4D-longctx-ob0.7 > $O/cl_c5_conn32_r02p.log 2>&1
