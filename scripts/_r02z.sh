set -u
O=gpurun_out; mkdir -p $O
timeout 600 python tests/golden/make_attn_golden.py $O/attn_libraries.npz > $O/attn_golden_r02z.log 2>&1
