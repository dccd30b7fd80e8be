set -u
O=gpurun_out; mkdir -p $O
timeout 600 python tests/golden/make_attn_golden.py $O/attn_libraries.npz > $O/attn_golden_r02y.log 2>&1
for i in 1 2 3; do
  timeout 900 python scripts/library_compare.py --only trt $O/library_compare_r02y_$i.json > $O/library_compare_r02y_$i.log 2>&1
done
