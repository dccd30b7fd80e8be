set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02o.log 2>&1; echo "rc=$?" >> $O/smoke_r02o.log
SHAPES="B8c1024k8 B32c4096k8" bash scripts/profile_ncu_split.sh r02o > $O/ncu_split_r02o.log 2>&1
