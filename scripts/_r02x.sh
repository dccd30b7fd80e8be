set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r02x.log 2>&1
bash scripts/gpu_round.sh r02x tests-all bench ref ncu
