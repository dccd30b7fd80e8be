set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r02end.log 2>&1
bash scripts/gpu_round.sh r02end tests-all bench
bash scripts/gpu_round.sh r02end ref
