set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r02final.log 2>&1
bash scripts/gpu_round.sh r02final tests-all bench
