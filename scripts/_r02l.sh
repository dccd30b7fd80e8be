set -u
O=gpurun_out; mkdir -p $O
bash scripts/gpu_round.sh r02l tests-all small capacity
TOOLS=initcheck CS_TIMEOUT=1800 bash scripts/sanitize.sh > $O/sanitize_r02l.log 2>&1
CURVES=profiles/coloc_curves_r02i.json CL_TIMEOUT=3000 CL_CASES="4P4D" bash scripts/gpu_round.sh r02l closed-loop
