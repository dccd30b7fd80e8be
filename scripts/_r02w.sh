O=gpurun_out
bash scripts/gpu_round.sh r02w tests-all calibrate
CURVES=$O/coloc_curves_r02w.json CL_TIMEOUT=3600 CL_CASES="4P4D" bash scripts/gpu_round.sh r02w closed-loop
