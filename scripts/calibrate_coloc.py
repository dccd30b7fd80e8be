#!/usr/bin/env python
"""On-box colocation calibration: sweep the attention
executor's green-context SM share beside a synthetic prefill GEMM load, fit the
B200 curves with fit_curves_from_samples, and derive the planner inputs.

    python scripts/calibrate_coloc.py [out.json]
"""
import dataclasses, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import coloc
from paper_2503_20552_b200.calibration import CalibrationCurves, min_sm_ratio_for_slo
from paper_2503_20552_b200.config import SimConfig
from paper_2503_20552_b200.specs import B200, LLAMA2_13B, LLAMA2_7B
from paper_2503_20552_b200.synthetic import DecodeShape, make_layer

out_path = Path(sys.argv[1]) if len(sys.argv) > 1 else Path("gpurun_out/coloc_curves.json")
dev = torch.device("cuda:0")
# executor workload: Llama-2-7B attention shapes, 32 requests x 4096 ctx (2 GiB KV per layer)
layer = make_layer(DecodeShape("exec", 32, 32, 32, 128, 1, 4096), dev)
# prefill load: Llama-2-7B layer GEMMs over a 4096-token prefill batch
pre = coloc.PrefillLoad(4096, 4096, 11008, dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
grid = [s for s in range(8, sms - 7, 8)]
sw = coloc.sweep_partitions(0, layer, pre, grid, iters=4, repeats=5)
alone = coloc.fit_curves(sw, shared=False)
shared = coloc.fit_curves(sw, shared=True)
res = {"total_sms": sw["total_sms"], "full_attn_gbs": sw["full_attn_gbs"],
       "full_prefill_s": sw["full_prefill_s"], "prefill_tflops_full": sw["prefill_tflops_full"],
       "samples": [dataclasses.asdict(s) for s in sw["samples"]],
       "curves_alone": alone.to_dict() if alone else None,
       "curves_shared": shared.to_dict() if shared else None}
for name, cur in (("alone", alone), ("shared", shared)):
    if cur is None:
        continue
    plan = {}
    for model in (LLAMA2_7B, LLAMA2_13B):
        cfg = SimConfig(gpu=B200, model=model, curves=cur, avg_context_tokens=4096)
        plan[model.name] = {"executor_bw_fraction@0.5": cur.attn_bw_fraction(0.5),
                            "prefill_slowdown@0.5": cur.prefill_slowdown(0.5),
                            "planner_bound": cfg.planner_bound(),
                            "min_prefill_sm_ratio_ttft2s": min_sm_ratio_for_slo(cur, 1.0, 2.0)}
    res[f"planner_{name}"] = plan
out_path.parent.mkdir(parents=True, exist_ok=True)
out_path.write_text(json.dumps(res, indent=1))
for s in sw["samples"]:
    print(f"attn {s.attn_sms:3d} SMs ({s.attn_ratio:.2f}): {s.attn_gbs_alone:7.0f} GB/s alone, "
          f"{s.attn_gbs_shared:7.0f} shared | prefill {s.prefill_s_alone*1e3:7.2f} ms alone, "
          f"{s.prefill_s_shared*1e3:7.2f} ms shared (full {sw['full_prefill_s']*1e3:.2f} ms) "
          f"[median of {s.repeats} overlapped windows, >= {s.prefill_reps_in_window} prefill "
          f"iterations inside each]")
print("full attention", round(sw["full_attn_gbs"]), "GB/s; prefill", round(sw["prefill_tflops_full"]), "TFLOP/s")
print("fit alone:", "ok" if alone else "violates curve shape", "| fit shared:", "ok" if shared else "violates curve shape")
