#!/usr/bin/env python
"""Closed-loop engine runs: the reference's event semantics
with decode attention priced by the real sm_100a kernel (runtime.MeasuredPricer)
vs the analytic roofline prices, offload on/off, for the C4 / C3 cluster shapes.

    python scripts/closed_loop.py [out.json]
"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_20552_b200 import config, engine, specs, workload
from paper_2503_20552_b200.kvcache import PagedKVMirror
from paper_2503_20552_b200.runtime import MeasuredPricer

out = Path(sys.argv[1]) if len(sys.argv) > 1 else Path("gpurun_out/closed_loop.json")
runs = []
cases = [
    # label, model, num_prefill, num_decode, offload_ratio, preset, rate, n
    ("C4-13B-2P2D-no-offload", specs.LLAMA2_13B, 2, 2, 0.0, "sharegpt_like", 20.0, 400),
    ("C4-13B-2P2D-ob0.7", specs.LLAMA2_13B, 2, 2, 0.7, "sharegpt_like", 20.0, 400),
    ("C3-8B-1P1D-no-offload", specs.LLAMA3_8B, 1, 1, 0.0, "sharegpt_like", 12.0, 300),
    ("C3-8B-1P1D-ob0.5", specs.LLAMA3_8B, 1, 1, 0.5, "sharegpt_like", 12.0, 300),
]
for label, model, npf, ndc, ob, pre, rate, n in cases:
    cfg = config.SimConfig(gpu=specs.B200, model=model, num_prefill=npf, num_decode=ndc,
                           offload_ratio=ob, avg_context_tokens=4096)
    reqs = workload.synth_requests(workload.preset(pre, rate, n), 0)
    row = {"label": label, "offload_ratio": ob, "requests": n}
    for pricer_name in ("analytic", "measured"):
        mirror = PagedKVMirror.for_config(cfg, slack_pages=2048, keep_log=False)
        pricer = MeasuredPricer(cfg, mirror) if pricer_name == "measured" else None
        t0 = time.time()
        r = engine.simulate(cfg, reqs, pricer=pricer, observer=mirror)
        toks = sum(q.output_tokens for q in r.requests)
        steps = r.steps
        row[pricer_name] = {
            "tokens_per_s": toks / r.end_time, "end_time_s": r.end_time,
            "max_batch": max(s.batch for s in steps),
            "mean_batch": sum(s.batch for s in steps) / len(steps),
            "offloaded_slot_share": sum(s.batch_offload for s in steps) / max(1, sum(s.batch for s in steps)),
            "mean_local_attn_ms": 1e3 * sum(s.local_attn for s in steps) / len(steps),
            "mean_stall_ms": 1e3 * sum(s.stall for s in steps) / len(steps),
            "steps": len(steps), "wall_s": time.time() - t0,
            "kernel_calls": getattr(pricer, "kernel_calls", 0),
        }
        print(label, pricer_name, json.dumps(row[pricer_name]), flush=True)
    runs.append(row)
out.parent.mkdir(parents=True, exist_ok=True)
out.write_text(json.dumps(runs, indent=1))
