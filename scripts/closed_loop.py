#!/usr/bin/env python
"""Closed-loop engine runs: the reference's event semantics
with decode attention priced by the real sm_100a kernel (runtime.MeasuredPricer)
vs the analytic roofline prices, offload on/off, for the C4 / C3 cluster shapes.

    python scripts/closed_loop.py [out.json] [--curves coloc_curves.json] [label-substring ...]

With --curves, SimConfig uses the B200 colocation curves measured under
interference (scripts/calibrate_coloc.py "curves_shared": executor bandwidth
fraction and prefill slowdown with both partitions busy) instead of the
reference's A100-anchored defaults (calibration.py:41-48).
"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_20552_b200 import config, engine, metrics, specs, workload
from paper_2503_20552_b200.kvcache import PagedKVMirror
from paper_2503_20552_b200.runtime import MeasuredPricer

args = sys.argv[1:]
curves = None
if "--curves" in args:
    i = args.index("--curves")
    from paper_2503_20552_b200.calibration import CalibrationCurves
    curves = CalibrationCurves.from_dict(json.loads(Path(args[i + 1]).read_text())["curves_shared"])
    del args[i:i + 2]
n_override = None
if "--requests" in args:  # fewer requests per case (diagnostics)
    i = args.index("--requests")
    n_override = int(args[i + 1])
    del args[i:i + 2]
out = Path(args[0]) if args else Path("gpurun_out/closed_loop.json")
runs = []
from paper_2503_20552_b200.capacity import LLAMA3_70B_TP8W, LONGCTX  # noqa: E402  (C5 model, length mix)

def spec(pre, rate, n):
    if pre == "longctx":
        return workload.WorkloadSpec(rate=rate, num_requests=n, prompt_dist=LONGCTX[0],
                                     output_dist=LONGCTX[1], name="longctx")
    return workload.preset(pre, rate, n)


cases = [
    # label, model, num_prefill, num_decode, offload_ratio, preset, rate, n
    ("C4-13B-2P2D-no-offload", specs.LLAMA2_13B, 2, 2, 0.0, "sharegpt_like", 20.0, 400),
    ("C4-13B-2P2D-ob0.7", specs.LLAMA2_13B, 2, 2, 0.7, "sharegpt_like", 20.0, 400),
    ("C3-8B-1P1D-no-offload", specs.LLAMA3_8B, 1, 1, 0.0, "sharegpt_like", 12.0, 300),
    ("C3-8B-1P1D-ob0.5", specs.LLAMA3_8B, 1, 1, 0.5, "sharegpt_like", 12.0, 300),
    # BASELINE config 3: 1 decode + 1 prefill-role GPU, offload ratio sweep 0-0.8
    *[(f"C3sweep-8B-1P1D-24rps-ob{ob / 10:.1f}", specs.LLAMA3_8B, 1, 1, ob / 10, "sharegpt_like", 24.0, 300)
      for ob in range(0, 9)],
    # 8 GPUs: 4 prefill + 4 decode roles
    ("C4-13B-4P4D-no-offload", specs.LLAMA2_13B, 4, 4, 0.0, "sharegpt_like", 80.0, 1600),
    ("C4-13B-4P4D-ob0.7", specs.LLAMA2_13B, 4, 4, 0.7, "sharegpt_like", 80.0, 1600),
    ("C4-13B-4P4D-openthoughts-no-offload", specs.LLAMA2_13B, 4, 4, 0.0, "openthoughts_like", 12.0, 600),
    ("C4-13B-4P4D-openthoughts-ob0.8", specs.LLAMA2_13B, 4, 4, 0.8, "openthoughts_like", 12.0, 600),
    ("C5-70B-4P4D-longctx-no-offload", LLAMA3_70B_TP8W, 4, 4, 0.0, "longctx", 10.0, 500),
    ("C5-70B-4P4D-longctx-ob0.7", LLAMA3_70B_TP8W, 4, 4, 0.7, "longctx", 10.0, 500),
]
only = args[1:]
for label, model, npf, ndc, ob, pre, rate, n in cases:
    if only and not any(o in label for o in only):
        continue
    extra = {"curves": curves} if curves is not None else {}
    cfg = config.SimConfig(gpu=specs.B200, model=model, num_prefill=npf, num_decode=ndc,
                           offload_ratio=ob, avg_context_tokens=4096, **extra)
    n = n_override or n
    reqs = workload.synth_requests(spec(pre, rate, n), 0)
    row = {"label": label, "offload_ratio": ob, "requests": n,
           "curves": "b200-measured-shared" if curves is not None else "reference-default",
           "executor_bw_Bps": cfg.executor_bw, "prefill_slowdown": cfg.prefill_slowdown_factor}
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
            "uncovered_steps": getattr(pricer, "uncovered_steps", 0),
            "stable_window": metrics.summarize(r),
        }
        print(label, pricer_name, json.dumps(row[pricer_name]), flush=True)
    runs.append(row)
out.parent.mkdir(parents=True, exist_ok=True)
out.write_text(json.dumps(runs, indent=1))
