"""Command line: ``python -m paper_2503_20552_b200.cli {run,calibrate}``.

The reference declares a ``cli`` entry point (pyproject.toml:25-26)
but ships none. Two commands cover the path:

  run        simulate a cluster config (JSON, SimConfig.from_dict keys) on a
             workload preset; ``--measured`` prices decode attention with the
             sm_100a kernel on this GPU (runtime.MeasuredPricer) instead of the
             analytic roofline
  bmax       B_max by sweep: time the non-attention layers over batch sizes,
             fit the knee of the reference's flat-then-linear model (bmax.py)
  calibrate  sweep green-context SM partitions on this GPU (executor decode
             attention beside a synthetic prefill GEMM), fit the B200 curves
             (fit_curves_from_samples) and write them as JSON that
             ``SimConfig.from_dict({"curves": ...})`` / ``CalibrationCurves.from_json_file`` load
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path


def _summary(result) -> dict:
    from . import metrics
    steps = result.steps
    toks = sum(r.output_tokens for r in result.requests)
    return {
        "bound": result.bound, "completed": result.completed, "end_time_s": result.end_time,
        "tokens_per_s": toks / result.end_time if result.end_time > 0 else 0.0,
        "steps": len(steps), "max_batch": max((s.batch for s in steps), default=0),
        "mean_batch": sum(s.batch for s in steps) / max(1, len(steps)),
        "offloaded_slot_share": sum(s.batch_offload for s in steps) / max(1, sum(s.batch for s in steps)),
        "preemptions": sum(1 for e in result.saturation if e.kind == "preempt"),
        "blocked": sum(1 for e in result.saturation if e.kind == "blocked"),
        "stable_window": metrics.summarize(result),  # SPEC metrics: TTFT / TPOT / P99
    }


def cmd_run(args) -> int:
    from . import config, engine, workload
    cfg_dict = json.loads(Path(args.config).read_text()) if args.config else {}
    if args.offload_ratio is not None:
        cfg_dict["offload_ratio"] = args.offload_ratio
    cfg = config.SimConfig.from_dict(cfg_dict)
    if args.trace:
        reqs = workload.load_trace_jsonl(args.trace)
    else:
        reqs = workload.synth_requests(workload.preset(args.preset, args.rate, args.requests),
                                       args.seed)
    pricer = observer = None
    if args.measured:
        from .kvcache import PagedKVMirror
        from .runtime import MeasuredPricer
        observer = PagedKVMirror.for_config(cfg, slack_pages=2048, keep_log=False)
        pricer = MeasuredPricer(cfg, observer, device=args.device)
    result = engine.simulate(cfg, reqs, pricer=pricer, observer=observer)
    out = {"pricer": "measured" if args.measured else "analytic", **_summary(result)}
    print(json.dumps(out, indent=1))
    return 0


def cmd_calibrate(args) -> int:
    import dataclasses

    import torch

    from . import coloc
    from .synthetic import DecodeShape, make_layer
    if not coloc.green_contexts_supported():
        print("calibrate: CUDA green contexts are not available on this device", file=sys.stderr)
        return 2
    dev = torch.device("cuda", args.device)
    layer = make_layer(DecodeShape("exec", args.batch, args.q_heads, args.kv_heads, 128, 1,
                                   args.ctx), dev)
    pre = coloc.PrefillLoad(args.prefill_tokens, args.hidden, args.intermediate, dev)
    sms = torch.cuda.get_device_properties(args.device).multi_processor_count
    sweep = coloc.sweep_partitions(args.device, layer, pre, list(range(8, sms - 7, 8)),
                                   iters=args.iters)
    curves = coloc.fit_curves(sweep, shared=args.shared)
    if curves is None:
        print("calibrate: measured points violate the curve-shape rules", file=sys.stderr)
        return 3
    Path(args.out).write_text(json.dumps(curves.to_dict(), indent=1))
    if args.samples:
        Path(args.samples).write_text(json.dumps(
            {"full_attn_gbs": sweep["full_attn_gbs"], "full_prefill_s": sweep["full_prefill_s"],
             "samples": [dataclasses.asdict(s) for s in sweep["samples"]]}, indent=1))
    print(f"wrote {args.out}: bw(0.2)={curves.attn_bw_fraction(0.2):.3f} "
          f"bw(0.5)={curves.attn_bw_fraction(0.5):.3f} slowdown(0.5)={curves.prefill_slowdown(0.5):.3f}")
    return 0


def cmd_bmax(args) -> int:
    """B_max by sweep: time the non-attention layers of
    ``--model`` over a batch sweep, fit the knee, report the GpuSpec that makes
    the reference's b_max formula give it."""
    import dataclasses

    import torch

    from . import bmax, specs
    from .costs import b_max as b_max_formula
    from .decoder import MODEL_DIMS
    dev = torch.device("cuda", args.device)
    batches = [int(b) for b in args.batches.split(",")]
    samples = bmax.sweep_nonattn(MODEL_DIMS[args.model], batches, dev, layers=args.layers)
    t0, knee = bmax.fit_knee(samples)
    model = specs.MODEL_PRESETS[args.model]
    gpu = bmax.gpu_for_bmax(specs.B200, model, knee)
    res = {"model": args.model, "samples_s_per_layer": samples, "flat_s_per_layer": t0,
           "b_max_measured": knee, "b_max_analytic": b_max_formula(specs.B200, model),
           "gpu": dataclasses.asdict(gpu)}
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(f"wrote {args.out}: B_max measured {knee:.1f} (analytic {res['b_max_analytic']}), "
          f"flat {t0 * 1e6:.1f} us/layer")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2503_20552_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="simulate a cluster on a workload")
    r.add_argument("--config", help="SimConfig JSON (keys of SimConfig.from_dict)")
    r.add_argument("--preset", default="sharegpt_like")
    r.add_argument("--rate", type=float, default=3.0)
    r.add_argument("--requests", type=int, default=300)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--trace", help="JSONL trace instead of a preset")
    r.add_argument("--offload-ratio", type=float, default=None)
    r.add_argument("--measured", action="store_true", help="price attention with the GPU kernel")
    r.add_argument("--device", type=int, default=0)
    r.set_defaults(fn=cmd_run)
    c = sub.add_parser("calibrate", help="measure SM-partition curves on this GPU")
    c.add_argument("--out", default="coloc_curves.json")
    c.add_argument("--samples", help="also write the raw sweep samples here")
    c.add_argument("--device", type=int, default=0)
    c.add_argument("--batch", type=int, default=32)
    c.add_argument("--ctx", type=int, default=4096)
    c.add_argument("--q-heads", type=int, default=32)
    c.add_argument("--kv-heads", type=int, default=32)
    c.add_argument("--prefill-tokens", type=int, default=4096)
    c.add_argument("--hidden", type=int, default=4096)
    c.add_argument("--intermediate", type=int, default=11008)
    c.add_argument("--iters", type=int, default=4)
    c.add_argument("--shared", action="store_true", help="fit the under-interference curves")
    c.set_defaults(fn=cmd_calibrate)
    b = sub.add_parser("bmax", help="B_max by sweep of the non-attention layers on this GPU")
    b.add_argument("--model", default="llama2-7b", choices=["llama2-7b", "llama2-13b", "llama3-8b"])
    b.add_argument("--batches", default="1,8,16,32,64,96,128,192,256,384,512,768,1024")
    b.add_argument("--layers", type=int, default=4)
    b.add_argument("--device", type=int, default=0)
    b.add_argument("--out", default="bmax.json")
    b.set_defaults(fn=cmd_bmax)
    args = ap.parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
