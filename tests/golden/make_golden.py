#!/usr/bin/env python
"""Generate the decision-path golden vectors from the reference itself.

Run in the build container (the only place /root/reference exists):
    python tests/golden/make_golden.py
It imports adrenaline_sim from /root/reference/pkg/src, evaluates it on seeded
inputs and writes tests/golden/*.json (floats via repr, so bit-exact). The
tests compare the package — and oracle/decision_oracle.py — against these.
"""
from __future__ import annotations

import dataclasses
import hashlib
import json
import math
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from adrenaline_sim import calibration, config, costs, engine, graphs, scheduling, specs, workload  # noqa: E402


def err(fn, *a, **k):
    try:
        return {"ok": fn(*a, **k)}
    except (ValueError, RuntimeError) as e:
        return {"error": type(e).__name__, "msg": str(e)}


def gpu_dict(g):
    return dataclasses.asdict(g)


GPUS = [
    specs.A100_80G,
    specs.GpuSpec("b200", 1669.3e12, 180e9, 6550.7e9, 900e9, 1.137e-3),
    specs.GpuSpec("b200-nominal", 2250e12, 180e9, 8000e9, 900e9, 1.137e-3),
    specs.GpuSpec("tiny", 10e12, 16e9, 500e9, 50e9, 0.0),
]
MODELS = [
    specs.LLAMA2_7B,
    specs.ModelSpec("llama2-13b", 40, 5120, 2, 26.032e9, 2.6032e10, 2.6032e10, 26.032e9),
    specs.ModelSpec("small", 4, 512, 2, 1e9, 1e9, 1e9, 1e9),
]


def need_offload_cases(n, seed):
    rng = random.Random(seed)
    out = []
    for i in range(n):
        def mk(k):
            rs = []
            for j in range(k):
                p = rng.randint(1, 4000)
                o = rng.randint(1, 2000)
                r = scheduling.Request(j, 0.0, p, o)
                r.used_token = rng.choice([0, rng.randint(0, p + o)])
                rs.append(r)
            return rs
        off = mk(rng.choice([0, 0, 1, 2, 5, 20]))
        loc = mk(rng.choice([0, 1, 3, 8, 40]))
        p = rng.randint(1, 8000)
        o = rng.randint(1, 4000)
        req = scheduling.Request(999, 0.0, p, o)
        req.used_token = rng.choice([0, 0, rng.randint(0, p + o)])
        bound = rng.choice([0.0, 0.1, 0.3, 0.5, 0.7, 0.8, 1.0, 2.5, rng.random()])
        c1max = rng.random() < 0.3
        d = scheduling.need_offload(req, off, loc, bound, c1_uses_max_tokens=c1max)
        out.append({
            "offloaded": [[r.prompt_tokens, r.output_tokens, r.used_token] for r in off],
            "local": [[r.prompt_tokens, r.output_tokens, r.used_token] for r in loc],
            "req": [p, o, req.used_token], "bound": bound, "c1_uses_max_tokens": c1max,
            "offload": d.offload, "rule": d.rule, "trace": d.trace,
        })
    # SURVEY §8c C1 selection golden: 8 requests, max_token 512, admitted in order, bound 0.5
    sel = []
    for used in (0, 512):
        off, loc, picks = [], [], []
        for k in range(8):
            r = scheduling.Request(k, 0.0, 256, 256)
            r.used_token = used
            dec = scheduling.need_offload(r, off, loc, 0.5)
            (off if dec.offload else loc).append(r)
            picks.append([k, dec.offload, dec.rule])
        sel.append({"used": used, "picks": picks})
    return out, sel


def bounds_cases(seed):
    rng = random.Random(seed)
    mem, comp, comb = [], [], []
    for _ in range(300):
        k = rng.choice([0, 1, 2, 4])
        hbm = [rng.uniform(0, 80e9) for _ in range(k)]
        bw = [rng.uniform(0, 3e12) for _ in range(k)]
        dh, db = rng.choice([rng.uniform(1e9, 80e9), 0.0]), rng.uniform(1e11, 8e12)
        mem.append({"args": [hbm, bw, dh, db], **err(scheduling.offload_bound_mem, hbm, bw, dh, db)})
    mem.append({"args": [[1.0], [1.0, 2.0], 1.0, 1.0],
                **err(scheduling.offload_bound_mem, [1.0], [1.0, 2.0], 1.0, 1.0)})
    mem.append({"args": [[-1.0], [1.0], 1.0, 1.0],
                **err(scheduling.offload_bound_mem, [-1.0], [1.0], 1.0, 1.0)})
    for _ in range(200):
        bm, bt = rng.randint(0, 600), rng.choice([-1, 0, rng.randint(0, 600)])
        comp.append({"args": [bm, bt], **err(scheduling.offload_bound_comp, bm, bt)})
    for _ in range(100):
        a, b = rng.choice([-0.1, rng.random() * 2]), rng.choice([math.inf, rng.random() * 2])
        comb.append({"args": [a, b], **err(scheduling.combined_offload_bound, a, b)})
    return {"mem": mem, "comp": comp, "combined": comb}


def cost_cases():
    out = []
    for g in GPUS:
        for m in MODELS:
            row = {"gpu": gpu_dict(g), "model": dataclasses.asdict(m),
                   "machine_balance": g.machine_balance, "kv_bytes_per_token": m.kv_bytes_per_token,
                   "b_max": costs.b_max(g, m),
                   "nonattn": [costs.nonattn_step_latency(g, m, b) for b in (1, 7, 64, 158, 159, 300, 1000, 5000)],
                   "prefill": [costs.prefill_latency(g, m, n, s) for n in (0, 1, 517, 4096) for s in (1.0, 1.4, 3.0)],
                   "launch": [costs.launch_overhead(m.num_layers, gr, g, w) for gr in (True, False)
                              for w in (0.0, 1e-4, 5e-4, 2e-3)],
                   "kv_bytes": [costs.kv_bytes(m, s) for s in (0, 1, 4096, 32768)],
                   "b_tpot": [[slo, ctx, scheduling.estimate_b_tpot(g, m, slo, ctx)]
                              for slo in (0.005, 0.01, 0.025, 0.03, 0.04, 0.05, 0.1, 0.5)
                              for ctx in (1, 512, 2048, 4096, 32768)]}
            out.append(row)
    misc = {
        "ai": [[h, b, costs.arithmetic_intensity_nonattn(h, b)] for h in (512, 4096, 5120) for b in (1, 3, 64, 999)],
        "attn": [[kv, bw, f, costs.attention_step_latency(kv, bw, f)]
                 for kv in (0.0, 1e6, 137.4e9) for bw in (2039e9, 6550.7e9) for f in (0.2, 0.72, 1.0)],
        "errors": [err(costs.kv_bytes, specs.LLAMA2_7B, -1), err(costs.attention_step_latency, 1.0, 1.0, 0.0),
                   err(costs.attention_step_latency, -1.0, 1.0), err(costs.nonattn_step_latency, GPUS[0], MODELS[0], 0),
                   err(costs.prefill_latency, GPUS[0], MODELS[0], 5, 0.5), err(costs.launch_overhead, 0, True, GPUS[0]),
                   err(scheduling.estimate_b_tpot, GPUS[0], MODELS[0], 0.0, 10),
                   err(scheduling.estimate_b_tpot, GPUS[0], MODELS[0], 1.0, 0)],
    }
    return {"grid": out, "misc": misc}


def graph_cases(seed):
    rng = random.Random(seed)
    out = []
    for _ in range(150):
        bi = rng.choice([1, 4, 8, 16, 64])
        md = rng.choice([1, 17, 64, 158, 512])
        mo = rng.choice([0, 0, md, rng.randint(0, 512)])
        bud = rng.choice([1, 4, 9, 20, 64])
        g = graphs.build_grid(bi, md, mo, bud)
        sel = []
        for _ in range(10):
            bd, bo = rng.randint(0, md + 40), rng.randint(0, mo + 40)
            sel.append([bd, bo, graphs.select_graph(g, bd, bo)])
        out.append({"args": [bi, md, mo, bud], "interval": g.interval, "decode_caps": list(g.decode_caps),
                    "offload_caps": list(g.offload_caps), "size": g.size, "select": sel})
    errors = [err(graphs.build_grid, 0, 1, 0, 1), err(graphs.build_grid, 1, 0, 0, 1),
              err(graphs.build_grid, 1, 1, -1, 1), err(graphs.build_grid, 1, 1, 0, 0)]
    return {"cases": out, "errors": errors}


def calibration_cases():
    cur = calibration.CalibrationCurves.default()
    xs = [i / 200 for i in range(201)] + [-0.5, 1.5, 0.123456789, 0.05]
    out = {
        "bw": [[x, cur.bw(x)] for x in xs],
        "slowdown": [[x, cur.slowdown(x)] for x in xs],
        "attn_bw_fraction": [[x, cur.attn_bw_fraction(x)] for x in xs if 0 <= x <= 1],
        "prefill_slowdown": [[x, cur.prefill_slowdown(x)] for x in xs if 0 < x <= 1],
        "min_sm": [[b, s, calibration.min_sm_ratio_for_slo(cur, b, s)]
                   for b in (0.1, 0.5, 1.0, 2.0) for s in (0.1, 0.5, 1.0, 1.4, 2.0, 5.0, 100.0)],
    }
    fits = []
    sample_sets = [
        ([[0.2, 0.6], [0.5, 0.8]], [[0.5, 1.4], [0.25, 2.5]]),
        ([[0.5, 0.72], [0.5, 0.75], [0.1, 0.3]], [[0.6, 1.3]]),
        ([[0.0, 0.0], [1.0, 1.0]], [[1.0, 1.0]]),
        ([[0.3, 0.2]], [[0.5, 1.4]]),               # sublinear -> error
        ([[0.3, 0.5], [0.4, 0.45]], [[0.5, 1.4]]),  # non-monotone -> error
        ([[0.3, 0.5]], [[0.5, 3.0]]),               # superlinear slowdown -> error
        ([[0.3, 0.5]], [[0.5, 0.9]]),               # below 1 -> error
        ([], [[0.5, 1.4]]),
        ([[0.3, 0.5]], []),
        ([[0.3, float("nan")]], [[0.5, 1.4]]),
        ([[0.3]], [[0.5, 1.4]]),
    ]
    for bw, sd in sample_sets:
        try:
            c = calibration.fit_curves_from_samples(bw, sd)
            fits.append({"bw": bw, "sd": sd, "ok": c.to_dict()})
        except calibration.CurveValidationError as e:
            fits.append({"bw": bw, "sd": sd, "error": str(e)})
    out["fits"] = fits
    return out


def config_cases():
    variants = [
        {},
        {"num_prefill": 2, "num_decode": 2},
        {"num_prefill": 4, "num_decode": 4, "attn_sm_ratio": 0.3},
        {"offload_ratio": 0.5},
        {"num_prefill": 0},
        {"tpot_slo": 0.02, "avg_context_tokens": 4096},
        {"gpu": gpu_dict(GPUS[1]), "model": dataclasses.asdict(MODELS[1])},
        {"gpu": gpu_dict(GPUS[1]), "model": dataclasses.asdict(MODELS[0]), "avg_context_tokens": 4096},
        {"gpu": gpu_dict(GPUS[1]), "model": dataclasses.asdict(MODELS[0])},
        {"gpu": gpu_dict(GPUS[2]), "model": dataclasses.asdict(MODELS[0]), "tpot_slo": 0.025},
        {"graph_max_batch": 100, "graph_interval": 8, "graph_budget": 64},
        {"mem_util": 0.9, "activation_reserve": 0.05, "prefill_inflight_fraction": 0.5},
    ]
    out = []
    for v in variants:
        c = config.SimConfig.from_dict(v)
        out.append({"input": v, "pool_bytes": c.pool_bytes, "executor_budget_bytes": c.executor_budget_bytes,
                    "prefill_inflight_budget_bytes": c.prefill_inflight_budget_bytes,
                    "b_max_ideal": c.b_max_ideal, "b_tpot": c.b_tpot, "graph_axis_max": c.graph_axis_max,
                    "executor_bw": c.executor_bw, "prefill_slowdown_factor": c.prefill_slowdown_factor,
                    "planner_bound": c.planner_bound(), "effective_bound": c.effective_bound(),
                    "to_dict": c.to_dict()})
    bad = [{"num_decode": 0}, {"attn_sm_ratio": 1.0}, {"offload_ratio": -1}, {"tpot_slo": 0},
           {"mem_util": 0.05, "activation_reserve": 0.0}, {"bogus": 1}, {"gpu": "h100"},
           {"curves": 3}, {"graph_max_batch": 0}]
    errors = [{"input": b, **err(config.SimConfig.from_dict, b)} for b in bad]
    return {"cases": out, "errors": errors}


def workload_cases():
    out = []
    for name in workload.PRESET_NAMES:
        for seed in (0, 1, 7):
            reqs = workload.synth_requests(workload.preset(name, 3.0, 40), seed)
            out.append({"preset": name, "seed": seed,
                        "requests": [[r.req_id, r.arrival_time, r.prompt_tokens, r.output_tokens] for r in reqs]})
    spec = workload.WorkloadSpec(5.0, 30, workload.Uniform(3, 900), workload.Constant(7), "mix")
    reqs = workload.synth_requests(spec, 11)
    out.append({"custom": spec.to_dict(), "seed": 11,
                "requests": [[r.req_id, r.arrival_time, r.prompt_tokens, r.output_tokens] for r in reqs]})
    return out


def sim_hash(r):
    h = hashlib.sha256()
    for s in r.steps:
        h.update(repr((s.decoder, s.t_start, s.t_end, s.batch_local, s.batch_offload,
                       s.graph_shape, s.stall)).encode())
    for rid in sorted(r.decisions):
        h.update(repr((rid, [(t, d.rule) for t, d in r.decisions[rid]])).encode())
    return h.hexdigest()[:16]


def full_hash(r):
    h = hashlib.sha256()
    for s in r.steps:
        h.update(repr((s.decoder, s.t_start, s.t_end, s.batch_local, s.batch_offload, s.graph_shape,
                       s.launch, s.nonattn, s.local_attn, s.stall, s.local_kv_bytes,
                       sorted(s.exec_kv_bytes.items()), sorted(s.exec_attn.items()), s.link_bytes,
                       s.completions)).encode())
    for p in r.prefill_records:
        h.update(repr(dataclasses.astuple(p)).encode())
    for t in r.transfers:
        h.update(repr(dataclasses.astuple(t)).encode())
    for e in r.saturation:
        h.update(repr(dataclasses.astuple(e)).encode())
    for q in r.requests:
        h.update(repr((q.req_id, q.first_token_time, q.finish_time, q.preempt_count, q.phase)).encode())
    for rid in sorted(r.decisions):
        h.update(repr((rid, [(t, d.rule, sorted(d.trace.items())) for t, d in r.decisions[rid]])).encode())
    return h.hexdigest()


SIM_RUNS = [
    # (label, config dict, preset, rate, n, seed)
    ("survey-hash", {}, "sharegpt_like", 3.0, 300, 7),
    ("openthoughts", {}, "openthoughts_like", 3.0, 120, 1),
    ("2p2d-ob0.5", {"num_prefill": 2, "num_decode": 2, "offload_ratio": 0.5}, "sharegpt_like", 6.0, 150, 3),
    ("c1max-ungraphed", {"c1_uses_max_tokens": True, "use_graphs": False}, "sharegpt_like", 4.0, 120, 5),
    ("no-offload", {"offload_ratio": 0.0}, "sharegpt_like", 3.0, 150, 7),
    ("tight-memory", {"gpu": {"name": "tight", "flops_peak": 312e12, "hbm_capacity_bytes": 24e9,
                              "hbm_bandwidth": 2039e9, "interconnect_bandwidth": 600e9,
                              "cpu_launch_per_layer": 1.137e-3}, "offload_ratio": 0.8},
     "sharegpt_like", 8.0, 150, 9),
    ("b200-13b-ob0.7", {"gpu": {"name": "b200", "flops_peak": 1669.3e12, "hbm_capacity_bytes": 180e9,
                                "hbm_bandwidth": 6550.7e9, "interconnect_bandwidth": 900e9,
                                "cpu_launch_per_layer": 1.137e-3},
                        "model": dataclasses.asdict(MODELS[1]), "offload_ratio": 0.7,
                        "num_prefill": 2, "num_decode": 2}, "sharegpt_like", 20.0, 300, 0),
    ("long-prompt", {"num_prefill": 2, "num_decode": 1}, "long_prompt", 2.0, 60, 2),
]


def sim_cases():
    out = []
    for label, cfgd, pre, rate, n, seed in SIM_RUNS:
        cfg = config.SimConfig.from_dict(cfgd)
        reqs = workload.synth_requests(workload.preset(pre, rate, n), seed)
        r = engine.simulate(cfg, reqs)
        out.append({"label": label, "config": cfgd, "preset": pre, "rate": rate, "n": n, "seed": seed,
                    "bound": r.bound, "end_time": r.end_time, "completed": r.completed,
                    "n_steps": len(r.steps), "n_saturation": len(r.saturation),
                    "max_batch": max(s.batch for s in r.steps),
                    "offloaded_rules": sum(1 for v in r.decisions.values() for _, d in v if d.offload),
                    "hash": sim_hash(r), "full_hash": full_hash(r),
                    "first_steps": [[s.decoder, s.t_start, s.t_end, s.batch_local, s.batch_offload,
                                     s.graph_shape, s.launch, s.nonattn, s.local_attn, s.stall,
                                     s.link_bytes, s.completions] for s in r.steps[:25]]})
    errors = []
    reqs = [scheduling.Request(1, 0.0, 10, 10), scheduling.Request(1, 1.0, 10, 10)]
    errors.append(err(engine.simulate, config.SimConfig(), reqs))
    errors.append(err(engine.simulate, config.SimConfig(num_prefill=0), [scheduling.Request(1, 0.0, 10, 10)]))
    return {"runs": out, "errors": errors}


def main():
    no, sel = need_offload_cases(3000, 20250320)
    files = {
        "need_offload.json": {"cases": no, "c1_selection": sel},
        "bounds.json": bounds_cases(1),
        "costs.json": cost_cases(),
        "graphs.json": graph_cases(2),
        "calibration.json": calibration_cases(),
        "config.json": config_cases(),
        "workload.json": workload_cases(),
        "simulate.json": sim_cases(),
    }
    for name, data in files.items():
        (OUT / name).write_text(json.dumps(data, indent=None, separators=(",", ":")) + "\n")
        print(name, (OUT / name).stat().st_size, "bytes")


if __name__ == "__main__":
    main()
