"""Bit-exact parity of the decision path (scheduler, bounds, planner, graph grid,
calibration, workload, engine) with the reference, via golden vectors generated
by tests/golden/make_golden.py from /root/reference itself."""
import dataclasses
import hashlib
import json
import math
from pathlib import Path

import pytest

from paper_2503_20552_b200 import (calibration, config, costs, engine, graphs, scheduling, specs,
                                   workload)

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())


def same(a, b):
    """Exact equality, NaN-aware, tuples vs lists tolerated (JSON)."""
    if isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b):
        return True
    if isinstance(a, (list, tuple)) and isinstance(b, (list, tuple)):
        return len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
    if isinstance(a, dict) and isinstance(b, dict):
        return a.keys() == b.keys() and all(same(a[k], b[k]) for k in a)
    return a == b and type(a) in (type(b), int, float) or (a is None and b is None)


def call(fn, *a, **k):
    try:
        return {"ok": fn(*a, **k)}
    except (ValueError, RuntimeError) as e:
        return {"error": type(e).__name__, "msg": str(e)}


def mkreq(p, o, used, rid=0):
    r = scheduling.Request(rid, 0.0, p, o)
    r.used_token = used
    return r


def test_need_offload_matches_reference():
    g = load("need_offload.json")
    for c in g["cases"]:
        off = [mkreq(*x) for x in c["offloaded"]]
        loc = [mkreq(*x) for x in c["local"]]
        req = mkreq(*c["req"], rid=999)
        d = scheduling.need_offload(req, off, loc, c["bound"],
                                    c1_uses_max_tokens=c["c1_uses_max_tokens"])
        assert (d.offload, d.rule) == (c["offload"], c["rule"]), c
        assert same(d.trace, c["trace"])
        led = scheduling.OffloadLedger.of(off, loc)
        d2 = led.decide(req, c["bound"], c1_uses_max_tokens=c["c1_uses_max_tokens"])
        assert (d2.offload, d2.rule) == (d.offload, d.rule) and same(d2.trace, d.trace)


def test_c1_selection_golden():
    """8 requests of max_token 512 admitted in order at bound 0.5."""
    for case in load("need_offload.json")["c1_selection"]:
        off, loc, picks = [], [], []
        for k in range(8):
            r = mkreq(256, 256, case["used"], rid=k)
            d = scheduling.need_offload(r, off, loc, 0.5)
            (off if d.offload else loc).append(r)
            picks.append([k, d.offload, d.rule])
        assert picks == case["picks"]
    assert [p[0] for p in load("need_offload.json")["c1_selection"][1]["picks"] if p[1]] == [3, 6]


def test_bounds_match_reference():
    g = load("bounds.json")
    for c in g["mem"]:
        assert same(call(scheduling.offload_bound_mem, *c["args"]), {k: v for k, v in c.items() if k != "args"})
    for c in g["comp"]:
        assert same(call(scheduling.offload_bound_comp, *c["args"]), {k: v for k, v in c.items() if k != "args"})
    for c in g["combined"]:
        assert same(call(scheduling.combined_offload_bound, *c["args"]),
                    {k: v for k, v in c.items() if k != "args"})


def test_costs_and_b_tpot_match_reference():
    g = load("costs.json")
    for row in g["grid"]:
        gpu = specs.GpuSpec(**row["gpu"])
        m = specs.ModelSpec(**row["model"])
        assert gpu.machine_balance == row["machine_balance"]
        assert m.kv_bytes_per_token == row["kv_bytes_per_token"]
        assert costs.b_max(gpu, m) == row["b_max"]
        assert [costs.nonattn_step_latency(gpu, m, b) for b in (1, 7, 64, 158, 159, 300, 1000, 5000)] == row["nonattn"]
        assert [costs.prefill_latency(gpu, m, n, s) for n in (0, 1, 517, 4096)
                for s in (1.0, 1.4, 3.0)] == row["prefill"]
        assert [costs.launch_overhead(m.num_layers, gr, gpu, w) for gr in (True, False)
                for w in (0.0, 1e-4, 5e-4, 2e-3)] == row["launch"]
        assert [costs.kv_bytes(m, s) for s in (0, 1, 4096, 32768)] == row["kv_bytes"]
        for slo, ctx, want in row["b_tpot"]:
            assert scheduling.estimate_b_tpot(gpu, m, slo, ctx) == want
    misc = g["misc"]
    for h, b, want in misc["ai"]:
        assert costs.arithmetic_intensity_nonattn(h, b) == want
    for kv, bw, f, want in misc["attn"]:
        assert costs.attention_step_latency(kv, bw, f) == want
    got = [call(costs.kv_bytes, specs.LLAMA2_7B, -1), call(costs.attention_step_latency, 1.0, 1.0, 0.0),
           call(costs.attention_step_latency, -1.0, 1.0),
           call(costs.nonattn_step_latency, specs.A100_80G, specs.LLAMA2_7B, 0),
           call(costs.prefill_latency, specs.A100_80G, specs.LLAMA2_7B, 5, 0.5),
           call(costs.launch_overhead, 0, True, specs.A100_80G),
           call(scheduling.estimate_b_tpot, specs.A100_80G, specs.LLAMA2_7B, 0.0, 10),
           call(scheduling.estimate_b_tpot, specs.A100_80G, specs.LLAMA2_7B, 1.0, 0)]
    assert got == misc["errors"]


def test_graph_grid_matches_reference():
    g = load("graphs.json")
    for c in g["cases"]:
        grid = graphs.build_grid(*c["args"])
        assert (grid.interval, list(grid.decode_caps), list(grid.offload_caps), grid.size) == \
            (c["interval"], c["decode_caps"], c["offload_caps"], c["size"])
        for bd, bo, want in c["select"]:
            got = graphs.select_graph(grid, bd, bo)
            assert (list(got) if got is not None else None) == want
    got = [call(graphs.build_grid, 0, 1, 0, 1), call(graphs.build_grid, 1, 0, 0, 1),
           call(graphs.build_grid, 1, 1, -1, 1), call(graphs.build_grid, 1, 1, 0, 0)]
    assert got == g["errors"]


def test_calibration_matches_reference():
    g = load("calibration.json")
    cur = calibration.CalibrationCurves.default()
    assert all(cur.bw(x) == y for x, y in g["bw"])
    assert all(cur.slowdown(x) == y for x, y in g["slowdown"])
    assert all(cur.attn_bw_fraction(x) == y for x, y in g["attn_bw_fraction"])
    assert all(cur.prefill_slowdown(x) == y for x, y in g["prefill_slowdown"])
    for b, s, want in g["min_sm"]:
        assert calibration.min_sm_ratio_for_slo(cur, b, s) == want
    for f in g["fits"]:
        try:
            got = {"ok": calibration.fit_curves_from_samples(f["bw"], f["sd"]).to_dict()}
        except calibration.CurveValidationError as e:
            got = {"error": str(e)}
        want = {k: v for k, v in f.items() if k in ("ok", "error")}
        assert same(got, want), (f, got)


def test_config_planner_matches_reference():
    g = load("config.json")
    for c in g["cases"]:
        cfg = config.SimConfig.from_dict(c["input"])
        for key in ("pool_bytes", "executor_budget_bytes", "prefill_inflight_budget_bytes",
                    "b_max_ideal", "b_tpot", "graph_axis_max", "executor_bw",
                    "prefill_slowdown_factor"):
            assert getattr(cfg, key) == c[key], key
        assert cfg.planner_bound() == c["planner_bound"]
        assert cfg.effective_bound() == c["effective_bound"]
        assert same(cfg.to_dict(), c["to_dict"])
        # round trip through JSON-able dict
        assert config.SimConfig.from_dict(cfg.to_dict()) == cfg
    for e in g["errors"]:
        got = call(config.SimConfig.from_dict, e["input"])
        assert got.get("error") == e["error"]


def test_workload_matches_reference():
    for c in load("workload.json"):
        if "preset" in c:
            reqs = workload.synth_requests(workload.preset(c["preset"], 3.0, 40), c["seed"])
        else:
            d = c["custom"]
            spec = workload.WorkloadSpec(d["rate"], d["num_requests"],
                                         workload.dist_from_dict(d["prompt_dist"]),
                                         workload.dist_from_dict(d["output_dist"]), d["name"])
            reqs = workload.synth_requests(spec, c["seed"])
        assert [[r.req_id, r.arrival_time, r.prompt_tokens, r.output_tokens] for r in reqs] == c["requests"]


def _sim_hash(r):
    h = hashlib.sha256()
    for s in r.steps:
        h.update(repr((s.decoder, s.t_start, s.t_end, s.batch_local, s.batch_offload,
                       s.graph_shape, s.stall)).encode())
    for rid in sorted(r.decisions):
        h.update(repr((rid, [(t, d.rule) for t, d in r.decisions[rid]])).encode())
    return h.hexdigest()[:16]


def _full_hash(r):
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


@pytest.mark.parametrize("label", [r["label"] for r in load("simulate.json")["runs"]])
def test_simulate_bit_identical_to_reference(label):
    run = next(r for r in load("simulate.json")["runs"] if r["label"] == label)
    cfg = config.SimConfig.from_dict(run["config"])
    reqs = workload.synth_requests(workload.preset(run["preset"], run["rate"], run["n"]), run["seed"])
    r = engine.simulate(cfg, reqs)
    assert r.bound == run["bound"]
    assert len(r.steps) == run["n_steps"] and r.completed == run["completed"]
    assert r.end_time == run["end_time"]
    first = [[s.decoder, s.t_start, s.t_end, s.batch_local, s.batch_offload,
              list(s.graph_shape) if s.graph_shape else None, s.launch, s.nonattn, s.local_attn,
              s.stall, s.link_bytes, s.completions] for s in r.steps[:25]]
    assert first == run["first_steps"]
    assert _sim_hash(r) == run["hash"]
    assert _full_hash(r) == run["full_hash"]


def test_survey_determinism_hash():
    r = engine.simulate(config.SimConfig(),
                        workload.synth_requests(workload.preset("sharegpt_like", 3.0, 300), 7))
    assert _sim_hash(r) == "322fc68d142ad349"


def test_simulate_input_errors():
    want = load("simulate.json")["errors"]
    reqs = [scheduling.Request(1, 0.0, 10, 10), scheduling.Request(1, 1.0, 10, 10)]
    got = [call(engine.simulate, config.SimConfig(), reqs),
           call(engine.simulate, config.SimConfig(num_prefill=0), [scheduling.Request(1, 0.0, 10, 10)])]
    assert got == want


def test_gqa_model_reduces_to_reference_formula_for_mha():
    mha = specs.ModelSpec("m", 32, 4096, 2, 1e9, 1e9, 1e9, 1e9, num_q_heads=32, num_kv_heads=32,
                          head_dim=128)
    assert mha.kv_bytes_per_token == specs.LLAMA2_7B.kv_bytes_per_token == 524288
    assert specs.LLAMA3_8B.kv_bytes_per_token == 131072
    assert specs.LLAMA3_70B.kv_bytes_per_token == 327680
