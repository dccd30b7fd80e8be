"""metrics.py: the SPEC's stable-window rule and summary (SPEC.md "[MODULE]
metrics" examples), and properties over real simulate() runs."""
import math
from types import SimpleNamespace

import pytest

from paper_2503_20552_b200 import config, engine, metrics, workload
from paper_2503_20552_b200.engine import SaturationEvent, StepRecord
from paper_2503_20552_b200.scheduling import Request


def step(t0, t1, bl, bo=0, dec=0):
    return StepRecord(dec, t0, t1, bl, bo, None, 0.0, 0.0, 0.0, 0.0, 0.0, {}, {}, 0.0)


def run_of(steps, saturation=(), requests=(), end=None):
    return SimpleNamespace(steps=list(steps), saturation=list(saturation),
                           requests=list(requests),
                           end_time=end if end is not None else max(s.t_end for s in steps))


def test_saturation_window():
    sat = [SaturationEvent(t, "preempt", 0, i) for i, t in enumerate((10.0, 30.0, 50.0))]
    w = metrics.stable_window(run_of([step(0, 60, 4)], sat))
    assert (w.t_start, w.t_end, w.rule, w.flagged) == (10.0, 50.0, "saturation", False)


def test_peak_batch_window():
    steps = [step(0, 5, 10), step(5, 10, 80), step(10, 30, 100), step(30, 40, 20)]
    w = metrics.stable_window(run_of(steps))
    assert (w.t_start, w.t_end, w.rule) == (5.0, 30.0, "peak-batch")


def test_single_request_full_run_flagged():
    w = metrics.stable_window(run_of([step(0, 0.02, 1), step(0.02, 0.04, 1)], end=0.05))
    assert (w.t_start, w.t_end, w.rule, w.flagged) == (0.0, 0.05, "full-run", True)


def test_constant_steps_tpot():
    steps = [step(0.02 * i, 0.02 * (i + 1), 8) for i in range(50)]
    s = metrics.summarize(run_of(steps), metrics.Window(0.0, 1.0, "full-run", True))
    assert s["mean_tpot_s"] == pytest.approx(0.02)
    assert s["p99_tpot_s"] == pytest.approx(0.02)
    assert s["throughput_tok_s"] == pytest.approx(400.0)


def test_one_token_per_second():
    s = metrics.summarize(run_of([step(0.2, 0.7, 1)]), metrics.Window(0.0, 1.0, "full-run", True))
    assert s["throughput_tok_s"] == 1.0 and s["output_tokens"] == 1


def test_empty_window():
    assert metrics.summarize(run_of([step(0, 1, 1)]), metrics.Window(2.0, 2.0, "full-run", True))["empty"]


def test_nearest_rank():
    vals = [(float(v), 1) for v in range(1, 101)]
    assert metrics.nearest_rank(vals, 0.99) == 99.0
    assert metrics.nearest_rank(vals, 0.5) == 50.0
    assert metrics.nearest_rank([(1.0, 99), (5.0, 1)], 0.99) == 1.0
    assert metrics.nearest_rank([(1.0, 98), (5.0, 2)], 0.99) == 5.0


@pytest.mark.parametrize("ratio", [0.0, 0.7])
def test_simulated_run_properties(ratio):
    cfg = config.SimConfig.from_dict({"offload_ratio": ratio})
    reqs = workload.synth_requests(workload.preset("sharegpt_like", 6.0, 200), 3)
    r = engine.simulate(cfg, reqs)
    s = metrics.summarize(r)
    assert not s["empty"]
    assert s["p99_tpot_s"] >= s["mean_tpot_s"] > 0
    assert s["p99_tpot_s"] >= s["p90_tpot_s"] >= s["p50_tpot_s"]
    assert s["throughput_tok_s"] > 0 and 0.0 <= s["offloaded_share"] <= 1.0
    assert s["mean_ttft_s"] > 0
    # a pure function of the run: recomputation is identical
    assert metrics.summarize(r) == s or all(
        (a == b) or (isinstance(a, float) and math.isnan(a) and math.isnan(b))
        for a, b in zip(metrics.summarize(r).values(), s.values()))
    if ratio == 0.0:
        assert s["offloaded_share"] == 0.0
