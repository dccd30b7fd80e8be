"""Evaluation metrics of a run: stable window, TTFT / TPOT / P99, throughput.

The reference package declares a ``metrics`` module (SPEC.md "[MODULE]
metrics") but does not ship it (pyproject.toml lists it; pkg/src has no file),
so this follows the SPEC's operations over the reference's own records
(engine.py:40-93: StepRecord, SaturationEvent; scheduling.py:38-88: Request):

* ``stable_window(run)`` — SPEC "[OP] stable_window" (paper §4.1, "between the
  first and last time when the HBM capacity of decoding instances is
  saturated"): first to last saturation event (preemption or budget-blocked
  admission); else the span where a decoder's batch is >= 80% of the peak
  batch; else the whole run, flagged.
* ``summarize(run, window)`` — SPEC "[OP] summarize": mean TTFT, mean / P50 /
  P90 / P99 TPOT (nearest rank, no interpolation) over the per-token step
  samples in the window (every request in a decode step receives one token
  after that step's duration), output-token throughput in the window, plus
  the decode batch and offloaded share. Pure function of the run.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

__all__ = ["Window", "stable_window", "nearest_rank", "summarize"]


@dataclass(frozen=True)
class Window:
    t_start: float
    t_end: float
    rule: str          # "saturation" | "peak-batch" | "full-run"
    flagged: bool      # True for the degenerate full-run fallback

    @property
    def length(self) -> float:
        return self.t_end - self.t_start


def stable_window(run, peak_fraction: float = 0.8) -> Window:
    """SPEC metrics.stable_window over a RunResult."""
    if run.saturation:
        ts = [e.time for e in run.saturation]
        if max(ts) > min(ts):
            return Window(min(ts), max(ts), "saturation", False)
    steps = run.steps
    if steps:
        peak = max(s.batch for s in steps)
        hot = [s for s in steps if s.batch >= peak_fraction * peak]
        if peak > 1 and hot:
            lo = min(s.t_start for s in hot)
            hi = max(s.t_end for s in hot)
            if hi > lo:
                return Window(lo, hi, "peak-batch", False)
    return Window(0.0, run.end_time, "full-run", True)


def nearest_rank(sorted_counts: list[tuple[float, int]], q: float) -> float:
    """q-quantile (0 < q <= 1) by nearest rank over (value, multiplicity) pairs
    sorted by value: the smallest value whose cumulative count >= ceil(q * n)."""
    n = sum(c for _, c in sorted_counts)
    if n == 0:
        return math.nan
    rank = max(1, math.ceil(q * n))
    acc = 0
    for v, c in sorted_counts:
        acc += c
        if acc >= rank:
            return v
    return sorted_counts[-1][0]


def summarize(run, window: Window | None = None) -> dict:
    """SPEC metrics.summarize. Returns {"empty": True, ...} for an empty window."""
    w = window if window is not None else stable_window(run)
    base = {"window": [w.t_start, w.t_end], "window_rule": w.rule, "flagged": w.flagged}
    if w.length <= 0:
        return dict(base, empty=True)
    inside = [s for s in run.steps if s.t_start >= w.t_start and s.t_end <= w.t_end]
    samples = sorted(((s.duration, s.batch) for s in inside if s.batch > 0))
    n_tok = sum(c for _, c in samples)
    if n_tok == 0:
        return dict(base, empty=True)
    ttft = [r.first_token_time - r.arrival_time for r in run.requests
            if not math.isnan(r.first_token_time) and w.t_start <= r.first_token_time <= w.t_end]
    req_tpot = [r.tpot() for r in run.requests
                if not math.isnan(r.tpot()) and w.t_start <= r.finish_time <= w.t_end]
    mean_tpot = sum(d * c for d, c in samples) / n_tok
    off = sum(s.batch_offload for s in inside)
    tot = sum(s.batch for s in inside)
    return dict(
        base, empty=False,
        output_tokens=n_tok,
        throughput_tok_s=n_tok / w.length,
        mean_ttft_s=sum(ttft) / len(ttft) if ttft else math.nan,
        p99_ttft_s=nearest_rank([(x, 1) for x in sorted(ttft)], 0.99) if ttft else math.nan,
        mean_tpot_s=mean_tpot,
        p50_tpot_s=nearest_rank(samples, 0.50),
        p90_tpot_s=nearest_rank(samples, 0.90),
        p99_tpot_s=nearest_rank(samples, 0.99),
        mean_request_tpot_s=sum(req_tpot) / len(req_tpot) if req_tpot else math.nan,
        max_decode_batch=max(s.batch for s in inside),
        mean_decode_batch=tot / len(inside),
        offloaded_share=off / tot if tot else 0.0,
        completed_in_window=sum(1 for r in run.requests
                                if not math.isnan(r.finish_time)
                                and w.t_start <= r.finish_time <= w.t_end),
    )
