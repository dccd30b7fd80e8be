"""Capacity-bound decode batches (capacity.plan_capacity): the no-offload fill
stops at the decoder's KV pool, the offload fill is Algorithm 1 (need_offload,
literal form) with the engine's budget gating, and for the BASELINE C4 shape on
B200 the offload batch exceeds the no-offload batch."""
import pytest

import decision_oracle as dor  # noqa: F401  (oracle module path check)

from paper_2503_20552_b200 import capacity, config, scheduling, specs, workload


def reqs(n=1500, seed=17):
    return capacity.snapshot_requests(
        workload.synth_requests(workload.preset("sharegpt_like", 10.0, n), seed), 0)


def test_snapshot_is_mid_decode_and_deterministic():
    a, b = reqs(200), reqs(200)
    assert [r.used_token for r in a] == [r.used_token for r in b]
    for r in a:
        assert r.prompt_tokens <= r.used_token < r.max_token


@pytest.mark.parametrize("model,nd", [(specs.LLAMA2_13B, 1), (specs.LLAMA2_13B, 4),
                                      (specs.LLAMA3_8B, 2)])
def test_plan_matches_literal_algorithm_1(model, nd):
    cfg = config.SimConfig(gpu=specs.B200, model=model, num_prefill=nd, num_decode=nd)
    rs = reqs()
    plan = capacity.plan_capacity(cfg, rs)
    kv = cfg.model.kv_bytes_per_token
    # no offload: a prefix of the stream that fits the pool, the next one does not
    n = plan.batch_no_offload
    used = sum((r.used_token + 1) * kv for r in rs[:n])
    assert used <= cfg.pool_bytes < used + (rs[n].used_token + 1) * kv
    # offload: replay with the literal need_offload over explicit lists
    off, loc = [], []
    ub = cfg.executor_budget_bytes * nd / nd
    ul = ux = 0
    for r in rs:
        d = scheduling.need_offload(r, off, loc, plan.bound,
                                    c1_uses_max_tokens=cfg.c1_uses_max_tokens)
        need = (r.used_token + 1) * kv
        if d.offload:
            if ux + need > ub:
                break
            ux += need
            off.append(r)
        else:
            if ul + need > cfg.pool_bytes:
                break
            ul += need
            loc.append(r)
    assert plan.local == [r.used_token + 1 for r in loc]
    assert plan.offloaded == [r.used_token + 1 for r in off]
    assert plan.bytes("local") <= cfg.pool_bytes
    assert plan.bytes("offloaded") <= plan.exec_budget_bytes


def test_c4_offload_raises_the_capacity_bound_batch():
    cfg = config.SimConfig(gpu=specs.B200, model=specs.LLAMA2_13B, num_prefill=4, num_decode=4)
    plan = capacity.plan_capacity(cfg, reqs())
    assert plan.batch_gain >= 1.4
    assert plan.offloaded and plan.local
    s = plan.summary()
    assert s["batch_offload"] == len(plan.local) + len(plan.offloaded)


def test_scale_shrinks_both_budgets():
    cfg = config.SimConfig(gpu=specs.B200, model=specs.LLAMA2_13B, num_prefill=1, num_decode=1)
    full, half = capacity.plan_capacity(cfg, reqs()), capacity.plan_capacity(cfg, reqs(), scale=0.5)
    assert half.pool_bytes == pytest.approx(full.pool_bytes / 2)
    assert half.batch_no_offload < full.batch_no_offload
