"""Block tables / KV slots driven by the engine's token accounting, checked
bit-exactly against the oracle replay, and invariants of the page layout."""
import pytest

import kv_oracle

from paper_2503_20552_b200 import config, engine, kvcache, workload
from paper_2503_20552_b200.kvcache import BlockTables, PagePool, PagedKVMirror


def test_pool_lowest_id_first_and_reuse():
    pool = PagePool(10)
    assert pool.alloc(3) == [0, 1, 2]
    pool.free([1])
    assert pool.alloc(2) == [1, 3]
    with pytest.raises(MemoryError):
        pool.alloc(100)


def test_block_table_growth_and_slots():
    bt = BlockTables(PagePool(64))
    bt.reserve(7, 17)           # 2 pages
    assert bt.tables[7] == [0, 1]
    bt.reserve(9, 1)
    bt.reserve(7, 33)           # grows to 3 pages
    assert bt.tables[7] == [0, 1, 3] and bt.tables[9] == [2]
    assert bt.slot(7, 0) == 0 and bt.slot(7, 16) == 16 and bt.slot(7, 32) == 48
    assert bt.release(7) == [0, 1, 3]
    bt.reserve(11, 40)
    assert bt.tables[11] == [0, 1, 3]
    arr = bt.table_array([9, 11])
    assert arr.shape == (2, 3) and list(arr[1]) == [0, 1, 3]


@pytest.mark.parametrize("cfgd,preset,rate,n,seed", [
    ({}, "sharegpt_like", 3.0, 200, 7),
    ({"num_prefill": 2, "num_decode": 2, "offload_ratio": 0.5}, "sharegpt_like", 6.0, 150, 3),
    ({"gpu": {"name": "tight", "flops_peak": 312e12, "hbm_capacity_bytes": 24e9,
              "hbm_bandwidth": 2039e9, "interconnect_bandwidth": 600e9,
              "cpu_launch_per_layer": 1.137e-3}, "offload_ratio": 0.8},
     "sharegpt_like", 8.0, 150, 9),
])
def test_engine_driven_tables_match_oracle_replay(cfgd, preset, rate, n, seed):
    cfg = config.SimConfig.from_dict(cfgd)
    mirror = PagedKVMirror.for_config(cfg, slack_pages=512)
    reqs = workload.synth_requests(workload.preset(preset, rate, n), seed)
    engine.simulate(cfg, reqs, observer=mirror)
    # every request finished: all pages back in every pool
    for bt in mirror.pools.values():
        assert bt.pool.free_pages == bt.pool.num_pages and not bt.tables
    sizes = {w: bt.pool.num_pages for w, bt in mirror.pools.items()}
    events = [(op, w, rid, tok) for op, w, rid, tok, _ in mirror.log]
    _, handed = kv_oracle.replay(events, sizes)
    got = [pages if op == "reserve" else None for op, _, _, _, pages in mirror.log]
    assert got == handed


def test_live_pages_never_exceed_token_budget_plus_slack():
    cfg = config.SimConfig.from_dict({"gpu": {"name": "tight", "flops_peak": 312e12,
                                              "hbm_capacity_bytes": 24e9,
                                              "hbm_bandwidth": 2039e9,
                                              "interconnect_bandwidth": 600e9,
                                              "cpu_launch_per_layer": 1.137e-3},
                                      "offload_ratio": 0.8})
    kv_tok = cfg.model.kv_bytes_per_token

    class Check(PagedKVMirror):
        peak = 0

        def reserve(self, req, where, tokens):
            super().reserve(req, where, tokens)
            bt = self.pools[where]
            live_tokens = sum(bt.tokens.values())
            budget = cfg.pool_bytes if where[0] == "decoder" else cfg.executor_budget_bytes
            assert live_tokens * kv_tok <= budget
            used_pages = bt.pool.num_pages - bt.pool.free_pages
            assert used_pages <= live_tokens // 16 + len(bt.tables)
            Check.peak = max(Check.peak, used_pages)

    mirror = Check.for_config(cfg, slack_pages=256, keep_log=False)
    engine.simulate(cfg, workload.synth_requests(workload.preset("sharegpt_like", 8.0, 150), 9),
                    observer=mirror)
    assert Check.peak > 0


def test_slot_mapping_matches_oracle():
    bt = BlockTables(PagePool(100))
    for rid, tok in [(1, 40), (2, 3), (3, 100), (1, 70)]:
        bt.reserve(rid, tok)
    for rid in (1, 2, 3):
        for pos in range(bt.tokens[rid]):
            assert bt.slot(rid, pos) == kv_oracle.slot(bt.tables[rid], pos)


@pytest.mark.parametrize("cfgd,preset,rate,n,seed", [
    ({}, "sharegpt_like", 3.0, 120, 7),
    ({"num_prefill": 2, "num_decode": 2, "offload_ratio": 0.5}, "sharegpt_like", 6.0, 120, 3),
    ({"gpu": {"name": "tight", "flops_peak": 312e12, "hbm_capacity_bytes": 24e9,
              "hbm_bandwidth": 2039e9, "interconnect_bandwidth": 600e9,
              "cpu_launch_per_layer": 1.137e-3}, "offload_ratio": 0.8},
     "sharegpt_like", 8.0, 120, 9),
])
def test_prefill_to_decode_handoff_matches_oracle(cfgd, preset, rate, n, seed):
    """Every local request's prompt KV is staged in prefill-GPU pages and
    migrated into the decoder pages reserved at admission (engine.py:231-249);
    the whole reserve / stage / transfer / unstage / release stream replays
    bit-exactly on the oracle's allocator, and observing it changes nothing."""
    cfg = config.SimConfig.from_dict(cfgd)
    seen = []
    mirror = PagedKVMirror.for_config(cfg, slack_pages=512, stage_pages=1 << 16,
                                      on_transfer=seen.append)
    reqs = workload.synth_requests(workload.preset(preset, rate, n), seed)
    with_obs = engine.simulate(cfg, reqs, observer=mirror)
    plain = engine.simulate(cfg, workload.synth_requests(workload.preset(preset, rate, n), seed))
    assert [(s.t_start, s.t_end, s.batch_local, s.batch_offload) for s in with_obs.steps] == \
        [(s.t_start, s.t_end, s.batch_local, s.batch_offload) for s in plain.steps]
    # one hand-off per transfer the engine priced, all staging pages returned
    assert len(seen) == mirror.transfers == len(with_obs.transfers) > 0
    assert sorted(t.req_id for t in seen) == sorted(t.req_id for t in with_obs.transfers)
    for where, bt in mirror.pools.items():
        assert bt.pool.free_pages == bt.pool.num_pages and not bt.tables, where
    sizes = {w: bt.pool.num_pages for w, bt in mirror.pools.items()}
    events = []
    for op, w, rid, tok, pages in mirror.log:
        events.append((op, w, rid, tok, pages.dst) if op == "transfer" else (op, w, rid, tok))
    _, expect = kv_oracle.replay_handoff(events, sizes)
    got = []
    for op, w, rid, tok, pages in mirror.log:
        if op in ("reserve", "stage"):
            got.append(tuple(pages))
        elif op == "transfer":
            got.append((pages.src_pages, pages.dst_pages))
        else:
            got.append(None)
    assert got == expect
    # a transfer moves exactly the prompt's pages, into distinct decoder pages
    for tr in seen:
        assert len(tr.src_pages) == len(tr.dst_pages) > 0
        assert len(set(tr.dst_pages)) == len(tr.dst_pages)
