"""GPU checks of the offloaded decode step (pack -> transport -> executor
append+attention -> return -> scatter) and of green-context colocation."""
import math

import numpy as np
import pytest
import torch

import oracle as orc
from paper_2503_20552_b200 import coloc, ops
from paper_2503_20552_b200.kvcache import BlockTables, PagePool
from paper_2503_20552_b200.runtime import AttentionExecutor, LayeredKV, OffloadedDecodeStep, StepPlan
from paper_2503_20552_b200.synthetic import CONFIGS, make_layer

pytestmark = pytest.mark.gpu


def u16(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def build_step(cuda, ctx_local, ctx_off, L=2, Hq=32, Hkv=8, D=128, partition=None, seed=0,
               zero_copy=False):
    g = torch.Generator(device=cuda).manual_seed(seed)
    NB = 64 + sum(-(-c // 16) for c in ctx_local + ctx_off)
    local_kv = LayeredKV(L, NB, Hkv, D, cuda, fill="randn", generator=g)
    exec_kv = LayeredKV(L, NB, Hkv, D, cuda, fill="randn", generator=g)
    lt, xt = BlockTables(PagePool(NB)), BlockTables(PagePool(NB))
    for i, c in enumerate(ctx_local):
        lt.reserve(i, c)
    for i, c in enumerate(ctx_off):
        xt.reserve(i, c)
    nl, no = len(ctx_local), len(ctx_off)
    B = nl + no
    plan = StepPlan(
        nl, no,
        torch.from_numpy(lt.table_array(list(range(nl)))).to(cuda),
        torch.tensor(ctx_local, dtype=torch.int32, device=cuda),
        torch.tensor([lt.slot(i, c - 1) for i, c in enumerate(ctx_local)], dtype=torch.int64, device=cuda),
        torch.from_numpy(xt.table_array(list(range(no)))).to(cuda) if no else None,
        torch.tensor(ctx_off, dtype=torch.int32, device=cuda) if no else None,
        torch.tensor([xt.slot(i, c - 1) for i, c in enumerate(ctx_off)], dtype=torch.int64, device=cuda) if no else None)
    mk = lambda *s: torch.randn(*s, generator=g, device=cuda).to(torch.bfloat16)
    qs = [mk(B, Hq, D) for _ in range(L)]
    ks = [mk(B, Hkv, D) for _ in range(L)]
    vs = [mk(B, Hkv, D) for _ in range(L)]
    outs = [torch.empty(B, Hq, D, dtype=torch.bfloat16, device=cuda) for _ in range(L)]
    local = AttentionExecutor(local_kv, Hq, B)
    if partition is not None:
        remote = AttentionExecutor(exec_kv, Hq, B, stream=partition.attn_stream,
                                   num_sms=partition.attn_sms)
    else:
        remote = AttentionExecutor(exec_kv, Hq, B)
    before = {n: (u16(kv.k), u16(kv.v)) for n, kv in (("local", local_kv), ("exec", exec_kv))}
    step = OffloadedDecodeStep(Hq, Hkv, D, local, remote if no else None, zero_copy=zero_copy)
    return step, plan, qs, ks, vs, outs, before, (local_kv, exec_kv)


def oracle_step(plan, qs, ks, vs, before, D):
    scale = 1.0 / math.sqrt(D)
    nl, no = plan.n_local, plan.n_off
    res = []
    for l in range(len(qs)):
        o = np.zeros((nl + no,) + tuple(qs[l].shape[1:]), dtype=np.float32)
        for name, rows, bt, seq, slots in (("local", slice(0, nl), plan.local_bt, plan.local_seq, plan.local_slots),
                                           ("exec", slice(nl, nl + no), plan.exec_bt, plan.exec_seq, plan.exec_slots)):
            if rows.stop == rows.start:
                continue
            k0, v0 = before[name]
            kc, vc = orc.kv_append(ks[l][rows], vs[l][rows], k0[l], v0[l], slots.cpu().numpy())
            o[rows], _ = orc.paged_decode_attn(qs[l][rows], kc, vc, bt, seq, scale)
        res.append(o)
    return res


def check(out, ref):
    g = out.float().cpu().numpy()
    assert np.abs(g - ref).max() <= 2e-2
    refb = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
    assert np.abs(g - refb).sum() / np.abs(refb).sum() <= 1e-3


@pytest.mark.parametrize("zero_copy", [False, True])
@pytest.mark.parametrize("ctx_local,ctx_off", [
    ([300, 17, 1024, 64, 5], [900, 33, 2000]),
    ([128, 129], []),
    ([], [77, 4096]),
])
def test_offloaded_step_loopback_matches_oracle(cuda, ctx_local, ctx_off, zero_copy):
    """Message path (pack / send / unpack / attention / send / scatter) and the
    zero-copy path (the executor's kernel reads the decode rows and writes the
    decode outputs through row maps) give the oracle's outputs and appends."""
    step, plan, qs, ks, vs, outs, before, kvs = build_step(cuda, ctx_local, ctx_off,
                                                           zero_copy=zero_copy)
    times = step.run(qs, ks, vs, plan, outs)
    ref = oracle_step(plan, qs, ks, vs, before, 128)
    for l in range(len(qs)):
        check(outs[l], ref[l])
    assert times.total > 0
    if not zero_copy:
        assert times.link_bytes == 2 * len(ctx_off) * (32 + 16 + 32) * 128 * 2
    # the executor's cache received exactly the appended rows
    if ctx_off:
        ek = u16(kvs[1].k)
        for l in range(len(qs)):
            for i, s in enumerate(plan.exec_slots.cpu().tolist()):
                assert np.array_equal(ek[l, s // 16, :, s % 16, :],
                                      u16(ks[l][plan.n_local + i]))


@pytest.mark.skipif(not coloc.green_contexts_supported(), reason="no green contexts")
def test_offloaded_step_on_green_context_partition(cuda):
    part = coloc.SmPartition(0, 64)
    # the executor's green context gets the requested multiple of 8, the prefill's the rest
    assert part.attn_sms == 64 and part.prefill_sms == part.total_sms - 64
    step, plan, qs, ks, vs, outs, before, _ = build_step(cuda, [500, 40, 3000], [1000, 2500, 9],
                                                        partition=part)
    step.run(qs, ks, vs, plan, outs)
    ref = oracle_step(plan, qs, ks, vs, before, 128)
    for l in range(len(qs)):
        check(outs[l], ref[l])


@pytest.mark.skipif(not coloc.green_contexts_supported(), reason="no green contexts")
def test_partition_sweep_produces_valid_samples(cuda):
    from paper_2503_20552_b200.synthetic import DecodeShape
    shape = DecodeShape("sweep", 16, 32, 8, 128, 1, 4096)
    layer = make_layer(shape, cuda)
    load = ops  # noqa: F841
    pre = coloc.PrefillLoad(2048, 4096, 11008, cuda)
    sw = coloc.sweep_partitions(0, layer, pre, [32, 72, 112], iters=2)
    assert sw["full_attn_gbs"] > 1000
    for s in sw["samples"]:
        assert s.attn_gbs_alone > 0 and s.prefill_s_alone >= sw["full_prefill_s"] * 0.9
    # more SMs for attention -> at least as much bandwidth (monotone within noise)
    bws = [s.attn_gbs_alone for s in sw["samples"]]
    assert bws[-1] >= 0.9 * bws[0]
