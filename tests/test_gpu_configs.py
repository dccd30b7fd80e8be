"""GPU oracle parity on every BASELINE.json config at its own shapes, and the
kernel's behaviour on bad block tables.

Tolerances are the north star's: max-abs <= 2e-2 against the fp32 oracle and
mean-rel <= 1e-3 (fp32-output mode against the fp32 oracle; bf16-output mode
against the bf16-rounded oracle).

  C1  tiny 8q/2kv D=64, B=8, ctx 512, 2 layers; Algorithm 1 at bound 0.5 picks
      requests {3, 6} (scheduling.py:176-221, golden need_offload.json), and the
      step runs end to end through OffloadedDecodeStep (message and zero-copy
      modes) against the oracle.
  C2  Llama-2-7B MHA 32x128, B=64, ctx 4096: 16 of the 64 requests re-paged
      for the oracle.
  C3  Llama-3-8B GQA 32q/8kv, B=64 (the bench's batch), ctx 4096: every request.
  C4  Llama-2-13B MHA 40x128, B=64 decode contexts drawn from the reference's
      ShareGPT-like length mix (workload.py:141-142): prompt + a uniform share
      of the output already generated; every request.
  C5  Llama-3-70B GQA-8 64q/8kv, B=16, ctx 32k: tests/test_gpu_attention.py.
"""
import math
import random

import numpy as np
import pytest
import torch

import oracle as orc
from paper_2503_20552_b200 import _ffi, ops, scheduling
from paper_2503_20552_b200.synthetic import CONFIGS, DecodeShape, make_layer
from paper_2503_20552_b200.workload import preset, synth_requests

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
MEAN_REL = 1e-3


def check(out, ref, bf16_out=False):
    g = out.float().cpu().numpy()
    assert np.isfinite(g).all()
    err = float(np.abs(g - ref).max())
    assert err <= MAX_ABS, f"max-abs {err}"
    cmp = torch.from_numpy(ref).to(torch.bfloat16).float().numpy() if bf16_out else ref
    mr = float(np.abs(g - cmp).sum() / np.abs(cmp).sum())
    assert mr <= MEAN_REL, f"mean-rel {mr}"
    return err, mr


def repaged_oracle(x, pick, scale, k_cache=None, v_cache=None):
    """Oracle over requests ``pick`` only: their pages copied into a compact cache."""
    kc0 = x["k_cache"] if k_cache is None else k_cache
    vc0 = x["v_cache"] if v_cache is None else v_cache
    pages = x["block_table"][pick].flatten().long()
    kc, vc = kc0[pages].cpu(), vc0[pages].cpu()
    bt = torch.arange(pages.numel(), dtype=torch.int32).view(len(pick), -1)
    return orc.paged_decode_attn(x["q"][pick].cpu(), kc, vc, bt, x["seq_lens"][pick].cpu(), scale)


def sharegpt_contexts(batch, seed=0):
    """Decode-time contexts of a ShareGPT-like batch: prompt + generated-so-far."""
    reqs = synth_requests(preset("sharegpt_like", 1.0, batch), seed)
    rng = random.Random(seed + 1)
    return tuple(r.prompt_tokens + 1 + rng.randrange(r.output_tokens) for r in reqs)


def test_c2_full_batch_sixteen_requests(cuda):
    shape = CONFIGS["C2"]
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(128)
    ws = ops.DecodeWorkspace(64, 32, 32, 128, cuda, max_blocks_per_seq=shape.max_pages)
    lse = torch.empty(64, 32, dtype=torch.float32, device=cuda)
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], lse=lse, scale=scale, out_dtype=torch.float32,
                                workspace=ws, k_new=x["k_new"], v_new=x["v_new"], pdl=True)
    torch.cuda.synchronize()
    pick = list(range(0, 64, 4))  # 16 requests spread over the batch (and the chunk grid)
    ref, ref_lse = repaged_oracle(x, pick, scale)
    check(out[pick], ref)
    np.testing.assert_allclose(lse[pick].cpu().numpy(), ref_lse, atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_c3_batch64_every_request(cuda, out_dtype):
    shape = CONFIGS["C3"]
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(128)
    ws = ops.DecodeWorkspace(64, 32, 8, 128, cuda, max_blocks_per_seq=shape.max_pages)
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], scale=scale, out_dtype=out_dtype, workspace=ws)
    torch.cuda.synchronize()
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], scale)
    check(out, ref, out_dtype == torch.bfloat16)


@pytest.mark.parametrize("grid", ["auto", "dynamic", "static", "split"])
def test_c4_sharegpt_lengths_every_request(cuda, grid):
    ctx = sharegpt_contexts(64)
    assert min(ctx) >= 17 and max(ctx) <= 8192 + 4096
    shape = DecodeShape("C4-llama2-13b", 64, 40, 40, 128, 1, ctx)
    x = make_layer(shape, cuda, seed=4)
    scale = 1.0 / math.sqrt(128)
    pos = x["seq_lens"].long() - 1
    slots = ops.slot_mapping(x["block_table"], pos)
    ref_k, ref_v = orc.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"],
                                 slots.cpu().numpy())
    ws = ops.DecodeWorkspace(64, 40, 40, 128, cuda, max_blocks_per_seq=shape.max_pages)
    lse = torch.empty(64, 40, dtype=torch.float32, device=cuda)
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], lse=lse, scale=scale, out_dtype=torch.float32,
                                workspace=ws, k_new=x["k_new"], v_new=x["v_new"], grid=grid)
    torch.cuda.synchronize()
    # the fused append wrote exactly the oracle's rows
    assert np.array_equal(x["k_cache"].cpu().view(torch.int16).numpy().view(np.uint16), ref_k)
    assert np.array_equal(x["v_cache"].cpu().view(torch.int16).numpy().view(np.uint16), ref_v)
    ref, ref_lse = orc.paged_decode_attn(x["q"], ref_k, ref_v, x["block_table"], x["seq_lens"],
                                         scale)
    check(out, ref)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_lse, atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("zero_copy", [False, True])
def test_c1_offload_selection_runs_end_to_end(cuda, zero_copy):
    """C1: 8 requests (prompt 256 + output 256 = max_token 512), all at their
    last token (used 512). Algorithm 1 at bound 0.5 offloads {3, 6} (the golden
    selection); the step then runs the 6 local rows on the decode executor and
    rows 3 and 6 on the remote executor, 2 layers, against the oracle."""
    from test_gpu_runtime import build_step, oracle_step, check as check_step
    off, loc, picks = [], [], []
    for k in range(8):
        r = scheduling.Request(req_id=k, arrival_time=0.0, prompt_tokens=256, output_tokens=256)
        r.used_token = 512
        d = scheduling.need_offload(r, off, loc, 0.5)
        (off if d.offload else loc).append(r)
        picks.append(d.offload)
    chosen = [k for k, p in enumerate(picks) if p]
    assert chosen == [3, 6]
    shape = CONFIGS["C1"]
    local_ids = [k for k in range(8) if k not in chosen]
    ctx = shape.ctx_list()
    step, plan, qs, ks, vs, outs, before, _ = build_step(
        cuda, [ctx[k] for k in local_ids], [ctx[k] for k in chosen], L=shape.num_layers,
        Hq=shape.num_q_heads, Hkv=shape.num_kv_heads, D=shape.head_dim, zero_copy=zero_copy)
    assert plan.n_local == 6 and plan.n_off == 2
    step.run(qs, ks, vs, plan, outs)
    ref = oracle_step(plan, qs, ks, vs, before, shape.head_dim)
    for l in range(shape.num_layers):
        check_step(outs[l], ref[l])


# ---- bad tables: rejected, never dereferenced ---------------------------------

def _bad_case(cuda):
    shape = DecodeShape("bad", 4, 8, 2, 128, 1, (40, 100, 16, 70))
    x = make_layer(shape, cuda)
    return shape, x


def test_check_tables_rejects_out_of_range_page(cuda):
    shape, x = _bad_case(cuda)
    ws = ops.DecodeWorkspace(4, 8, 2, 128, cuda)
    NB = x["k_cache"].shape[0]
    ops.check_decode_tables(x["block_table"], x["seq_lens"], NB, ws)  # valid: no error
    bt = x["block_table"].clone()
    bt[1, 3] = NB  # request 1's 4th page (of 7) points past the cache
    with pytest.raises(_ffi.AdrError) as e:
        ops.check_decode_tables(bt, x["seq_lens"], NB, ws)
    assert e.value.code == _ffi.ADR_ERR_INVALID and "request 1" in str(e.value)
    bt[1, 3] = -5
    with pytest.raises(_ffi.AdrError):
        ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], bt, x["seq_lens"],
                              workspace=ws, check_tables=True)
    # entries past the request's pages are never used, so never checked
    bt2 = x["block_table"].clone()
    bt2[2, 1:] = 1 << 30
    ops.check_decode_tables(bt2, x["seq_lens"], NB, ws)


def test_check_tables_rejects_seq_len_past_table_row(cuda):
    shape, x = _bad_case(cuda)
    ws = ops.DecodeWorkspace(4, 8, 2, 128, cuda)
    NB = x["k_cache"].shape[0]
    width = x["block_table"].shape[1]
    for bad in (width * 16 + 1, -1):
        sl = x["seq_lens"].clone()
        sl[2] = bad
        with pytest.raises(_ffi.AdrError) as e:
            ops.check_decode_tables(x["block_table"], sl, NB, ws)
        assert e.value.code == _ffi.ADR_ERR_INVALID and "request 2" in str(e.value)
    sl = x["seq_lens"].clone()
    sl[2] = width * 16  # exactly the row: valid
    ops.check_decode_tables(x["block_table"], sl, NB, ws)


@pytest.mark.parametrize("grid", ["dynamic", "static", "split"])
def test_kernel_never_dereferences_bad_entries(cuda, grid):
    """Without the check, the kernel neither reads nor writes outside the cache
    on bad tables: the bad request's append is skipped, a request whose
    seq_len runs past its row gets a zero row / lse -inf, the good requests
    match the oracle, and the workspace records the status bits."""
    shape, x = _bad_case(cuda)
    NB = x["k_cache"].shape[0]
    ws = ops.DecodeWorkspace(4, 8, 2, 128, cuda)
    bt = x["block_table"].clone()
    last_page = (int(x["seq_lens"][1]) - 1) // 16
    bt[1, last_page] = NB + 1000  # the append page of request 1 is out of range
    sl = x["seq_lens"].clone()
    sl[3] = bt.shape[1] * 16 + 5  # request 3 runs past its row
    kc, vc = x["k_cache"].clone(), x["v_cache"].clone()
    lse = torch.empty(4, 8, dtype=torch.float32, device=cuda)
    out = ops.paged_decode_attn(x["q"], kc, vc, bt, sl, lse=lse, out_dtype=torch.float32,
                                workspace=ws, k_new=x["k_new"], v_new=x["v_new"], grid=grid)
    st = ops.decode_status(ws)
    assert st == _ffi.ADR_STATUS_BAD_PAGE | _ffi.ADR_STATUS_BAD_SEQ_LEN
    assert ops.decode_status(ws) == 0  # cleared
    assert torch.all(out[3] == 0) and bool(torch.isneginf(lse[3]).all())
    # good requests 0 and 2: appended and attended exactly as the oracle does
    good = [0, 2]
    pos = x["seq_lens"].long() - 1
    slots = ops.slot_mapping(x["block_table"], pos)
    ref_k, ref_v = orc.kv_append(x["k_new"][good], x["v_new"][good], x["k_cache"], x["v_cache"],
                                 slots[good].cpu().numpy())
    got_k = kc.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got_k, ref_k)  # nothing else in the cache changed
    ref, _ = orc.paged_decode_attn(x["q"][good], ref_k, ref_v, x["block_table"][good],
                                   x["seq_lens"][good], 1.0 / math.sqrt(128))
    check(out[good], ref)
    # the counters are clean for the next call
    counters = ws.buf[: (1 << 17) * 4 * 2 + 256].view(torch.int32)
    assert int(counters.abs().sum()) == 0


def test_workspace_sized_by_batch(cuda):
    """A workspace sized with max_blocks_per_seq scales with the batch; a call
    wider than it was sized for is refused with ADR_ERR_WORKSPACE."""
    small = ops.DecodeWorkspace(8, 32, 8, 128, cuda, max_blocks_per_seq=64)
    big = ops.DecodeWorkspace(8, 32, 8, 128, cuda)
    assert small.buf.numel() < big.buf.numel() // 8
    shape = DecodeShape("ws", 8, 32, 8, 128, 1, 1024)
    x = make_layer(shape, cuda)
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], out_dtype=torch.float32, workspace=small)
    torch.cuda.synchronize()
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], 1.0 / math.sqrt(128))
    check(out, ref)
    wide = torch.zeros(8, 200, dtype=torch.int32, device=cuda)
    wide[:, :64] = x["block_table"]
    with pytest.raises(_ffi.AdrError) as e:
        ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], wide, x["seq_lens"],
                              workspace=small)
    assert e.value.code == _ffi.ADR_ERR_WORKSPACE
