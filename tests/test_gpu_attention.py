"""GPU parity of adr_paged_decode_attn against the CPU oracle (fp32, double acc).

Tolerances (BASELINE.json north star): max-abs <= 2e-2 and mean-rel <= 1e-3 with
mean-rel = sum|gpu - ref| / sum|ref|. The mean-rel gate is applied to the
kernel's fp32-output mode: rounding a perfect fp32 result to bf16 alone gives
mean-rel ~1.4e-3 (measured on N(0,1)-like outputs), so the bf16-output mode is
gated at max-abs 2e-2 and mean-rel 1e-3 against the bf16-rounded oracle.
"""
import math

import numpy as np
import pytest
import torch

import oracle as orc
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.synthetic import CONFIGS, DecodeShape, make_layer

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
MEAN_REL = 1e-3


def mean_rel(a, ref):
    return float(np.abs(a - ref).sum() / max(np.abs(ref).sum(), 1e-30))


def check(gpu_out, ref, bf16_out):
    g = gpu_out.float().cpu().numpy()
    if bf16_out:
        ref_cmp = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
    else:
        ref_cmp = ref
    assert np.isfinite(g).all()
    err = float(np.abs(g - ref).max())
    assert err <= MAX_ABS, f"max-abs {err}"
    mr = mean_rel(g, ref_cmp)
    assert mr <= MEAN_REL, f"mean-rel {mr}"
    return err, mr


def run_case(shape, device, num_workers=0, out_dtype=torch.float32, with_lse=True, seed=0,
             grid="auto"):
    x = make_layer(shape, device, seed=seed)
    scale = 1.0 / math.sqrt(shape.head_dim)
    ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                             device, num_workers=num_workers)
    lse = torch.empty(shape.batch, shape.num_q_heads, dtype=torch.float32, device=device) \
        if with_lse else None
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], lse=lse, scale=scale, out_dtype=out_dtype,
                                workspace=ws, grid=grid)
    torch.cuda.synchronize()
    ref, ref_lse = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                         x["seq_lens"], scale)
    return x, out, lse, ref, ref_lse


CASES = {
    "C1": CONFIGS["C1"],
    "C2-b4": DecodeShape("C2-b4", 4, 32, 32, 128, 1, 4096),
    "C3-b8": DecodeShape("C3-b8", 8, 32, 8, 128, 1, 4096),
    "C5-b2-ctx8k": DecodeShape("C5-b2", 2, 64, 8, 128, 1, 8192),
    "ragged-mha": DecodeShape("rag", 7, 8, 8, 128, 1, (1, 15, 16, 17, 100, 1000, 2049)),
    "ragged-gqa2-d64": DecodeShape("rag64", 5, 4, 2, 64, 1, (3, 31, 32, 33, 777)),
}


GRIDS = ["auto", "dynamic", "static", "split"]


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_decode_attention_matches_oracle(cuda, name, out_dtype, grid):
    shape = CASES[name]
    x, out, lse, ref, ref_lse = run_case(shape, cuda, out_dtype=out_dtype, grid=grid)
    check(out, ref, out_dtype == torch.bfloat16)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_lse, atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("grid", ["dynamic", "static"])
@pytest.mark.parametrize("workers", [4, 12, 100, 1000, 5000])
def test_split_pairs_merge_exactly(cuda, workers, grid):
    # small worker counts keep whole pairs; large counts cut every pair into
    # several warp ranges that the LSE merge must recombine (static grid with
    # more warps than fit on the GPU: late CTAs delay, never deadlock, the merge)
    shape = DecodeShape("split", 3, 16, 4, 128, 1, (700, 64, 1500))
    x, out, lse, ref, ref_lse = run_case(shape, cuda, num_workers=workers, grid=grid)
    check(out, ref, False)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_lse, atol=1e-3, rtol=1e-4)


def test_empty_and_single_token_requests(cuda):
    shape = DecodeShape("edge", 4, 8, 2, 128, 1, (0, 1, 0, 16))
    x, out, lse, ref, ref_lse = run_case(shape, cuda)
    g = out.cpu().numpy()
    assert np.all(g[0] == 0) and np.all(g[2] == 0)
    assert np.all(np.isneginf(lse.cpu().numpy()[[0, 2]]))
    check(out[[1, 3]], ref[[1, 3]], False)


def test_no_lse_and_repeatable(cuda):
    shape = CASES["C3-b8"]
    _, out1, _, ref, _ = run_case(shape, cuda, with_lse=False, out_dtype=torch.bfloat16)
    _, out2, _, _, _ = run_case(shape, cuda, with_lse=False, out_dtype=torch.bfloat16)
    assert torch.equal(out1, out2)  # deterministic (no atomics)
    check(out1, ref, True)


def test_full_c2_subsample_against_oracle(cuda):
    """C2 at full size (B=64, 32 heads, ctx 4096: 4 GiB KV). The oracle checks a
    sample of 4 requests by re-paging just their pages into a compact cache."""
    shape = CONFIGS["C2"]
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(128)
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                workspace=ops.DecodeWorkspace(64, 32, 32, 128, cuda))
    torch.cuda.synchronize()
    pick = [0, 17, 42, 63]
    bt = x["block_table"][pick]
    pages = bt.flatten().long()
    kc = x["k_cache"][pages].cpu()
    vc = x["v_cache"][pages].cpu()
    compact_bt = torch.arange(pages.numel(), dtype=torch.int32).view(len(pick), -1)
    ref, _ = orc.paged_decode_attn(x["q"][pick].cpu(), kc, vc, compact_bt, x["seq_lens"][pick],
                                   scale)
    check(out[pick], ref, False)
    # size-independent property on all rows: outputs are convex combinations of V rows
    o = out.abs().amax().item()
    assert math.isfinite(o) and o <= x["v_cache"].abs().amax().item() + 1e-3


def test_workspace_reuse_across_shapes(cuda):
    """The split-pair counters are self-cleaning: one workspace serves calls of
    different shapes / worker counts back to back."""
    ws = ops.DecodeWorkspace(16, 32, 8, 128, cuda, num_workers=37)
    for shape in [DecodeShape("a", 3, 32, 8, 128, 1, (900, 33, 2000)),
                  DecodeShape("b", 16, 8, 8, 128, 1, 300),
                  DecodeShape("c", 3, 32, 8, 128, 1, (900, 33, 2000))]:
        x = make_layer(shape, cuda)
        scale = 1.0 / math.sqrt(128)
        out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                    x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                    workspace=ws)
        torch.cuda.synchronize()
        ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                       x["seq_lens"], scale)
        check(out, ref, False)
    counters = ws.buf[: (1 << 17) * 4 + 256].view(torch.int32)  # pair arrivals + chunk claims
    assert int(counters.abs().sum()) == 0


@pytest.mark.parametrize("grid", ["auto", "static", "split"])
@pytest.mark.parametrize("workers", [0, 7, 3000])
@pytest.mark.parametrize("pdl", [False, True])
def test_fused_append_matches_separate_append(cuda, workers, pdl, grid):
    """k_new/v_new fused into the attention pass == kv_append then attention:
    identical (bit-exact) caches, outputs within tolerance of the oracle, and the
    same bits as the unfused path."""
    shape = DecodeShape("fused", 6, 32, 8, 128, 1, (1, 16, 17, 700, 2048, 4095))
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(128)
    pos = x["seq_lens"].long() - 1
    slots = ops.slot_mapping(x["block_table"], pos)
    ref_k, ref_v = orc.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"],
                                 slots.cpu().numpy())
    ws = ops.DecodeWorkspace(shape.batch, 32, 8, 128, cuda, num_workers=workers)
    kc, vc = x["k_cache"].clone(), x["v_cache"].clone()
    fused = ops.paged_decode_attn(x["q"], kc, vc, x["block_table"], x["seq_lens"], scale=scale,
                                  out_dtype=torch.float32, workspace=ws, k_new=x["k_new"],
                                  v_new=x["v_new"], pdl=pdl, grid=grid)
    torch.cuda.synchronize()
    assert np.array_equal(kc.cpu().view(torch.int16).numpy().view(np.uint16), ref_k)
    assert np.array_equal(vc.cpu().view(torch.int16).numpy().view(np.uint16), ref_v)
    ref, _ = orc.paged_decode_attn(x["q"], ref_k, ref_v, x["block_table"], x["seq_lens"], scale)
    check(fused, ref, False)
    ops.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
    plain = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                  x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                  workspace=ws, grid=grid)
    torch.cuda.synchronize()
    assert torch.equal(fused, plain)


def test_pdl_chain_of_layers(cuda):
    """Back-to-back PDL launches on one stream (the decode step's layer chain)
    give the same bits as plain launches."""
    shape = DecodeShape("chain", 8, 32, 32, 128, 6, 1500)
    from paper_2503_20552_b200.synthetic import make_block_table
    bt = make_block_table(shape)
    layers = [make_layer(shape, cuda, seed=l, block_table=bt) for l in range(shape.num_layers)]
    ws = ops.DecodeWorkspace(8, 32, 32, 128, cuda)

    def run(pdl):
        outs = []
        for x in layers:
            outs.append(ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                              x["seq_lens"], workspace=ws, pdl=pdl))
        torch.cuda.synchronize()
        return outs
    a, b = run(False), run(True)
    for u, v in zip(a, b):
        assert torch.equal(u, v)


def test_padding_rows_do_not_change_results(cuda):
    """Empty padding requests (seq_len 0, as CUDA-graph grid padding produces)
    leave the real rows' bits unchanged: the work split depends only on the
    non-empty requests."""
    shape = DecodeShape("pad", 5, 8, 2, 64, 1, (300, 77, 512, 40, 129))
    x = make_layer(shape, cuda)
    ws = ops.DecodeWorkspace(8, 8, 2, 64, cuda)
    base = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                 x["seq_lens"], workspace=ws)
    pad = 3
    q = torch.cat([x["q"], torch.zeros(pad, 8, 64, dtype=torch.bfloat16, device=cuda)])
    bt = torch.cat([x["block_table"], torch.zeros(pad, x["block_table"].shape[1],
                                                  dtype=torch.int32, device=cuda)])
    sl = torch.cat([x["seq_lens"], torch.zeros(pad, dtype=torch.int32, device=cuda)])
    padded = ops.paged_decode_attn(q, x["k_cache"], x["v_cache"], bt, sl, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(padded[:5], base) and torch.all(padded[5:] == 0)


def _subsample_check(x, pick, scale, out):
    pages = x["block_table"][pick].flatten().long()
    kc = x["k_cache"][pages].cpu()
    vc = x["v_cache"][pages].cpu()
    compact_bt = torch.arange(pages.numel(), dtype=torch.int32).view(len(pick), -1)
    ref, _ = orc.paged_decode_attn(x["q"][pick].cpu(), kc, vc, compact_bt, x["seq_lens"][pick],
                                   scale)
    check(out[pick], ref, False)


def test_full_c5_subsample_against_oracle(cuda):
    """C5 at full size: B=16, 64q/8kv GQA-8, ctx 32768 (2 GiB KV per layer), with
    the fused append; 3 requests re-paged for the oracle."""
    shape = CONFIGS["C5"]
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(128)
    pos = x["seq_lens"].long() - 1
    slots = ops.slot_mapping(x["block_table"], pos)
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                k_new=x["k_new"], v_new=x["v_new"], pdl=True,
                                workspace=ops.DecodeWorkspace(16, 64, 8, 128, cuda))
    torch.cuda.synchronize()
    # the appended rows landed in the cache
    kc = x["k_cache"].view(-1, 8, 128)
    for b in (0, 15):
        s = int(slots[b])
        page, off = s // 16, s % 16
        assert torch.equal(x["k_cache"][page, :, off, :], x["k_new"][b])
    _subsample_check(x, [0, 7, 15], scale, out)


def test_max_batch_ragged(cuda):
    """B = 2048 (the per-call limit), ragged short contexts, GQA-4."""
    g = torch.Generator().manual_seed(11)
    ctx = tuple(int(c) for c in torch.randint(1, 200, (2048,), generator=g))
    shape = DecodeShape("maxb", 2048, 16, 4, 128, 1, ctx)
    x, out, lse, ref, ref_lse = run_case(shape, cuda)
    check(out, ref, False)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_lse, atol=1e-3, rtol=1e-4)


def test_bitwise_repeatable_under_dynamic_claims(cuda):
    """Chunks are claimed dynamically (which warp gets which chunk varies from
    run to run), but the chunk grid fixes every piece's slot and the merge
    order: outputs and lse must be bit-identical across repeated calls."""
    shape = DecodeShape("rep", 6, 32, 8, 128, 1, (4096, 333, 2048, 17, 4000, 1024))
    x = make_layer(shape, cuda)
    ws = ops.DecodeWorkspace(shape.batch, 32, 8, 128, cuda)
    outs = []
    for _ in range(5):
        lse = torch.empty(shape.batch, 32, dtype=torch.float32, device=cuda)
        o = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                  x["seq_lens"], lse=lse, scale=0.088, out_dtype=torch.float32,
                                  workspace=ws)
        outs.append((o.clone(), lse.clone()))
    torch.cuda.synchronize()
    for o, l in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(l, outs[0][1])


@pytest.mark.parametrize("grid", ["auto", "dynamic", "static", "split"])
def test_concurrent_calls_on_two_streams(cuda, grid):
    """Two full-device persistent grids running at once (the 1-GPU offload path
    runs local and executor attention concurrently): on the dynamic grid no
    chunk is owned in advance, on the static grid no warp ever waits on
    another, so neither call can wait on warps the other keeps off the SMs."""
    shapes = [DecodeShape("s0", 16, 32, 8, 128, 1, 4096), DecodeShape("s1", 8, 32, 32, 128, 1, 2048)]
    xs = [make_layer(s, cuda, seed=i) for i, s in enumerate(shapes)]
    wss = [ops.DecodeWorkspace(s.batch, s.num_q_heads, s.num_kv_heads, 128, cuda) for s in shapes]
    streams = [torch.cuda.Stream(cuda) for _ in shapes]
    torch.cuda.synchronize()
    outs = [[], []]
    for rep in range(4):
        for i, (x, ws, st) in enumerate(zip(xs, wss, streams)):
            with torch.cuda.stream(st):
                outs[i].append(ops.paged_decode_attn(
                    x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                    scale=0.088, out_dtype=torch.float32, workspace=ws, stream=st, grid=grid))
    torch.cuda.synchronize()
    for i, x in enumerate(xs):
        ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                       x["seq_lens"], 0.088)
        for o in outs[i]:
            check(o, ref, False)
            assert torch.equal(o, outs[i][0])


def test_cross_check_against_trtllm_gen_decode(cuda):
    """Secondary check of the attention semantics (scale, GQA head mapping,
    masking of the last page) against an independent production kernel:
    FlashInfer's TRT-LLM-gen paged decode (same HND page layout). Both the
    oracle and our kernel must agree with it to bf16 output rounding."""
    try:
        import flashinfer
        fn = flashinfer.decode.trtllm_batch_decode_with_kv_cache
    except Exception as exc:  # library absent on this box: the oracle gate still stands
        pytest.skip(f"flashinfer unavailable: {exc!r}")
    shape = DecodeShape("xc", 6, 32, 8, 128, 1, (4096, 333, 2048, 17, 4000, 1))
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(128)
    ws_fi = torch.zeros(128 << 20, dtype=torch.uint8, device=cuda)
    try:
        theirs = fn(x["q"], (x["k_cache"], x["v_cache"]), ws_fi, x["block_table"], x["seq_lens"],
                    int(x["seq_lens"].max()), bmm1_scale=scale, bmm2_scale=1.0, kv_layout="HND")
        torch.cuda.synchronize()
    except Exception as exc:
        pytest.skip(f"trtllm-gen decode not runnable here: {exc!r}")
    ours = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                 x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                 workspace=ops.DecodeWorkspace(6, 32, 8, 128, cuda))
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], scale)
    t = theirs.float().cpu().numpy()
    # theirs is bf16: compare at bf16 resolution (rounding alone is ~1.4e-3 mean-rel)
    assert float(np.abs(t - ref).max()) <= MAX_ABS
    assert mean_rel(t, ref) <= 3e-3
    o = ours.cpu().numpy()
    assert float(np.abs(o - t).max()) <= MAX_ABS
    assert mean_rel(o, t) <= 3e-3


def test_row_maps_match_gathered_call_bitwise(cuda):
    """adr_paged_decode_attn_rows (zero-copy offload): reading q/k_new/v_new rows
    through in_rows and writing out/lse rows through out_rows is bit-identical to
    the plain call on gathered inputs, and leaves every other output row alone."""
    shape = DecodeShape("rows", 5, 32, 8, 128, 1, (700, 16, 4096, 1, 2500))
    x = make_layer(shape, cuda)
    g = torch.Generator(device=cuda).manual_seed(5)
    Bsrc, Bdst = 9, 11
    in_rows = torch.tensor([7, 0, 3, 8, 5], dtype=torch.int32, device=cuda)
    out_rows = torch.tensor([2, 10, 4, 0, 6], dtype=torch.int32, device=cuda)
    rnd = lambda *s: torch.randn(*s, generator=g, device=cuda).to(torch.bfloat16)
    q_src, k_src, v_src = rnd(Bsrc, 32, 128), rnd(Bsrc, 8, 128), rnd(Bsrc, 8, 128)
    idx = in_rows.long()
    kc0, vc0 = x["k_cache"].clone(), x["v_cache"].clone()
    ws = ops.DecodeWorkspace(shape.batch, 32, 8, 128, cuda)
    ref_lse = torch.empty(5, 32, dtype=torch.float32, device=cuda)
    ref = ops.paged_decode_attn(q_src[idx].contiguous(), kc0, vc0, x["block_table"], x["seq_lens"],
                                lse=ref_lse, scale=0.088, out_dtype=torch.float32, workspace=ws,
                                k_new=k_src[idx].contiguous(), v_new=v_src[idx].contiguous())
    out = torch.full((Bdst, 32, 128), 7.0, dtype=torch.float32, device=cuda)
    lse = torch.full((Bdst, 32), 7.0, dtype=torch.float32, device=cuda)
    ops.paged_decode_attn(q_src, x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                          out=out, lse=lse, scale=0.088, out_dtype=torch.float32, workspace=ws,
                          k_new=k_src, v_new=v_src, in_rows=in_rows, out_rows=out_rows)
    torch.cuda.synchronize()
    oi = out_rows.long()
    assert torch.equal(out[oi], ref) and torch.equal(lse[oi], ref_lse)
    rest = torch.ones(Bdst, dtype=torch.bool, device=cuda)
    rest[oi] = False
    assert bool((out[rest] == 7.0).all()) and bool((lse[rest] == 7.0).all())
    assert torch.equal(x["k_cache"], kc0) and torch.equal(x["v_cache"], vc0)  # same appends


@pytest.mark.parametrize("shape", [DecodeShape("s1", 8, 32, 8, 128, 1, 1024),
                                   DecodeShape("s2", 5, 16, 16, 64, 1, (1, 40, 0, 900, 17)),
                                   DecodeShape("s3", 64, 32, 8, 128, 1, 1024)])
@pytest.mark.parametrize("grid", ["static", "split"])
def test_static_grid_matches_oracle_and_leaves_workspace_clean(cuda, shape, grid):
    """Static grid (one chunk per warp, last-arriving warp merges) and split-pair
    CTA kernel (last-arriving CTA merges): oracle parity, bitwise repeatable,
    PDL chain == plain, and every counter back at zero."""
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(shape.head_dim)
    ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                             cuda)
    outs = []
    for pdl in (False, True, True):
        lse = torch.empty(shape.batch, shape.num_q_heads, dtype=torch.float32, device=cuda)
        outs.append((ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                           x["seq_lens"], lse=lse, scale=scale,
                                           out_dtype=torch.float32, workspace=ws, pdl=pdl,
                                           grid=grid), lse))
    torch.cuda.synchronize()
    ref, ref_lse = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                         x["seq_lens"], scale)
    check(outs[0][0], ref, False)
    live = np.asarray(shape.ctx_list()) > 0
    np.testing.assert_allclose(outs[0][1].cpu().numpy()[live], ref_lse[live], atol=1e-3, rtol=1e-4)
    for o, l in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(l, outs[0][1])
    counters = ws.buf[: (1 << 17) * 4 * 2 + 256].view(torch.int32)
    assert int(counters.abs().sum()) == 0


def test_cross_check_against_vllm_paged_attention_v2(cuda):
    """The paper's prototype runs vLLM v0.6.3's decode attention (PAPER.md:163,
    not vendored in the reference): the same batch through vLLM's
    paged_attention_v2 (this image's vLLM; its cache layout converted once) must
    agree with the oracle and with our kernel to bf16 output rounding."""
    try:
        import vllm._custom_ops as vops
    except Exception as exc:  # library absent on this box: the oracle gate still stands
        pytest.skip(f"vllm unavailable: {exc!r}")
    shape = DecodeShape("xv", 5, 32, 8, 128, 1, (4096, 333, 17, 2000, 1))
    x = make_layer(shape, cuda)
    B, Hq, Hkv, D = 5, 32, 8, 128
    scale = 1.0 / math.sqrt(D)
    vk = x["k_cache"].view(-1, Hkv, 16, D // 8, 8).permute(0, 1, 3, 2, 4).contiguous()
    vv = x["v_cache"].permute(0, 1, 3, 2).contiguous()
    max_len = int(x["seq_lens"].max())
    parts = (max_len + 511) // 512
    theirs = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=cuda)
    es = torch.empty(B, Hq, parts, dtype=torch.float32, device=cuda)
    ml = torch.empty_like(es)
    tmp = torch.empty(B, Hq, parts, D, dtype=torch.bfloat16, device=cuda)
    one = torch.ones((), dtype=torch.float32, device=cuda)
    try:
        vops.paged_attention_v2(theirs, es, ml, tmp, x["q"], vk, vv, Hkv, scale, x["block_table"],
                                x["seq_lens"], 16, max_len, None, "auto", one, one)
        torch.cuda.synchronize()
    except Exception as exc:
        pytest.skip(f"vllm paged_attention_v2 not runnable here: {exc!r}")
    ours = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                 x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                 workspace=ops.DecodeWorkspace(B, Hq, Hkv, D, cuda))
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], scale)
    t = theirs.float().cpu().numpy()
    assert float(np.abs(t - ref).max()) <= MAX_ABS
    assert mean_rel(t, ref) <= 3e-3
    o = ours.cpu().numpy()
    assert float(np.abs(o - t).max()) <= MAX_ABS
    assert mean_rel(o, t) <= 3e-3


@pytest.mark.parametrize("shape", [
    DecodeShape("sp1", 1, 32, 8, 128, 1, 64),                        # one pair per kv-head, few pages
    DecodeShape("sp2", 3, 64, 8, 128, 1, (32768, 5, 7000)),           # long pair cut into many items
    DecodeShape("sp3", 40, 32, 32, 128, 1, 2048),                     # more items than CTAs (rounds)
    DecodeShape("sp4", 9, 8, 1, 64, 1, (1, 2, 15, 16, 17, 31, 33, 4095, 0)),  # G=8 D=64 ragged, empty
    DecodeShape("sp5", 200, 16, 2, 128, 1, 33),                      # many short pairs
])
def test_split_kernel_shapes_match_oracle(cuda, shape):
    """The split-pair CTA kernel over item layouts the small-call rule produces
    and ones it does not (multi-round grids, a 32k pair in dozens of items,
    GQA-8 at D=64, empty and 1-token requests): oracle parity with lse, fused
    append bit-exact, repeatable bits, clean counters."""
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(shape.head_dim)
    pos = x["seq_lens"].long() - 1
    live = pos >= 0
    slots = ops.slot_mapping(x["block_table"], pos)
    ref_k, ref_v = orc.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"],
                                 slots.cpu().numpy())
    ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                             cuda, max_blocks_per_seq=shape.max_pages)
    outs = []
    for rep in range(2):
        kc, vc = x["k_cache"].clone(), x["v_cache"].clone()
        lse = torch.empty(shape.batch, shape.num_q_heads, dtype=torch.float32, device=cuda)
        o = ops.paged_decode_attn(x["q"], kc, vc, x["block_table"], x["seq_lens"], lse=lse,
                                  scale=scale, out_dtype=torch.float32, workspace=ws,
                                  k_new=x["k_new"] if bool(live.all()) else None,
                                  v_new=x["v_new"] if bool(live.all()) else None,
                                  grid="split", pdl=rep == 1)
        outs.append((o, lse, kc, vc))
    torch.cuda.synchronize()
    o, lse, kc, vc = outs[0]
    if bool(live.all()):
        assert np.array_equal(kc.cpu().view(torch.int16).numpy().view(np.uint16), ref_k)
        assert np.array_equal(vc.cpu().view(torch.int16).numpy().view(np.uint16), ref_v)
        kref, vref = ref_k, ref_v
    else:
        kref, vref = x["k_cache"], x["v_cache"]
    ref, ref_lse = orc.paged_decode_attn(x["q"], kref, vref, x["block_table"], x["seq_lens"], scale)
    check(o, ref, False)
    lv = np.asarray(shape.ctx_list()) > 0
    np.testing.assert_allclose(lse.cpu().numpy()[lv], ref_lse[lv], atol=1e-3, rtol=1e-4)
    assert bool(torch.isneginf(lse[~torch.from_numpy(lv).to(cuda)]).all())
    assert torch.equal(outs[1][0], o) and torch.equal(outs[1][1], lse)
    counters = ws.buf[: (1 << 17) * 4 * 2 + 256].view(torch.int32)
    assert int(counters.abs().sum()) == 0


@pytest.mark.parametrize("case", ["C1_layer0", "C1_ragged", "C2_mha", "C3_gqa4", "C4_mha40",
                                  "C5_gqa8"])
@pytest.mark.parametrize("grid", ["auto", "dynamic", "split"])
def test_against_committed_library_outputs(cuda, case, grid):
    """Our kernel (fused append from the pre-append cache) on the inputs of
    tests/golden/attn_libraries.npz — the outputs vLLM paged_attention_v2 and
    FlashInfer TRT-LLM-gen produced on a B200 — agrees with both libraries the
    way the libraries agree with each other, and with the fp32 oracle at the
    north-star gate; the appended slots are bit-identical to the oracle's."""
    import sys
    from pathlib import Path
    gold = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(gold))
    import make_attn_golden as mk
    blob = np.load(gold / "attn_libraries.npz")
    (name, shape, seed), = [c for c in mk.CASES if c[0] == case]
    x = mk.inputs(shape, seed)
    assert mk.digest(x) == blob[f"{case}/sha256"].tobytes().hex()
    kc, vc = x["k_cache"].clone(), x["v_cache"].clone()
    for b, n in enumerate(shape.ctx_list()):  # undo the append: the kernel fuses it
        p = n - 1
        page = int(x["block_table"][b, p // 16])
        kc[page, :, p % 16] = 0
        vc[page, :, p % 16] = 0
    g = {k: v.to(cuda) for k, v in x.items()}
    kc, vc = kc.to(cuda), vc.to(cuda)
    ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                             cuda)
    ours = ops.paged_decode_attn(g["q"], kc, vc, g["block_table"], g["seq_lens"],
                                 k_new=g["k_new"], v_new=g["v_new"], out_dtype=torch.float32,
                                 workspace=ws, grid=grid)
    torch.cuda.synchronize()
    assert torch.equal(kc, g["k_cache"]) and torch.equal(vc, g["v_cache"])
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], 1.0 / math.sqrt(shape.head_dim))
    o = ours.cpu().numpy()
    check(ours, ref, False)
    f = lambda k: (blob[f"{case}/{k}"].astype(np.uint32) << 16).view(np.float32).reshape(o.shape)
    v, t = f("vllm_paged_attention_v2"), f("flashinfer_trtllm_gen")
    between = mean_rel(v, t)
    for lib in (v, t):
        assert float(np.abs(o - lib).max()) <= MAX_ABS
        assert mean_rel(lib, o) <= max(3e-3, 1.1 * between)


@pytest.mark.parametrize("shape", [
    DecodeShape("coarse9", 4, 32, 8, 128, 1, 32768),             # ~0.6 chunks per warp: variant 9
    DecodeShape("coarse9r", 3, 64, 8, 128, 1, (32768, 20000, 9)),  # ragged, GQA-8
])
def test_coarse_grid_variants_match_oracle(cuda, shape):
    """Coarse chunk grids launch the fewer, deeper-warp variants (pick_variant:
    < 2 chunks per default warp -> 8 warps x 2 pages; the C5 full-size test covers
    the 8 x 3 one): oracle parity with lse, fused append bit-exact, repeatable bits."""
    x = make_layer(shape, cuda)
    scale = 1.0 / math.sqrt(shape.head_dim)
    kc, vc = x["k_cache"].clone(), x["v_cache"].clone()
    ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                             cuda, max_blocks_per_seq=shape.max_pages)
    lse = torch.empty(shape.batch, shape.num_q_heads, dtype=torch.float32, device=cuda)
    out = ops.paged_decode_attn(x["q"], kc, vc, x["block_table"], x["seq_lens"], lse=lse,
                                scale=scale, out_dtype=torch.float32, workspace=ws,
                                k_new=x["k_new"], v_new=x["v_new"], grid="dynamic")
    again = ops.paged_decode_attn(x["q"], kc, vc, x["block_table"], x["seq_lens"], scale=scale,
                                  out_dtype=torch.float32, workspace=ws, k_new=x["k_new"],
                                  v_new=x["v_new"], grid="dynamic")
    torch.cuda.synchronize()
    assert torch.equal(out, again)
    pos = x["seq_lens"].long() - 1
    slots = orc.slot_mapping(x["block_table"].cpu(), pos.cpu())
    ek, ev = orc.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
    assert np.array_equal(kc.cpu().view(torch.int16).numpy().view(np.uint16), ek)
    assert np.array_equal(vc.cpu().view(torch.int16).numpy().view(np.uint16), ev)
    ref, ref_lse = orc.paged_decode_attn(x["q"], kc, vc, x["block_table"], x["seq_lens"], scale)
    check(out, ref, False)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_lse, atol=1e-3, rtol=1e-4)
