"""Full decode layers (decoder.SyntheticDecoder): the attention inside a layer is
the product kernel on the layer's own projections — checked against the oracle
— and a CUDA-graph replay of the whole step is bit-identical to eager."""
import math

import numpy as np
import pytest
import torch

import oracle as orc
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.decoder import LayerDims, SyntheticDecoder
from paper_2503_20552_b200.runtime import CapturedStep
from paper_2503_20552_b200.synthetic import DecodeShape, make_block_table, make_layer

pytestmark = pytest.mark.gpu

DIMS = LayerDims(hidden=256, intermediate=512, num_q_heads=8, num_kv_heads=2, head_dim=64)
SHAPE = DecodeShape("dec", 8, 8, 2, 64, 2, (1, 15, 16, 17, 100, 260, 513, 47), spare_pages=4)


def build(cuda):
    bt = make_block_table(SHAPE)
    layers = [make_layer(SHAPE, cuda, seed=l, block_table=bt) for l in range(SHAPE.num_layers)]
    kv = [(x["k_cache"], x["v_cache"]) for x in layers]
    dec = SyntheticDecoder(DIMS, kv, SHAPE.batch, cuda, seed=5)
    g = torch.Generator(device=cuda).manual_seed(9)
    x = torch.randn(SHAPE.batch, DIMS.hidden, generator=g, device=cuda).to(torch.bfloat16)
    return dec, layers, x


def u16(t):
    return t.cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def test_layer_attention_matches_oracle(cuda):
    dec, layers, x = build(cuda)
    bt, seq = layers[0]["block_table"], layers[0]["seq_lens"]
    k0, v0 = u16(layers[0]["k_cache"]), u16(layers[0]["v_cache"])
    dec.layer(0, x, bt, seq)
    torch.cuda.synchronize()
    # the layer's own k/v projections were appended at position seq_len - 1
    slots = ops.slot_mapping(bt, seq.to(torch.int64) - 1).cpu().numpy()
    ref_k, ref_v = orc.kv_append(dec.k, dec.v, k0, v0, slots)
    assert np.array_equal(u16(layers[0]["k_cache"]), ref_k)
    assert np.array_equal(u16(layers[0]["v_cache"]), ref_v)
    # and the attention output is the oracle's on the layer's q (bf16-rounded gate)
    ref, _ = orc.paged_decode_attn(dec.q, ref_k, ref_v, bt, seq, 1.0 / math.sqrt(DIMS.head_dim))
    ref_bf = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
    got = dec.attn.float().cpu().numpy()
    assert np.abs(got - ref_bf).max() <= 2e-2
    assert np.abs(got - ref_bf).sum() / np.abs(ref_bf).sum() <= 1e-3
    assert bool(torch.isfinite(x).all())


@pytest.mark.parametrize("pdl", [False, True])
def test_graph_replay_matches_eager(cuda, pdl):
    dec, layers, x0 = build(cuda)
    bt, seq = layers[0]["block_table"], layers[0]["seq_lens"]
    x = x0.clone()
    dec.step(x, bt, seq)
    torch.cuda.synchronize()
    eager = x.clone()
    xs = x0.clone()

    def step():
        xs.copy_(x0)
        dec.step(xs, bt, seq, pdl=pdl)
    graph = CapturedStep(step)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(xs, eager)
    assert bool(torch.isfinite(eager).all())


# ---- full layers with attention offloading (decoder.OffloadedDecoder) -----------

N_LOCAL = 5


def build_offloaded(cuda, mha=False, nonattn=True):
    from paper_2503_20552_b200.decoder import OffloadedDecoder
    dims = LayerDims(256, 512, 4, 4, 64) if mha else DIMS
    shape = DecodeShape("odec", 8, dims.num_q_heads, dims.num_kv_heads, 64, 2,
                        (1, 15, 16, 17, 100, 260, 513, 47), spare_pages=4)
    bt = make_block_table(shape)
    layers = [make_layer(shape, cuda, seed=l, block_table=bt) for l in range(shape.num_layers)]
    kv = [(x["k_cache"], x["v_cache"]) for x in layers]
    # the executor holds its own caches (same page ids for simplicity, separate memory)
    exec_kv = [(x["k_cache"].clone(), x["v_cache"].clone()) for x in layers]
    dec = OffloadedDecoder(dims, kv, exec_kv, shape.batch, N_LOCAL, cuda, seed=5, nonattn=nonattn)
    g = torch.Generator(device=cuda).manual_seed(9)
    x = torch.randn(shape.batch, dims.hidden, generator=g, device=cuda).to(torch.bfloat16)
    b, s = layers[0]["block_table"], layers[0]["seq_lens"]
    tabs = (b[:N_LOCAL].contiguous(), s[:N_LOCAL].contiguous(), b[N_LOCAL:].contiguous(),
            s[N_LOCAL:].contiguous())
    return dec, layers, exec_kv, x, tabs, dims


@pytest.mark.parametrize("mha,nonattn", [(False, True), (True, True), (False, False)])
def test_offloaded_layer_attention_matches_oracle(cuda, mha, nonattn):
    """Local rows attend over the decoder's caches, offloaded rows over the
    executor's (zero-copy row maps into the decoder's QKV output / attention
    buffer): every row matches the oracle and each cache received exactly its
    own rows' appends. nonattn=False: the attention-only layers of the C5
    capacity run (fixed random q / k / v rows, no GEMMs)."""
    dec, layers, exec_kv, x, tabs, dims = build_offloaded(cuda, mha, nonattn)
    assert dec.weight_bytes() == (dims.weight_bytes_per_layer() * 2 if nonattn else 0)
    bt, seq = layers[0]["block_table"], layers[0]["seq_lens"]
    k0, v0 = u16(layers[0]["k_cache"]), u16(layers[0]["v_cache"])
    dec._exec_tables = (tabs[2], tabs[3])
    dec.layer(0, x, tabs[0], tabs[1])
    torch.cuda.synchronize()
    q = dec.q[dec.rows.long()] if mha else dec.q
    k = dec.k[dec.rows.long()] if mha else dec.k
    v = dec.v[dec.rows.long()] if mha else dec.v
    slots = ops.slot_mapping(bt, seq.to(torch.int64) - 1).cpu().numpy()
    loc, off = slice(0, N_LOCAL), slice(N_LOCAL, 8)
    ref_lk, ref_lv = orc.kv_append(k[loc], v[loc], k0, v0, slots[loc])
    ref_xk, ref_xv = orc.kv_append(k[off], v[off], k0, v0, slots[off])
    assert np.array_equal(u16(layers[0]["k_cache"]), ref_lk)
    assert np.array_equal(u16(layers[0]["v_cache"]), ref_lv)
    assert np.array_equal(u16(exec_kv[0][0]), ref_xk)
    assert np.array_equal(u16(exec_kv[0][1]), ref_xv)
    all_k, all_v = orc.kv_append(k, v, k0, v0, slots)
    ref, _ = orc.paged_decode_attn(q, all_k, all_v, bt, seq, 1.0 / math.sqrt(64))
    ref_bf = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
    got = dec.attn.float().cpu().numpy()
    assert np.abs(got - ref).max() <= 2e-2
    assert np.abs(got - ref_bf).sum() / np.abs(ref_bf).sum() <= 1e-3


@pytest.mark.parametrize("pdl", [False, True])
def test_offloaded_step_graph_replay_matches_eager(cuda, pdl):
    """The whole offloaded step (both streams, every layer) captures into one
    CUDA graph whose replay is bit-identical to eager execution."""
    dec, layers, exec_kv, x0, tabs, _ = build_offloaded(cuda)
    x = x0.clone()
    dec.step(x, *tabs)
    torch.cuda.synchronize()
    eager = x.clone()
    xs = x0.clone()

    def step():
        xs.copy_(x0)
        dec.step(xs, *tabs, pdl=pdl)
    graph = CapturedStep(step)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(xs, eager)
    assert bool(torch.isfinite(eager).all())
