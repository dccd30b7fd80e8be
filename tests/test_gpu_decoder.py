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
