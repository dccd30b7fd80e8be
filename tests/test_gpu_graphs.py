"""CUDA-graph capture of decode steps: replay is bit-identical to eager
execution, and the 2-D grid pads steps to captured shapes correctly."""
import math
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))

import numpy as np
import pytest
import torch

from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.graphs import build_grid
from paper_2503_20552_b200.runtime import CapturedStep, DecodeGraphCache
from paper_2503_20552_b200.synthetic import DecodeShape, make_block_table, make_layer

pytestmark = pytest.mark.gpu


def test_captured_local_step_matches_eager(cuda):
    shape = DecodeShape("g", 16, 32, 8, 128, 4, (100, 2000, 17, 900) * 4)
    bt = make_block_table(shape)
    layers = [make_layer(shape, cuda, seed=l, block_table=bt) for l in range(shape.num_layers)]
    slots = ops.slot_mapping(layers[0]["block_table"], layers[0]["seq_lens"].long() - 1)
    ws = ops.DecodeWorkspace(shape.batch, 32, 8, 128, cuda)
    outs = [torch.empty(shape.batch, 32, 128, dtype=torch.bfloat16, device=cuda) for _ in layers]

    def step():
        for x, o in zip(layers, outs):
            ops.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
            ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                  x["seq_lens"], out=o, workspace=ws)

    step()
    torch.cuda.synchronize()
    eager = [o.clone() for o in outs]
    cap = CapturedStep(step)
    for o in outs:
        o.zero_()
    cap.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, outs):
        assert torch.equal(a, b)
    # new inputs flow through the same graph
    for x in layers:
        x["q"].mul_(-1)
    cap.replay()
    step_ref = [o.clone() for o in outs]
    step()
    torch.cuda.synchronize()
    for a, b in zip(step_ref, outs):
        assert torch.equal(a, b)


def test_graph_grid_padding(cuda):
    Hq, Hkv, D, L = 8, 2, 64, 2
    grid = build_grid(4, 12, 0, 8)   # decode caps (4, 8, 12), offload axis off
    full = DecodeShape("pool", 12, Hq, Hkv, D, L, 300)
    bt_all = make_block_table(full)
    data = [make_layer(full, cuda, seed=l, block_table=bt_all) for l in range(L)]
    scale = 1 / math.sqrt(D)

    def make(cd, co):
        inp = {"q": [torch.zeros(cd, Hq, D, dtype=torch.bfloat16, device=cuda) for _ in range(L)],
               "bt": torch.zeros(cd, bt_all.shape[1], dtype=torch.int32, device=cuda),
               "seq": torch.zeros(cd, dtype=torch.int32, device=cuda),
               "out": [torch.empty(cd, Hq, D, dtype=torch.bfloat16, device=cuda) for _ in range(L)],
               "ws": ops.DecodeWorkspace(cd, Hq, Hkv, D, cuda)}

        def fn():
            for l in range(L):
                ops.paged_decode_attn(inp["q"][l], data[l]["k_cache"], data[l]["v_cache"], inp["bt"],
                                      inp["seq"], out=inp["out"][l], scale=scale, workspace=inp["ws"])
        return inp, fn

    cache = DecodeGraphCache(grid, make)
    for bd in (3, 4, 7, 12, 5):
        def fill(inp, shape, bd=bd):
            n = shape[0]
            for l in range(L):
                inp["q"][l].zero_()
                inp["q"][l][:bd].copy_(data[l]["q"][:bd])
            inp["bt"].zero_()
            inp["bt"][:bd].copy_(data[0]["block_table"][:bd])
            inp["seq"].zero_()
            inp["seq"][:bd].copy_(data[0]["seq_lens"][:bd])
        shape = cache.run(bd, 0, fill)
        assert shape == (-(-bd // 4) * 4, 0)
        inp = cache.graphs[shape][0]
        torch.cuda.synchronize()
        for l in range(L):
            ref = ops.paged_decode_attn(data[l]["q"][:bd].contiguous(), data[l]["k_cache"], data[l]["v_cache"],
                                        data[l]["block_table"][:bd].contiguous(),
                                        data[l]["seq_lens"][:bd].contiguous(), scale=scale,
                                        workspace=ops.DecodeWorkspace(bd, Hq, Hkv, D, cuda))
            torch.cuda.synchronize()
            assert torch.equal(inp["out"][l][:bd], ref)
            assert torch.all(inp["out"][l][bd:] == 0)  # padding rows are empty
    assert cache.graphed_steps == 5 and len(cache.graphs) == 3


def test_captured_offloaded_step_matches_eager(cuda):
    """The full offloaded step (exchange + executor streams) is graph-capturable:
    one replay gives the eager step's bits."""
    from test_gpu_runtime import build_step
    step, plan, qs, ks, vs, outs, before, kvs = build_step(cuda, [300, 17, 1024], [900, 33, 2000])
    step.timing = False
    k0, v0 = [t.clone() for t in (kvs[0].k, kvs[0].v)], [t.clone() for t in (kvs[1].k, kvs[1].v)]
    step.run(qs, ks, vs, plan, outs)
    torch.cuda.synchronize()
    eager = [o.clone() for o in outs]
    # restore the caches (the step appended into them) and capture
    kvs[0].k.copy_(k0[0]); kvs[0].v.copy_(k0[1]); kvs[1].k.copy_(v0[0]); kvs[1].v.copy_(v0[1])
    cap = CapturedStep(lambda: step.run(qs, ks, vs, plan, outs), warmup=1)
    kvs[0].k.copy_(k0[0]); kvs[0].v.copy_(k0[1]); kvs[1].k.copy_(v0[0]); kvs[1].v.copy_(v0[1])
    for o in outs:
        o.zero_()
    cap.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, outs):
        assert torch.equal(a, b)
