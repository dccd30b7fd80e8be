"""Self-checks of the CPU oracle (oracle/attn_oracle.c) before it is trusted as
the parity checker. Attention parity against the reference is unpinned (the
reference has no attention arithmetic), so the oracle is pinned here against an
independent float64 dense restatement and known-answer cases."""
import math

import numpy as np
import pytest
import torch

import oracle as orc
from paper_2503_20552_b200.synthetic import CONFIGS, DecodeShape, make_block_table, make_layer


def _bf16_f64(t):
    return t.float().double().numpy()


def _unpage(cache, bt_row, n):
    # [NB,Hkv,bs,D] -> [n,Hkv,D]
    bs = cache.shape[2]
    rows = [cache[bt_row[t // bs], :, t % bs, :] for t in range(n)]
    return torch.stack(rows, 0)


@pytest.mark.parametrize("cfg", ["C1"])
def test_oracle_matches_dense_fp64(built, cfg):
    shape = CONFIGS[cfg]
    x = make_layer(shape, "cpu")
    scale = 1.0 / math.sqrt(shape.head_dim)
    out, lse = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                     x["seq_lens"], scale)
    for b in range(shape.batch):
        n = int(x["seq_lens"][b])
        k = _unpage(x["k_cache"], x["block_table"][b], n)
        v = _unpage(x["v_cache"], x["block_table"][b], n)
        ref = orc.dense_attention_fp64(_bf16_f64(x["q"][b]), _bf16_f64(k), _bf16_f64(v), scale)
        np.testing.assert_allclose(out[b], ref, rtol=1e-5, atol=1e-6)


def test_oracle_known_answers(built):
    # identical keys -> uniform softmax -> mean of V; lse = s + log(n)
    Hq, Hkv, D, n = 4, 2, 64, 37
    shape = DecodeShape("kat", 1, Hq, Hkv, D, 1, n)
    bt = make_block_table(shape)
    NB = shape.num_pages
    k = torch.zeros(NB, Hkv, 16, D, dtype=torch.bfloat16)
    k[..., 0] = 1.0
    v = torch.randn(NB, Hkv, 16, D).to(torch.bfloat16)
    q = torch.ones(1, Hq, D, dtype=torch.bfloat16)
    out, lse = orc.paged_decode_attn(q, k, v, bt, torch.tensor([n], dtype=torch.int32), 0.5)
    vv = _unpage(v, bt[0], n).double()
    for h in range(Hq):
        np.testing.assert_allclose(out[0, h], vv[:, h // (Hq // Hkv)].mean(0).numpy(), rtol=1e-5,
                                   atol=1e-6)
        assert lse[0, h] == pytest.approx(0.5 + math.log(n), rel=1e-6)


def test_oracle_empty_request(built):
    shape = DecodeShape("empty", 2, 2, 2, 64, 1, (0, 20))
    x = make_layer(shape, "cpu")
    out, lse = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                     x["seq_lens"], 0.125)
    assert np.all(out[0] == 0) and np.all(np.isneginf(lse[0]))
    assert np.all(np.isfinite(out[1]))


def test_oracle_kv_append_and_slots(built):
    shape = DecodeShape("app", 3, 4, 2, 64, 1, (5, 16, 33))
    x = make_layer(shape, "cpu")
    pos = np.array([4, 15, -1])
    slots = orc.slot_mapping(x["block_table"], pos)
    bt = x["block_table"].numpy()
    assert slots[0] == bt[0, 0] * 16 + 4 and slots[1] == bt[1, 0] * 16 + 15 and slots[2] == -1
    kc, vc = orc.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
    kn = x["k_new"].view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(kc[bt[0, 0], :, 4, :], kn[0])
    assert np.array_equal(kc[bt[1, 0], :, 15, :], kn[1])
    # untouched rows unchanged
    ko = x["k_cache"].view(torch.int16).numpy().view(np.uint16)
    mask = np.ones(kc.shape[0], bool)
    mask[[bt[0, 0], bt[1, 0]]] = False
    assert np.array_equal(kc[mask], ko[mask])


def test_oracle_threads_deterministic(built):
    shape = CONFIGS["C1"]
    x = make_layer(shape, "cpu")
    a, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                 x["seq_lens"], 0.125, num_threads=1)
    b, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                 x["seq_lens"], 0.125, num_threads=0)
    assert np.array_equal(a, b)
