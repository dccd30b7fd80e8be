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


def _load_library_golden():
    import sys
    from pathlib import Path
    gold = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(gold))
    import make_attn_golden as mk
    blob = np.load(gold / "attn_libraries.npz")
    return mk, blob


def _bits_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("case", ["C1_layer0", "C1_layer1", "C1_ragged", "C2_mha", "C3_gqa4",
                                  "C4_mha40", "C5_gqa8"])
def test_oracle_pinned_to_library_outputs(built, case):
    """Pins the attention restatement to the paper prototype's kernel family:
    tests/golden/attn_libraries.npz holds vLLM paged_attention_v2 (vLLM 0.22; the
    PagedAttention v2 algorithm the paper ran as vLLM v0.6.3) and
    FlashInfer TRT-LLM-gen outputs for the same seeded inputs (regenerated here,
    digest-checked), produced on a B200 by tests/golden/make_attn_golden.py.

    Tolerance: the north star's max-abs 2e-2 against the fp32 oracle, and
    mean-rel (sum|lib - oracle| / sum|oracle|) <= 3e-3. The libraries emit bf16:
    rounding a perfect fp32 result to bf16 alone gives ~1.4e-3, and vLLM also
    keeps its 512-token partition outputs in bf16 (measured 0.9-2.9e-3 here;
    TRT-LLM-gen 0.8-2.5e-3; the two libraries differ from each other by 1.0-3.1e-3).

    Append: vLLM's reshape_and_cache must write the appended token to exactly
    the oracle's slot (page = block_table[b][p // 16], offset p % 16). It fills
    only the first 4096 elements of a token (32 kv-heads at D=128): at Llama-2-13B's
    40 kv-heads, heads 32-39 stay unwritten (recorded by the generator; the
    attention outputs above use the correctly appended cache). Rows inside its
    4096-element reach are checked; ours (adr_kv_append / fused append) writes
    every head and is bit-exact against the oracle in the GPU suite."""
    mk, blob = _load_library_golden()
    (name, shape, seed), = [c for c in mk.CASES if c[0] == case]
    x = mk.inputs(shape, seed)
    assert mk.digest(x) == blob[f"{case}/sha256"].tobytes().hex(), "input regeneration drifted"
    out, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], 1.0 / math.sqrt(shape.head_dim))
    for lib in ("vllm_paged_attention_v2", "flashinfer_trtllm_gen"):
        theirs = _bits_to_f32(blob[f"{case}/{lib}"]).reshape(out.shape)
        assert float(np.abs(theirs - out).max()) <= 2e-2, lib
        rel = float(np.abs(theirs - out).sum() / np.abs(out).sum())
        assert rel <= 3e-3, (lib, rel)
    bad = blob[f"{case}/vllm_reshape_and_cache_bad_rows"]
    assert bad.shape == (shape.batch, shape.num_kv_heads)
    reach = 4096 // shape.head_dim
    assert not bad[:, :reach].any()
