"""Golden decode-attention outputs from the paper prototype's kernel family.

Run on a GPU box (the libraries need one):  python tests/golden/make_attn_golden.py [OUT]
Writes tests/golden/attn_libraries.npz, read by tests/test_oracle_cpu.py on CPU.

Why: the reference (adrenaline_sim) has no attention arithmetic — it only prices
attention (costs.py:73-80) — so the oracle's attention restatement
(oracle/attn_oracle.c) cannot be pinned to the reference. The paper's prototype
runs the attention on vLLM v0.6.3, a dependency that is not
vendored or pinned in /root/reference. This script pins the oracle to that
kernel family instead: the same seeded inputs go through
  * vLLM ``paged_attention_v2`` (this image: vLLM 0.22, the PagedAttention v2
    algorithm of v0.6.3: partitioned softmax over 512-token partitions + a
    max/exp-sum reduction), its cache layout converted once, and
  * vLLM ``reshape_and_cache`` for the appended token (the slot convention
    slot = block_table[b][p // 16] * 16 + p % 16),
  * FlashInfer ``trtllm_batch_decode_with_kv_cache`` (NVIDIA TRT-LLM-gen
    cubins, HND layout = ours) as a second, independent implementation,
and their bf16 outputs are committed. The inputs are NOT committed: they are
regenerated on CPU from the seeds (``synthetic.make_layer(shape, "cpu", seed)``,
torch's CPU generator), and a SHA-256 of the input bytes is stored so a test
notices if regeneration ever drifts.

Cases cover every BASELINE config's head geometry at small batch, with ragged
lengths (1 token, partial last pages, > 512-token partitions):
C1 (8q/2kv D64, both layers), C2/C4 MHA (32x128, 40x128), C3 GQA-4, C5 GQA-8.
"""
from __future__ import annotations

import hashlib
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2503_20552_b200.synthetic import DecodeShape, make_layer  # noqa: E402

OUT = Path(__file__).resolve().parent / "attn_libraries.npz"

# (case name, shape, data seed). ctx = tokens after this step's append.
CASES = [
    ("C1_layer0", DecodeShape("C1-tiny", 8, 8, 2, 64, 2, 512), 0),
    ("C1_layer1", DecodeShape("C1-tiny", 8, 8, 2, 64, 2, 512), 1),
    ("C1_ragged", DecodeShape("C1r", 6, 8, 2, 64, 1, (512, 1, 17, 300, 16, 513)), 2),
    ("C2_mha", DecodeShape("C2s", 3, 32, 32, 128, 1, (4096, 1000, 33)), 3),
    ("C3_gqa4", DecodeShape("C3s", 5, 32, 8, 128, 1, (4096, 333, 17, 2000, 1)), 4),
    ("C4_mha40", DecodeShape("C4s", 3, 40, 40, 128, 1, (1100, 777, 16)), 5),
    ("C5_gqa8", DecodeShape("C5s", 2, 64, 8, 128, 1, (5000, 65)), 6),
]


def inputs(shape: DecodeShape, seed: int) -> dict:
    """CPU inputs with this step's token appended at position seq_len - 1."""
    x = make_layer(shape, "cpu", seed=seed)
    for b, n in enumerate(shape.ctx_list()):
        if n <= 0:
            continue
        p = n - 1
        page = int(x["block_table"][b, p // shape.block_size])
        x["k_cache"][page, :, p % shape.block_size] = x["k_new"][b]
        x["v_cache"][page, :, p % shape.block_size] = x["v_new"][b]
    return x


def digest(x: dict) -> str:
    h = hashlib.sha256()
    for key in ("q", "k_new", "v_new", "k_cache", "v_cache", "block_table", "seq_lens"):
        h.update(x[key].contiguous().view(torch.uint8).numpy().tobytes())
    return h.hexdigest()


def bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def run_vllm(shape: DecodeShape, x: dict, dev) -> tuple[np.ndarray, np.ndarray]:
    import vllm._custom_ops as vops
    B, Hq, Hkv, D = shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
    bs = shape.block_size
    g = {k: v.to(dev) for k, v in x.items()}
    # vLLM layouts: key [NB, Hkv, D/8, bs, 8], value [NB, Hkv, D, bs]
    vk = g["k_cache"].view(-1, Hkv, bs, D // 8, 8).permute(0, 1, 3, 2, 4).contiguous()
    vv = g["v_cache"].permute(0, 1, 3, 2).contiguous()
    one = torch.ones((), dtype=torch.float32, device=dev)
    # append check on a copy: zero the appended slots, let reshape_and_cache write
    # them back from k_new / v_new through the slot mapping; the (request, kv-head)
    # rows it did not reproduce are recorded. Attention then runs on the correctly
    # appended cache, so a library append quirk cannot leak into the outputs.
    sl = [n - 1 for n in shape.ctx_list()]
    slots = torch.tensor([int(x["block_table"][b, p // bs]) * bs + p % bs if p >= 0 else -1
                          for b, p in enumerate(sl)], dtype=torch.int64, device=dev)
    ak, av = vk.clone(), vv.clone()
    for b, p in enumerate(sl):
        if p >= 0:
            page, off = int(x["block_table"][b, p // bs]), p % bs
            ak[page, :, :, off, :] = 0
            av[page, :, :, off] = 0
    vops.reshape_and_cache(g["k_new"], g["v_new"], ak, av, slots, "auto", one, one)
    torch.cuda.synchronize()
    bad = np.zeros((B, Hkv), dtype=bool)
    for b, p in enumerate(sl):
        if p >= 0:
            page, off = int(x["block_table"][b, p // bs]), p % bs
            for h in range(Hkv):
                bad[b, h] = not (torch.equal(ak[page, h, :, off, :], vk[page, h, :, off, :])
                                 and torch.equal(av[page, h, :, off], vv[page, h, :, off]))
    max_len = int(g["seq_lens"].max())
    parts = (max_len + 511) // 512
    out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev)
    es = torch.empty(B, Hq, parts, dtype=torch.float32, device=dev)
    ml = torch.empty_like(es)
    tmp = torch.empty(B, Hq, parts, D, dtype=torch.bfloat16, device=dev)
    vops.paged_attention_v2(out, es, ml, tmp, g["q"], vk, vv, Hkv, 1.0 / math.sqrt(D),
                            g["block_table"], g["seq_lens"], bs, max_len, None, "auto", one, one)
    torch.cuda.synchronize()
    return bits(out), bad


def run_trtllm(shape: DecodeShape, x: dict, dev) -> np.ndarray:
    import flashinfer
    B, Hq, D = shape.batch, shape.num_q_heads, shape.head_dim
    g = {k: v.to(dev) for k, v in x.items()}
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev)
    flashinfer.decode.trtllm_batch_decode_with_kv_cache(
        g["q"], (g["k_cache"], g["v_cache"]), ws, g["block_table"], g["seq_lens"],
        int(g["seq_lens"].max()), bmm1_scale=1.0 / math.sqrt(D), bmm2_scale=1.0, out=out,
        kv_layout="HND")
    torch.cuda.synchronize()
    return bits(out)


def main() -> None:
    dev = torch.device("cuda:0")
    blob: dict[str, np.ndarray] = {}
    meta = []
    for name, shape, seed in CASES:
        x = inputs(shape, seed)
        blob[f"{name}/sha256"] = np.frombuffer(bytes.fromhex(digest(x)), dtype=np.uint8)
        try:
            o, bad = run_vllm(shape, x, dev)
            blob[f"{name}/vllm_paged_attention_v2"] = o
            blob[f"{name}/vllm_reshape_and_cache_bad_rows"] = bad
            rows = np.argwhere(bad).tolist()
            meta.append(f"{name}: vllm ok, append " + ("bit-exact" if not rows else
                        f"rows not reproduced (request, kv-head): {rows}"))
        except Exception as exc:  # noqa: BLE001 — record which library could not run
            meta.append(f"{name}: vllm unavailable: {exc!r}"[:200])
        try:
            blob[f"{name}/flashinfer_trtllm_gen"] = run_trtllm(shape, x, dev)
            meta.append(f"{name}: trtllm-gen ok")
        except Exception as exc:  # noqa: BLE001 — e.g. head_dim 64 has no cubin
            meta.append(f"{name}: trtllm-gen unavailable: {exc!r}"[:200])
    import vllm
    versions = f"torch {torch.__version__}; vllm {vllm.__version__}"
    try:
        import flashinfer
        versions += f"; flashinfer {flashinfer.__version__}"
    except Exception:  # noqa: BLE001
        pass
    blob["versions"] = np.frombuffer(versions.encode(), dtype=np.uint8)
    blob["log"] = np.frombuffer("\n".join(meta).encode(), dtype=np.uint8)
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else OUT
    np.savez_compressed(out, **blob)
    print(versions)
    print("\n".join(meta))
    print("wrote", out)


if __name__ == "__main__":
    main()
