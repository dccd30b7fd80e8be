"""Python front end of the CPU oracle (oracle/attn_oracle.c + numpy restatements).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm as the checker. The product package
never imports this module.

Attention parity is UNPINNED against the reference (it has no attention
arithmetic; costs.py:73-80 only prices it) — see the header of attn_oracle.c.
It is pinned instead to the paper prototype's kernel family: committed vLLM
paged_attention_v2 / reshape_and_cache and FlashInfer TRT-LLM-gen outputs on
seeded inputs (tests/golden/attn_libraries.npz, tests/golden/make_attn_golden.py),
checked by tests/test_oracle_cpu.py::test_oracle_pinned_to_library_outputs.
The byte/index restatements below follow the reference's token accounting
(engine.py:331, 416-421) and the paged-slot convention of include/adrenaline.h.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            import sys
            sys.path.insert(0, str(HERE.parent))
            from paper_2503_20552_b200._build import build_oracle
            build_oracle()
        lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        i32 = ctypes.c_int
        lib.oracle_paged_decode_attn.restype = i32
        lib.oracle_paged_decode_attn.argtypes = [P, P, P, P, P, P, P, i32, i32, i32, i32, i32, i32,
                                                 ctypes.c_float, i32]
        lib.oracle_kv_append.restype = i32
        lib.oracle_kv_append.argtypes = [P, P, P, P, P, i32, i32, i32, i32, ctypes.c_longlong]
        lib.oracle_max_threads.restype = i32
        _lib = lib
    return _lib


def _u16(a) -> np.ndarray:
    """bf16 torch tensor / uint16 array -> contiguous uint16 numpy view."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(a, dtype=np.uint16)


def _np(a, dtype) -> np.ndarray:
    try:
        import torch
        if isinstance(a, torch.Tensor):
            a = a.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(a, dtype=dtype)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def paged_decode_attn(q, k_cache, v_cache, block_table, seq_lens, scale: float,
                      num_threads: int = 0):
    """fp32 (double-accumulated) decode attention. Returns (out [B,Hq,D] f32, lse [B,Hq] f32)."""
    qn = _u16(q)
    kc = _u16(k_cache)
    vc = _u16(v_cache)
    bt = _np(block_table, np.int32)
    sl = _np(seq_lens, np.int32)
    B, Hq, D = qn.shape
    _, Hkv, bs, _ = kc.shape
    out = np.zeros((B, Hq, D), dtype=np.float32)
    lse = np.zeros((B, Hq), dtype=np.float32)
    rc = _load().oracle_paged_decode_attn(
        qn.ctypes.data, kc.ctypes.data, vc.ctypes.data, bt.ctypes.data, sl.ctypes.data,
        out.ctypes.data, lse.ctypes.data, B, Hq, Hkv, D, bs, bt.shape[1], float(scale), num_threads)
    if rc != 0:
        raise ValueError("oracle_paged_decode_attn: invalid arguments")
    return out, lse


def kv_append(k_new, v_new, k_cache, v_cache, slots):
    """Returns new (k_cache, v_cache) uint16 arrays with the rows scattered in."""
    kn, vn = _u16(k_new), _u16(v_new)
    kc, vc = _u16(k_cache).copy(), _u16(v_cache).copy()
    sl = _np(slots, np.int64)
    B, Hkv, D = kn.shape
    NB, _, bs, _ = kc.shape
    rc = _load().oracle_kv_append(kn.ctypes.data, vn.ctypes.data, kc.ctypes.data, vc.ctypes.data,
                                  sl.ctypes.data, B, Hkv, D, bs, NB)
    if rc < 0:
        raise ValueError("oracle_kv_append: invalid arguments")
    return kc, vc


def slot_mapping(block_table, positions, block_size: int = 16) -> np.ndarray:
    """slot[b] = bt[b, p // bs] * bs + p % bs (int64), -1 for p < 0."""
    bt = _np(block_table, np.int64)
    pos = _np(positions, np.int64)
    out = np.full(pos.shape, -1, dtype=np.int64)
    for b, p in enumerate(pos):
        if p >= 0:
            out[b] = bt[b, p // block_size] * block_size + p % block_size
    return out


def pack_qkv(q, k, v, rows) -> np.ndarray:
    """Message rows [ q[r] | k[r] | v[r] ] as uint16 (bf16 bits)."""
    qn, kn, vn = _u16(q), _u16(k), _u16(v)
    r = _np(rows, np.int64)
    return np.concatenate([qn[r].reshape(len(r), -1), kn[r].reshape(len(r), -1),
                           vn[r].reshape(len(r), -1)], axis=1)


def scatter_out(src, rows, out) -> np.ndarray:
    o = _u16(out).copy()
    s = _u16(src)
    r = _np(rows, np.int64)
    o[r] = s.reshape((len(r),) + o.shape[1:])
    return o


def dense_attention_fp64(q, k, v, scale: float) -> np.ndarray:
    """Unpaged float64 reference for small self-checks: q [Hq,D], k/v [T,Hkv,D]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    Hq, D = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    out = np.zeros((Hq, D))
    for h in range(Hq):
        s = k[:, h // G, :] @ q[h] * scale
        p = np.exp(s - s.max())
        out[h] = (p / p.sum()) @ v[:, h // G, :]
    return out
