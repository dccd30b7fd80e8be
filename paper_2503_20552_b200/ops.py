"""Torch-tensor front end of the sm_100a kernels (thin; all work is in CUDA).

Each function validates dtypes/shapes/devices, takes pointers with
``data_ptr()`` and launches on ``torch.cuda.current_stream()`` (or an explicit
stream), so the calls compose with torch streams, events and CUDA graphs.
"""
from __future__ import annotations

import contextlib
import math

import torch

from . import _ffi
from ._ffi import ADR_DTYPE_BF16, ADR_DTYPE_F32

PAGE = 16  # tokens per KV page (block_size)

__all__ = [
    "PAGE", "DecodeWorkspace", "paged_decode_attn", "kv_append", "pack_qkv", "unpack_qkv",
    "scatter_out", "slot_mapping", "device_info", "kv_transfer", "check_decode_tables",
    "decode_status",
]


def _stream_ptr(stream: torch.cuda.Stream | None, device: torch.device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _on_device(device: torch.device):
    """Make ``device`` current for the C call (the C entry points launch on the
    current device; a kernel cannot be launched into another device's stream)."""
    if device.index is None or torch.cuda.current_device() == device.index:
        return contextlib.nullcontext()
    return torch.cuda.device(device)


def _require(t: torch.Tensor, name: str, dtype: torch.dtype, ndim: int | None = None) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def device_info(device: int = 0) -> dict:
    sms, major, minor = (_ffi.ctypes.c_int32() for _ in range(3))
    _ffi.call("adr_device_info", device, _ffi.ctypes.byref(sms), _ffi.ctypes.byref(major),
              _ffi.ctypes.byref(minor))
    return {"num_sms": sms.value, "cc": (major.value, minor.value)}


class DecodeWorkspace:
    """Caller-owned scratch for adr_paged_decode_attn (split-pair partials).

    Sized once for the largest batch it will serve (and, with
    ``max_blocks_per_seq``, the widest block table: the partial slots then scale
    with the batch instead of the device's whole grid); reusing it across layers
    and steps keeps the call allocation-free (and so CUDA-graph capturable).
    Every decode call must be given one (no hidden allocation per call).
    """

    def __init__(self, max_batch: int, Hq: int, Hkv: int, D: int, device: torch.device,
                 num_workers: int = 0, max_blocks_per_seq: int = 0) -> None:
        device = torch.device(device)
        with _on_device(device):
            nbytes = _ffi.lib().adr_decode_workspace_size(max_batch, Hq, Hkv, D,
                                                          max_blocks_per_seq, num_workers)
        if nbytes == 0:
            raise _ffi.AdrError("adr_decode_workspace_size", _ffi.ADR_ERR_INVALID,
                                f"bad shape B={max_batch} Hq={Hq} Hkv={Hkv} D={D}")
        self.max_batch = max_batch
        self.max_blocks_per_seq = max_blocks_per_seq
        self.num_workers = num_workers
        self.device = device
        # zero-filled once: the kernel keeps its split-pair counters at zero between calls
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)


_GRID_FLAGS = {"auto": 0, "dynamic": 2, "static": 4, "split": 8}  # _ffi.ADR_DECODE_GRID_*


def paged_decode_attn(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                      block_table: torch.Tensor, seq_lens: torch.Tensor, *,
                      out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                      scale: float | None = None, out_dtype: torch.dtype = torch.bfloat16,
                      workspace: DecodeWorkspace | None = None,
                      stream: torch.cuda.Stream | None = None,
                      num_sms: int = 0, k_new: torch.Tensor | None = None,
                      v_new: torch.Tensor | None = None, pdl: bool = False,
                      grid: str = "auto",
                      in_rows: torch.Tensor | None = None,
                      out_rows: torch.Tensor | None = None,
                      check_tables: bool = False) -> torch.Tensor:
    """Decode attention of q [B,Hq,D] over paged K/V [NB,Hkv,16,D] (bf16).

    Returns ``out`` [B,Hq,D] (bf16, or fp32 with ``out_dtype=torch.float32``).
    ``lse`` [B,Hq] fp32 receives the natural-log log-sum-exp when given.
    ``num_sms`` > 0 confines the persistent grid to an SM partition of that size
    (pass the partition's stream); the workspace's ``num_workers`` is a testing knob.
    ``k_new``/``v_new`` [B,Hkv,D]: fused append of each request's token at
    position seq_lens-1 (written into the caches and attended in the same pass).
    ``grid``: work split, "auto" (default), "dynamic", "static" or "split" (testing /
    tuning; see ADR_DECODE_GRID_* in include/adrenaline.h).
    ``pdl``: programmatic dependent launch (see include/adrenaline.h for the
    contract on what the preceding kernel may write).
    ``in_rows`` / ``out_rows`` [B] int32 (zero-copy offload): request b reads
    q / k_new / v_new row ``in_rows[b]`` and writes out / lse row
    ``out_rows[b]``; q, k_new, v_new, out and lse may then live on a peer GPU
    (peer access enabled) — B is the block table's batch, the launch device and
    stream are the cache's.
    ``workspace`` is required (``DecodeWorkspace``; see its docstring).
    ``check_tables``: validate block_table / seq_lens first (synchronises the
    stream; raises ``AdrError`` with ADR_ERR_INVALID on a page outside the
    cache or a seq_len past the table row). Without it bad entries are still
    never dereferenced (see ``decode_status``).
    """
    _require(q, "q", torch.bfloat16, 3)
    _require(k_cache, "k_cache", torch.bfloat16, 4)
    _require(v_cache, "v_cache", torch.bfloat16, 4)
    _require(block_table, "block_table", torch.int32, 2)
    _require(seq_lens, "seq_lens", torch.int32, 1)
    Bq, Hq, D = q.shape
    B = block_table.shape[0]
    NB, Hkv, bs, Dk = k_cache.shape
    for name, rows in (("in_rows", in_rows), ("out_rows", out_rows)):
        if rows is not None:
            _require(rows, name, torch.int32, 1)
            if rows.shape[0] != B or rows.device != k_cache.device:
                raise ValueError(f"{name} must be [B] on the cache's device")
    if in_rows is None and Bq != B:
        raise ValueError("q batch differs from the block table's (pass in_rows)")
    if out_rows is not None and out is None:
        raise ValueError("out_rows needs an explicit out tensor")
    if v_cache.shape != k_cache.shape:
        raise ValueError("k_cache and v_cache shapes differ")
    if Dk != D:
        raise ValueError(f"head_dim mismatch q {D} vs cache {Dk}")
    if seq_lens.shape[0] != B:
        raise ValueError("block_table / seq_lens batch mismatch")
    if out_dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("out_dtype must be bfloat16 or float32")
    if grid not in _GRID_FLAGS:
        raise ValueError(f"grid must be one of {sorted(_GRID_FLAGS)}")
    if out is None:
        with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
            out = torch.empty((B, Hq, D), dtype=out_dtype, device=k_cache.device)
    else:
        _require(out, "out", out_dtype, 3)
    if lse is not None:
        _require(lse, "lse", torch.float32, 2)
    if (k_new is None) != (v_new is None):
        raise ValueError("k_new and v_new go together")
    if k_new is not None:
        _require(k_new, "k_new", torch.bfloat16, 3)
        _require(v_new, "v_new", torch.bfloat16, 3)
        if tuple(k_new.shape[1:]) != (Hkv, D) or k_new.shape[0] != Bq or v_new.shape != k_new.shape:
            raise ValueError("k_new / v_new must be [rows of q, Hkv, D]")
    dev = k_cache.device
    for name, t in (("q", q), ("block_table", block_table), ("seq_lens", seq_lens)):
        if (in_rows is None or name != "q") and t.device != dev:
            raise ValueError(f"{name} must be on the cache's device {dev}")
    if tuple(out.shape[1:]) != (Hq, D) or (out_rows is None and out.shape[0] < B):
        raise ValueError(f"out must be [rows, {Hq}, {D}], got {tuple(out.shape)}")
    if lse is not None and (lse.shape[1] != Hq or lse.shape[0] != out.shape[0]):
        raise ValueError(f"lse must be [{out.shape[0]}, {Hq}], got {tuple(lse.shape)}")
    if workspace is None:
        raise ValueError("paged_decode_attn needs a DecodeWorkspace (no per-call allocation)")
    if workspace.max_batch < B:
        raise ValueError(f"workspace sized for B <= {workspace.max_batch}, call has B={B}")
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    sp = _stream_ptr(stream, dev)
    if check_tables:
        with _on_device(dev):
            _ffi.call("adr_check_decode_tables", block_table.data_ptr(), seq_lens.data_ptr(), B,
                      block_table.shape[1], NB, workspace.buf.data_ptr(), workspace.buf.numel(), sp)
    with _on_device(dev):
        _ffi.call(
        "adr_paged_decode_attn_rows", q.data_ptr(),
        k_new.data_ptr() if k_new is not None else None,
        v_new.data_ptr() if v_new is not None else None,
        in_rows.data_ptr() if in_rows is not None else None,
        k_cache.data_ptr(), v_cache.data_ptr(),
        block_table.data_ptr(), seq_lens.data_ptr(), out.data_ptr(),
        lse.data_ptr() if lse is not None else None,
        out_rows.data_ptr() if out_rows is not None else None,
        B, Hq, Hkv, D, bs, block_table.shape[1], NB,
        float(scale), num_sms, workspace.num_workers,
        ADR_DTYPE_F32 if out_dtype == torch.float32 else ADR_DTYPE_BF16,
        (_ffi.ADR_DECODE_PDL if pdl else 0) | _GRID_FLAGS[grid],
        workspace.buf.data_ptr(), workspace.buf.numel(), sp)
    return out


def check_decode_tables(block_table: torch.Tensor, seq_lens: torch.Tensor, num_blocks: int,
                        workspace: DecodeWorkspace, *,
                        stream: torch.cuda.Stream | None = None) -> None:
    """Raise ``AdrError`` (ADR_ERR_INVALID) if a seq_len is negative or runs past
    its block-table row, or a used block-table entry lies outside [0, num_blocks).
    Synchronises the stream (diagnostic; not for the per-layer hot path)."""
    _require(block_table, "block_table", torch.int32, 2)
    _require(seq_lens, "seq_lens", torch.int32, 1)
    dev = block_table.device
    with _on_device(dev):
        _ffi.call("adr_check_decode_tables", block_table.data_ptr(), seq_lens.data_ptr(),
                  block_table.shape[0], block_table.shape[1], num_blocks, workspace.buf.data_ptr(),
                  workspace.buf.numel(), _stream_ptr(stream, dev))


def decode_status(workspace: DecodeWorkspace, *, clear: bool = True,
                  stream: torch.cuda.Stream | None = None) -> int:
    """ADR_STATUS_* bits recorded by the decode calls on ``workspace`` (bad
    seq_len / page entries they refused to dereference). Synchronises."""
    st = _ffi.ctypes.c_int32()
    with _on_device(workspace.device):
        _ffi.call("adr_decode_status", workspace.buf.data_ptr(), workspace.buf.numel(), int(clear),
                  _ffi.ctypes.byref(st), _stream_ptr(stream, workspace.device))
    return st.value


def kv_append(k_new: torch.Tensor, v_new: torch.Tensor, k_cache: torch.Tensor,
              v_cache: torch.Tensor, slots: torch.Tensor, *,
              stream: torch.cuda.Stream | None = None) -> None:
    """Scatter the step's new K/V rows [B,Hkv,D] into their paged slots (int64)."""
    _require(k_new, "k_new", torch.bfloat16, 3)
    _require(v_new, "v_new", torch.bfloat16, 3)
    _require(k_cache, "k_cache", torch.bfloat16, 4)
    _require(v_cache, "v_cache", torch.bfloat16, 4)
    _require(slots, "slots", torch.int64, 1)
    B, Hkv, D = k_new.shape
    NB, Hc, bs, Dc = k_cache.shape
    if (Hc, Dc) != (Hkv, D) or v_new.shape != k_new.shape or slots.shape[0] != B:
        raise ValueError("kv_append shape mismatch")
    with _on_device(k_cache.device):
        _ffi.call("adr_kv_append", k_new.data_ptr(), v_new.data_ptr(), k_cache.data_ptr(),
                  v_cache.data_ptr(), slots.data_ptr(), B, Hkv, D, bs, NB,
                  _stream_ptr(stream, k_cache.device))


def pack_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, row_idx: torch.Tensor, *,
             out: torch.Tensor | None = None,
             stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Gather rows row_idx of q [B,Hq,D], k/v [B,Hkv,D] into one [n,(Hq+2Hkv)*D] message."""
    _require(q, "q", torch.bfloat16, 3)
    _require(k, "k", torch.bfloat16, 3)
    _require(v, "v", torch.bfloat16, 3)
    _require(row_idx, "row_idx", torch.int32, 1)
    _, Hq, D = q.shape
    Hkv = k.shape[1]
    n = row_idx.shape[0]
    width = (Hq + 2 * Hkv) * D
    if out is None:
        out = torch.empty((n, width), dtype=torch.bfloat16, device=q.device)
    else:
        _require(out, "out", torch.bfloat16)
        if out.numel() < n * width:
            raise ValueError("pack_qkv output too small")
    with _on_device(q.device):
        _ffi.call("adr_pack_qkv", q.data_ptr(), k.data_ptr(), v.data_ptr(), row_idx.data_ptr(), n,
                  Hq, Hkv, D, out.data_ptr(), _stream_ptr(stream, q.device))
    return out


def unpack_qkv(msg: torch.Tensor, n_rows: int, Hq: int, Hkv: int, D: int, *,
               q: torch.Tensor | None = None, k: torch.Tensor | None = None,
               v: torch.Tensor | None = None,
               stream: torch.cuda.Stream | None = None):
    """Split a packed message into dense q [n,Hq,D], k [n,Hkv,D], v [n,Hkv,D]."""
    _require(msg, "msg", torch.bfloat16)
    dev = msg.device
    q = q if q is not None else torch.empty((n_rows, Hq, D), dtype=torch.bfloat16, device=dev)
    k = k if k is not None else torch.empty((n_rows, Hkv, D), dtype=torch.bfloat16, device=dev)
    v = v if v is not None else torch.empty((n_rows, Hkv, D), dtype=torch.bfloat16, device=dev)
    with _on_device(dev):
        _ffi.call("adr_unpack_qkv", msg.data_ptr(), n_rows, Hq, Hkv, D, q.data_ptr(), k.data_ptr(),
                  v.data_ptr(), _stream_ptr(stream, dev))
    return q, k, v


def scatter_out(src: torch.Tensor, row_idx: torch.Tensor, out: torch.Tensor, *,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """out[row_idx[i]] = src[i] for the executor-returned rows [n,Hq,D]."""
    _require(src, "src", torch.bfloat16)
    _require(out, "out", torch.bfloat16, 3)
    _require(row_idx, "row_idx", torch.int32, 1)
    n = row_idx.shape[0]
    _, Hq, D = out.shape
    if src.numel() < n * Hq * D:
        raise ValueError("scatter_out source too small")
    with _on_device(out.device):
        _ffi.call("adr_scatter_out", src.data_ptr(), row_idx.data_ptr(), n, Hq, D, out.data_ptr(),
                  _stream_ptr(stream, out.device))
    return out


def slot_mapping(block_table: torch.Tensor, positions: torch.Tensor) -> torch.Tensor:
    """Slot of token ``positions[b]`` of each request: bt[b, p // 16] * 16 + p % 16 (int64).

    Pure index arithmetic on the device tensors (no host sync); positions < 0
    map to slot -1 (padding rows that kv_append skips).
    """
    pos = positions.to(torch.int64)
    page_col = torch.clamp(pos, min=0) // PAGE
    pages = torch.gather(block_table.to(torch.int64), 1, page_col.unsqueeze(1)).squeeze(1)
    slots = pages * PAGE + torch.remainder(pos, PAGE)
    return torch.where(pos >= 0, slots, torch.full_like(slots, -1))


def kv_transfer(src_k: torch.Tensor, src_v: torch.Tensor, src_pages: torch.Tensor,
                dst_k: torch.Tensor, dst_v: torch.Tensor, dst_pages: torch.Tensor, *,
                stream: torch.cuda.Stream | None = None) -> None:
    """Copy whole KV pages src_pages[i] -> dst_pages[i] (per layer cache tensors
    [NB, Hkv, 16, D]); the source may be a peer GPU's cache (NVLink pull)."""
    for t, n in ((src_k, "src_k"), (src_v, "src_v"), (dst_k, "dst_k"), (dst_v, "dst_v")):
        _require(t, n, torch.bfloat16, 4)
    _require(src_pages, "src_pages", torch.int32, 1)
    _require(dst_pages, "dst_pages", torch.int32, 1)
    if src_pages.shape != dst_pages.shape or src_k.shape[1:] != dst_k.shape[1:]:
        raise ValueError("kv_transfer shape mismatch")
    _, Hkv, bs, D = dst_k.shape
    with _on_device(dst_k.device):  # the copy runs on the destination GPU (pulls over NVLink)
        _ffi.call("adr_kv_transfer", src_k.data_ptr(), src_v.data_ptr(), src_pages.data_ptr(),
                  dst_k.data_ptr(), dst_v.data_ptr(), dst_pages.data_ptr(), src_pages.numel(), Hkv,
                  D, bs, _stream_ptr(stream, dst_k.device))
