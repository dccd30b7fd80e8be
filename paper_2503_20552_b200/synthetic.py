"""Seeded synthetic decode batches of the BASELINE.json shapes.

q, k, v ~ N(0, 1) rounded to bf16 (seed 0 for data); block tables are a seeded
random permutation of the physical pages (seed 1) so the page indirection is
real, not contiguous. Context lengths may be uniform or ragged.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import torch

from .ops import PAGE

__all__ = ["DecodeShape", "CONFIGS", "make_block_table", "make_layer", "kv_read_bytes",
           "algorithmic_bytes"]


@dataclass(frozen=True)
class DecodeShape:
    name: str
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    num_layers: int
    ctx: int | tuple[int, ...]      # tokens per request (after this step's append)
    block_size: int = PAGE
    spare_pages: int = 0            # extra physical pages beyond the live ones

    def ctx_list(self) -> list[int]:
        if isinstance(self.ctx, int):
            return [self.ctx] * self.batch
        if len(self.ctx) != self.batch:
            raise ValueError("ctx list length must equal batch")
        return list(self.ctx)

    def pages_per_request(self) -> list[int]:
        return [-(-c // self.block_size) for c in self.ctx_list()]

    @property
    def num_pages(self) -> int:
        return sum(self.pages_per_request()) + self.spare_pages

    @property
    def max_pages(self) -> int:
        return max(1, max(self.pages_per_request()))


# Decode shapes of BASELINE.json:configs (C1..C5). C1 is the tiny CPU-oracle case.
CONFIGS: dict[str, DecodeShape] = {
    "C1": DecodeShape("C1-tiny", 8, 8, 2, 64, 2, 512),
    "C2": DecodeShape("C2-llama2-7b", 64, 32, 32, 128, 32, 4096),
    "C3": DecodeShape("C3-llama3-8b", 64, 32, 8, 128, 32, 4096),
    "C5": DecodeShape("C5-llama3-70b", 16, 64, 8, 128, 80, 32768),
}


def make_block_table(shape: DecodeShape, seed: int = 1) -> torch.Tensor:
    """[B, max_pages] int32: each request owns a disjoint random set of pages."""
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(shape.num_pages, generator=g).to(torch.int32)
    bt = torch.zeros((shape.batch, shape.max_pages), dtype=torch.int32)
    off = 0
    for b, n in enumerate(shape.pages_per_request()):
        bt[b, :n] = perm[off:off + n]
        off += n
    return bt


def make_layer(shape: DecodeShape, device: torch.device | str, seed: int = 0,
               block_table: torch.Tensor | None = None) -> dict:
    """One layer's decode inputs on ``device`` (bf16 data, int32 tables)."""
    device = torch.device(device)
    g = torch.Generator(device=device).manual_seed(seed)
    B, Hq, Hkv, D = shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
    NB = shape.num_pages
    def randn(*s):
        return torch.randn(*s, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    k_cache = torch.empty((NB, Hkv, shape.block_size, D), dtype=torch.bfloat16, device=device)
    v_cache = torch.empty_like(k_cache)
    # fill in chunks so the fp32 staging stays small for multi-GiB caches
    step = max(1, (1 << 28) // max(1, Hkv * shape.block_size * D))
    for lo in range(0, NB, step):
        hi = min(NB, lo + step)
        k_cache[lo:hi] = randn(hi - lo, Hkv, shape.block_size, D)
        v_cache[lo:hi] = randn(hi - lo, Hkv, shape.block_size, D)
    bt = block_table if block_table is not None else make_block_table(shape)
    return {
        "q": randn(B, Hq, D),
        "k_new": randn(B, Hkv, D),
        "v_new": randn(B, Hkv, D),
        "k_cache": k_cache,
        "v_cache": v_cache,
        "block_table": bt.to(device),
        "seq_lens": torch.tensor(shape.ctx_list(), dtype=torch.int32, device=device),
    }


def kv_read_bytes(shape: DecodeShape) -> int:
    """K+V bytes one layer of decode attention must stream (the KV GB/s numerator)."""
    return sum(shape.ctx_list()) * shape.num_kv_heads * shape.head_dim * 2 * 2


def algorithmic_bytes(shape: DecodeShape) -> int:
    """SURVEY.md §8d per-layer algorithmic bytes: KV read + q + out + append + tables."""
    B, Hq, Hkv, D = shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
    e = 2
    tables = 4 * sum(shape.pages_per_request()) + 4 * B
    return kv_read_bytes(shape) + 2 * B * Hq * D * e + B * Hkv * D * 2 * e + tables
