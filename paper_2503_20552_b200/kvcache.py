"""Paged KV memory: deterministic page allocator, block tables, slot mapping.

The reference keeps KV as token counters only (engine.py:331-349, 416-421).
Here the same token-granular reservations drive real 16-token pages:

  * ``PagePool`` hands out the lowest free page ids first (a min-heap), so a
    given reservation sequence always yields the same block tables;
  * ``BlockTables`` grows each request's page list as its reservation grows
    and releases it whole on completion / preemption;
  * ``PagedKVMirror`` is an ``engine.MemoryObserver``: attached to ``simulate``
    it keeps one ``BlockTables`` per decoder pool, per executor and per prefill
    GPU's staging area, so an engine run produces the exact page layout the
    device caches use — including the prefill -> decode hand-off: a local
    request's prompt KV is staged in prefill-GPU pages and migrated page by
    page into the decoder pages reserved at admission (``Transfer``: the
    block-table remap that ``ops.kv_transfer`` executes).

Admission stays token-granular (decisions bit-identical to the reference);
pages add at most one partial page of slack per live request, which the pool
sizes for (``slack_pages``).
"""
from __future__ import annotations

import heapq
from typing import Iterable

import numpy as np

from .engine import MemoryObserver
from .scheduling import Request

PAGE_TOKENS = 16

__all__ = ["PAGE_TOKENS", "PagePool", "BlockTables", "PagedKVMirror", "Transfer",
           "pages_for_budget"]


def pages_for_budget(budget_bytes: float, kv_bytes_per_token: int, slack_pages: int) -> int:
    """Physical pages for a token budget: whole pages of it plus partial-page slack."""
    return int(budget_bytes // (kv_bytes_per_token * PAGE_TOKENS)) + slack_pages


class PagePool:
    """Fixed set of page ids [0, num_pages); lowest free id first."""

    def __init__(self, num_pages: int) -> None:
        if num_pages <= 0:
            raise ValueError("num_pages must be positive")
        self.num_pages = num_pages
        self._free = list(range(num_pages))  # already a valid min-heap

    @property
    def free_pages(self) -> int:
        return len(self._free)

    def alloc(self, n: int) -> list[int]:
        if n < 0:
            raise ValueError("n must be >= 0")
        if n > len(self._free):
            raise MemoryError(f"page pool exhausted: need {n}, have {len(self._free)}")
        return [heapq.heappop(self._free) for _ in range(n)]

    def free(self, pages: Iterable[int]) -> None:
        for p in pages:
            heapq.heappush(self._free, p)


class BlockTables:
    """Per-request page lists over one PagePool."""

    def __init__(self, pool: PagePool, page_tokens: int = PAGE_TOKENS) -> None:
        self.pool = pool
        self.page_tokens = page_tokens
        self.tables: dict[int, list[int]] = {}
        self.tokens: dict[int, int] = {}

    def reserve(self, req_id: int, tokens: int) -> None:
        """Ensure ``req_id`` owns ceil(tokens / page) pages (never shrinks)."""
        have = self.tables.setdefault(req_id, [])
        need = -(-tokens // self.page_tokens)
        if need > len(have):
            have.extend(self.pool.alloc(need - len(have)))
        self.tokens[req_id] = max(tokens, self.tokens.get(req_id, 0))

    def release(self, req_id: int) -> list[int]:
        pages = self.tables.pop(req_id, [])
        self.tokens.pop(req_id, None)
        self.pool.free(pages)
        return pages

    def slot(self, req_id: int, pos: int) -> int:
        """Cache slot of token ``pos``: page * page_tokens + pos % page_tokens."""
        pages = self.tables[req_id]
        return pages[pos // self.page_tokens] * self.page_tokens + pos % self.page_tokens

    def table_array(self, req_ids: list[int], width: int | None = None) -> np.ndarray:
        """[len(req_ids), width] int32 block table (unused entries 0)."""
        width = width or max((len(self.tables[r]) for r in req_ids), default=1)
        out = np.zeros((len(req_ids), max(width, 1)), dtype=np.int32)
        for i, r in enumerate(req_ids):
            t = self.tables[r]
            out[i, :len(t)] = t
        return out


class Transfer(tuple):
    """One prefill -> decode page migration: (req_id, src, dst, src_pages, dst_pages).

    ``src`` = ("prefill", p), ``dst`` = ("decoder", d); page i of the request's
    staged prompt KV (``src_pages[i]``) lands in ``dst_pages[i]``, the decoder
    pages reserved for the same token range at admission."""

    __slots__ = ()

    def __new__(cls, req_id, src, dst, src_pages, dst_pages):
        return super().__new__(cls, (req_id, src, dst, tuple(src_pages), tuple(dst_pages)))

    req_id = property(lambda self: self[0])
    src = property(lambda self: self[1])
    dst = property(lambda self: self[2])
    src_pages = property(lambda self: self[3])
    dst_pages = property(lambda self: self[4])


class PagedKVMirror(MemoryObserver):
    """Engine observer maintaining the page layout of every device pool.

    ``log`` records (op, where, req_id, tokens, pages) for replay / checking;
    op is "reserve" / "release" (decoder and executor pools), "stage" /
    "unstage" (a prefill GPU's staging pages) or "transfer" (``pages`` is then
    the ``Transfer``). ``on_transfer`` (optional callable) is invoked with each
    ``Transfer`` as the engine starts it — the device-side hook
    (``runtime.KVTransferRunner``) copies the pages there.
    """

    def __init__(self, pages_per_decoder: int, pages_per_executor: int,
                 num_decode: int, num_prefill: int, keep_log: bool = True,
                 pages_per_prefill: int = 0, on_transfer=None) -> None:
        self.pools = {("decoder", i): BlockTables(PagePool(pages_per_decoder))
                      for i in range(num_decode)}
        self.pools.update({("executor", i): BlockTables(PagePool(pages_per_executor))
                           for i in range(num_prefill)})
        if pages_per_prefill > 0:
            self.pools.update({("prefill", i): BlockTables(PagePool(pages_per_prefill))
                               for i in range(num_prefill)})
        self.keep_log = keep_log
        self.on_transfer = on_transfer
        self.log: list[tuple] = []
        self.transfers: int = 0

    @classmethod
    def for_config(cls, cfg, slack_pages: int = 4096, keep_log: bool = True,
                   stage_pages: int | None = None, on_transfer=None) -> "PagedKVMirror":
        """``stage_pages``: staging pages per prefill GPU (default: its in-flight
        budget plus the slack; a lone prompt larger than the budget still runs
        in the engine, so size it for the longest prompt when that is larger)."""
        kv_tok = cfg.model.kv_bytes_per_token
        if stage_pages is None:
            stage_pages = pages_for_budget(cfg.prefill_inflight_budget_bytes, kv_tok, slack_pages)
        return cls(pages_for_budget(cfg.pool_bytes, kv_tok, slack_pages),
                   pages_for_budget(cfg.executor_budget_bytes, kv_tok, slack_pages),
                   cfg.num_decode, cfg.num_prefill, keep_log, stage_pages, on_transfer)

    def reserve(self, req: Request, where: tuple[str, int], tokens: int) -> None:
        bt = self.pools[where]
        before = len(bt.tables.get(req.req_id, ()))
        bt.reserve(req.req_id, tokens)
        if self.keep_log:
            self.log.append(("reserve", where, req.req_id, tokens,
                             tuple(bt.tables[req.req_id][before:])))

    def release(self, req: Request, where: tuple[str, int]) -> None:
        pages = self.pools[where].release(req.req_id)
        if self.keep_log:
            self.log.append(("release", where, req.req_id, 0, tuple(pages)))

    # ---- prefill -> decode hand-off (no-ops without staging pools) ----

    def prefill_start(self, req: Request, p_idx: int, tokens: int) -> None:
        where = ("prefill", p_idx)
        bt = self.pools.get(where)
        if bt is None:
            return
        bt.reserve(req.req_id, tokens)
        if self.keep_log:
            self.log.append(("stage", where, req.req_id, tokens, tuple(bt.tables[req.req_id])))

    def transfer(self, req: Request, p_idx: int, d_idx: int, tokens: int) -> None:
        src, dst = ("prefill", p_idx), ("decoder", d_idx)
        st = self.pools.get(src)
        if st is None:
            return
        n = -(-tokens // st.page_tokens)
        tr = Transfer(req.req_id, src, dst, st.tables[req.req_id][:n],
                      self.pools[dst].tables[req.req_id][:n])
        self.transfers += 1
        if self.keep_log:
            self.log.append(("transfer", src, req.req_id, tokens, tr))
        if self.on_transfer is not None:
            self.on_transfer(tr)

    def transfer_done(self, req: Request, p_idx: int) -> None:
        where = ("prefill", p_idx)
        bt = self.pools.get(where)
        if bt is None:
            return
        pages = bt.release(req.req_id)
        if self.keep_log:
            self.log.append(("unstage", where, req.req_id, 0, tuple(pages)))
