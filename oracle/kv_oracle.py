"""CPU restatement of the paged-KV bookkeeping (TEST INFRASTRUCTURE ONLY).

The reference has token counters only (engine.py:331 reserve prefill_len+1 at
admission, 416-421 +1 per running request per step, 274-283 / 364-377 free on
completion / preemption). This replays those reservation events onto
16-token pages with a sorted free list (lowest id first) — a different data
structure from kvcache.PagePool's heap, same contract — so block tables and
slot mappings can be checked bit-exactly.
"""
from __future__ import annotations

import bisect


class ListAllocator:
    def __init__(self, num_pages: int) -> None:
        self.free = list(range(num_pages))   # kept sorted

    def take(self, n: int) -> list[int]:
        if n > len(self.free):
            raise MemoryError("exhausted")
        got, self.free = self.free[:n], self.free[n:]
        return got

    def give(self, pages) -> None:
        for p in pages:
            bisect.insort(self.free, p)


def replay(events, pages_per_pool: dict, page_tokens: int = 16):
    """events: (op, where, req_id, tokens). Returns {where: {req_id: [pages]}} at the end
    and the list of pages handed out per reserve event."""
    alloc = {w: ListAllocator(n) for w, n in pages_per_pool.items()}
    tables: dict = {w: {} for w in pages_per_pool}
    handed = []
    for op, where, rid, tokens in events:
        tab = tables[where]
        if op == "reserve":
            have = tab.setdefault(rid, [])
            need = -(-tokens // page_tokens)
            new = alloc[where].take(max(0, need - len(have)))
            have.extend(new)
            handed.append(tuple(new))
        else:
            alloc[where].give(tab.pop(rid, []))
            handed.append(None)
    return tables, handed


def slot(table: list[int], pos: int, page_tokens: int = 16) -> int:
    return table[pos // page_tokens] * page_tokens + pos % page_tokens
