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


def replay_handoff(events, pages_per_pool: dict, page_tokens: int = 16):
    """Like ``replay`` with the prefill -> decode hand-off: events are
    (op, where, req_id, tokens[, dst]) with op in reserve / release (decoder and
    executor pools), stage / unstage (a prefill GPU's staging pages, same
    allocator contract) and transfer (``where`` = the prefill pool, ``dst`` the
    decoder pool; the staged prompt's first ceil(tokens / 16) pages go to the
    decoder's first ceil(tokens / 16) reserved pages, in order — engine.py:231-249
    moves prefill_len tokens of KV into the slots reserved at admission, 331).
    Returns the expected output per event: pages handed (reserve / stage),
    (src_pages, dst_pages) (transfer) or None (release / unstage)."""
    alloc = {w: ListAllocator(n) for w, n in pages_per_pool.items()}
    tables: dict = {w: {} for w in pages_per_pool}
    out = []
    for ev in events:
        op, where, rid, tokens = ev[:4]
        tab = tables[where]
        if op in ("reserve", "stage"):
            have = tab.setdefault(rid, [])
            need = -(-tokens // page_tokens)
            new = alloc[where].take(max(0, need - len(have)))
            have.extend(new)
            out.append(tuple(new))
        elif op in ("release", "unstage"):
            alloc[where].give(tab.pop(rid, []))
            out.append(None)
        elif op == "transfer":
            n = -(-tokens // page_tokens)
            src = tab[rid]
            dst = tables[ev[4]][rid]
            if n > len(src) or n > len(dst):
                raise ValueError(f"transfer of {n} pages for request {rid} exceeds its tables")
            out.append((tuple(src[:n]), tuple(dst[:n])))
        else:
            raise ValueError(f"unknown op {op}")
    return tables, out


def slot(table: list[int], pos: int, page_tokens: int = 16) -> int:
    return table[pos // page_tokens] * page_tokens + pos % page_tokens
