"""Literal CPU restatement of the reference's placement arithmetic.

TEST INFRASTRUCTURE ONLY (imported by tests/). Pinned: tests/test_oracle_decisions.py
checks it against the golden vectors that tests/golden/make_golden.py produced
by running the reference itself. Each function cites the reference lines it
restates (files under /root/reference/pkg/src/adrenaline_sim/).
"""
from __future__ import annotations

import math


def algorithm1(req_used, req_max, offloaded, local, bound, c1_uses_max_tokens=False):
    """scheduling.py:176-221. offloaded/local: lists of (used_token, max_token).
    Returns (offload, rule)."""
    attn_used = sum(u for u, _ in offloaded)       # :188-191
    attn_max = sum(m for _, m in offloaded)
    decode_used = sum(u for u, _ in local)         # :194-197
    n_off, n_loc = len(offloaded), len(local)
    budget = decode_used * bound                   # :199
    c1_load = attn_max if c1_uses_max_tokens else attn_used   # :200
    if c1_load + req_max < budget:                 # :210 (C1, strict)
        return True, "C1"
    if attn_used + req_used < budget and n_off + 1 < n_loc * bound:   # :212 (C2)
        return True, "C2"
    return False, "local"


def eq1_mem(exec_hbm, exec_bw, dec_hbm, dec_bw):
    """scheduling.py:91-111 (Eq. 1)."""
    if not exec_hbm:
        return 0.0
    return min(sum(exec_hbm) / dec_hbm, sum(exec_bw) / dec_bw)


def eq2_comp(b_max_ideal, b_tpot):
    """scheduling.py:114-124 (Eq. 2); inf when b_tpot == 0."""
    if b_tpot == 0:
        return math.inf
    return max(0.0, (b_max_ideal - b_tpot) / b_tpot)


def eq3(mem, comp):
    """scheduling.py:127-130 (Eq. 3)."""
    return min(mem, comp)


def graph_caps(max_batch, interval):
    """graphs.py:22-27."""
    if max_batch == 0:
        return (0,)
    top = -(-max_batch // interval) * interval
    return tuple(range(interval, top + 1, interval))


def pick_graph(decode_caps, offload_caps, bd, bo):
    """graphs.py:67-84: smallest cap >= batch on each axis, None on overflow."""
    d = next((c for c in decode_caps if c >= bd), None)
    o = next((c for c in offload_caps if c >= bo), None)
    return None if d is None or o is None else (d, o)
