"""Pin oracle/decision_oracle.py to the reference goldens, then use it to
property-test the package's incremental OffloadLedger on random event streams."""
import json
import random
from pathlib import Path

import decision_oracle as dor

from paper_2503_20552_b200 import scheduling

GOLD = Path(__file__).resolve().parent / "golden"


def test_oracle_pinned_to_reference_goldens():
    g = json.loads((GOLD / "need_offload.json").read_text())
    for c in g["cases"]:
        off = [(u, p + o) for p, o, u in c["offloaded"]]
        loc = [(u, p + o) for p, o, u in c["local"]]
        p, o, u = c["req"]
        assert dor.algorithm1(u, p + o, off, loc, c["bound"], c["c1_uses_max_tokens"]) == \
            (c["offload"], c["rule"])
    b = json.loads((GOLD / "bounds.json").read_text())
    for c in b["mem"]:
        if "ok" in c:
            assert dor.eq1_mem(*c["args"]) == c["ok"]
    for c in b["comp"]:
        if "ok" in c:
            assert dor.eq2_comp(*c["args"]) == c["ok"]
    gr = json.loads((GOLD / "graphs.json").read_text())
    for c in gr["cases"]:
        dc = dor.graph_caps(c["args"][1], c["interval"])
        oc = dor.graph_caps(c["args"][2], c["interval"])
        assert list(dc) == c["decode_caps"] and list(oc) == c["offload_caps"]
        for bd, bo, want in c["select"]:
            got = dor.pick_graph(dc, oc, bd, bo)
            assert (list(got) if got else None) == want


def test_ledger_tracks_random_event_streams():
    """Placements, token growth, completions and preemptions applied to the O(1)
    ledger always yield the oracle's decision on the explicit sets."""
    rng = random.Random(5)
    for trial in range(20):
        led = scheduling.OffloadLedger()
        off, loc = [], []
        for step in range(400):
            op = rng.random()
            if op < 0.4:
                r = scheduling.Request(step, 0.0, rng.randint(1, 3000), rng.randint(1, 1500))
                r.used_token = rng.choice([0, rng.randint(0, r.max_token)])
                bound = rng.choice([0.3, 0.5, 0.7, 0.8, 1.2])
                d = led.decide(r, bound)
                want = dor.algorithm1(r.used_token, r.max_token,
                                      [(x.used_token, x.max_token) for x in off],
                                      [(x.used_token, x.max_token) for x in loc], bound)
                assert (d.offload, d.rule) == want
                (off if d.offload else loc).append(r)
                led.add(r, offloaded=d.offload)
            elif op < 0.8 and (off or loc):
                side_off = bool(off) and (not loc or rng.random() < 0.5)
                grp = off if side_off else loc
                for x in grp:
                    x.used_token += 1
                led.grow(len(grp), offloaded=side_off)
            elif off or loc:
                side_off = bool(off) and (not loc or rng.random() < 0.5)
                grp = off if side_off else loc
                victim = grp.pop(rng.randrange(len(grp)))
                led.remove(victim, offloaded=side_off)
        ref = scheduling.OffloadLedger.of(off, loc)
        assert (led.attn_used, led.attn_max, led.n_off, led.decode_used, led.decode_max,
                led.n_local) == (ref.attn_used, ref.attn_max, ref.n_off, ref.decode_used,
                                 ref.decode_max, ref.n_local)
