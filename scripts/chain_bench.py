#!/usr/bin/env python
"""Per-launch time of adr_paged_decode_attn on C2 layers under different
chaining styles (diagnostic for the bench step)."""
import json, os, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.synthetic import CONFIGS, make_block_table, make_layer

L = int(os.environ.get("CHAIN_LAYERS", "16"))
shape = CONFIGS["C2"]
dev = torch.device("cuda:0")
bt = make_block_table(shape)
layers = [make_layer(shape, dev, seed=l, block_table=bt) for l in range(L)]
ws = [ops.DecodeWorkspace(64, 32, 32, 128, dev) for _ in range(2)]
outs = [torch.empty(64, 32, 128, dtype=torch.bfloat16, device=dev) for _ in range(L)]
slots = ops.slot_mapping(layers[0]["block_table"], layers[0]["seq_lens"].long() - 1)

def call(l, fused=True, pdl=False):
    x = layers[l]
    kw = dict(k_new=x["k_new"], v_new=x["v_new"]) if fused else {}
    ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                          out=outs[l], workspace=ws[l % 2], pdl=pdl, **kw)

def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / L * 1e3   # us per layer

res = {}
res["chain_fused"] = timed(lambda: [call(l) for l in range(L)])
res["chain_fused_pdl"] = timed(lambda: [call(l, pdl=True) for l in range(L)])
res["chain_plain_noappend"] = timed(lambda: [call(l, fused=False) for l in range(L)])
def sep():
    for l in range(L):
        x = layers[l]
        ops.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
        call(l, fused=False)
res["chain_separate_append"] = timed(sep)
def with_events():
    for l in range(L):
        torch.cuda.Event().record()
        call(l)
res["chain_fused_events"] = timed(with_events)
def synced():
    for l in range(L):
        call(l); torch.cuda.synchronize()
res["synced_fused"] = timed(synced)
def same_layer():
    for l in range(L):
        call(0)
res["chain_same_layer"] = timed(same_layer)
res["variant"] = os.environ.get("ADR_DECODE_VARIANT", "default")
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}))
