#!/usr/bin/env python
"""Chained (PDL) per-call time of adr_paged_decode_attn over a set of decode
shapes, for chunk-grid knob tuning (knobs come from the environment).
One compact line per shape; the fit separates fixed cost and streaming rate."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.synthetic import DecodeShape, kv_read_bytes, make_block_table, make_layer

dev = torch.device("cuda:0")
SHAPES = [(8, 4, 512), (8, 16, 1024), (8, 40, 2048), (8, 64, 1024), (8, 64, 4096), (8, 128, 4096),
          (32, 4, 512), (32, 8, 1024), (32, 16, 1024), (32, 64, 1024), (32, 64, 4096), (8, 16, 32768)]
rows = []
for Hkv, B, ctx in SHAPES:
    Hq = 64 if ctx == 32768 else 32
    sh = DecodeShape("s", B, Hq, Hkv, 128, 6, ctx)
    bt = make_block_table(sh)
    ls = [make_layer(sh, dev, seed=l, block_table=bt) for l in range(6)]
    ws = [ops.DecodeWorkspace(B, Hq, Hkv, 128, dev) for _ in range(2)]
    out = torch.empty(B, Hq, 128, dtype=torch.bfloat16, device=dev)
    def run():
        for l, x in enumerate(ls):
            ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                                  out=out, workspace=ws[l % 2], k_new=x["k_new"], v_new=x["v_new"], pdl=True)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 60 * 1e3
    mb = kv_read_bytes(sh) / 1e6
    rows.append((mb, us))
    print(f"Hkv={Hkv:2d} B={B:3d} ctx={ctx:5d} {mb:8.1f} MB {us:8.1f} us {mb / us:6.2f} TB/s", flush=True)
    del ls, ws
    torch.cuda.empty_cache()
x = np.array([r[0] for r in rows]); y = np.array([r[1] for r in rows])
(a, b), *_ = np.linalg.lstsq(np.vstack([np.ones_like(x), x]).T, y, rcond=None)
print(f"knobs {dict((k, v) for k, v in os.environ.items() if k.startswith('ADR_'))} fixed {a:.2f} us stream {1e3 / b:.0f} GB/s total {y.sum():.1f} us")
