#!/usr/bin/env python
"""Time adr_paged_decode_attn for one kernel variant (ADR_DECODE_VARIANT env) on
C2 shapes over several distinct layer caches (>> L2). Prints one JSON line."""
import json, math, os, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.synthetic import CONFIGS, algorithmic_bytes, kv_read_bytes, make_block_table, make_layer

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nlayers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
shape = CONFIGS[cfg]
dev = torch.device("cuda:0")
bt = make_block_table(shape)
layers = [make_layer(shape, dev, seed=l, block_table=bt) for l in range(nlayers)]
ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, dev)
out = torch.empty(shape.batch, shape.num_q_heads, shape.head_dim, dtype=torch.bfloat16, device=dev)
def call(x):
    ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"], out=out, workspace=ws)
for _ in range(3):
    for x in layers: call(x)
torch.cuda.synchronize()
times = []
for rep in range(10):
    for x in layers:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); call(x); e.record()
        times.append((s, e))
torch.cuda.synchronize()
ms = [s.elapsed_time(e) for s, e in times]
med = statistics.median(ms)
print(json.dumps({"variant": int(os.environ.get("ADR_DECODE_VARIANT", "0")), "config": cfg,
                  "median_ms": med, "min_ms": min(ms),
                  "alg_GBps": algorithmic_bytes(shape) / (med / 1e3) / 1e9,
                  "kv_GBps_best": kv_read_bytes(shape) / (min(ms) / 1e3) / 1e9}))
