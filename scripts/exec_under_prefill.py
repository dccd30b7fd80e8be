#!/usr/bin/env python
"""Executor attention on a green-context partition, alone and beside a prefill
GEMM load (diagnostic for the measured pricer): per shape, µs per call of the
offloaded batch's decode attention on the partition's stream.

    python scripts/exec_under_prefill.py [attn_sms] [grids, e.g. auto,split,dynamic]
"""
import math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import coloc, ops, specs
from paper_2503_20552_b200.capacity import LLAMA3_70B_TP8W
from paper_2503_20552_b200.synthetic import DecodeShape, kv_read_bytes, make_layer

dev = torch.device("cuda:0")
sms = int(sys.argv[1]) if len(sys.argv) > 1 else 72
grids = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"]
part = coloc.SmPartition(0, sms)
loads = {"none": None, "13B": coloc.prefill_load_for(specs.LLAMA2_13B, dev),
         "70B-tp8w": coloc.prefill_load_for(LLAMA3_70B_TP8W, dev)}
shapes = [DecodeShape("C5-exec B8 ctx16k", 8, 64, 8, 128, 1, 16384),
          DecodeShape("C5-exec B4 ctx24k", 4, 64, 8, 128, 1, 24576),
          DecodeShape("C4-exec B24 ctx1.5k", 24, 40, 40, 128, 1, 1536),
          DecodeShape("C3-exec B16 ctx4k", 16, 32, 8, 128, 1, 4096)]
for sh, grid in [(sh, g) for sh in shapes for g in grids]:
    x = make_layer(sh, dev)
    ws = ops.DecodeWorkspace(sh.batch, sh.num_q_heads, sh.num_kv_heads, 128, dev)
    out = torch.empty(sh.batch, sh.num_q_heads, 128, dtype=torch.bfloat16, device=dev)
    fn = lambda: ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                       x["seq_lens"], out=out, scale=1 / math.sqrt(128),
                                       workspace=ws, stream=part.attn_stream,
                                       num_sms=part.attn_sms, pdl=True, grid=grid)
    for name, pre in loads.items():
        if pre is None:
            fn(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(part.attn_stream)
            for _ in range(20):
                fn()
            e1.record(part.attn_stream)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            print(f"{sh.name:22s} {grid:7s} prefill {name:9s}: {us:8.1f} us  {kv_read_bytes(sh) / us / 1e3:7.0f} GB/s", flush=True)
            continue
        ov = coloc.run_under_prefill(part.attn_stream, fn, 20, part.prefill_stream, pre, 12)
        us = ov.attn_s * 1e6
        print(f"{sh.name:22s} {grid:7s} prefill {name:9s}: {us:8.1f} us  {kv_read_bytes(sh) / us / 1e3:7.0f} GB/s"
              f"  (prefill iter {ov.prefill_s * 1e3:.2f} ms, covered {ov.covered})", flush=True)
