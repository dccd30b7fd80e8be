#!/usr/bin/env python
"""Per-call cost of executor attention on a green-context partition while a
prefill GEMM load runs on the rest (diagnostic): call size sweep, PDL on/off.

    python scripts/exec_latency.py [attn_sms]
"""
import math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import coloc, ops, specs
from paper_2503_20552_b200.synthetic import DecodeShape, kv_read_bytes, make_layer

dev = torch.device("cuda:0")
sms = int(sys.argv[1]) if len(sys.argv) > 1 else 72
part = coloc.SmPartition(0, sms)
pre = coloc.prefill_load_for(specs.LLAMA2_13B, dev)
shapes = [DecodeShape("B8 ctx1k GQA-4", 8, 32, 8, 128, 1, 1024),
          DecodeShape("B16 ctx4k GQA-4", 16, 32, 8, 128, 1, 4096),
          DecodeShape("B32 ctx4k GQA-4", 32, 32, 8, 128, 1, 4096),
          DecodeShape("B32 ctx4k MHA", 32, 32, 32, 128, 1, 4096)]
for sh in shapes:
    x = make_layer(sh, dev)
    ws = ops.DecodeWorkspace(sh.batch, sh.num_q_heads, sh.num_kv_heads, 128, dev)
    out = torch.empty(sh.batch, sh.num_q_heads, 128, dtype=torch.bfloat16, device=dev)
    for pdl in (True, False):
        fn = lambda: ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                           x["seq_lens"], out=out, scale=1 / math.sqrt(128),
                                           workspace=ws, stream=part.attn_stream,
                                           num_sms=part.attn_sms, pdl=pdl)
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(part.attn_stream)
        for _ in range(20):
            fn()
        e1.record(part.attn_stream)
        torch.cuda.synchronize()
        alone = e0.elapsed_time(e1) / 20 * 1e3
        ov = coloc.run_under_prefill(part.attn_stream, fn, 20, part.prefill_stream, pre, 16)
        shared = ov.attn_s * 1e6
        mb = kv_read_bytes(sh) / 1e6
        print(f"{sh.name:18s} {mb:7.0f} MB pdl={int(pdl)}: alone {alone:8.1f} us ({mb / alone:5.2f} TB/s) | "
              f"beside prefill {shared:8.1f} us ({mb / shared:5.2f} TB/s), prefill iter {ov.prefill_s * 1e3:.2f} ms", flush=True)
