#!/usr/bin/env python
"""Does CTA-dispatch priority remove the per-call cost of executor attention
beside a prefill GEMM load? Plain streams (no green contexts): attention
(grid sized for 72 SMs) on a stream of priority P_attn, prefill on a default-
priority stream (diagnostic)."""
import math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import coloc, ops, specs
from paper_2503_20552_b200.synthetic import DecodeShape, kv_read_bytes, make_layer

dev = torch.device("cuda:0")
pre = coloc.prefill_load_for(specs.LLAMA2_13B, dev)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
print("priority range", lo, hi)
pre_stream = torch.cuda.Stream(dev, priority=0)
for prio in (0, -1, -2, -5):
    st = torch.cuda.Stream(dev, priority=prio)
    for sh in (DecodeShape("B8 ctx1k GQA-4", 8, 32, 8, 128, 1, 1024),
               DecodeShape("B32 ctx4k GQA-4", 32, 32, 8, 128, 1, 4096)):
        x = make_layer(sh, dev)
        ws = ops.DecodeWorkspace(sh.batch, sh.num_q_heads, sh.num_kv_heads, 128, dev)
        out = torch.empty(sh.batch, sh.num_q_heads, 128, dtype=torch.bfloat16, device=dev)
        fn = lambda: ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                           x["seq_lens"], out=out, scale=1 / math.sqrt(128),
                                           workspace=ws, stream=st, num_sms=72, pdl=True)
        ov = coloc.run_under_prefill(st, fn, 20, pre_stream, pre, 16)
        mb = kv_read_bytes(sh) / 1e6
        print(f"attn priority {prio:3d} {sh.name:16s}: beside prefill {ov.attn_s * 1e6:8.1f} us "
              f"({mb / (ov.attn_s * 1e6):5.2f} TB/s), prefill iter {ov.prefill_s * 1e3:.2f} ms", flush=True)
