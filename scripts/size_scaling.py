#!/usr/bin/env python
"""Per-launch time of chained adr_paged_decode_attn calls vs problem size:
fit t = a + bytes / BW to separate the fixed per-call cost from streaming."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.synthetic import DecodeShape, kv_read_bytes, make_block_table, make_layer

dev = torch.device("cuda:0")
rows = []
for Hkv in (8, 32):
    for B, ctx in ((4, 512), (8, 1024), (16, 1024), (40, 2048), (64, 1024), (64, 4096), (128, 4096)):
        sh = DecodeShape("s", B, 32, Hkv, 128, 8, ctx)
        bt = make_block_table(sh)
        ls = [make_layer(sh, dev, seed=l, block_table=bt) for l in range(8)]
        ws = [ops.DecodeWorkspace(B, 32, Hkv, 128, dev) for _ in range(2)]
        out = torch.empty(B, 32, 128, dtype=torch.bfloat16, device=dev)
        res = {}
        for pdl in (False, True):
            def run():
                for l, x in enumerate(ls):
                    ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                                          out=out, workspace=ws[l % 2], k_new=x["k_new"], v_new=x["v_new"], pdl=pdl)
            run(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): run()
            e1.record(); torch.cuda.synchronize()
            res[pdl] = e0.elapsed_time(e1) / 80 * 1e3
        nbytes = kv_read_bytes(sh)
        rows.append({"Hkv": Hkv, "B": B, "ctx": ctx, "MB": nbytes / 1e6, "us": res[False], "us_pdl": res[True],
                     "GBps_pdl": nbytes / res[True] / 1e3})
        print(json.dumps(rows[-1]), flush=True)
        del ls, ws
        torch.cuda.empty_cache()
for key in ("us", "us_pdl"):
    x = np.array([r["MB"] for r in rows]); y = np.array([r[key] for r in rows])
    A = np.vstack([np.ones_like(x), x]).T
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    print(key, "fixed us", round(a, 2), "stream GB/s", round(1e3 / b, 0))
