#!/usr/bin/env python
"""Per-call time of adr_paged_decode_attn (fused append, PDL chain over 8
distinct layer caches) on the BASELINE decode shapes, for the kernel knobs
in the environment (ADR_PREFETCH_UNITS, ADR_CHUNK_MIN, ADR_CHUNKS_PER_WARP,
ADR_SPLIT_RULE, ADR_DECODE_VARIANT). Runs each setting in a fresh process:

    python scripts/knob_sweep.py ADR_PREFETCH_UNITS=0,4,8,16 [--configs C2,C3,C5,B8c1024k8]
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(configs, layers=8, reps=10):
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_2503_20552_b200 import ops
    from paper_2503_20552_b200.synthetic import CONFIGS, kv_read_bytes, make_block_table, make_layer
    dev = torch.device("cuda:0")
    res = {}
    import re
    from paper_2503_20552_b200.synthetic import DecodeShape
    for name in configs:
        m = re.fullmatch(r"B(\d+)c(\d+)k(\d+)", name)  # e.g. B8c1024k8: Hq 32, D 128
        sh = CONFIGS[name] if m is None else DecodeShape(name, int(m[1]), 32, int(m[3]), 128, 8,
                                                         int(m[2]))
        bt = make_block_table(sh)
        ls = [make_layer(sh, dev, seed=l, block_table=bt) for l in range(layers)]
        workers = int(os.environ.get("KS_WORKERS", "0"))  # explicit grid warps (0: persistent)
        ws = [ops.DecodeWorkspace(sh.batch, sh.num_q_heads, sh.num_kv_heads, sh.head_dim, dev,
                                  num_workers=workers) for _ in range(2)]
        out = torch.empty(sh.batch, sh.num_q_heads, sh.head_dim, dtype=torch.bfloat16, device=dev)

        def run():
            for l, x in enumerate(ls):
                ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                      x["seq_lens"], out=out, workspace=ws[l % 2],
                                      k_new=x["k_new"], v_new=x["v_new"], pdl=True)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
        res[name] = {"us": round(us, 1), "kv_GBps": round(kv_read_bytes(sh) / us / 1e3, 1)}
        del ls, ws, out
        torch.cuda.empty_cache()
    print(json.dumps(res))


def main():
    args = sys.argv[1:]
    if args and args[0] == "--child":
        child(args[1].split(","))
        return
    configs = "C2,C3,C5"
    if "--configs" in args:
        i = args.index("--configs")
        configs = args[i + 1]
        args = args[:i] + args[i + 2:]
    settings = [{}]
    for spec in args:
        key, vals = spec.split("=")
        settings = [dict(s, **{key: v}) for s in settings for v in vals.split(",")]
    for s in settings:
        env = dict(os.environ, **s)
        r = subprocess.run([sys.executable, __file__, "--child", configs], env=env,
                           capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
        print(json.dumps(s), line, flush=True)


if __name__ == "__main__":
    main()
