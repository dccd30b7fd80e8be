#!/usr/bin/env python
"""Small decode calls: how much of the per-call time is the GPU, how much the host.

For each shape, per call (µs), 8 distinct layer caches cycled:
  * ``loop``  — calls issued from a Python loop (what library_compare / size_scaling time:
    includes the host cost of each call if it exceeds the GPU's)
  * ``graph`` — the same chain captured once in a CUDA graph and replayed (GPU-side cost only)
for our kernel (PDL chain and plain) and FlashInfer's TRT-LLM-gen decode, plus the host
cost of one ``ops.paged_decode_attn`` call and a trivial-kernel graph chain (the floor).

    python scripts/small_call_bench.py [--shapes B8c1024k8,...] [--reps 20] [out.json]
"""
from __future__ import annotations

import argparse
import json
import math
import re
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_20552_b200 import ops  # noqa: E402
from paper_2503_20552_b200.synthetic import DecodeShape, kv_read_bytes, make_block_table, make_layer  # noqa: E402

DEFAULT = ("B4c512k8,B8c1024k8,B16c1024k8,B4c512k32,B8c1024k32,B16c1024k32,B64c1024k8,"
           "B32c2048k8,B64c4096k8,B64c4096k32")


def graph_time(fn, n_layers: int, reps: int) -> float:
    """µs per call of fn(0..n_layers-1) x reps captured in one CUDA graph."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(n_layers):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            for i in range(n_layers):
                fn(i)
    g.replay()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (reps * n_layers))
    return best


def loop_time(fn, n_layers: int, reps: int) -> float:
    for i in range(3 * n_layers):
        fn(i % n_layers)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for i in range(n_layers):
            fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n_layers)


def host_time(fn, n: int = 400) -> float:
    """µs of host time per call (GPU kept ahead: measured on a long chain)."""
    fn(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        fn(i & 7)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) * 1e6 / n


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--no-trt", action="store_true")
    ap.add_argument("--grids", default="auto", help="comma list of ops grid modes to time")
    ap.add_argument("--no-floor", action="store_true")
    ap.add_argument("--no-host", action="store_true")
    ap.add_argument("out", nargs="?")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []

    if not a.no_floor:
        # floor: a trivial kernel of ours (one-row kv_append) chained in a graph
        sh = DecodeShape("floor", 1, 8, 8, 128, 1, 16)
        x = make_layer(sh, dev, seed=0)
        slots = torch.zeros(1, dtype=torch.int64, device=dev)
        floor = graph_time(lambda i: ops.kv_append(x["k_new"], x["v_new"], x["k_cache"],
                                                   x["v_cache"], slots), 8, 50)
        print(json.dumps({"floor_kernel_graph_us": floor}), flush=True)
        rows.append({"floor_kernel_graph_us": floor})

    for name in a.shapes.split(","):
        m = re.fullmatch(r"B(\d+)c(\d+)k(\d+)(?:q(\d+))?", name)  # q: Hq (default 32)
        B, ctx, Hkv = int(m[1]), int(m[2]), int(m[3])
        Hq = int(m[4]) if m[4] else 32
        sh = DecodeShape(name, B, Hq, Hkv, 128, 1, ctx)
        bt = make_block_table(sh)
        ls = [make_layer(sh, dev, seed=l, block_table=bt) for l in range(a.layers)]
        bt, sl = ls[0]["block_table"], ls[0]["seq_lens"]
        ws = ops.DecodeWorkspace(B, Hq, Hkv, 128, dev, max_blocks_per_seq=bt.shape[1])
        out = torch.empty(B, Hq, 128, dtype=torch.bfloat16, device=dev)
        scale = 1.0 / math.sqrt(128)
        row = {"shape": name, "MB": kv_read_bytes(sh) / 1e6}

        for grid in a.grids.split(","):
            def ours(i, pdl=True, grid=grid):
                y = ls[i]
                ops.paged_decode_attn(y["q"], y["k_cache"], y["v_cache"], bt, sl, out=out,
                                      scale=scale, workspace=ws, k_new=y["k_new"],
                                      v_new=y["v_new"], pdl=pdl, grid=grid)
            sfx = "" if grid == "auto" else "_" + grid
            row["ours_graph_pdl" + sfx] = graph_time(ours, a.layers, a.reps)
            row["ours_graph_nopdl" + sfx] = graph_time(lambda i: ours(i, False), a.layers, a.reps)
            if not a.no_host:
                row["ours_loop_pdl" + sfx] = loop_time(ours, a.layers, a.reps)
                row["ours_host_us" + sfx] = host_time(ours)
        if not a.no_trt:
            try:
                import flashinfer
                fw = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
                fo = torch.empty(B, Hq, 128, dtype=torch.bfloat16, device=dev)
                max_len = int(sl.max())

                def trt(i):
                    y = ls[i]
                    flashinfer.decode.trtllm_batch_decode_with_kv_cache(
                        y["q"], (y["k_cache"], y["v_cache"]), fw, bt, sl, max_len,
                        bmm1_scale=scale, bmm2_scale=1.0, out=fo, kv_layout="HND")
                try:
                    row["trt_graph"] = graph_time(trt, a.layers, a.reps)
                except Exception as ex:  # noqa: BLE001
                    row["trt_graph"] = repr(ex)[:200]
                if not a.no_host:
                    row["trt_loop"] = loop_time(trt, a.layers, a.reps)
                    row["trt_host_us"] = host_time(trt)
            except Exception as ex:  # noqa: BLE001
                row["trt_error"] = repr(ex)[:200]
        for k in [k for k in row if "graph" in k]:
            if isinstance(row.get(k), float):
                row[k.replace("graph", "GBps")] = row["MB"] / row[k] * 1e3
        print(json.dumps(row), flush=True)
        rows.append(row)
        del ls, ws
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
