#!/usr/bin/env python
"""Per-layer CPU launch cost vs GPU time of a small decode step, ungraphed vs
graphed (the reference's launch_overhead model, costs.py:94-108; PAPER.md:378:
0.38 ms GPU vs 1.137 ms CPU per layer on A100 at batch 8, seq 1K)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.runtime import CapturedStep
from paper_2503_20552_b200.synthetic import DecodeShape, make_block_table, make_layer

def measure(B, ctx, L=32, iters=50):
    dev = torch.device("cuda:0")
    shape = DecodeShape("small", B, 32, 32, 128, L, ctx)
    bt = make_block_table(shape)
    layers = [make_layer(shape, dev, seed=l, block_table=bt) for l in range(L)]
    slots = ops.slot_mapping(layers[0]["block_table"], layers[0]["seq_lens"].long() - 1)
    ws = ops.DecodeWorkspace(B, 32, 32, 128, dev)
    outs = [torch.empty(B, 32, 128, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    def step():
        for x, o in zip(layers, outs):
            ops.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
            ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"], out=o, workspace=ws)
    for _ in range(3): step()
    torch.cuda.synchronize()
    # CPU issue cost per layer (host wall time of enqueueing, GPU not waited)
    t0 = time.perf_counter(); step(); cpu_issue = (time.perf_counter() - t0) / L
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): step()
    e.record(); torch.cuda.synchronize()
    eager = s.elapsed_time(e) / iters / 1e3
    cap = CapturedStep(step)
    s.record()
    for _ in range(iters): cap.replay()
    e.record(); torch.cuda.synchronize()
    graphed = s.elapsed_time(e) / iters / 1e3
    return {"batch": B, "ctx": ctx, "layers": L, "cpu_issue_s_per_layer": cpu_issue,
            "eager_step_s": eager, "graphed_step_s": graphed, "graph_speedup": eager / graphed,
            "gpu_s_per_layer_graphed": graphed / L}

res = [measure(8, 1024), measure(64, 1024), measure(64, 4096)]
print(json.dumps(res, indent=1))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/launch_overhead.json").write_text(json.dumps(res, indent=1))
