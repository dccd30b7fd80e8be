#!/usr/bin/env python
"""C3 offload sweep on ONE B200 (BASELINE configs[2] needs 1 decode + 1 prefill
GPU; with one GPU the executor runs in a green-context partition of the same
GPU and the q/k/v / output messages go through the loopback transport).

For each offloaded share of a 64-request Llama-3-8B decode batch (ctx 4096, 32
layers) it times the full offloaded step (pack -> send -> executor fused
append + attention -> return -> scatter, overlapped with local attention) and
reports step time, tokens/s, link bytes and the measured stall. Both sides
share one HBM here, so this measures the exchange/overlap machinery, not the
capacity gain of a second GPU.
"""
import json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2503_20552_b200 import coloc, ops
from paper_2503_20552_b200.kvcache import BlockTables, PagePool
from paper_2503_20552_b200.runtime import AttentionExecutor, LayeredKV, OffloadedDecodeStep, StepPlan

dev = torch.device("cuda:0")
B, Hq, Hkv, D, L, ctx = 64, 32, 8, 128, 32, 4096
pages_per_req = ctx // 16
g = torch.Generator(device=dev).manual_seed(0)
local_kv = LayeredKV(L, B * pages_per_req + 64, Hkv, D, dev, fill="randn", generator=g)
exec_kv = LayeredKV(L, B * pages_per_req + 64, Hkv, D, dev, fill="randn", generator=g)
mk = lambda *s: torch.randn(*s, generator=g, device=dev).to(torch.bfloat16)
qs = [mk(B, Hq, D) for _ in range(L)]
ks = [mk(B, Hkv, D) for _ in range(L)]
vs = [mk(B, Hkv, D) for _ in range(L)]
outs = [torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev) for _ in range(L)]
part = coloc.SmPartition(0, 64) if coloc.green_contexts_supported() else None
res = {"shape": f"B={B} ctx={ctx} Hq={Hq} Hkv={Hkv} D={D} L={L}",
       "executor": f"green context {part.attn_sms} SMs" if part else "side stream", "points": []}
for n_off in (0, 8, 16, 24, 32):
    nl = B - n_off
    lt, xt = BlockTables(PagePool(local_kv.num_pages)), BlockTables(PagePool(exec_kv.num_pages))
    for i in range(nl):
        lt.reserve(i, ctx)
    for i in range(n_off):
        xt.reserve(i, ctx)
    t = lambda a: torch.from_numpy(a).to(dev)
    plan = StepPlan(nl, n_off, t(lt.table_array(list(range(nl)))) if nl else None,
                    torch.full((nl,), ctx, dtype=torch.int32, device=dev),
                    torch.zeros(nl, dtype=torch.int64, device=dev),
                    t(xt.table_array(list(range(n_off)))) if n_off else None,
                    torch.full((n_off,), ctx, dtype=torch.int32, device=dev) if n_off else None,
                    torch.zeros(n_off, dtype=torch.int64, device=dev) if n_off else None)
    local = AttentionExecutor(local_kv, Hq, B)
    remote = AttentionExecutor(exec_kv, Hq, B, stream=part.attn_stream if part else None,
                               num_sms=part.attn_sms if part else 0) if n_off else None
    step = OffloadedDecodeStep(Hq, Hkv, D, local, remote)
    for _ in range(2):
        step.run(qs, ks, vs, plan, outs)
    times = [step.run(qs, ks, vs, plan, outs) for _ in range(5)]
    tot = sorted(x.total for x in times)[2]
    pt = {"n_offloaded": n_off, "offload_ratio": n_off / max(1, nl), "step_ms": tot * 1e3,
          "tokens_per_s": B / tot, "local_attn_ms": times[2].local_attn * 1e3,
          "exec_attn_ms": times[2].exec_attn * 1e3, "stall_ms": times[2].stall * 1e3,
          "link_bytes_per_step": times[2].link_bytes,
          "kv_GBps": B * ctx * Hkv * D * 4 * L / tot / 1e9}
    res["points"].append(pt)
    print(json.dumps(pt), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/offload_sweep.json").write_text(json.dumps(res, indent=1))
