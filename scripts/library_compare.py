#!/usr/bin/env python
"""Same decode batches through our kernel and through the library decode kernels in
this image, timed the same way (GPU box only; secondary evidence, not the product):

* vLLM ``paged_attention_v2`` — the kernel family the paper's prototype runs
  (vLLM v0.6.3); its cache layout is converted once, outside the timing.
* FlashInfer ``trtllm_batch_decode_with_kv_cache`` (TRT-LLM-gen cubins for sm_100,
  HND layout = ours, zero conversion).
* FlashInfer ``BatchDecodeWithPagedKVCacheWrapper`` (its own CUDA decode kernel).

Each library output is also compared with ours (a cross-check of the attention
arithmetic beside the oracle gate). Every timing cycles ``--layers`` distinct
layer caches (>> L2) with CUDA events, after warm-up.

    python scripts/library_compare.py [--configs C2,C3,C5] [--layers 8] [out.json]
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import traceback
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_20552_b200 import ops  # noqa: E402
from paper_2503_20552_b200.synthetic import (CONFIGS, algorithmic_bytes, kv_read_bytes,  # noqa: E402
                                              make_layer)


def timeit(fn, n_layers: int, reps: int, warm: int = 3) -> float:
    """Average ms per call over reps x n_layers calls (layer index cycles)."""
    for i in range(warm * n_layers):
        fn(i % n_layers)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for r in range(reps):
        for i in range(n_layers):
            fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (reps * n_layers)


def diff(a: torch.Tensor, ref: torch.Tensor) -> dict:
    a, ref = a.float(), ref.float()
    return {"max_abs": float((a - ref).abs().max()),
            "mean_rel": float((a - ref).abs().sum() / ref.abs().sum())}


def run_config(name: str, n_layers: int, reps: int, only: str = "") -> dict:
    import re
    from paper_2503_20552_b200.synthetic import DecodeShape
    m = re.fullmatch(r"B(\d+)c(\d+)k(\d+)", name)  # ad-hoc shape, e.g. B8c1024k8 (Hq 32, D 128)
    shape = CONFIGS[name] if m is None else DecodeShape(name, int(m[1]), 32, int(m[3]), 128, 1,
                                                        int(m[2]))
    dev = torch.device("cuda:0")
    B, Hq, Hkv, D = shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
    scale = 1.0 / math.sqrt(D)
    layers = [make_layer(shape, dev, seed=i) for i in range(n_layers)]
    bt, sl = layers[0]["block_table"], layers[0]["seq_lens"]
    kvb, algb = kv_read_bytes(shape), algorithmic_bytes(shape)
    res = {"shape": f"B={B} ctx={shape.ctx} Hq={Hq} Hkv={Hkv} D={D} page=16",
           "layers_cycled": n_layers, "kv_bytes_per_call": kvb, "impls": {}}

    def record(impl, ms, out=None, note=None):
        row = {"us_per_call": 1e3 * ms, "kv_GBps": kvb / ms / 1e6}
        if out is not None:
            row["vs_ours"] = diff(out, ours_out)
        if note:
            row["note"] = note
        res["impls"][impl] = row
        print(name, impl, json.dumps(row), flush=True)

    ws = ops.DecodeWorkspace(B, Hq, Hkv, D, dev)
    outs = [torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev) for _ in range(2)]

    def ours(i, pdl=True):
        x = layers[i]
        ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], bt, sl, out=outs[i & 1],
                              scale=scale, workspace=ws, pdl=pdl)
    ours(0, pdl=False)
    torch.cuda.synchronize()
    ours_out = outs[0].clone()
    record("ours (adr_paged_decode_attn)", timeit(ours, n_layers, reps))
    record("ours, no PDL", timeit(lambda i: ours(i, pdl=False), n_layers, reps))

    # --- FlashInfer TRT-LLM-gen decode (HND == our layout) ---
    try:
        if only and only != "trt":
            raise RuntimeError("skipped (--only)")
        import flashinfer
        fw = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
        fo = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev)
        max_len = int(sl.max())

        def trt(i):
            x = layers[i]
            flashinfer.decode.trtllm_batch_decode_with_kv_cache(
                x["q"], (x["k_cache"], x["v_cache"]), fw, bt, sl, max_len,
                bmm1_scale=scale, bmm2_scale=1.0, out=fo, kv_layout="HND")
        trt(0)
        torch.cuda.synchronize()
        first = fo.clone()
        record("flashinfer trtllm-gen decode", timeit(trt, n_layers, reps), first)
    except Exception as ex:  # library path unavailable on this box: say so
        res["impls"]["flashinfer trtllm-gen decode"] = {"error": repr(ex)[:300]}
        traceback.print_exc()

    # --- FlashInfer BatchDecode wrapper (auto backend) ---
    try:
        if only and only != "fi":
            raise RuntimeError("skipped (--only)")
        import flashinfer
        fw2 = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(fw2, kv_layout="HND",
                                                          use_tensor_cores=Hq // Hkv >= 4)
        npg = (sl + 15) // 16
        indptr = torch.zeros(B + 1, dtype=torch.int32, device=dev)
        indptr[1:] = torch.cumsum(npg, 0)
        idx = torch.cat([bt[b, :int(npg[b])] for b in range(B)]).to(torch.int32)
        last = ((sl - 1) % 16 + 1).to(torch.int32)
        w.plan(indptr, idx, last, Hq, Hkv, D, 16, q_data_type=torch.bfloat16,
               kv_data_type=torch.bfloat16, sm_scale=scale)
        fo2 = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev)

        def fib(i):
            x = layers[i]
            w.run(x["q"], (x["k_cache"], x["v_cache"]), out=fo2)
        fib(0)
        torch.cuda.synchronize()
        first = fo2.clone()
        record("flashinfer BatchDecode", timeit(fib, n_layers, reps), first)
    except Exception as ex:
        res["impls"]["flashinfer BatchDecode"] = {"error": repr(ex)[:300]}
        traceback.print_exc()

    # --- vLLM paged_attention_v2 (the paper prototype's kernel family) ---
    try:
        if only and only != "vllm":
            raise RuntimeError("skipped (--only)")
        import vllm._custom_ops as vops
        x8 = 8
        vk = [l["k_cache"].view(-1, Hkv, 16, D // x8, x8).permute(0, 1, 3, 2, 4).contiguous()
              for l in layers[:min(n_layers, 4)]]
        vv = [l["v_cache"].permute(0, 1, 3, 2).contiguous() for l in layers[:min(n_layers, 4)]]
        nl = len(vk)
        max_len = int(sl.max())
        P = 512
        nparts = (max_len + P - 1) // P
        vo = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev)
        es = torch.empty(B, Hq, nparts, dtype=torch.float32, device=dev)
        ml = torch.empty_like(es)
        tmp = torch.empty(B, Hq, nparts, D, dtype=torch.bfloat16, device=dev)
        one = torch.ones((), dtype=torch.float32, device=dev)

        def vl(i):
            vops.paged_attention_v2(vo, es, ml, tmp, layers[i]["q"], vk[i], vv[i], Hkv, scale,
                                    bt, sl, 16, max_len, None, "auto", one, one)
        vl(0)
        torch.cuda.synchronize()
        first = vo.clone()
        record("vllm paged_attention_v2", timeit(vl, nl, max(1, reps * n_layers // nl)), first,
               note=f"{nl} layer caches cycled (converted layout copies)")
        del vk, vv
    except Exception as ex:
        res["impls"]["vllm paged_attention_v2"] = {"error": repr(ex)[:300]}
        traceback.print_exc()
    del layers
    torch.cuda.empty_cache()
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C5")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="", help="trt | fi | vllm: run ours + that library only")
    ap.add_argument("out", nargs="?", default="gpurun_out/library_compare.json")
    a = ap.parse_args()
    out = {"gpu": torch.cuda.get_device_name(0), "configs": {}}
    for name in a.configs.split(","):
        out["configs"][name] = run_config(name, a.layers, a.reps, a.only)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
