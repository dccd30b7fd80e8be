#!/usr/bin/env python
"""Benchmark of the offloaded decode-attention hot path on B200.

One *step* = one decode step of the attention path over one batch: for each of
the L layers, one adr_paged_decode_attn call that appends the step's new K/V
rows into the paged cache and attends over every request's context (fused),
the layers chained with programmatic dependent launch. Workload (BASELINE.json
configs[1], "C2"): Llama-2-7B attention shapes, 32 heads MHA x 128, batch 64,
context 4096, 32 layers, bf16 paged KV (137 GB of KV, resident in HBM).

metric  = decode-attn KV GB/s: KV bytes read per step / step time (whole job,
          summed over ranks; N>1 runs independent request shards, weak scaling)
e2e     = the same metric through the public API with HOST buffers: the step's
          q/k/v rows are copied from pinned memory and the outputs copied back
          inside the timed region
roofline= algorithmic bytes of one adr_paged_decode_attn call /
          its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs

`--impl reference` times the reference arm: the CPU restatement of the path
(oracle/attn_oracle.c; the reference itself is a Python simulator with no
attention arithmetic) on this host's cores, on bounded samples of the same
workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2503_20552_b200.synthetic import (CONFIGS, algorithmic_bytes, kv_read_bytes,  # noqa: E402
                                             make_block_table, make_layer)

METRIC = "decode-attn KV GB/s"
UNIT = "GB/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        if self.proc is None or self.path is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [n for i, n in enumerate(names) if any(r[2 + i] == "Active" for r in rows)]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        # one process per GPU over NCCL; ranks sharing a GPU (a 1-GPU smoke run of
        # the zero-copy role split, whose data path is CUDA IPC) fall back to gloo
        backend = "nccl" if ndev >= world else "gloo"
        if ndev:
            local = local % ndev
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU side (oracle): cpu_baseline leg and the reference arm
# ---------------------------------------------------------------------------

_CPU_SAMPLES: dict = {}


def cpu_sample_rate(shape, budget_s: float, seed: int = 0, max_requests: int = 8) -> dict:
    """KV GB/s of the CPU restatement (oracle/attn_oracle.c, all host threads) on
    a bounded sample of `shape`: the first `max_requests` requests of one layer,
    run repeatedly until `budget_s` seconds of CPU work are spent."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    from dataclasses import replace
    threads = orc.max_threads()
    scale = 1.0 / math.sqrt(shape.head_dim)
    nreq = min(max_requests, shape.batch)
    sub = replace(shape, batch=nreq,
                  ctx=shape.ctx if isinstance(shape.ctx, int) else tuple(shape.ctx_list()[:nreq]))
    key = (shape.name, nreq, seed)
    if key not in _CPU_SAMPLES:  # build the sample once per process
        _CPU_SAMPLES[key] = make_layer(sub, "cpu", seed=seed)
    x = _CPU_SAMPLES[key]
    done_bytes, done_s, runs = 0, 0.0, 0
    while done_s < budget_s:
        t0 = time.perf_counter()
        orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                              scale, num_threads=threads)
        done_s += time.perf_counter() - t0
        done_bytes += kv_read_bytes(sub)
        runs += 1
    return {"value": done_bytes / done_s / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{runs} runs of the CPU restatement over {nreq} of {shape.batch} requests of "
                      f"one {shape.name} layer ({kv_read_bytes(sub) / 1e9:.2f} GB of bf16 KV per "
                      f"run, {done_s:.1f} s total, double accumulation, {threads} threads)"}


def host_cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def decision_timings(budget_s: float = 2.0) -> dict:
    """BASELINE.md §4 CPU items 2-3, single-threaded on this host: Algorithm 1
    (need_offload, scheduling.py:176-221; this package's restatement is the
    reference's code path, pinned bit-exact to it) in microseconds per decision
    at |offloaded| = |local| = 8 / 64 / 256 — literal form and the O(1)
    OffloadLedger — and simulate() wall time on the survey's determinism case
    (sharegpt_like, rate 3, 300 requests, seed 7, A100 defaults)."""
    from paper_2503_20552_b200 import config, engine, scheduling, workload
    res = {"need_offload_us": {}, "ledger_us": {}}
    for n in (8, 64, 256):
        mk = lambda i: scheduling.Request(i, 0.0, 200 + i % 50, 100 + i % 30)
        off, loc = [mk(i) for i in range(n)], [mk(n + i) for i in range(n)]
        for r in off + loc:
            r.used_token = r.prompt_tokens
        req = mk(2 * n)
        led = scheduling.OffloadLedger.of(off, loc)
        for key, fn in (("need_offload_us", lambda: scheduling.need_offload(req, off, loc, 0.5)),
                        ("ledger_us", lambda: led.decide(req, 0.5))):
            k, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < budget_s / 6:
                for _ in range(100):
                    fn()
                k += 100
            res[key][str(n)] = (time.perf_counter() - t0) / k * 1e6
    cfg = config.SimConfig()
    reqs = workload.synth_requests(workload.preset("sharegpt_like", 3.0, 300), 7)
    t0 = time.perf_counter()
    engine.simulate(cfg, reqs)
    res["simulate_s"] = time.perf_counter() - t0
    res["simulate_case"] = "sharegpt_like rate 3, 300 requests, seed 7, SimConfig() defaults"
    return res


def run_reference(args, shape, world, rank):
    if rank != 0:
        return
    budget = max(1.0, min(10.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample_rate(shape, 0.1, max_requests=shape.batch)
    vals = []
    t0 = time.perf_counter()
    info = None
    for _ in range(args.steps):
        info = cpu_sample_rate(shape, budget, max_requests=shape.batch)
        vals.append(info["value"])
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    cpu = dict(info, value=value, cpu_model=host_cpu_model(), decisions=decision_timings())
    # one real step of this workload = every layer's KV at the measured CPU rate
    step_ms = kv_read_bytes(shape) * shape.num_layers / (value * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "sample_wall_ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": config_dict(shape, args),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "CPU restatement of the path (oracle/attn_oracle.c): the reference "
                "(adrenaline_sim) prices attention analytically and has no attention kernel",
    }
    print(json.dumps(line), flush=True)


def config_dict(shape, args) -> dict:
    return {"workload": f"{shape.name}: decode attention (KV append + paged attention), "
                        f"B={shape.batch} ctx={shape.ctx if isinstance(shape.ctx, int) else 'ragged'}"
                        f" Hq={shape.num_q_heads} Hkv={shape.num_kv_heads} D={shape.head_dim} "
                        f"L={shape.num_layers} page=16 bf16, local-only per GPU",
            "global_batch": shape.batch * args.gpus, "seq_len": shape.ctx if isinstance(shape.ctx, int) else None,
            "layers": shape.num_layers, "parallelism": f"request-sharded x{args.gpus} (no collective)",
            "l2": "inputs larger than L2 (KV per layer >> 126 MB; 32 distinct layer caches)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(args, shape, world, rank, local):
    from paper_2503_20552_b200 import ops
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    L = shape.num_layers
    B, Hq, Hkv, D = shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim
    scale = 1.0 / math.sqrt(D)
    bt = make_block_table(shape, seed=1 + rank)
    log(f"[rank {rank}] allocating {L} layers x {2 * shape.num_pages * Hkv * 16 * D * 2 / 2**30:.1f}"
        f" GiB of paged KV")
    layers = [make_layer(shape, dev, seed=1000 * rank + l, block_table=bt) for l in range(L)]
    # two workspaces, alternated by layer: a PDL-launched layer may start while the
    # previous one drains, so consecutive calls never share split-pair scratch
    ws = [ops.DecodeWorkspace(B, Hq, Hkv, D, dev) for _ in range(2)]
    outs = [torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    stream = torch.cuda.current_stream(dev)

    def layer_call(l, x, seq):
        # fused KV append of this step's token + paged attention, chained with PDL
        ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], seq,
                              out=outs[l], scale=scale, workspace=ws[l % 2],
                              k_new=x["k_new"], v_new=x["v_new"], pdl=not args.no_pdl)

    def step():
        for l, x in enumerate(layers):
            layer_call(l, x, x["seq_lens"])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timing ----
    # The step is nothing but L adr_paged_decode_attn launches on `stream`, so the
    # kernel's average launch duration is the event-timed region / launches
    # (per-launch events would break the PDL chain).
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    local_ms = t_start.elapsed_time(t_end)
    elapsed_ms = max_over_ranks(local_ms, world, dev)
    attn_avg_ms = local_ms / (args.steps * L)
    # isolated single-call duration (plain launch, events around each call), for reference
    iso = []
    for l, x in enumerate(layers[:8]):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                              x["seq_lens"], out=outs[l], scale=scale, workspace=ws[0],
                              k_new=x["k_new"], v_new=x["v_new"])
        e1.record(stream)
        iso.append((e0, e1))
    torch.cuda.synchronize()
    iso_ms = statistics.median(a.elapsed_time(b) for a, b in iso)

    kv_bytes_step = kv_read_bytes(shape) * L
    ms_per_step = elapsed_ms / args.steps
    value = kv_bytes_step * world / (ms_per_step / 1e3) / 1e9
    tokens_per_s = B * world / (ms_per_step / 1e3)

    # ---- end-to-end through the public API with host buffers ----
    # Every step copies all its inputs (each layer's q / k_new / v_new rows and
    # the lengths) from pinned host memory and every layer's output back. The
    # copies run on their own streams (H2D and D2H copy engines) beside the
    # attention chain: a layer's kernel waits for its inputs, its output leaves
    # as soon as its group of layers is done. Steps stay serialised like real
    # decoding: a step's first input copy waits until the previous step's last
    # output has reached the host.
    h_q = [x["q"].cpu().pin_memory() for x in layers]
    h_k = [x["k_new"].cpu().pin_memory() for x in layers]
    h_v = [x["v_new"].cpu().pin_memory() for x in layers]
    h_out = [torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory() for _ in range(L)]
    h_seq = layers[0]["seq_lens"].cpu().pin_memory()
    d_seq = torch.empty_like(layers[0]["seq_lens"])
    h2d = sum(t.numel() * t.element_size() for t in h_q + h_k + h_v) + h_seq.numel() * 4
    d2h = sum(t.numel() * t.element_size() for t in h_out)
    in_groups = e2e_groups(L, [1, 4])          # layer 0 | 1-3 | the rest
    out_groups = e2e_groups(L, [L // 2, L - 4, L - 1])
    cs_in, cs_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in in_groups]
    ev_k = [torch.cuda.Event() for _ in out_groups]
    d2h_done = torch.cuda.Event()
    d2h_done.record(cs_out)
    in_first = {g[0]: i for i, g in enumerate(in_groups)}
    out_last = {g[-1]: i for i, g in enumerate(out_groups)}

    def e2e_step():
        cs_in.wait_event(d2h_done)  # the previous step's results are on the host
        with torch.cuda.stream(cs_in):
            for i, grp in enumerate(in_groups):
                if i == 0:
                    d_seq.copy_(h_seq, non_blocking=True)
                for l in grp:
                    layers[l]["q"].copy_(h_q[l], non_blocking=True)
                    layers[l]["k_new"].copy_(h_k[l], non_blocking=True)
                    layers[l]["v_new"].copy_(h_v[l], non_blocking=True)
                ev_in[i].record(cs_in)
        for l, x in enumerate(layers):
            if l in in_first:
                stream.wait_event(ev_in[in_first[l]])
            layer_call(l, x, d_seq)
            if l in out_last:
                j = out_last[l]
                ev_k[j].record(stream)
                cs_out.wait_event(ev_k[j])
                with torch.cuda.stream(cs_out):
                    for m in out_groups[j]:
                        h_out[m].copy_(outs[m], non_blocking=True)
        d2h_done.record(cs_out)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    # bit-exact check of the overlapped path: the host copies hold this step's outputs
    for l in (0, L - 1):
        assert torch.equal(h_out[l], outs[l].cpu()), "e2e host output differs from the device output"
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    stream.wait_event(d2h_done)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    e2e_value = kv_bytes_step * world / (e2e_ms / 1e3) / 1e9

    # ---- full decode layers: synthetic non-attention GEMMs around the same attention ----
    full = None
    if not args.no_full_layer:
        try:
            full = full_layer_step(args, shape, layers, dev, stream, ms_per_step, world)
        except (RuntimeError, ValueError) as e:  # secondary measurement: never lose the line
            full = {"error": str(e)[:300]}
            torch.cuda.empty_cache()

    # ---- the other decode shapes of BASELINE.json (kernel-level, 8 chained layers) ----
    del layers, outs, h_q, h_k, h_v, h_out
    torch.cuda.empty_cache()
    extra = {} if args.no_extra else other_configs(dev, scale_for=lambda D: 1.0 / math.sqrt(D))
    if not args.no_extra:
        try:
            extra["executor_calls"] = executor_calls(dev)
        except (RuntimeError, ValueError) as e:  # secondary measurement: never lose the line
            extra["executor_calls"] = {"error": str(e)[:300]}

    pk = peaks()
    alg = algorithmic_bytes(shape)
    achieved = alg / (attn_avg_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": config_dict(shape, args),
        "tokens_per_s": tokens_per_s,
        "frac_of_hbm_peak": {"measured": value / world / pk["hbm_gbs"], "nominal_8tbs": value / world / 8000.0},
        "roofline": {"bound": "hbm", "kernel": "adr_paged_decode_attn (fused KV append + stream-K attention + in-kernel LSE merge)",
                     "achieved": achieved, "peak": pk["hbm_gbs"], "peak_source": pk["source"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                     "frac_of_nominal_8tbs": achieved / 8000.0,
                     "traffic": load_traffic(), "bytes_per_launch": alg,
                     "avg_launch_ms": attn_avg_ms, "isolated_launch_ms": iso_ms,
                     "pdl": not args.no_pdl},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "copies": "pinned host <-> HBM on two copy streams beside the attention chain; "
                          "steps serialised (a step's inputs wait for the previous step's outputs)"},
        "gpu_launches": args.steps * L,
        "full_layer": full,
        "other_configs": extra,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample_rate(shape, args.cpu_budget, max_requests=shape.batch)
        cpu["cpu_model"] = host_cpu_model()
        cpu["decisions"] = decision_timings()
        line["cpu_baseline"] = cpu
    return line if rank == 0 else None


def full_layer_step(args, shape, layers, dev, stream, attn_ms_per_step, world) -> dict:
    """Decode tokens/s of full layers: decoder.SyntheticDecoder (RMSNorm, Q/K/V/O
    and gated-MLP cuBLAS GEMMs with random weights of the model's shapes, every
    layer its own weights) around the same adr_paged_decode_attn calls on the
    same KV caches, the whole step captured in one CUDA graph."""
    from paper_2503_20552_b200.decoder import MODEL_DIMS, SyntheticDecoder
    from paper_2503_20552_b200.runtime import CapturedStep
    model = {"C2": "llama2-7b", "C3": "llama3-8b"}.get(args.config)
    if model is None:  # 70B weights (141 GB) beside 172 GB of KV need tensor parallelism
        return {"skipped": f"no single-GPU full-layer model for {args.config}"}
    dims = MODEL_DIMS[model]
    if (dims.num_q_heads, dims.num_kv_heads, dims.head_dim) != (
            shape.num_q_heads, shape.num_kv_heads, shape.head_dim):
        raise ValueError("model dims differ from the decode shape")
    kv = [(x["k_cache"], x["v_cache"]) for x in layers]
    dec = SyntheticDecoder(dims, kv, shape.batch, dev, seed=7)
    bt, seq = layers[0]["block_table"], layers[0]["seq_lens"]
    g = torch.Generator(device=dev).manual_seed(3)
    x0 = torch.randn(shape.batch, dims.hidden, generator=g, device=dev).to(torch.bfloat16)
    x = x0.clone()

    def step():
        x.copy_(x0)
        dec.step(x, bt, seq, pdl=not args.no_pdl)
    graph = CapturedStep(step)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if not bool(torch.isfinite(x).all()):
        raise RuntimeError("full-layer step produced non-finite activations")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    wbytes = dec.weight_bytes()
    res = {"model": f"{model} layer shapes (synthetic weights, no RoPE), {dec.num_layers} layers",
           "ms_per_step": ms, "tokens_per_s": shape.batch * world / (ms / 1e3),
           "attention_share": attn_ms_per_step / ms,
           "nonattn_ms_per_step": ms - attn_ms_per_step,
           "weight_GB": wbytes / 1e9,
           "nonattn_weight_GBps": wbytes / ((ms - attn_ms_per_step) / 1e3) / 1e9,
           "graphed": True, "pdl": not args.no_pdl}
    del dec, graph
    torch.cuda.empty_cache()
    try:
        res["offload_loopback"] = full_layer_offload_step(args, shape, layers, dev, stream, ms,
                                                          world, dims, model)
    except (RuntimeError, ValueError) as e:  # secondary measurement: never lose the line
        res["offload_loopback"] = {"error": str(e)[:300]}
    return res


def full_layer_offload_step(args, shape, layers, dev, stream, plain_ms, world, dims, model) -> dict:
    """The same full-layer step with a quarter of the batch offloaded
    (decoder.OffloadedDecoder): per layer the executor attends the offloaded
    rows on its own stream with the zero-copy row-mapped kernel, beside the
    local attention, and the step is one CUDA graph over both streams. On one
    GPU (loopback) the executor shares this GPU's SMs and HBM and reads the
    offloaded requests' pages of the same caches (their pages are disjoint from
    the local rows'), so the KV bytes equal the plain step's: the difference to
    the plain step is the cost of the offload machinery (two grids per layer,
    cross-stream fork/join, row maps), not a capacity gain (which needs the
    second GPU)."""
    from paper_2503_20552_b200.decoder import OffloadedDecoder
    from paper_2503_20552_b200.runtime import CapturedStep
    B = shape.batch
    no = B // 4
    nl = B - no
    kv = [(x["k_cache"], x["v_cache"]) for x in layers]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    dec = OffloadedDecoder(dims, kv, kv, B, nl, dev, exec_sms=max(8, round(sms * no / B)), seed=7)
    bt, seq = layers[0]["block_table"], layers[0]["seq_lens"]
    tabs = (bt[:nl].contiguous(), seq[:nl].contiguous(), bt[nl:].contiguous(), seq[nl:].contiguous())
    g = torch.Generator(device=dev).manual_seed(3)
    x0 = torch.randn(B, dims.hidden, generator=g, device=dev).to(torch.bfloat16)
    x = x0.clone()

    def step():
        x.copy_(x0)
        dec.step(x, *tabs, pdl=not args.no_pdl)
    graph = CapturedStep(step)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if not bool(torch.isfinite(x).all()):
        raise RuntimeError("offloaded full-layer step produced non-finite activations")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    res = {"model": f"{model} layer shapes, {dec.num_layers} layers", "n_local": nl,
           "n_offloaded": no, "executor_sms": dec.exec_sms, "ms_per_step": ms,
           "tokens_per_s": B * world / (ms / 1e3), "vs_plain_full_layer": plain_ms / ms,
           "graphed": True, "streams": 2,
           "note": "1-GPU loopback: executor on a second stream of the same GPU, same KV bytes"}
    del dec, graph
    torch.cuda.empty_cache()
    return res


def e2e_groups(L: int, cuts) -> list:
    """Split layers 0..L-1 at the given cut points into consecutive groups."""
    edges = [0] + sorted({c for c in cuts if 0 < c < L}) + [L]
    return [list(range(a, b)) for a, b in zip(edges, edges[1:])]


def other_configs(dev, scale_for, layers: int = 8, reps: int = 5) -> dict:
    """KV GB/s of adr_paged_decode_attn (fused append, PDL chain) on the C3 and C5
    decode shapes: 8 distinct layer caches, chained, event-timed."""
    from paper_2503_20552_b200 import ops
    res = {}
    for name in ("C3", "C5"):
        sh = CONFIGS[name]
        bt = make_block_table(sh)
        ls = [make_layer(sh, dev, seed=l, block_table=bt) for l in range(layers)]
        ws = [ops.DecodeWorkspace(sh.batch, sh.num_q_heads, sh.num_kv_heads, sh.head_dim, dev)
              for _ in range(2)]
        out = torch.empty(sh.batch, sh.num_q_heads, sh.head_dim, dtype=torch.bfloat16, device=dev)

        def run():
            for l, x in enumerate(ls):
                ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                      x["seq_lens"], out=out, scale=scale_for(sh.head_dim),
                                      workspace=ws[l % 2], k_new=x["k_new"], v_new=x["v_new"],
                                      pdl=True)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        per_launch = e0.elapsed_time(e1) / 1e3 / (reps * layers)
        res[name] = {"shape": f"B={sh.batch} ctx={sh.ctx} Hq={sh.num_q_heads} Hkv={sh.num_kv_heads} "
                              f"D={sh.head_dim}", "us_per_layer": per_launch * 1e6,
                     "kv_GBps": kv_read_bytes(sh) / per_launch / 1e9,
                     "alg_GBps": algorithmic_bytes(sh) / per_launch / 1e9,
                     "tokens_per_s_attention_only": sh.batch / (per_launch * sh.num_layers)}
        del ls, ws, out
        torch.cuda.empty_cache()
    return res


# Offloaded batches an executor attends per layer (C3 / C4 head shapes): small calls,
# where the dispatcher picks the split-pair kernel (DESIGN §3 "small calls").
EXECUTOR_SHAPES = (("B8 ctx1024 GQA-4", 8, 32, 8, 1024), ("B16 ctx2048 GQA-4", 16, 32, 8, 2048),
                   ("B32 ctx4096 GQA-4", 32, 32, 8, 4096), ("B8 ctx1024 MHA-40", 8, 40, 40, 1024))


def executor_calls(dev, layers: int = 8, reps: int = 20) -> dict:
    """µs per call and KV GB/s of small decode calls: a PDL chain over 8 distinct
    layer caches captured in one CUDA graph (the GPU-side cost per call, as an
    executor replays it; an eager loop would time the host)."""
    from paper_2503_20552_b200 import ops
    from paper_2503_20552_b200.synthetic import DecodeShape
    res = {}
    for name, B, Hq, Hkv, ctx in EXECUTOR_SHAPES:
        sh = DecodeShape(name, B, Hq, Hkv, 128, 1, ctx)
        bt = make_block_table(sh)
        ls = [make_layer(sh, dev, seed=l, block_table=bt) for l in range(layers)]
        bt, sl = ls[0]["block_table"], ls[0]["seq_lens"]
        ws = [ops.DecodeWorkspace(B, Hq, Hkv, 128, dev, max_blocks_per_seq=bt.shape[1])
              for _ in range(2)]
        out = torch.empty(B, Hq, 128, dtype=torch.bfloat16, device=dev)

        def chain():
            for l, x in enumerate(ls):
                ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], bt, sl, out=out,
                                      scale=1.0 / math.sqrt(128), workspace=ws[l % 2],
                                      k_new=x["k_new"], v_new=x["v_new"], pdl=True)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            chain()
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                chain()
        g.replay()
        torch.cuda.synchronize(dev)
        best = float("inf")
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1) * 1e3 / (reps * layers))
        units = B * bt.shape[1] * Hkv
        res[name] = {"us_per_call": best, "kv_GBps": kv_read_bytes(sh) / best / 1e3,
                     "kernel": "split-pair" if units <= (131072 if Hq // Hkv > 4 else 65536)
                     else "stream-K"}
        del ls, ws, out, g
        torch.cuda.empty_cache()
    return res


def run_roles(args, world, rank, local):
    """N >= 2: even ranks decode, odd ranks are the executors of prefill-role GPUs
    (rank 2i pairs with 2i+1). Each decoder keeps `batch` local requests and
    offloads round(batch * offload_ratio) more (offload ratio = offloaded:local,
    scheduling.py:176-221) whose KV lives on its executor; per layer q/k/v go out
    and outputs come back over NCCL (exchange.DistTransport) while the decoder
    attends its local rows. value = KV bytes streamed by all ranks / step time."""
    from paper_2503_20552_b200 import ops
    from paper_2503_20552_b200.exchange import DistTransport
    from paper_2503_20552_b200.runtime import RoleSplitStep
    from dataclasses import replace
    if world < 2 or world % 2:
        raise SystemExit("--roles needs an even number of ranks")
    dev = torch.device("cuda", local)
    base = CONFIGS[args.config]
    L, Hq, Hkv, D = base.num_layers, base.num_q_heads, base.num_kv_heads, base.head_dim
    n_local = base.batch
    n_off = int(round(base.batch * args.offload_ratio))
    decoder = rank % 2 == 0
    peer = rank + 1 if decoder else rank - 1
    mine = replace(base, batch=n_local if decoder else max(1, n_off))
    bt = make_block_table(mine, seed=1 + rank)
    layers = [make_layer(mine, dev, seed=100 * rank + l, block_table=bt) for l in range(L)]
    ws = [ops.DecodeWorkspace(mine.batch, Hq, Hkv, D, dev) for _ in range(2)]
    scale = 1.0 / math.sqrt(D)

    def attend(l, q, k, v, out):
        x = layers[l]
        ops.paged_decode_attn(q, x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                              out=out, scale=scale, workspace=ws[l % 2], k_new=k, v_new=v)

    B = n_local + n_off
    g = torch.Generator(device=dev).manual_seed(rank)
    mk = lambda *sh: torch.randn(*sh, generator=g, device=dev).to(torch.bfloat16)
    if decoder:
        qs = [mk(B, Hq, D) for _ in range(L)]
        ks = [mk(B, Hkv, D) for _ in range(L)]
        vs = [mk(B, Hkv, D) for _ in range(L)]
        outs = [torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    link_step = n_off * L * ((Hq + 2 * Hkv) * D * 2 + Hq * D * 2)
    if args.zero_copy:
        # no messages: the executor's kernel reads the decoder's q/k/v rows and
        # writes its out rows over NVLink (CUDA IPC mappings + stream flags)
        from types import SimpleNamespace
        from paper_2503_20552_b200.runtime import ZeroCopyRoleStep
        zc = ZeroCopyRoleStep("decoder" if decoder else "executor", L, peer)
        counter = [0]
        if decoder:
            zc.setup_decoder(qs, ks, vs, outs)
            main_s = torch.cuda.current_stream(dev)

            def one():
                counter[0] += 1
                zc.decoder_step(counter[0], n_local, lambda l: attend(
                    l, qs[l][:n_local], ks[l][:n_local], vs[l][:n_local], outs[l][:n_local]),
                    outs, stream=main_s)
                return link_step
        else:
            zc.setup_executor(dev)

            class _Exec:
                stream = torch.cuda.Stream(device=dev)
                kv = SimpleNamespace(device=dev)

                def run_layer(self, l, q, k, v, bt_, seq_, slots, out, stream=None, in_rows=None,
                              out_rows=None):
                    x = layers[l]
                    ops.paged_decode_attn(q, x["k_cache"], x["v_cache"], x["block_table"],
                                          x["seq_lens"], out=out, scale=scale, workspace=ws[l % 2],
                                          stream=stream, k_new=k, v_new=v, in_rows=in_rows,
                                          out_rows=out_rows)
            ex = _Exec()

            def one():
                counter[0] += 1
                if n_off:
                    zc.executor_step(counter[0], n_local, B, ex, layers[0]["block_table"],
                                     layers[0]["seq_lens"])
                return 0
    else:
        step = RoleSplitStep("decoder" if decoder else "executor", Hq, Hkv, D,
                             DistTransport(peer), attend=attend)
        if decoder:
            one = lambda: step.run_decoder(qs, ks, vs, n_local, outs)
        else:
            one = lambda: step.run_executor(L, n_off, torch.bfloat16, dev) if n_off else 0
    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(args.steps):
            link = one()
        e1.record()
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world, dev) / args.steps
    kv_mine = kv_read_bytes(mine) * L if (decoder or n_off) else 0
    import torch.distributed as dist
    tot = torch.tensor([kv_mine, B if decoder else 0], dtype=torch.float64, device=dev)
    dist.all_reduce(tot)
    if rank == 0:
        line = {
            "metric": METRIC, "value": tot[0].item() / (ms / 1e3) / 1e9, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"{base.name} decode with offloaded attention: {world // 2} "
                                   f"decoder + {world // 2} executor ranks, {n_local} local + "
                                   f"{n_off} offloaded requests per decoder (offload ratio "
                                   f"{args.offload_ratio}), ctx {base.ctx}, L={L}",
                       "global_batch": int(tot[1].item()), "seq_len": base.ctx,
                       "parallelism": f"roles {world // 2}D+{world // 2}P "
                                      + ("(zero-copy: CUDA IPC + kernel peer loads/stores)"
                                         if args.zero_copy else "(NCCL p2p exchange)")},
            "tokens_per_s": tot[1].item() / (ms / 1e3),
            "nvlink_GBps_per_decoder": (link or 0) / (ms / 1e3) / 1e9,
            "nvlink_frac_of_900": (link or 0) / (ms / 1e3) / 900e9,
            "gpu_launches": args.steps * L * ((1 if args.zero_copy else 4) if n_off else 1),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Capacity-bound decode with and without offloading (the north-star comparison)
# ---------------------------------------------------------------------------



def _contig_tables(ctxs, dev):
    """Block table [n, max_pages] over pages laid out request after request, and lengths."""
    pages = [-(-c // 16) for c in ctxs]
    width = max(pages + [1])
    bt = torch.zeros((max(1, len(ctxs)), width), dtype=torch.int32)
    off = 0
    for i, n in enumerate(pages):
        bt[i, :n] = torch.arange(off, off + n, dtype=torch.int32)
        off += n
    return bt[:len(ctxs)].to(dev), torch.tensor(ctxs, dtype=torch.int32, device=dev), max(1, off)


def _zero_kv(L, NB, Hkv, D, dev):
    return [(torch.zeros((NB, Hkv, 16, D), dtype=torch.bfloat16, device=dev),
             torch.zeros((NB, Hkv, 16, D), dtype=torch.bfloat16, device=dev)) for _ in range(L)]


def _timed_steps(fn, steps, warmup, stream):
    for _ in range(warmup):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    return e0, e1


def run_capacity(args, world, rank, local):
    """Capacity-bound decode, no offload vs offload (BASELINE.json north star:
    "offloaded decoding on 8xB200 raising decode batch size and tokens/s by at
    least 1.5x over the no-offload configuration").

    Roles: even ranks decode, odd ranks are prefill GPUs whose SM partition
    (attn_sm_ratio of the SMs, a green context) runs the offloaded attention
    beside a continuous prefill GEMM load on the rest. Each decoder's batch is
    the steady state of its KV pool (capacity.plan_capacity: SimConfig
    pool_bytes, Algorithm 1 at the planner bound through the OffloadLedger,
    executor budget; engine.py:326-355), over ShareGPT-like requests caught
    mid-decode. Both runs execute full Llama-2-13B decode layers (40 layers of
    cuBLAS GEMMs with synthetic weights around our attention, fused append):
      no offload  the decoder's whole batch attends locally;
      offload     rows placed locally attend on the decoder, offloaded rows on
                  the executor GPU (decoder.RemoteOffloadedDecoder /
                  OffloadServer: zero-copy over CUDA IPC, stream-ordered flags).
    N = 1 is the degenerate single-GPU run of the same code (both roles on one
    GPU, budgets scaled by --capacity-scale, executor in a green-context
    partition of the same GPU): the machinery runs, the gain is not a capacity
    gain (one HBM)."""
    import torch.distributed as dist
    from paper_2503_20552_b200 import capacity, coloc, config, specs, workload
    from paper_2503_20552_b200.decoder import (MODEL_DIMS, OffloadedDecoder, OffloadServer,
                                               RemoteOffloadedDecoder, SyntheticDecoder)
    if world > 1 and world % 2:
        raise SystemExit("--capacity needs an even number of ranks (decoder, executor pairs)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    nd = max(1, world // 2)
    case = capacity.CAPACITY_CASES[args.capacity_config]
    model = case.model
    dims = MODEL_DIMS[case.dims]
    Hq, Hkv, D = dims.num_q_heads, dims.num_kv_heads, dims.head_dim
    L = model.num_layers
    cfg = config.SimConfig(gpu=specs.B200, model=model, num_prefill=nd, num_decode=nd,
                           offload_ratio=case.offload_ratio)
    # budgets scaled down when the roles share a GPU (N=1, or a 1-GPU smoke of N=2)
    shared = world == 1 or torch.cuda.device_count() < world
    scale = args.capacity_scale if shared else 1.0
    d_idx = rank // 2
    reqs = capacity.case_requests(case, d_idx)
    plan = capacity.plan_capacity(cfg, reqs, scale=scale)
    decoder = world == 1 or rank % 2 == 0
    stream = torch.cuda.current_stream(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    part = None
    if (world == 1 or not decoder) and coloc.green_contexts_supported():
        part = coloc.SmPartition(local, int(round(cfg.attn_sm_ratio * sms)))
    res = {}
    g = torch.Generator(device=dev).manual_seed(3)

    # The prefill load runs on the executor (prefill-role) GPUs. When the roles
    # share one GPU (N = 1) it is off by default: it would take the SMs of the
    # decoder's own kernels, which a decode GPU never shares with prefill.
    use_prefill = args.capacity_prefill == "on" or (args.capacity_prefill == "auto" and not shared)

    def prefill_cover(ms_needed):
        """Enqueue enough prefill iterations on the prefill partition to keep it
        busy for ms_needed (it starts at once); returns the iterations enqueued."""
        if part is None or not use_prefill:
            return 0
        pre = coloc.prefill_load_for(model, dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pre.run(part.prefill_stream)
        e0.record(part.prefill_stream)
        pre.run(part.prefill_stream)
        e1.record(part.prefill_stream)
        e1.synchronize()
        reps = int(math.ceil(ms_needed / max(1e-3, e0.elapsed_time(e1)))) + 2
        pre.run(part.prefill_stream, repeats=reps)
        return reps

    # ---- run A: no offload (decoders only; prefill GPUs only prefill) ----
    weights = None
    step_a = 0.0
    if decoder:
        bt, seq, NB = _contig_tables(plan.no_offload, dev)
        kv = _zero_kv(L, NB, Hkv, D, dev)
        dec = SyntheticDecoder(dims, kv, plan.batch_no_offload, dev, seed=7, nonattn=case.nonattn)
        weights = dec.layers
        x = torch.randn(plan.batch_no_offload, dims.hidden, generator=g, device=dev).to(torch.bfloat16)
        x0 = x.clone()

        def step_a_fn():
            x.copy_(x0)
            dec.step(x, bt, seq, pdl=True)
        barrier(world)
        e0, e1 = _timed_steps(step_a_fn, args.steps, args.warmup, stream)
        torch.cuda.synchronize()
        step_a = e0.elapsed_time(e1) / args.steps
        res["no_offload"] = {"batch": plan.batch_no_offload, "ms_per_step": step_a,
                             "tokens_per_s_per_decoder": plan.batch_no_offload / (step_a / 1e3),
                             "kv_GB": plan.bytes("no_offload") / 1e9}
        del dec, kv, x, x0
        torch.cuda.empty_cache()
    else:
        barrier(world)
    step_a = max_over_ranks(step_a, world, dev)
    barrier(world)

    # ---- run B: offload ----
    nl, no = len(plan.local), len(plan.offloaded)
    B = nl + no
    est_ms = step_a * (args.warmup + args.steps) * 2.0 + 2000.0  # prefill cover (ms)
    link = 0
    step_b = 0.0
    if world == 1:
        lbt, lseq, NBl = _contig_tables(plan.local, dev)
        xbt, xseq, NBx = _contig_tables(plan.offloaded, dev)
        kv = _zero_kv(L, NBl, Hkv, D, dev)
        xkv = _zero_kv(L, NBx, Hkv, D, dev)
        dec = OffloadedDecoder(dims, kv, xkv, B, nl, dev,
                               exec_stream=part.attn_stream if part else None,
                               exec_sms=part.attn_sms if part else 0, seed=7, weights=weights,
                               nonattn=case.nonattn)
        x = torch.randn(B, dims.hidden, generator=g, device=dev).to(torch.bfloat16)
        x0 = x.clone()

        def step_b_fn():
            x.copy_(x0)
            dec.step(x, lbt, lseq, xbt, xseq, pdl=True)
        reps = prefill_cover(est_ms)
        e0, e1 = _timed_steps(step_b_fn, args.steps, args.warmup, stream)
        torch.cuda.synchronize()
        step_b = e0.elapsed_time(e1) / args.steps
        link = no * L * ((Hq + 2 * Hkv) * D * 2 + Hq * D * 2)
        res["offload"] = {"batch": B, "n_local": nl, "n_offloaded": no, "ms_per_step": step_b,
                          "tokens_per_s_per_decoder": B / (step_b / 1e3),
                          "executor_sms": part.attn_sms if part else sms, "prefill_reps": reps}
    elif decoder:
        lbt, lseq, NBl = _contig_tables(plan.local, dev)
        kv = _zero_kv(L, NBl, Hkv, D, dev)
        dec = RemoteOffloadedDecoder(dims, kv, B, nl, dev, seed=7, weights=weights,
                                     nonattn=case.nonattn)
        dist.send_object_list([dec.export()], dst=rank + 1)
        x = torch.randn(B, dims.hidden, generator=g, device=dev).to(torch.bfloat16)
        x0 = x.clone()

        def step_b_fn():
            x.copy_(x0)
            dec.step(x, lbt, lseq, pdl=True)
        barrier(world)
        e0, e1 = _timed_steps(step_b_fn, args.steps, args.warmup, stream)
        torch.cuda.synchronize()
        step_b = e0.elapsed_time(e1) / args.steps
        link = no * L * ((Hq + 2 * Hkv) * D * 2 + Hq * D * 2)
        res["offload"] = {"batch": B, "n_local": nl, "n_offloaded": no, "ms_per_step": step_b,
                          "tokens_per_s_per_decoder": B / (step_b / 1e3)}
        barrier(world)
    else:
        box = [None]
        dist.recv_object_list(box, src=rank - 1)
        xbt, xseq, NBx = _contig_tables(plan.offloaded, dev)
        xkv = _zero_kv(L, NBx, Hkv, D, dev)
        srv = OffloadServer(box[0], xkv, dev, stream=part.attn_stream if part else None,
                            num_sms=part.attn_sms if part else 0)
        sid = [0]

        def step_b_fn():
            sid[0] += 1
            srv.step(sid[0], xbt, xseq)
        barrier(world)
        prefill_cover(est_ms)
        e0, e1 = _timed_steps(step_b_fn, args.steps, args.warmup, srv.stream)
        torch.cuda.synchronize()
        step_b = e0.elapsed_time(e1) / args.steps
        barrier(world)
        srv.close()
    step_b = max_over_ranks(step_b, world, dev)
    if rank != 0:
        return
    tok_a = nd * plan.batch_no_offload / (step_a / 1e3)
    tok_b = nd * B / (step_b / 1e3)
    line = {
        "metric": "decode tokens/s (capacity-bound, " + ("full layers)" if case.nonattn else
                                                          "attention-only layers)"),
        "value": tok_b,
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_b, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (" + ("ShareGPT-like" if case.preset != "longctx" else "long-context") +
                " lengths caught mid-decode; random weights, zero KV)",
        "config": {"workload": f"{case.name} {case.note}; KV-capacity-bound batch per decoder "
                               f"(SimConfig pool {plan.pool_bytes / 1e9:.1f} GB, executor budget "
                               f"{plan.exec_budget_bytes / 1e9:.1f} GB, Algorithm 1 bound "
                               f"{plan.bound:.3f}), {L} layers",
                   "global_batch": nd * B, "parallelism": f"roles {nd}D+{nd}P" if world > 1 else
                   "1 GPU: decoder + executor partition on one GPU (degenerate)",
                   "capacity_scale": scale, "prefill_load_on_executor": use_prefill},
        "no_offload": dict(res.get("no_offload", {}), tokens_per_s=tok_a),
        "offload": dict(res.get("offload", {}), tokens_per_s=tok_b),
        "batch_gain": plan.batch_gain, "tokens_per_s_gain": tok_b / tok_a,
        "nvlink_GBps_per_decoder": link / (step_b / 1e3) / 1e9,
        "nvlink_frac_of_900": link / (step_b / 1e3) / 900e9,
        "plan": plan.summary(),
        # our kernels in the timed region of the offload run: per decoder and layer one
        # local attention launch and one executor (row-mapped) launch
        "gpu_launches": nd * args.steps * L * (1 + (1 if no else 0)),
    }
    print(json.dumps(line), flush=True)


ROLE_RUNS = (  # (offload ratio, zero-copy): no-offload baseline, message exchange, zero-copy
    (0.0, False), (0.5, False), (0.5, True))
# capacity-bound comparisons run after the role splits (even N): the north star's
# "decode batch size and tokens/s >= 1.5x over no offload" at C4 and C5
CAPACITY_RUNS = ("C4", "C5")


def role_split_runs(args, world, rank) -> list | None:
    """N > 1: after the request-sharded line, the same N GPUs split into decode
    and prefill (executor) roles (BASELINE.json: "at 2, 4 and 8 GPUs split into
    decode and prefill roles"), C3 shapes, no offload vs offload ratio 0.5.
    Each run is a separate torchrun of ``bench.py --roles`` (its own NCCL
    world), in its own process group under a timeout, so a failing exchange
    cannot take the main line with it. The main ranks wait on a CPU (gloo)
    barrier meanwhile and hold no GPU memory beyond their contexts."""
    import signal
    import socket
    import torch.distributed as dist
    torch.cuda.empty_cache()
    cpu = dist.new_group(backend="gloo")
    dist.barrier(group=cpu)
    res = None
    if rank == 0:
        res = []
        env = {k: v for k, v in os.environ.items()
               if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "GROUP_RANK",
                            "ROLE_RANK", "ROLE_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")
               and not k.startswith("TORCHELASTIC")}
        runs = [({"offload_ratio": ratio, "exchange": "zero-copy" if zc else "nccl"},
                 ["--roles", "--config", args.role_config, "--steps", "20", "--warmup", "3",
                  "--offload-ratio", str(ratio)] + (["--zero-copy"] if zc else []))
                for ratio, zc in ROLE_RUNS]
        if world % 2 == 0:
            runs += [({"capacity": c}, ["--capacity", "--capacity-config", c, "--steps", "10",
                                        "--warmup", "3"]) for c in CAPACITY_RUNS]
        for tag, extra in runs:
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
                   "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", str(world)] + extra
            proc = subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                    text=True, start_new_session=True)
            try:
                out, err = proc.communicate(timeout=args.role_timeout)
                lines = [l for l in out.splitlines() if l.startswith("{")]
                if proc.returncode == 0 and lines:
                    res.append(dict(tag, **json.loads(lines[-1])))
                else:
                    res.append(dict(tag, error=f"rc={proc.returncode}: {err.strip()[-300:]}"))
            except subprocess.TimeoutExpired:
                os.killpg(proc.pid, signal.SIGKILL)
                proc.communicate()
                res.append(dict(tag, error=f"timed out after {args.role_timeout} s"))
            log(f"roles {tag}: {res[-1].get('tokens_per_s', res[-1].get('error'))}")
    dist.barrier(group=cpu)
    return res


def load_traffic():
    """dram bytes per launch from the committed ncu capture summary, if present."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except (ValueError, OSError):
            return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of CPU oracle work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pdl", action="store_true", help="plain launches instead of PDL chaining")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3/C5 kernel measurements")
    ap.add_argument("--no-full-layer", action="store_true",
                    help="skip the full-layer (synthetic non-attention GEMMs) measurement")
    ap.add_argument("--roles", action="store_true",
                    help="N>=2: decoder / executor role split with the offload exchange")
    ap.add_argument("--offload-ratio", type=float, default=0.5, help="offloaded:local (roles)")
    ap.add_argument("--zero-copy", action="store_true",
                    help="roles: executor kernels read/write the decoder's rows over NVLink")
    ap.add_argument("--no-role-runs", action="store_true",
                    help="N>1: skip the decode/prefill role-split runs after the main line")
    ap.add_argument("--role-config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--role-timeout", type=float, default=300.0)
    ap.add_argument("--capacity", action="store_true",
                    help="capacity-bound decode, no offload vs offload (roles; N=1 degenerate)")
    ap.add_argument("--capacity-config", default="C4", choices=["C4", "C5"],
                    help="capacity case (paper_2503_20552_b200.capacity.CAPACITY_CASES)")
    ap.add_argument("--capacity-prefill", default="auto", choices=["auto", "on", "off"],
                    help="prefill GEMM load beside the executor partition (auto: on unless the "
                         "roles share one GPU)")
    ap.add_argument("--capacity-scale", type=float, default=0.45,
                    help="N=1 only: fraction of the per-GPU budgets (both roles share one GPU)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("warning: fewer than 3 warm-up steps")
    world, rank, local = dist_setup()
    shape = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, shape, world, rank)
    elif args.capacity:
        run_capacity(args, world, rank, local)
    elif args.roles:
        run_roles(args, world, rank, local)
    else:
        line = run_ours(args, shape, world, rank, local)
        if world > 1 and not args.no_role_runs:
            roles = role_split_runs(args, world, rank)
            if line is not None:
                line["role_split"] = roles
        if line is not None:
            print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
