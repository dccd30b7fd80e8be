"""B_max by sweep: the batch where the non-attention layers stop being
weight-streaming bound, measured on this GPU.

The reference derives B_max analytically from the machine balance
(costs.py:41-55 ``b_max``: floor(1 / (1/balance - 1/hidden))) and prices the
non-attention step as flat up to B_max and linear beyond (costs.py:77-91
``nonattn_step_latency``); its SPEC leaves a
``calibrate`` path that "estimates B_max by sweep" instead. Here:

  * ``sweep_nonattn`` times the real non-attention work of decode layers
    (decoder.SyntheticDecoder's RMSNorm + QKV / O / gated-MLP cuBLAS GEMMs,
    synthetic weights, distinct per layer, CUDA-graph captured) at a range of
    batch sizes;
  * ``fit_knee`` fits the reference's own shape t(B) = t0 for B <= B_max,
    t0 * B / B_max beyond, to the samples;
  * ``gpu_for_bmax`` returns the GpuSpec whose effective machine balance makes
    the reference's ``b_max`` formula give the measured knee, so
    ``SimConfig(gpu=...)`` plans with it (Eq. 2's OB_comp, the graph grid).
"""
from __future__ import annotations

import dataclasses
import math
import statistics

from .costs import b_max
from .specs import GpuSpec, ModelSpec

__all__ = ["sweep_nonattn", "fit_knee", "gpu_for_bmax"]


def fit_knee(samples, flat_batches: int = 3) -> tuple[float, float]:
    """(t0, B_max) of t(B) = max(t0, t0 * B / B_max) fitted to [(B, seconds)].

    t0 = median time of the ``flat_batches`` smallest batches; the slope s of
    the linear regime is a least-squares fit through the origin over the
    batches whose time exceeds 1.15 t0, and B_max = t0 / s (no such batch:
    B_max = the largest batch swept, a lower bound)."""
    pts = sorted((int(b), float(t)) for b, t in samples)
    if len(pts) < 2:
        raise ValueError("need at least two (batch, time) samples")
    t0 = statistics.median(t for _, t in pts[:max(1, flat_batches)])
    lin = [(b, t) for b, t in pts if t > 1.15 * t0]
    if not lin:
        return t0, float(pts[-1][0])
    s = sum(b * t for b, t in lin) / sum(b * b for b, _ in lin)
    return t0, t0 / s


def gpu_for_bmax(gpu: GpuSpec, model: ModelSpec, knee: float) -> GpuSpec:
    """``gpu`` with flops_peak set so costs.b_max(gpu, model) == floor(knee):
    balance = 1 / (1/(knee + 0.5) + 1/hidden) (the +0.5 keeps the formula's
    floor on the measured integer)."""
    k = max(1, int(math.floor(knee)))
    balance = 1.0 / (1.0 / (k + 0.5) + 1.0 / model.hidden_size)
    out = dataclasses.replace(gpu, name=f"{gpu.name}-bmax{k}", flops_peak=balance * gpu.hbm_bandwidth)
    assert b_max(out, model) == k
    return out


def sweep_nonattn(dims, batches, device, layers: int = 4, reps: int = 10) -> list[tuple[int, float]]:
    """Seconds per decode layer of the non-attention work at each batch
    (mean over ``layers`` distinct layers, CUDA-graph replays, event-timed)."""
    import torch
    import torch.nn.functional as F

    from .decoder import SyntheticDecoder
    out = []
    for B in batches:
        dec = SyntheticDecoder(dims, [(None, None)] * layers, B, device, seed=1)
        x = torch.randn(B, dims.hidden, device=device).to(torch.bfloat16)
        I = dims.intermediate

        def step():
            for W in dec.layers:
                h = F.rms_norm(x, (dims.hidden,), W["n1"], dec.eps)
                if dec.mha:
                    torch.matmul(h, W["wqkv"].t(), out=dec.qkv[:3 * B].view(B, -1))
                else:
                    torch.matmul(h, W["wq"].t(), out=dec.q.view(B, -1))
                    torch.matmul(h, W["wk"].t(), out=dec.k.view(B, -1))
                    torch.matmul(h, W["wv"].t(), out=dec.v.view(B, -1))
                torch.matmul(dec.attn.view(B, -1), W["wo"].t(), out=dec.o)
                x.add_(dec.o)
                h = F.rms_norm(x, (dims.hidden,), W["n2"], dec.eps)
                torch.matmul(h, W["wgu"].t(), out=dec.gate_up)
                act = F.silu(dec.gate_up[:, :I]).mul_(dec.gate_up[:, I:])
                torch.matmul(act, W["wd"].t(), out=dec.o)
                x.add_(dec.o)
        dec.attn.zero_()
        s = torch.cuda.Stream(device)
        s.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream(device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        g.replay()
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize(device)
        out.append((B, e0.elapsed_time(e1) / 1e3 / (reps * layers)))
        del dec, g, x
        torch.cuda.empty_cache()
    return out
