"""Prefill colocation on B200: SM partitions for the attention executor.

The reference models a prefill GPU split into an attention share r and a
prefill share 1 - r by two curves (calibration.py:1-219; used at
config.py:125-132, engine.py:159-160), anchored to A100/MPS measurements
(PAPER.md:436). Here the split is real:

  * ``SmPartition`` carves the GPU into two CUDA green contexts — the executor's
    (``attn_sms``, a multiple of 8 as sm_90+ partitions require) and the
    prefill engine's (the rest) — each exposing a stream whose kernels only run
    on its SMs, the executor's at the highest stream priority. Decode attention launched with ``num_sms=attn_sms`` sizes its
    persistent grid to the partition and uses the 12-warps/SM variant.
  * ``PrefillLoad`` is the synthetic prefill: bf16 GEMMs of a prefill batch's
    QKV / O / MLP shapes on the prefill stream.
  * ``sweep_partitions`` measures executor bandwidth vs SM share and prefill
    slowdown vs SM share (alone and under interference), and
    ``fit_curves`` feeds the samples to ``fit_curves_from_samples`` — the
    B200 replacement for the A100-anchored default curves.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import ops
from .calibration import CalibrationCurves, CurveValidationError, fit_curves_from_samples

__all__ = ["green_contexts_supported", "SmPartition", "PrefillLoad", "sweep_partitions",
           "fit_curves", "PartitionSample", "Overlap", "PrefillCover", "run_under_prefill",
           "prefill_load_for"]


def green_contexts_supported() -> bool:
    try:
        from torch.cuda import green_contexts as gc
        return bool(gc.SUPPORTED) and torch.cuda.is_available()
    except ImportError:  # pragma: no cover
        return False


class SmPartition:
    """Attention / prefill split of one GPU's SMs: two green contexts created by
    the C-ABI (``adr_sm_partition_create``), each with one stream whose kernels
    only run on its SMs. The executor's stream gets the device's highest stream
    priority and the prefill's the lowest: the block scheduler otherwise hands
    out a grid's CTAs only after every CTA of the grids launched before it, and
    an attention call queued behind a prefill GEMM waits for that GEMM
    (measured +100-350 µs per call, ``profiles/exec_prio_r02u.txt``)."""

    def __init__(self, device: int, attn_sms: int, prioritize_attention: bool = True) -> None:
        if not green_contexts_supported():
            raise RuntimeError("CUDA green contexts unavailable")
        from . import _ffi
        total = torch.cuda.get_device_properties(device).multi_processor_count
        attn = max(8, min(total - 8, (attn_sms // 8) * 8))
        lowest, greatest = torch.cuda.Stream.priority_range()
        s_attn, s_pre, h = _ffi.ctypes.c_void_p(), _ffi.ctypes.c_void_p(), _ffi.ctypes.c_void_p()
        n_attn, n_pre = _ffi.ctypes.c_int32(), _ffi.ctypes.c_int32()
        _ffi.call("adr_sm_partition_create", device, attn,
                  greatest if prioritize_attention else lowest, lowest,
                  _ffi.ctypes.byref(s_attn), _ffi.ctypes.byref(s_pre), _ffi.ctypes.byref(n_attn),
                  _ffi.ctypes.byref(n_pre), _ffi.ctypes.byref(h))
        self._handle = h.value
        self.device = device
        self.total_sms = total
        self.attn_sms = n_attn.value
        self.prefill_sms = n_pre.value
        self.attn_stream = torch.cuda.ExternalStream(s_attn.value, device=torch.device("cuda", device))
        self.prefill_stream = torch.cuda.ExternalStream(s_pre.value, device=torch.device("cuda", device))

    @property
    def attn_ratio(self) -> float:
        return self.attn_sms / self.total_sms

    def close(self) -> None:
        """Release the green contexts (after the streams' work is done)."""
        if self._handle:
            from . import _ffi
            torch.cuda.synchronize(self.device)
            _ffi.call("adr_sm_partition_destroy", self._handle)
            self._handle = None


class PrefillLoad:
    """Synthetic prefill compute: per layer QKV, O and gated-MLP GEMMs of a
    ``tokens``-token prefill batch (bf16, random weights)."""

    def __init__(self, tokens: int, hidden: int, intermediate: int, device: torch.device,
                 seed: int = 0) -> None:
        self.device = torch.device(device)
        g = torch.Generator(device=device).manual_seed(seed)
        mk = lambda *s: (torch.randn(*s, generator=g, device=device) * 0.02).to(torch.bfloat16)
        self.x = mk(tokens, hidden)
        self.w_qkv = mk(hidden, 3 * hidden)
        self.w_o = mk(hidden, hidden)
        self.w_up = mk(hidden, 2 * intermediate)
        self.w_down = mk(intermediate, hidden)
        self.flops = 2 * tokens * hidden * (3 * hidden + hidden + 2 * intermediate) + \
            2 * tokens * intermediate * hidden

    def run(self, stream: torch.cuda.Stream, repeats: int = 1) -> None:
        with torch.cuda.stream(stream):
            for _ in range(repeats):
                h = self.x @ self.w_qkv
                h = h[:, : self.x.shape[1]] @ self.w_o
                u = h @ self.w_up
                self.x.copy_((u[:, : self.w_down.shape[0]] @ self.w_down))


# FFN widths of the reference's model presets (specs.py:73-82 and the GQA ones)
_INTERMEDIATE = {4096: 11008, 5120: 13824, 8192: 28672}


def prefill_load_for(model, device: torch.device, tokens: int = 2048) -> PrefillLoad:
    """A PrefillLoad of ``model``'s layer GEMM shapes (hidden size; FFN width of
    the Llama family: 11008 / 13824 / 28672, 14336 for Llama-3-8B)."""
    h = model.hidden_size
    inter = 14336 if (h == 4096 and model.num_kv_heads not in (None, model.q_heads)) else \
        _INTERMEDIATE.get(h, (h * 8 // 3 + 255) // 256 * 256)
    return PrefillLoad(tokens, h, inter, device)


@dataclass
class PartitionSample:
    attn_sms: int
    prefill_sms: int
    attn_ratio: float
    attn_gbs_alone: float
    attn_gbs_shared: float
    prefill_s_alone: float
    prefill_s_shared: float
    repeats: int = 1                 # overlapped windows measured (median reported)
    prefill_reps_in_window: int = 0  # prefill iterations fully inside each window (min)


def _time_on(stream: torch.cuda.Stream, fn, iters: int) -> float:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record(stream)
    for _ in range(iters):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / iters


@dataclass
class Overlap:
    """One overlapped window: attention calls on the executor partition while
    prefill iterations run back to back on the prefill partition."""

    attn_s: float            # per attention call inside the window
    prefill_s: float         # per prefill iteration fully inside the window (mean)
    prefill_in_window: int   # prefill iterations fully inside the window
    covered: bool            # prefill was running from before the window to after it


class PrefillCover:
    """Keep the prefill partition busy across a region of attention work:
    ``start(reps)`` enqueues ``reps`` back-to-back prefill iterations on the
    prefill stream (an event after each) and returns the event of the first
    one, which the attention streams wait on, so the region opens with prefill
    running. After a synchronize, ``covered(t0, t1)`` tells whether prefill
    ran from before event t0 to after event t1, and ``inside(t0, t1)`` gives
    the durations of the iterations wholly inside [t0, t1].

    The prefill starts running as soon as it is enqueued, so the caller sizes
    ``reps`` to cover the host's enqueue time of the region as well as its GPU
    time (a device-side hold on a flag would be simpler but can deadlock: a
    stream blocked in cuStreamWaitValue32 may share a hardware queue with the
    stream that would release it)."""

    def __init__(self, prefill_stream: torch.cuda.Stream, prefill: "PrefillLoad") -> None:
        self.stream = prefill_stream
        self.prefill = prefill
        self.ev: list = []

    def start(self, reps: int) -> torch.cuda.Event:
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        self.ev[0].record(self.stream)
        for i in range(reps):
            self.prefill.run(self.stream)
            self.ev[i + 1].record(self.stream)
        return self.ev[1]

    def _rel(self, t0) -> list[float]:
        return [t0.elapsed_time(e) / 1e3 for e in self.ev]

    def covered(self, t0, t1) -> bool:
        rel = self._rel(t0)
        return rel[1] <= 0.0 and rel[-1] >= t0.elapsed_time(t1) / 1e3

    def inside(self, t0, t1) -> list[float]:
        rel = self._rel(t0)
        w = t0.elapsed_time(t1) / 1e3
        return [rel[i + 1] - rel[i] for i in range(len(rel) - 1) if rel[i] >= 0.0 and rel[i + 1] <= w]


def run_under_prefill(attn_stream: torch.cuda.Stream, attn_fn, attn_iters: int,
                      prefill_stream: torch.cuda.Stream, prefill: "PrefillLoad",
                      prefill_reps: int) -> Overlap:
    """Time ``attn_iters`` calls of ``attn_fn`` (enqueued on ``attn_stream``)
    while ``prefill`` runs ``prefill_reps`` iterations back to back on
    ``prefill_stream`` (``PrefillCover``). The caller sizes ``prefill_reps`` so
    prefill is still running when the window closes (``covered``). Only the
    overlapped span is timed: attention over its window, prefill over the
    iterations that lie wholly inside it."""
    torch.cuda.synchronize()
    cover = PrefillCover(prefill_stream, prefill)
    gate = cover.start(prefill_reps)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    attn_stream.wait_event(gate)
    s0.record(attn_stream)
    for _ in range(attn_iters):
        attn_fn()
    s1.record(attn_stream)
    torch.cuda.synchronize()
    inside = cover.inside(s0, s1)
    return Overlap(s0.elapsed_time(s1) / 1e3 / attn_iters,
                   sum(inside) / len(inside) if inside else math.nan, len(inside),
                   cover.covered(s0, s1))


def sweep_partitions(device: int, layer: dict, prefill: PrefillLoad, attn_sm_list,
                     iters: int = 5, kv_bytes: int | None = None, repeats: int = 5,
                     min_prefill_in_window: int = 3) -> dict:
    """Measure executor KV GB/s and prefill time per attention SM share, each
    partition alone and both busy at once.

    ``layer`` is one decode-attention input set (synthetic.make_layer). The
    shared numbers come from ``run_under_prefill``: the attention chain is
    long enough to hold at least ``min_prefill_in_window`` whole prefill
    iterations, prefill runs continuously from before the window to after it
    (checked; the window is re-run with more prefill otherwise), and each
    partition's value is the median over ``repeats`` windows.
    """
    import statistics
    dev = torch.device("cuda", device)
    scale = 1.0 / math.sqrt(layer["q"].shape[-1])
    B, Hq, D = layer["q"].shape
    Hkv = layer["k_cache"].shape[1]
    kv_bytes = kv_bytes or int(layer["seq_lens"].sum().item()) * Hkv * D * 4
    out = torch.empty_like(layer["q"])

    ws = ops.DecodeWorkspace(B, Hq, Hkv, D, dev)

    def attn(stream, num_sms):
        return lambda: ops.paged_decode_attn(layer["q"], layer["k_cache"], layer["v_cache"],
                                             layer["block_table"], layer["seq_lens"], out=out,
                                             scale=scale, workspace=ws, stream=stream,
                                             num_sms=num_sms, pdl=True)

    full = torch.cuda.Stream(device=dev)
    t_attn_full = _time_on(full, attn(full, 0), iters)
    t_pre_full = _time_on(full, lambda: prefill.run(full), iters)
    samples = []
    for sms in attn_sm_list:
        part = SmPartition(device, sms)
        fa = attn(part.attn_stream, part.attn_sms)
        ta = _time_on(part.attn_stream, fa, iters)
        tp = _time_on(part.prefill_stream, lambda: prefill.run(part.prefill_stream), iters)
        # window: >= min_prefill_in_window prefill iterations even if interference
        # doubles the prefill time; prefill: the window (even if attention slows
        # 3x) plus slack on both sides
        n_attn = max(iters, math.ceil((min_prefill_in_window + 1) * 2.0 * tp / ta))
        reps = math.ceil(3.0 * n_attn * ta / tp) + 3
        a_s, p_s, inside = [], [], []
        for _ in range(repeats):
            for _attempt in range(4):
                ov = run_under_prefill(part.attn_stream, fa, n_attn, part.prefill_stream,
                                       prefill, reps)
                if ov.covered and ov.prefill_in_window >= min_prefill_in_window:
                    break
                if not ov.covered:
                    reps *= 2
                else:
                    n_attn *= 2
            a_s.append(ov.attn_s)
            p_s.append(ov.prefill_s)
            inside.append(ov.prefill_in_window)
        samples.append(PartitionSample(part.attn_sms, part.prefill_sms, part.attn_ratio,
                                       kv_bytes / ta / 1e9,
                                       kv_bytes / statistics.median(a_s) / 1e9, tp,
                                       statistics.median(p_s), repeats, min(inside)))
    return {"full_attn_gbs": kv_bytes / t_attn_full / 1e9, "full_prefill_s": t_pre_full,
            "prefill_tflops_full": prefill.flops / t_pre_full / 1e12,
            "samples": samples, "total_sms": torch.cuda.get_device_properties(device).multi_processor_count}


def fit_curves(sweep: dict, shared: bool = False) -> CalibrationCurves | None:
    """Fit validated curves from a sweep: bandwidth fraction vs attention SM
    share, prefill slowdown vs prefill SM share. Returns None if the measured
    points violate the reference's curve-shape rules (reported, not forced)."""
    full_bw, full_pre = sweep["full_attn_gbs"], sweep["full_prefill_s"]
    total = sweep["total_sms"]
    samples = sorted(sweep["samples"], key=lambda s: s.attn_sms)
    bw, sd = [], []
    best = 0.0
    for s in samples:
        gbs = s.attn_gbs_shared if shared else s.attn_gbs_alone
        r = s.attn_sms / total
        # monotone envelope: an executor with more SMs can always leave some idle
        best = max(best, min(1.0, gbs / full_bw))
        bw.append((round(r, 4), max(r, best)))
    worst = math.inf
    for s in reversed(samples):  # prefill share ascending as attention share descends
        tp = s.prefill_s_shared if shared else s.prefill_s_alone
        x = round(s.prefill_sms / total, 4) if hasattr(s, "prefill_sms") else round(1 - s.attn_sms / total, 4)
        y = min(max(1.0, tp / full_pre), 1.0 / x)
        worst = min(worst, y)
        sd.append((x, worst))
    sd.sort()
    try:
        return fit_curves_from_samples(bw, sd)
    except CurveValidationError:
        return None
