"""B200 decode-step runtime: local attention + offloaded attention exchange.

This is the real counterpart of the reference's step pricing
(engine.py:423-456). For every layer of one decode step:

  decode GPU   pack q/k/v of the offloaded rows (adr_pack_qkv) and send them
               on the exchange stream; kv_append + paged_decode_attn over the
               local rows on the main stream; receive the executor's outputs
               and place them beside the local ones (adr_scatter_out)
  executor     receive, unpack, kv_append into its own paged cache, paged
               decode attention on its stream (a green-context SM partition on
               a prefill GPU), send the outputs back

so the per-layer critical path is max(local_attn, send + remote_attn + recv),
the reference's ``stall = max(0, worst_path - local_attn)`` made real per layer.
All launches are asynchronous; CUDA events give the StepRecord-style timings.

Rows of a decode batch are ordered local-first ([0, B_local) local,
[B_local, B) offloaded) so the local kernel reads a contiguous prefix.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import torch

from . import _ffi, ops
from .exchange import LoopbackTransport, TAG_OUT, TAG_QKV

__all__ = ["LayeredKV", "AttentionExecutor", "StepPlan", "StepTimes", "two_sided_step", "OffloadedDecodeStep",
           "CapturedStep", "DecodeGraphCache", "MeasuredPricer", "step_record", "RoleSplitStep",
           "ZeroCopyRoleStep", "KVTransferRunner"]


class LayeredKV:
    """Paged K/V caches of one device pool for all layers: [L, NB, Hkv, 16, D] bf16."""

    def __init__(self, num_layers: int, num_pages: int, Hkv: int, D: int,
                 device: torch.device, fill: str = "empty", generator=None) -> None:
        shape = (num_layers, num_pages, Hkv, ops.PAGE, D)
        if fill == "randn":
            self.k = torch.empty(shape, dtype=torch.bfloat16, device=device)
            self.v = torch.empty(shape, dtype=torch.bfloat16, device=device)
            for t in (self.k, self.v):
                for l in range(num_layers):
                    t[l].copy_(torch.randn(shape[1:], generator=generator, device=device,
                                           dtype=torch.float32))
        else:
            self.k = torch.zeros(shape, dtype=torch.bfloat16, device=device)
            self.v = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.num_layers, self.num_pages, self.Hkv, self.D = num_layers, num_pages, Hkv, D
        self.device = device

    def layer(self, l: int):
        return self.k[l], self.v[l]


class KVTransferRunner:
    """Executes the prefill -> decode KV hand-off that ``kvcache.PagedKVMirror``
    plans (pass it as the mirror's ``on_transfer``): the request's staged prompt
    pages on prefill GPU p move into the decoder pages reserved for it at
    admission — the block-table remap — for every layer in ONE ``adr_kv_transfer``
    launch (the [L, NB] caches are addressed as L x NB pages). With the caches
    on two GPUs (peer access on) the kernel pulls the pages over NVLink. The
    reference prices this step as prefill_len x kv_bytes_per_token over the link
    (engine.py:231-249); ``pages`` / ``bytes`` count what was actually moved.
    """

    def __init__(self, src: dict, dst: dict, stream: torch.cuda.Stream | None = None,
                 before=None) -> None:
        self.src, self.dst = src, dst          # prefill idx -> LayeredKV, decoder idx -> LayeredKV
        self.stream = stream
        self.before = before                   # optional hook(transfer) run first (tests: fill the prompt KV)
        self.pages = 0
        self.bytes = 0
        self.launches = 0

    def __call__(self, tr) -> None:
        if self.before is not None:
            self.before(tr)
        s, d = self.src[tr.src[1]], self.dst[tr.dst[1]]
        n = len(tr.src_pages)
        if n == 0:
            return
        if (s.num_layers, s.Hkv, s.D) != (d.num_layers, d.Hkv, d.D):
            raise ValueError("source and destination caches differ in layers / heads / head_dim")
        L = s.num_layers
        sp = torch.tensor(tr.src_pages, dtype=torch.int64)
        dp = torch.tensor(tr.dst_pages, dtype=torch.int64)
        lay = torch.arange(L, dtype=torch.int64).unsqueeze(1)
        src_idx = (lay * s.num_pages + sp).reshape(-1).to(torch.int32)
        dst_idx = (lay * d.num_pages + dp).reshape(-1).to(torch.int32)
        shape = lambda kv: (kv.num_layers * kv.num_pages, kv.Hkv, ops.PAGE, kv.D)
        with torch.cuda.device(d.device):
            stream = self.stream or torch.cuda.current_stream(d.device)
            with torch.cuda.stream(stream):
                si = src_idx.pin_memory().to(d.device, non_blocking=True)
                di = dst_idx.pin_memory().to(d.device, non_blocking=True)
            ops.kv_transfer(s.k.view(shape(s)), s.v.view(shape(s)), si, d.k.view(shape(d)),
                            d.v.view(shape(d)), di, stream=stream)
        self.pages += n * L
        self.bytes += n * L * 2 * s.Hkv * ops.PAGE * s.D * 2
        self.launches += 1


class AttentionExecutor:
    """kv_append + paged decode attention for a set of rows on one stream.

    On a prefill GPU the stream belongs to the attention partition (see
    coloc.SmPartition) and ``num_sms`` is its SM count so the persistent grid
    fits the partition.
    """

    def __init__(self, kv: LayeredKV, Hq: int, max_batch: int,
                 stream: torch.cuda.Stream | None = None, num_sms: int = 0) -> None:
        self.kv = kv
        self.Hq = Hq
        self.stream = stream if stream is not None else torch.cuda.Stream(device=kv.device)
        self.num_sms = num_sms
        self.fused_append = True
        self.ws = ops.DecodeWorkspace(max(1, max_batch), Hq, kv.Hkv, kv.D, kv.device)
        self.scale = 1.0 / math.sqrt(kv.D)

    def run_layer(self, l: int, q, k_new, v_new, block_table, seq_lens, slots, out,
                  lse=None, stream: torch.cuda.Stream | None = None,
                  in_rows=None, out_rows=None) -> None:
        """Append each row's new token (position seq_len - 1) and attend.

        The append is fused into the attention pass; ``slots`` (the explicit slot
        mapping) is only used when ``fused_append`` is off. ``in_rows`` /
        ``out_rows``: zero-copy mode — q/k/v/out are the decode GPU's full
        tensors and these [n] maps pick this executor's rows (fused path only)."""
        if block_table.shape[0] == 0:
            return
        s = stream if stream is not None else self.stream
        kc, vc = self.kv.layer(l % self.kv.num_layers)  # a 1-layer pool serves a chain of layers
        if self.fused_append or in_rows is not None or out_rows is not None:
            ops.paged_decode_attn(q, kc, vc, block_table, seq_lens, out=out, lse=lse,
                                  scale=self.scale, workspace=self.ws, stream=s,
                                  num_sms=self.num_sms, k_new=k_new, v_new=v_new,
                                  in_rows=in_rows, out_rows=out_rows)
        else:
            ops.kv_append(k_new, v_new, kc, vc, slots, stream=s)
            ops.paged_decode_attn(q, kc, vc, block_table, seq_lens, out=out, lse=lse,
                                  scale=self.scale, workspace=self.ws, stream=s,
                                  num_sms=self.num_sms)


@dataclass
class StepPlan:
    """Device-side tables of one decode step (local rows first)."""

    n_local: int
    n_off: int
    local_bt: torch.Tensor        # [n_local, P] int32 (decode device)
    local_seq: torch.Tensor       # [n_local] int32
    local_slots: torch.Tensor     # [n_local] int64
    exec_bt: torch.Tensor | None = None     # [n_off, P] int32 (executor device)
    exec_seq: torch.Tensor | None = None
    exec_slots: torch.Tensor | None = None

    @property
    def batch(self) -> int:
        return self.n_local + self.n_off


@dataclass
class StepTimes:
    """Per-step timings from CUDA events (seconds) — the measured StepRecord fields."""

    total: float = 0.0
    local_attn: float = 0.0       # sum over layers, main stream
    exec_attn: float = 0.0        # sum over layers, executor stream
    stall: float = 0.0            # sum over layers of max(0, out_ready - local_done)
    link_bytes: int = 0
    per_layer_stall: list = field(default_factory=list)
    per_layer_local: list = field(default_factory=list)


def two_sided_step(loc: StepTimes, rem: StepTimes) -> StepTimes:
    """A step timed as on two GPUs (MeasuredPricer under prefill interference):
    ``loc`` = the decoder's local attention run alone, ``rem`` = the executor's
    side run alone (no local rows: its per-layer stall is the whole remote path,
    exchange included). Per layer, the decoder waits max(0, remote path -
    local attention) (engine.py:441-456)."""
    if len(loc.per_layer_local) != len(rem.per_layer_stall):
        raise ValueError("the two sides ran different layer counts")
    times = StepTimes(local_attn=loc.local_attn, exec_attn=rem.exec_attn,
                      link_bytes=rem.link_bytes)
    for la, path in zip(loc.per_layer_local, rem.per_layer_stall):
        st = max(0.0, path - la)
        times.stall += st
        times.per_layer_stall.append(st)
    times.per_layer_local = list(loc.per_layer_local)
    times.total = loc.total + times.stall
    return times


class OffloadedDecodeStep:
    """Drives one decode step across a local executor and (optionally) a remote
    one reached through a transport. Both executors may live on the same GPU
    (loopback: 1-GPU testing and the colocated-partition measurement).

    ``zero_copy=True`` (one process driving both GPUs, peer access on, or the
    same GPU): no messages at all — the executor's attention kernel reads the
    offloaded rows' q/k/v straight from the decode GPU's tensors and writes their
    outputs straight into the decode GPU's output rows (adr_paged_decode_attn_rows
    over NVLink), ordered by two cross-device events per layer. Same bytes on the
    link, none of the pack / copy / unpack / copy / scatter launches."""

    def __init__(self, Hq: int, Hkv: int, D: int, local: AttentionExecutor,
                 remote: AttentionExecutor | None = None, transport=None,
                 back_transport=None, timing: bool = True, zero_copy: bool = False) -> None:
        self.Hq, self.Hkv, self.D = Hq, Hkv, D
        self.local = local
        self.remote = remote
        dev = local.kv.device
        self.device = dev
        self.transport = transport if transport is not None else LoopbackTransport(
            remote.kv.device if remote is not None else dev)
        self.back = back_transport if back_transport is not None else LoopbackTransport(dev)
        self.exch = torch.cuda.Stream(device=dev)
        self.timing = timing
        self.zero_copy = zero_copy
        if zero_copy and remote is not None and remote.kv.device != dev:
            from . import _ffi
            _ffi.call("adr_peer_open", remote.kv.device.index, dev.index)

    def run(self, q_layers, k_layers, v_layers, plan: StepPlan, outs,
            on_enqueued=None) -> StepTimes:
        """q_layers[l] [B,Hq,D], k/v_layers[l] [B,Hkv,D], outs[l] [B,Hq,D] (all bf16 on the
        decode device). Enqueues the whole step; returns event timings after a sync.
        ``on_enqueued()`` runs once everything is enqueued, before the sync (e.g.
        ``PrefillCover.release``)."""
        main = torch.cuda.current_stream(self.device)
        L = len(q_layers)
        nl, no = plan.n_local, plan.n_off
        if no and self.remote is None:
            raise ValueError("offloaded rows need a remote executor")
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if self.timing else (lambda: None)
        t0, t1 = ev(), ev()
        rec = []
        if t0 is not None:
            t0.record(main)
        rows_off = torch.arange(nl, nl + no, dtype=torch.int32, device=self.device)
        rdev = self.remote.kv.device if self.remote is not None else self.device
        if self.zero_copy and no:
            return self._run_zero_copy(q_layers, k_layers, v_layers, plan, outs, rdev, ev,
                                       on_enqueued)
        msg_width = (self.Hq + 2 * self.Hkv) * self.D
        exec_msg = torch.empty((no, msg_width), dtype=torch.bfloat16, device=rdev) if no else None
        exec_out = torch.empty((no, self.Hq, self.D), dtype=torch.bfloat16, device=rdev) if no else None
        back_buf = torch.empty((no, self.Hq, self.D), dtype=torch.bfloat16, device=self.device) if no else None
        link = 0
        for l in range(L):
            q, k, v, out = q_layers[l], k_layers[l], v_layers[l], outs[l]
            e_local0, e_local1, e_exec0, e_exec1, e_out = ev(), ev(), ev(), ev(), ev()
            if no:
                # decode side: pack + send on the exchange stream once q/k/v exist
                produced = torch.cuda.Event()
                produced.record(main)
                self.exch.wait_event(produced)
                with torch.cuda.stream(self.exch):  # allocation belongs to the exchange stream
                    msg = ops.pack_qkv(q, k, v, rows_off, stream=self.exch)
                self.transport.send(TAG_QKV, l, msg, stream=self.exch)
                link += msg.numel() * 2
                # executor side
                xs = self.remote.stream
                self.transport.recv(TAG_QKV, l, exec_msg, stream=xs)
                with torch.cuda.stream(xs):
                    qo, ko, vo = ops.unpack_qkv(exec_msg, no, self.Hq, self.Hkv, self.D, stream=xs)
                if e_exec0 is not None:
                    e_exec0.record(xs)
                self.remote.run_layer(l, qo, ko, vo, plan.exec_bt, plan.exec_seq,
                                      plan.exec_slots, exec_out)
                if e_exec1 is not None:
                    e_exec1.record(xs)
                self.back.send(TAG_OUT, l, exec_out, stream=xs)
                link += exec_out.numel() * 2
            # decode side: local rows on the main stream
            if e_local0 is not None:
                e_local0.record(main)
            if nl:
                self.local.run_layer(l, q[:nl], k[:nl], v[:nl], plan.local_bt, plan.local_seq,
                                     plan.local_slots, out[:nl], stream=main)
            if e_local1 is not None:
                e_local1.record(main)
            if no:
                self.back.recv(TAG_OUT, l, back_buf, stream=main)
                ops.scatter_out(back_buf, rows_off, out, stream=main)
            if e_out is not None:
                e_out.record(main)
            rec.append((e_local0, e_local1, e_exec0, e_exec1, e_out))
        if t1 is not None:
            t1.record(main)
        if on_enqueued is not None:
            on_enqueued()
        times = StepTimes(link_bytes=link)
        if not self.timing:
            return times
        torch.cuda.synchronize(self.device)
        if rdev != self.device:
            torch.cuda.synchronize(rdev)
        times.total = t0.elapsed_time(t1) / 1e3
        for e_l0, e_l1, e_x0, e_x1, e_o in rec:
            la = e_l0.elapsed_time(e_l1) / 1e3
            times.local_attn += la
            times.per_layer_local.append(la)
            if no:
                times.exec_attn += e_x0.elapsed_time(e_x1) / 1e3
                # time the main stream spent waiting for the executor after its local work
                st = max(0.0, e_l1.elapsed_time(e_o) / 1e3)
                times.stall += st
                times.per_layer_stall.append(st)
        return times


    def _run_zero_copy(self, q_layers, k_layers, v_layers, plan: StepPlan, outs, rdev, ev,
                       on_enqueued=None):
        main = torch.cuda.current_stream(self.device)
        nl, no = plan.n_local, plan.n_off
        t0, t1 = ev(), ev()
        if t0 is not None:
            t0.record(main)
        rows = torch.arange(nl, nl + no, dtype=torch.int32, device=rdev)
        per_row = (self.Hq + 2 * self.Hkv) * self.D * 2 + self.Hq * self.D * 2
        xs = self.remote.stream
        rec = []
        for l in range(len(q_layers)):
            q, k, v, out = q_layers[l], k_layers[l], v_layers[l], outs[l]
            e_local0, e_local1, e_exec0, e_exec1, e_out = ev(), ev(), ev(), ev(), ev()
            produced = torch.cuda.Event()
            produced.record(main)
            xs.wait_event(produced)
            if e_exec0 is not None:
                e_exec0.record(xs)
            self.remote.run_layer(l, q, k, v, plan.exec_bt, plan.exec_seq, plan.exec_slots, out,
                                  in_rows=rows, out_rows=rows)
            if e_exec1 is not None:
                e_exec1.record(xs)
            done = torch.cuda.Event()
            done.record(xs)
            if e_local0 is not None:
                e_local0.record(main)
            if nl:
                self.local.run_layer(l, q[:nl], k[:nl], v[:nl], plan.local_bt, plan.local_seq,
                                     plan.local_slots, out[:nl], stream=main)
            if e_local1 is not None:
                e_local1.record(main)
            main.wait_event(done)
            if e_out is not None:
                e_out.record(main)
            rec.append((e_local0, e_local1, e_exec0, e_exec1, e_out))
        if t1 is not None:
            t1.record(main)
        if on_enqueued is not None:
            on_enqueued()
        times = StepTimes(link_bytes=per_row * no * len(q_layers))  # bytes the executor moves over the link
        if not self.timing:
            return times
        torch.cuda.synchronize(self.device)
        if rdev != self.device:
            torch.cuda.synchronize(rdev)
        times.total = t0.elapsed_time(t1) / 1e3
        for e_l0, e_l1, e_x0, e_x1, e_o in rec:
            la = e_l0.elapsed_time(e_l1) / 1e3
            times.local_attn += la
            times.per_layer_local.append(la)
            times.exec_attn += e_x0.elapsed_time(e_x1) / 1e3
            st = max(0.0, e_l1.elapsed_time(e_o) / 1e3)
            times.stall += st
            times.per_layer_stall.append(st)
        return times


class CapturedStep:
    """A CUDA graph of one enqueue function (warm-up on a side stream first, as
    graph capture requires). ``replay()`` re-issues every kernel of the step
    with one launch — the graphed branch of costs.launch_overhead
    (costs.py:94-108)."""

    def __init__(self, fn, warmup: int = 2) -> None:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()

    def replay(self) -> None:
        self.graph.replay()


class DecodeGraphCache:
    """2-D graph grid (graphs.build_grid / select_graph, graphs.py:41-84) of a
    decode step: one captured graph per (decode cap, offload cap) shape, built on
    first use. ``make(cd, co)`` returns (static_inputs, enqueue_fn) for a step
    padded to cd local and co offloaded rows (padding rows: seq_len 0 and slot
    -1, which every kernel treats as empty). Steps overflowing the grid run
    eagerly, like the reference's ungraphed path."""

    def __init__(self, grid, make) -> None:
        from .graphs import select_graph
        self.grid = grid
        self._select = select_graph
        self._make = make
        self.graphs: dict[tuple[int, int], tuple[dict, CapturedStep]] = {}
        self.eager_steps = 0
        self.graphed_steps = 0

    def shape_for(self, bd: int, bo: int):
        return self._select(self.grid, bd, bo)

    def run(self, bd: int, bo: int, fill) -> tuple[int, int] | None:
        """``fill(static_inputs, shape)`` copies the real step's inputs into the
        padded static buffers (shape None: build eager buffers for bd, bo)."""
        shape = self.shape_for(bd, bo)
        if shape is None:
            inputs, fn = self._make(bd, bo)
            fill(inputs, (bd, bo))
            fn()
            self.eager_steps += 1
            return None
        if shape not in self.graphs:
            inputs, fn = self._make(*shape)
            fill(inputs, shape)
            self.graphs[shape] = (inputs, CapturedStep(fn))
        inputs, cap = self.graphs[shape]
        fill(inputs, shape)
        cap.replay()
        self.graphed_steps += 1
        return shape


def step_record(idx: int, t: float, times: "StepTimes", layers_timed: int, num_layers: int,
                batch_local: int, batch_off: int, graph_shape, launch: float, nonattn: float,
                local_kv_bytes: float, exec_kv_bytes: dict, exec_attn: dict):
    """engine.StepRecord (engine.py:40-64) of one decode step from the CUDA-event
    timings of ``layers_timed`` executed layers (StepTimes), scaled to the
    model's ``num_layers``: local_attn, stall and link_bytes are the measured
    per-layer sums x num_layers / layers_timed; duration = launch + nonattn +
    local_attn + stall exactly as the reference composes it (engine.py:457)."""
    from .engine import StepRecord
    k = num_layers / layers_timed
    local_attn = times.local_attn * k
    stall = times.stall * k
    dur = launch + nonattn + local_attn + stall
    return StepRecord(idx, t, t + dur, batch_local, batch_off, graph_shape, launch, nonattn,
                      local_attn, stall, local_kv_bytes, exec_kv_bytes, exec_attn,
                      float(times.link_bytes) * k)


class MeasuredPricer:
    """engine.StepPricer that prices a decode step by running it.

    Closed loop (reference step pricing engine.py:423-456):
    every simulated step of a decoder runs the real offloaded decode step —
    ``OffloadedDecodeStep`` over ``chain`` layers with the decoder's running
    local requests on this GPU's main stream and, per executor, its offloaded
    requests on the executor stream: a green-context partition of
    ``attn_sm_ratio`` of the SMs while a model-shaped ``PrefillLoad`` keeps the
    complementary prefill partition busy (``prefill_interference``; the
    colocated prefill GPU of PAPER.md:436). Block tables come from the
    engine-driven ``PagedKVMirror``; contexts are the requests' resident tokens
    plus the appended one. The exchange is real too: the zero-copy row-mapped
    executor kernel by default (``zero_copy``), or the pack / send / unpack /
    scatter message path. ``local_attn``, ``exec_attn``, ``stall`` and
    ``link_bytes`` of the StepRecord are the CUDA-event measurements of that
    step (``step_record``) scaled from ``chain`` to the model's layers; launch
    and non-attention stay analytic, as in the reference (engine.py:447-456).
    ``records`` keeps (StepRecord, [StepTimes per executor group]) for checks.
    """

    def __init__(self, cfg, mirror, device: int = 0, use_partition: bool = True,
                 prefill_interference: bool = True, zero_copy: bool = True,
                 chain: int = 4, keep_records: int = 0) -> None:
        from . import coloc
        m = cfg.model
        self.cfg = cfg
        self.mirror = mirror
        self.dev = torch.device("cuda", device)
        self.Hq, self.Hkv, self.D = m.q_heads, m.kv_heads, m.dim_per_head
        self.L = m.num_layers
        g = torch.Generator(device=self.dev).manual_seed(0)
        pages = {w: bt.pool.num_pages for w, bt in mirror.pools.items()}
        self.kv = {}
        for kind in ("decoder", "executor"):
            n = max([v for (k, _), v in pages.items() if k == kind] + [1])
            self.kv[kind] = LayeredKV(1, n, self.Hkv, self.D, self.dev, fill="randn", generator=g)
        self.part = None
        self.prefill = None
        if use_partition and coloc.green_contexts_supported():
            total = torch.cuda.get_device_properties(device).multi_processor_count
            self.part = coloc.SmPartition(device, int(round(cfg.attn_sm_ratio * total)))
            if prefill_interference:
                self.prefill = coloc.prefill_load_for(m, self.dev)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.local = AttentionExecutor(self.kv["decoder"], self.Hq, 2048, stream=self.stream)
        xs, xsms = (self.part.attn_stream, self.part.attn_sms) if self.part else (None, 0)
        self.remote = AttentionExecutor(self.kv["executor"], self.Hq, 2048, stream=xs, num_sms=xsms)
        self.step = OffloadedDecodeStep(self.Hq, self.Hkv, self.D, self.local, self.remote,
                                        zero_copy=zero_copy)
        self.chain = chain
        self.kernel_calls = 0
        self.uncovered_steps = 0      # steps the prefill load did not fully cover (after retries)
        self.retried_steps = 0        # step runs re-done because the cover fell short
        self._prefill_s = None
        self._enqueue_s = 5e-3        # host time to enqueue a step (decaying max)
        self._last_step_s = 1e-3
        self.keep_records = keep_records
        self.records: list = []

    def _tables(self, where, reqs):
        bt = self.mirror.pools[where]
        ids = [r.req_id for r in reqs]
        table = torch.from_numpy(bt.table_array(ids)).to(self.dev)
        seq = torch.tensor([r.used_token + 1 for r in reqs], dtype=torch.int32, device=self.dev)
        return table, seq

    def run_step(self, local_reqs, where_local, off_reqs, where_exec) -> StepTimes:
        """One real offloaded step (``chain`` layers) of these requests; returns
        its StepTimes (sums over the executed layers)."""
        nl, no = len(local_reqs), len(off_reqs)
        B = nl + no
        if nl:
            lbt, lseq = self._tables(where_local, local_reqs)
        else:
            lbt = torch.zeros((0, 1), dtype=torch.int32, device=self.dev)
            lseq = torch.zeros(0, dtype=torch.int32, device=self.dev)
        xbt = xseq = None
        if no:
            xbt, xseq = self._tables(where_exec, off_reqs)
        plan = StepPlan(nl, no, lbt, lseq, None, xbt, xseq, None)
        mk = lambda *s: torch.randn(*s, device=self.dev).to(torch.bfloat16)
        qs = [mk(B, self.Hq, self.D) for _ in range(self.chain)]
        ks = [mk(B, self.Hkv, self.D) for _ in range(self.chain)]
        vs = [mk(B, self.Hkv, self.D) for _ in range(self.chain)]
        outs = [torch.empty(B, self.Hq, self.D, dtype=torch.bfloat16, device=self.dev)
                for _ in range(self.chain)]
        if no and self.prefill is not None and nl:
            # Two GPUs emulated on one: the decoder's local attention runs alone
            # (a decode GPU hosts no prefill), the executor's attention runs on
            # its SM partition beside the prefill load (the prefill GPU). Run
            # concurrently on this one GPU, the local kernels would take the
            # executor partition's SMs and HBM instead. Per layer, the stall is
            # the reference's max(0, remote path - local attention)
            # (engine.py:441-456) from the two measured sides.
            none = StepPlan(nl, 0, lbt, lseq, None, None, None, None)
            loc = self._timed(qs, ks, vs, none, outs, covered=False)
            remote = StepPlan(0, no, lbt[:0], lseq[:0], None, xbt, xseq, None)
            rem = self._timed([q[nl:] for q in qs], [k[nl:] for k in ks], [v[nl:] for v in vs],
                              remote, [o[nl:] for o in outs], covered=True)
            times = two_sided_step(loc, rem)
        else:
            times = self._timed(qs, ks, vs, plan, outs, covered=bool(no))
        self._last_step_s = max(times.total, 1e-5)
        return times

    def _timed(self, qs, ks, vs, plan: StepPlan, outs, covered: bool) -> StepTimes:
        """Run one step; with ``covered`` (and a prefill load) the prefill runs on
        its partition across the whole step (PrefillCover)."""
        nl, no = plan.n_local, plan.n_off
        main = torch.cuda.current_stream(self.dev)
        covered = covered and self.prefill is not None
        if covered and self._prefill_s is None:
            # first covered step: one untimed run of the step first (first-use
            # host work — workspaces, kernel attributes — would otherwise
            # stretch its enqueue past the estimate), then time the prefill
            self.step.run(qs, ks, vs, plan, outs)
            torch.cuda.synchronize(self.dev)
            ps = self.part.prefill_stream
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self.prefill.run(ps)
            e0.record(ps)
            self.prefill.run(ps)
            e1.record(ps)
            e1.synchronize()
            self._prefill_s = e0.elapsed_time(e1) / 1e3
        # A step the prefill did not cover from its first kernel to its last (a
        # host hiccup stretched the enqueue past the estimate) is re-run with a
        # longer cover; the step's inputs are the same, so re-running it (fused
        # append included) writes the same bytes.
        for attempt in range(3):
            cover = None
            if covered:
                from .coloc import PrefillCover
                cover = PrefillCover(self.part.prefill_stream, self.prefill)
                # the prefill runs from before the step's first kernel to after its
                # last: enough iterations for the host's enqueue time of the step
                # (it starts running at once) plus twice the step's GPU time
                need = (2.0 * self._enqueue_s + 2.0 * self._last_step_s) * (2 ** attempt)
                gate = cover.start(int(math.ceil(need / self._prefill_s)) + 2)
                main.wait_event(gate)
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(main)
            h0 = time.perf_counter()
            t1 = torch.cuda.Event(enable_timing=True)

            def enqueued():
                # the step's end on the main stream: recorded before step.run
                # synchronises (which also waits for the rest of the prefill cover)
                t1.record(main)
                self._enqueue_s = max(0.8 * self._enqueue_s, time.perf_counter() - h0)
            times = self.step.run(qs, ks, vs, plan, outs, on_enqueued=enqueued)
            self.kernel_calls += self.chain * ((1 if nl else 0) + (1 if no else 0))
            if cover is None:
                break
            torch.cuda.synchronize(self.dev)
            if cover.covered(t0, t1):
                break
            self.retried_steps += 1
        else:
            self.uncovered_steps += 1
        return times

    def price(self, sim, d, t):
        from .costs import launch_overhead, nonattn_step_latency
        from .graphs import select_graph
        cfg = sim.cfg
        kv_tok = sim.kv_tok
        bd, bo = len(d.run_local), len(d.run_off)
        kv_local = float(sum(r.used_token for r in d.run_local)) * kv_tok
        where_local = ("decoder", d.idx)
        groups = [(e, [r for r in d.run_off if r.executor_id == e])
                  for e in sorted({r.executor_id for r in d.run_off})]
        runs = []
        if not groups:
            runs.append(self.run_step(d.run_local, where_local, [], None))
        for e, group in groups:  # one executor at a time (one partition on this GPU)
            runs.append(self.run_step(d.run_local, where_local, group, ("executor", e)))
        k = self.L / self.chain
        exec_kv = {e: float(sum(r.used_token for r in g)) * kv_tok for e, g in groups}
        exec_attn = {e: tm.exec_attn * k for (e, _), tm in zip(groups, runs)}
        # the decoder's local attention (same rows every run: their mean) and
        # its stall on the slowest executor
        agg = StepTimes(local_attn=sum(tm.local_attn for tm in runs) / len(runs),
                        stall=max(tm.stall for tm in runs),
                        link_bytes=sum(tm.link_bytes for tm in runs))
        L = cfg.model.num_layers
        shape = select_graph(sim.grid, bd, bo) if cfg.use_graphs else None
        if shape is not None:
            nonattn = nonattn_step_latency(cfg.gpu, cfg.model, shape[0] + shape[1])
            launch = launch_overhead(L, True, cfg.gpu)
        else:
            nonattn = nonattn_step_latency(cfg.gpu, cfg.model, bd + bo)
            launch = launch_overhead(L, False, cfg.gpu, (nonattn + agg.local_attn * k) / L)
        rec = step_record(d.idx, t, agg, self.chain, L, bd, bo, shape, launch, nonattn, kv_local,
                          exec_kv, exec_attn)
        if len(self.records) < self.keep_records:
            self.records.append((rec, runs))
        return rec


class RoleSplitStep:
    """One decode step across two processes: a *decoder* rank and the *executor*
    rank of a prefill-role GPU (one process per GPU).

    Per layer the decoder packs the offloaded rows' q/k/v into one message and
    sends it, runs the fused-append attention of its local rows, receives the
    executor's outputs and scatters them beside its own; the executor receives,
    unpacks, runs fused-append attention over its paged cache (on its SM
    partition) and sends the outputs back. Messages travel through ``transport``
    (exchange.DistTransport: NCCL isend/irecv over NVLink on GPUs).

    The compute callables default to the sm_100a ops; they are parameters so the
    exact protocol can run under gloo on CPU in tests.
    """

    def __init__(self, role: str, Hq: int, Hkv: int, D: int, transport, *, attend=None,
                 pack=None, unpack=None, scatter=None) -> None:
        if role not in ("decoder", "executor"):
            raise ValueError("role must be 'decoder' or 'executor'")
        self.role = role
        self.Hq, self.Hkv, self.D = Hq, Hkv, D
        self.t = transport
        self.attend = attend
        self.pack = pack or (lambda q, k, v, rows: ops.pack_qkv(q, k, v, rows))
        self.unpack = unpack or (lambda msg, n: ops.unpack_qkv(msg, n, Hq, Hkv, D))
        self.scatter = scatter or (lambda src, rows, out: ops.scatter_out(src, rows, out))

    def run_decoder(self, q_layers, k_layers, v_layers, n_local: int, outs) -> int:
        """Rows [0, n_local) are local, the rest offloaded. Returns link bytes."""
        from .exchange import TAG_OUT, TAG_QKV
        B = q_layers[0].shape[0]
        n_off = B - n_local
        dev = q_layers[0].device
        rows = torch.arange(n_local, B, dtype=torch.int32, device=dev)
        back = torch.empty((n_off, self.Hq, self.D), dtype=q_layers[0].dtype, device=dev)
        link = 0
        for l in range(len(q_layers)):
            if n_off:
                msg = self.pack(q_layers[l], k_layers[l], v_layers[l], rows)
                self.t.send(TAG_QKV, l, msg)
                link += msg.numel() * msg.element_size()
            if n_local:
                self.attend(l, q_layers[l][:n_local], k_layers[l][:n_local],
                            v_layers[l][:n_local], outs[l][:n_local])
            if n_off:
                self.t.recv(TAG_OUT, l, back)
                link += back.numel() * back.element_size()
                self.scatter(back, rows, outs[l])
        if hasattr(self.t, "flush"):
            self.t.flush()
        return link

    def run_executor(self, num_layers: int, n_rows: int, dtype, device) -> None:
        from .exchange import TAG_OUT, TAG_QKV
        msg = torch.empty((n_rows, (self.Hq + 2 * self.Hkv) * self.D), dtype=dtype, device=device)
        out = torch.empty((n_rows, self.Hq, self.D), dtype=dtype, device=device)
        for l in range(num_layers):
            self.t.recv(TAG_QKV, l, msg)
            q, k, v = self.unpack(msg, n_rows)
            self.attend(l, q, k, v, out)
            self.t.send(TAG_OUT, l, out)
        if hasattr(self.t, "flush"):
            self.t.flush()


class ZeroCopyRoleStep:
    """The decode/executor role split with no messages at all (one process per
    GPU, PAPER.md:371 steps 2-3 fused into the attention kernel).

    Setup (once): the decoder exports, over CUDA IPC, its per-layer q/k/v/out
    tensors and a [2, L] uint32 flag array (q ready / out ready per layer); the
    executor maps them. Per step ``s`` and layer ``l``:

      decoder   adr_signal(q_ready[l] = s) once the layer's q/k/v exist, runs its
                local rows, then adr_wait(out_ready[l] >= s) before using out
      executor  adr_wait(q_ready[l] >= s) on its (partition) stream, runs
                adr_paged_decode_attn_rows reading rows [n_local, B) of the
                decode GPU's q/k/v over NVLink and writing their outputs into the
                decode GPU's out rows, then adr_signal(out_ready[l] = s) — a
                fenced stream write into the decode GPU's memory

    Flags are stream-ordered (cuStreamWrite/WaitValue32): no host round trip and
    no SM spins. The descriptors travel once over ``torch.distributed``
    (object send/recv; gloo or NCCL).
    """

    def __init__(self, role: str, num_layers: int, peer_rank: int, group=None) -> None:
        if role not in ("decoder", "executor"):
            raise ValueError("role must be 'decoder' or 'executor'")
        self.role, self.L, self.peer, self.group = role, num_layers, peer_rank, group
        self.flags = None
        self.remote = None

    def _flag(self, which: int, l: int) -> int:
        f = self.flags
        return f.data_ptr() + (which * self.L + l) * 4

    def setup_decoder(self, q_layers, k_layers, v_layers, outs) -> None:
        import torch.distributed as dist
        from .exchange import ipc_export
        dev = q_layers[0].device
        self.flags = torch.zeros((2, self.L), dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        desc = {"q": [ipc_export(t) for t in q_layers], "k": [ipc_export(t) for t in k_layers],
                "v": [ipc_export(t) for t in v_layers], "out": [ipc_export(t) for t in outs],
                "flags": ipc_export(self.flags)}
        dist.send_object_list([desc], dst=self.peer, group=self.group)

    def setup_executor(self, device: torch.device) -> None:
        import torch.distributed as dist
        from .exchange import ipc_import
        box = [None]
        dist.recv_object_list(box, src=self.peer, group=self.group)
        d = box[0]
        self.remote = {k: [ipc_import(x, device) for x in d[k]] for k in ("q", "k", "v", "out")}
        self.flags = ipc_import(d["flags"], device)

    def decoder_step(self, step: int, n_local: int, attend_local, outs,
                     stream: torch.cuda.Stream | None = None) -> None:
        """attend_local(l) runs the local rows of layer l on ``stream``."""
        s = stream if stream is not None else torch.cuda.current_stream()
        for l in range(self.L):
            _ffi.call("adr_signal", self._flag(0, l), step, s.cuda_stream)
            if n_local:
                attend_local(l)
            _ffi.call("adr_wait", self._flag(1, l), step, s.cuda_stream)

    def executor_step(self, step: int, n_local: int, batch: int, executor: "AttentionExecutor",
                      block_table, seq_lens) -> None:
        """Attend rows [n_local, batch) of the decode GPU with ``executor``'s cache."""
        xs = executor.stream
        rows = torch.arange(n_local, batch, dtype=torch.int32, device=executor.kv.device)
        xs.wait_stream(torch.cuda.current_stream(executor.kv.device))
        for l in range(self.L):
            _ffi.call("adr_wait", self._flag(0, l), step, xs.cuda_stream)
            executor.run_layer(l, self.remote["q"][l], self.remote["k"][l], self.remote["v"][l],
                               block_table, seq_lens, None, self.remote["out"][l], stream=xs,
                               in_rows=rows, out_rows=rows)
            _ffi.call("adr_signal", self._flag(1, l), step, xs.cuda_stream)

    def close(self) -> None:
        if self.remote is not None:
            for lst in self.remote.values():
                for p in lst:
                    p.close()
            self.flags.close()
            self.remote = None
