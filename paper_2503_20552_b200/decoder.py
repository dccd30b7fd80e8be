"""Full decode layers around the attention path, for full-layer tokens/s.

The reference prices the non-attention part of a decode step analytically
(``costs.nonattn_step_latency``, costs.py:77-91: every weight byte read once
per step, flat below b_max) and the paper's prototype runs it with vLLM's
model code. Here it is real GPU work with the model's shapes: per layer

    h = rms_norm(x);  q, k, v = h Wq^T, h Wk^T, h Wv^T   (cuBLAS bf16; one GEMM for MHA)
    attn = adr_paged_decode_attn(q, K_l, V_l, k_new=k, v_new=v)  (ours, fused append)
    x += attn Wo^T;  h = rms_norm(x);  g|u = h [Wg|Wu]^T (one GEMM);  x += (silu(g) * u) Wd^T

with synthetic random weights (no checkpoints offline; "the
non-attention layers in the tokens/s bench are real bf16 GEMMs with synthetic
weights"), every layer its own weights so nothing is L2-resident across layers.
No rotary embedding (elementwise, immaterial to the step's HBM traffic). The
GEMMs are plain library GEMMs (cuBLAS); the attention is the product path.
The whole step is captured into one CUDA graph (runtime.CapturedStep), the
graphed branch of costs.launch_overhead (costs.py:94-108).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import ops

__all__ = ["LayerDims", "MODEL_DIMS", "SyntheticDecoder", "OffloadedDecoder", "RemoteOffloadedDecoder",
           "OffloadServer"]


@dataclass(frozen=True)
class LayerDims:
    hidden: int
    intermediate: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int

    def weight_bytes_per_layer(self, elem: int = 2) -> int:
        h, i = self.hidden, self.intermediate
        qkv = (self.num_q_heads + 2 * self.num_kv_heads) * self.head_dim * h
        o = h * self.num_q_heads * self.head_dim
        return elem * (qkv + o + 3 * h * i + 2 * h)


# Public architecture shapes of the BASELINE.json models.
MODEL_DIMS = {
    "llama2-7b": LayerDims(4096, 11008, 32, 32, 128),
    "llama3-8b": LayerDims(4096, 14336, 32, 8, 128),
    "llama2-13b": LayerDims(5120, 13824, 40, 40, 128),
    "llama3-70b": LayerDims(8192, 28672, 64, 8, 128),
}


class SyntheticDecoder:
    """L decode layers of ``dims`` on ``device`` for a fixed batch B.

    ``kv`` is a list of per-layer (k_cache, v_cache) [NB, Hkv, 16, D] bf16; the
    block table and lengths are shared by all layers (one page allocation per
    request, as in a paged engine). ``step(x)`` advances the residual stream x
    [B, hidden] bf16 in place through every layer.
    """

    def __init__(self, dims: LayerDims, kv: list, batch: int, device: torch.device,
                 seed: int = 0, eps: float = 1e-5, weights: list | None = None,
                 nonattn: bool = True) -> None:
        self.dims, self.kv, self.B, self.device, self.eps = dims, kv, batch, device, eps
        # nonattn=False: attention-only layers (no weights; q / k / v rows are
        # random and fixed, each layer is its fused-append attention call)
        self.nonattn = nonattn
        L = len(kv)
        h, I = dims.hidden, dims.intermediate
        Hq, Hkv, D = dims.num_q_heads, dims.num_kv_heads, dims.head_dim
        g = torch.Generator(device=device).manual_seed(seed)
        # MHA: one fused QKV GEMM; the attention reads q / k / v as rows 3b, 3b+1,
        # 3b+2 of its output through the kernel's row maps (no split copies)
        self.mha = Hq == Hkv

        def w(n, k):  # N(0, 1/k): activations keep unit scale through the GEMM
            t = torch.empty((n, k), dtype=torch.bfloat16, device=device)
            step = max(1, (1 << 26) // k)
            for lo in range(0, n, step):
                hi = min(n, lo + step)
                t[lo:hi] = torch.randn((hi - lo, k), generator=g, device=device) / math.sqrt(k)
            return t

        self.layers = weights if weights is not None else []
        if not nonattn and weights is None:
            self.layers = [{} for _ in range(L)]
        for _ in range(0 if (weights is not None or not nonattn) else L):
            qkv = ({"wqkv": w(3 * Hq * D, h)} if self.mha else
                   {"wq": w(Hq * D, h), "wk": w(Hkv * D, h), "wv": w(Hkv * D, h)})
            self.layers.append({
                **qkv,
                "wo": w(h, Hq * D), "wgu": w(2 * I, h), "wd": w(h, I),  # gate | up fused
                "n1": torch.ones(h, dtype=torch.bfloat16, device=device),
                "n2": torch.ones(h, dtype=torch.bfloat16, device=device),
            })
        B = batch
        bf = dict(dtype=torch.bfloat16, device=device)
        if self.mha:
            self.qkv = torch.empty(3 * B + 2, Hq * D, **bf)  # + 2 rows: the shifted k / v views
            self.q = self.qkv[:3 * B].view(3 * B, Hq, D)
            self.k = self.qkv[1:3 * B + 1].view(3 * B, Hkv, D)
            self.v = self.qkv[2:3 * B + 2].view(3 * B, Hkv, D)
            self.rows = torch.arange(0, 3 * B, 3, dtype=torch.int32, device=device)
        else:
            self.q = torch.empty(B, Hq, D, **bf)
            self.k = torch.empty(B, Hkv, D, **bf)
            self.v = torch.empty(B, Hkv, D, **bf)
            self.rows = None
        if not nonattn:
            for t in ((self.qkv,) if self.mha else (self.q, self.k, self.v)):
                t.copy_(torch.randn(t.shape, generator=g, device=device))
        self.attn = torch.empty(B, Hq, D, **bf)
        self.o = torch.empty(B, h, **bf)
        self.gate_up = torch.empty(B, 2 * I, **bf)
        self.ws = [ops.DecodeWorkspace(B, Hq, Hkv, D, device) for _ in range(2)]
        self.scale = 1.0 / math.sqrt(D)

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    def weight_bytes(self) -> int:
        return self.dims.weight_bytes_per_layer() * self.num_layers if self.nonattn else 0

    def layer(self, l: int, x: torch.Tensor, block_table, seq_lens, pdl: bool = False) -> None:
        if not self.nonattn:
            self.attention(l, block_table, seq_lens, pdl)
            return
        W = self.layers[l]
        B, hdim = x.shape
        h = F.rms_norm(x, (hdim,), W["n1"], self.eps)
        if self.mha:
            torch.matmul(h, W["wqkv"].t(), out=self.qkv[:3 * B].view(B, -1))
        else:
            torch.matmul(h, W["wq"].t(), out=self.q.view(B, -1))
            torch.matmul(h, W["wk"].t(), out=self.k.view(B, -1))
            torch.matmul(h, W["wv"].t(), out=self.v.view(B, -1))
        self.attention(l, block_table, seq_lens, pdl)
        torch.matmul(self.attn.view(B, -1), W["wo"].t(), out=self.o)
        x.add_(self.o)
        h = F.rms_norm(x, (hdim,), W["n2"], self.eps)
        torch.matmul(h, W["wgu"].t(), out=self.gate_up)
        I = self.dims.intermediate
        act = F.silu(self.gate_up[:, :I]).mul_(self.gate_up[:, I:])
        torch.matmul(act, W["wd"].t(), out=self.o)
        x.add_(self.o)

    def attention(self, l: int, block_table, seq_lens, pdl: bool) -> None:
        """Fused-append decode attention of layer l over all B rows."""
        kc, vc = self.kv[l]
        ops.paged_decode_attn(self.q, kc, vc, block_table, seq_lens, out=self.attn,
                              scale=self.scale, workspace=self.ws[l % 2],
                              k_new=self.k, v_new=self.v, pdl=pdl, in_rows=self.rows)

    def step(self, x: torch.Tensor, block_table, seq_lens, pdl: bool = False) -> torch.Tensor:
        if x.shape != (self.B, self.dims.hidden) or x.dtype != torch.bfloat16:
            raise ValueError(f"x must be [{self.B}, {self.dims.hidden}] bf16")
        for l in range(self.num_layers):
            self.layer(l, x, block_table, seq_lens, pdl=pdl)
        return x


class OffloadedDecoder(SyntheticDecoder):
    """Full decode layers with attention offloading (the
    reference's step composition engine.py:423-456 made real): rows
    [0, n_local) of the batch attend over the decode GPU's caches on the main
    stream; rows [n_local, B) attend on an executor — its own per-layer caches
    ``exec_kv`` and stream (a green-context partition of a prefill GPU, or of
    this GPU for the 1-GPU loopback) — through the zero-copy row-mapped kernel:
    it reads the offloaded rows' q / k / v straight out of the decoder's QKV
    projection output and writes their attention rows straight into the
    decoder's attention buffer (no pack / send / unpack / scatter launches).
    Per layer the executor forks from the main stream after the QKV GEMM and
    joins before the O projection, so its attention overlaps the local
    attention; the whole step captures into one CUDA graph (both streams).

    ``step(x, local_bt, local_seq, exec_bt, exec_seq)``: tables of the local
    and the offloaded rows (executor pages), contexts including the appended
    token. ``exec_device``: the executor's device (peer access is enabled; the
    caches and tables of the executor live there)."""

    def __init__(self, dims: LayerDims, kv: list, exec_kv: list, batch: int, n_local: int,
                 device: torch.device, exec_stream: torch.cuda.Stream | None = None,
                 exec_sms: int = 0, seed: int = 0, eps: float = 1e-5,
                 weights: list | None = None, nonattn: bool = True) -> None:
        super().__init__(dims, kv, batch, device, seed=seed, eps=eps, weights=weights,
                         nonattn=nonattn)
        if not 0 <= n_local <= batch:
            raise ValueError("n_local must be in [0, batch]")
        if len(exec_kv) != len(kv):
            raise ValueError("exec_kv needs one cache pair per layer")
        self.n_local = n_local
        self.exec_kv = exec_kv
        xdev = exec_kv[0][0].device
        self.exec_device = xdev
        if xdev != torch.device(device):
            from . import _ffi
            _ffi.call("adr_peer_open", torch.device(device).index, xdev.index)
        # (the executor's grid is dispatched ahead of kernels queued before it: coloc.SmPartition)
        self.exec_stream = exec_stream if exec_stream is not None else torch.cuda.Stream(
            device=xdev, priority=torch.cuda.Stream.priority_range()[1])
        self.exec_sms = exec_sms
        B, no = batch, batch - n_local
        Hq, Hkv, D = dims.num_q_heads, dims.num_kv_heads, dims.head_dim
        self.exec_ws = [ops.DecodeWorkspace(max(1, no), Hq, Hkv, D, xdev) for _ in range(2)]
        # executor row maps: offloaded request i reads q/k/v row n_local + i (x3 in
        # the MHA fused-QKV layout) and writes attention row n_local + i
        off = torch.arange(n_local, B, dtype=torch.int32)
        self.exec_in = (off * 3 if self.mha else off).to(xdev)
        self.exec_out = off.to(xdev)
        self.local_rows = self.rows[:n_local] if self.mha else None
        self._exec_tables = None

    def attention(self, l: int, block_table, seq_lens, pdl: bool) -> None:
        main = torch.cuda.current_stream(self.device)
        nl, no = self.n_local, self.B - self.n_local
        xs = self.exec_stream
        if no:
            xbt, xseq = self._exec_tables
            ready = torch.cuda.Event()
            ready.record(main)
            xs.wait_event(ready)
            kc, vc = self.exec_kv[l]
            ops.paged_decode_attn(self.q, kc, vc, xbt, xseq, out=self.attn, scale=self.scale,
                                  workspace=self.exec_ws[l % 2], stream=xs, num_sms=self.exec_sms,
                                  k_new=self.k, v_new=self.v, pdl=pdl, in_rows=self.exec_in,
                                  out_rows=self.exec_out)
            done = torch.cuda.Event()
            done.record(xs)
        if nl:
            kc, vc = self.kv[l]
            if self.mha:
                ops.paged_decode_attn(self.q, kc, vc, block_table, seq_lens, out=self.attn,
                                      scale=self.scale, workspace=self.ws[l % 2], k_new=self.k,
                                      v_new=self.v, pdl=pdl, in_rows=self.local_rows)
            else:
                ops.paged_decode_attn(self.q[:nl], kc, vc, block_table, seq_lens,
                                      out=self.attn[:nl], scale=self.scale,
                                      workspace=self.ws[l % 2], k_new=self.k[:nl],
                                      v_new=self.v[:nl], pdl=pdl)
        if no:
            main.wait_event(done)

    def step(self, x: torch.Tensor, block_table, seq_lens, exec_block_table=None,
             exec_seq_lens=None, pdl: bool = False) -> torch.Tensor:
        no = self.B - self.n_local
        if no and (exec_block_table is None or exec_seq_lens is None):
            raise ValueError("offloaded rows need the executor's block table and lengths")
        if block_table.shape[0] != self.n_local or (no and exec_block_table.shape[0] != no):
            raise ValueError("table rows must match n_local / the offloaded count")
        self._exec_tables = (exec_block_table, exec_seq_lens)
        return super().step(x, block_table, seq_lens, pdl=pdl)


class RemoteOffloadedDecoder(SyntheticDecoder):
    """Full decode layers with the offloaded rows' attention on ANOTHER PROCESS's
    GPU (one process per GPU; the 8-GPU decode/prefill role split of
    PAPER.md:361-371 and engine.py:423-456). Rows [0, n_local) attend locally;
    rows [n_local, B) are attended by an ``OffloadServer`` on the executor GPU,
    which reads their q / k / v straight out of this process's QKV projection
    buffer and writes their attention rows straight into this process's
    attention buffer over NVLink (CUDA IPC mappings + adr_paged_decode_attn_rows).
    Per layer and step s, on the main stream:

        QKV GEMM -> adr_signal(q_ready[l] = s) -> local attention
                 -> adr_wait(out_ready[l] >= s) -> O projection, MLP

    so the executor's attention overlaps the local attention, and the step
    stalls only when it is the longer of the two (the reference's
    ``stall = max(0, remote - local)``, engine.py:441-456, made real).
    ``export()`` gives the picklable descriptors for the server process."""

    def __init__(self, dims: LayerDims, kv: list, batch: int, n_local: int,
                 device: torch.device, seed: int = 0, eps: float = 1e-5,
                 weights: list | None = None, nonattn: bool = True) -> None:
        super().__init__(dims, kv, batch, device, seed=seed, eps=eps, weights=weights,
                         nonattn=nonattn)
        if not 0 <= n_local <= batch:
            raise ValueError("n_local must be in [0, batch]")
        self.n_local = n_local
        self.flags = torch.zeros((2, len(kv)), dtype=torch.int32, device=device)
        self.step_id = 0
        self.local_rows = self.rows[:n_local] if self.mha else None

    def _flag(self, which: int, l: int) -> int:
        return self.flags.data_ptr() + (which * self.flags.shape[1] + l) * 4

    def export(self) -> dict:
        from .exchange import ipc_export
        torch.cuda.synchronize(self.device)
        qkv = self.qkv if self.mha else None
        return {"mha": self.mha, "B": self.B, "n_local": self.n_local,
                "dims": (self.dims.num_q_heads, self.dims.num_kv_heads, self.dims.head_dim),
                "qkv": ipc_export(qkv) if qkv is not None else None,
                "q": None if qkv is not None else ipc_export(self.q),
                "k": None if qkv is not None else ipc_export(self.k),
                "v": None if qkv is not None else ipc_export(self.v),
                "attn": ipc_export(self.attn), "flags": ipc_export(self.flags),
                "layers": len(self.kv)}

    def attention(self, l: int, block_table, seq_lens, pdl: bool) -> None:
        from . import _ffi
        main = torch.cuda.current_stream(self.device)
        nl, no = self.n_local, self.B - self.n_local
        if no:
            _ffi.call("adr_signal", self._flag(0, l), self.step_id, main.cuda_stream)
        if nl:
            kc, vc = self.kv[l]
            if self.mha:
                ops.paged_decode_attn(self.q, kc, vc, block_table, seq_lens, out=self.attn,
                                      scale=self.scale, workspace=self.ws[l % 2], k_new=self.k,
                                      v_new=self.v, pdl=pdl, in_rows=self.local_rows)
            else:
                ops.paged_decode_attn(self.q[:nl], kc, vc, block_table, seq_lens,
                                      out=self.attn[:nl], scale=self.scale,
                                      workspace=self.ws[l % 2], k_new=self.k[:nl],
                                      v_new=self.v[:nl], pdl=pdl)
        if no:
            _ffi.call("adr_wait", self._flag(1, l), self.step_id, main.cuda_stream)

    def step(self, x: torch.Tensor, block_table, seq_lens, pdl: bool = False) -> torch.Tensor:
        if block_table.shape[0] != self.n_local:
            raise ValueError("block_table rows must match n_local")
        self.step_id += 1
        return super().step(x, block_table, seq_lens, pdl=pdl)


class OffloadServer:
    """Executor side of ``RemoteOffloadedDecoder`` (runs in the prefill-role
    GPU's process): per step s and layer l, on its stream (an SM partition of
    the prefill GPU), adr_wait(q_ready[l] >= s), the row-mapped decode
    attention of the offloaded rows over this GPU's caches ``exec_kv`` (reading
    q / k / v from the decoder and writing attention rows into it, over
    NVLink), then adr_signal(out_ready[l] = s) into the decoder's memory."""

    def __init__(self, desc: dict, exec_kv: list, device: torch.device,
                 stream: torch.cuda.Stream | None = None, num_sms: int = 0) -> None:
        from .exchange import DevicePtr, ipc_import
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.Stream(
            device=self.device, priority=torch.cuda.Stream.priority_range()[1])
        self.num_sms = num_sms
        self.kv = exec_kv
        Hq, Hkv, D = desc["dims"]
        B, nl = desc["B"], desc["n_local"]
        self.B, self.n_local, self.no = B, nl, B - nl
        self.mapped = []
        if desc["mha"]:
            qkv = ipc_import(desc["qkv"], self.device)
            self.mapped.append(qkv)
            row = Hq * D * 2
            self.q = DevicePtr(qkv.ptr, (3 * B, Hq, D), torch.bfloat16, self.device)
            self.k = DevicePtr(qkv.ptr + row, (3 * B, Hkv, D), torch.bfloat16, self.device)
            self.v = DevicePtr(qkv.ptr + 2 * row, (3 * B, Hkv, D), torch.bfloat16, self.device)
            self.in_rows = (torch.arange(nl, B, dtype=torch.int32) * 3).to(self.device)
        else:
            self.q, self.k, self.v = (ipc_import(desc[n], self.device) for n in ("q", "k", "v"))
            self.mapped += [self.q, self.k, self.v]
            self.in_rows = torch.arange(nl, B, dtype=torch.int32, device=self.device)
        self.attn = ipc_import(desc["attn"], self.device)
        self.flags = ipc_import(desc["flags"], self.device)
        self.mapped += [self.attn, self.flags]
        self.L = desc["layers"]
        self.out_rows = torch.arange(nl, B, dtype=torch.int32, device=self.device)
        self.ws = [ops.DecodeWorkspace(max(1, self.no), Hq, Hkv, D, self.device) for _ in range(2)]
        self.scale = 1.0 / math.sqrt(D)

    def _flag(self, which: int, l: int) -> int:
        return self.flags.ptr + (which * self.L + l) * 4

    def step(self, step_id: int, block_table, seq_lens) -> None:
        """Enqueue step ``step_id``'s offloaded attention (all layers) on the stream."""
        from . import _ffi
        xs = self.stream
        if self.no == 0:
            return
        for l in range(self.L):
            _ffi.call("adr_wait", self._flag(0, l), step_id, xs.cuda_stream)
            kc, vc = self.kv[l]
            ops.paged_decode_attn(self.q, kc, vc, block_table, seq_lens, out=self.attn,
                                  scale=self.scale, workspace=self.ws[l % 2], stream=xs,
                                  num_sms=self.num_sms, k_new=self.k, v_new=self.v,
                                  in_rows=self.in_rows, out_rows=self.out_rows)
            _ffi.call("adr_signal", self._flag(1, l), step_id, xs.cuda_stream)

    def link_bytes_per_step(self) -> int:
        """q/k/v rows read and attention rows written over the link per step."""
        Hq, Hkv, D = self.q.shape[1], self.k.shape[1], self.q.shape[2]
        return self.no * self.L * ((Hq + 2 * Hkv) * D * 2 + Hq * D * 2)

    def close(self) -> None:
        for p in self.mapped:
            p.close()
        self.mapped = []
