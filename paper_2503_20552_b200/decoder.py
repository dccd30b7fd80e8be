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

__all__ = ["LayerDims", "MODEL_DIMS", "SyntheticDecoder"]


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
                 seed: int = 0, eps: float = 1e-5) -> None:
        self.dims, self.kv, self.B, self.device, self.eps = dims, kv, batch, device, eps
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

        self.layers = []
        for _ in range(L):
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
        self.attn = torch.empty(B, Hq, D, **bf)
        self.o = torch.empty(B, h, **bf)
        self.gate_up = torch.empty(B, 2 * I, **bf)
        self.ws = [ops.DecodeWorkspace(B, Hq, Hkv, D, device) for _ in range(2)]
        self.scale = 1.0 / math.sqrt(D)

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    def weight_bytes(self) -> int:
        return self.dims.weight_bytes_per_layer() * self.num_layers

    def layer(self, l: int, x: torch.Tensor, block_table, seq_lens, pdl: bool = False) -> None:
        W = self.layers[l]
        B, hdim = x.shape
        h = F.rms_norm(x, (hdim,), W["n1"], self.eps)
        if self.mha:
            torch.matmul(h, W["wqkv"].t(), out=self.qkv[:3 * B].view(B, -1))
        else:
            torch.matmul(h, W["wq"].t(), out=self.q.view(B, -1))
            torch.matmul(h, W["wk"].t(), out=self.k.view(B, -1))
            torch.matmul(h, W["wv"].t(), out=self.v.view(B, -1))
        kc, vc = self.kv[l]
        ops.paged_decode_attn(self.q, kc, vc, block_table, seq_lens, out=self.attn,
                              scale=self.scale, workspace=self.ws[l % 2],
                              k_new=self.k, v_new=self.v, pdl=pdl, in_rows=self.rows)
        torch.matmul(self.attn.view(B, -1), W["wo"].t(), out=self.o)
        x.add_(self.o)
        h = F.rms_norm(x, (hdim,), W["n2"], self.eps)
        torch.matmul(h, W["wgu"].t(), out=self.gate_up)
        I = self.dims.intermediate
        act = F.silu(self.gate_up[:, :I]).mul_(self.gate_up[:, I:])
        torch.matmul(act, W["wd"].t(), out=self.o)
        x.add_(self.o)

    def step(self, x: torch.Tensor, block_table, seq_lens, pdl: bool = False) -> torch.Tensor:
        if x.shape != (self.B, self.dims.hidden) or x.dtype != torch.bfloat16:
            raise ValueError(f"x must be [{self.B}, {self.dims.hidden}] bf16")
        for l in range(self.num_layers):
            self.layer(l, x, block_table, seq_lens, pdl=pdl)
        return x
