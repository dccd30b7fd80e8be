"""Hardware and model descriptions (API of adrenaline_sim.specs, specs.py:1-85).

Units are SI throughout: bytes, bytes/s, FLOP/s, seconds.

Differences from the reference, all additive:
  * ``ModelSpec`` takes optional ``num_q_heads`` / ``num_kv_heads`` /
    ``head_dim`` so grouped-query models size their KV correctly; left unset,
    ``kv_bytes_per_token`` is the reference's MHA formula
    ``2 * elem_bytes * hidden_size * num_layers`` (specs.py:54-57) bit for bit.
  * B200 and Llama-2-13B / Llama-3 presets next to the reference's A100 and
    Llama-2-7B ones.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

__all__ = [
    "GpuSpec", "ModelSpec", "A100_80G", "B200", "B200_NOMINAL", "LLAMA2_7B", "LLAMA2_13B",
    "LLAMA3_8B", "LLAMA3_70B", "GPU_PRESETS", "MODEL_PRESETS",
]


@dataclass(frozen=True)
class GpuSpec:
    """Per-GPU capability figures (peaks, not achieved rates)."""

    name: str
    flops_peak: float
    hbm_capacity_bytes: float
    hbm_bandwidth: float
    interconnect_bandwidth: float
    cpu_launch_per_layer: float

    def __post_init__(self) -> None:
        positive = ("flops_peak", "hbm_capacity_bytes", "hbm_bandwidth", "interconnect_bandwidth")
        for attr in positive:
            if getattr(self, attr) <= 0:
                raise ValueError(f"GpuSpec.{attr} must be positive")
        if self.cpu_launch_per_layer < 0:
            raise ValueError("GpuSpec.cpu_launch_per_layer must be >= 0")

    @property
    def machine_balance(self) -> float:
        """FLOP the GPU can issue per byte it can stream from HBM."""
        return self.flops_peak / self.hbm_bandwidth


@dataclass(frozen=True)
class ModelSpec:
    """Decoder shape and the per-token cost coefficients of the cost model."""

    name: str
    num_layers: int
    hidden_size: int
    elem_bytes: int
    weight_bytes: float
    flops_per_prompt_token: float
    flops_per_decode_token_nonattn: float
    bytes_per_decode_step_nonattn: float
    # grouped-query attention (None: multi-head with hidden_size = heads * head_dim)
    num_q_heads: Optional[int] = None
    num_kv_heads: Optional[int] = None
    head_dim: Optional[int] = None

    def __post_init__(self) -> None:
        if min(self.num_layers, self.hidden_size, self.elem_bytes) <= 0:
            raise ValueError("ModelSpec shape fields must be positive")
        if self.weight_bytes <= 0:
            raise ValueError("ModelSpec.weight_bytes must be positive")
        gqa = (self.num_q_heads, self.num_kv_heads, self.head_dim)
        if any(v is not None for v in gqa):
            if any(v is None or v <= 0 for v in gqa):
                raise ValueError("num_q_heads, num_kv_heads and head_dim go together and "
                                 "must be positive")
            if self.num_q_heads % self.num_kv_heads != 0:
                raise ValueError("num_q_heads must be a multiple of num_kv_heads")

    @property
    def kv_width(self) -> int:
        """Elements of one K (or V) vector per token per layer."""
        if self.num_kv_heads is None:
            return self.hidden_size
        return self.num_kv_heads * self.head_dim

    @property
    def kv_bytes_per_token(self) -> int:
        # one K and one V vector per layer
        return 2 * self.elem_bytes * self.kv_width * self.num_layers

    @property
    def q_heads(self) -> int:
        return self.num_q_heads if self.num_q_heads is not None else self.hidden_size // 128

    @property
    def kv_heads(self) -> int:
        return self.num_kv_heads if self.num_kv_heads is not None else self.q_heads

    @property
    def dim_per_head(self) -> int:
        return self.head_dim if self.head_dim is not None else self.hidden_size // self.q_heads


# Reference desk-scale pair (specs.py:64-82): one 80 GB A100 and Llama-2-7B in
# 16-bit weights; the shipped calibration curves are anchored to it.
A100_80G = GpuSpec(name="a100-80g", flops_peak=312e12, hbm_capacity_bytes=80e9,
                   hbm_bandwidth=2039e9, interconnect_bandwidth=600e9,
                   cpu_launch_per_layer=1.137e-3)

# B200 with the pool's measured roofline denominators (MEASURED_PEAKS.json:
# cuBLAS bf16 burst, STREAM copy) and NVLink 5 per direction. The per-layer
# CPU launch cost is inherited from the A100 figure until measured on-box.
B200 = GpuSpec(name="b200", flops_peak=1669.3e12, hbm_capacity_bytes=180e9,
               hbm_bandwidth=6550.7e9, interconnect_bandwidth=900e9,
               cpu_launch_per_layer=1.137e-3)
# Datasheet figures (dense bf16, HBM3e), for context.
B200_NOMINAL = GpuSpec(name="b200-nominal", flops_peak=2250e12, hbm_capacity_bytes=180e9,
                       hbm_bandwidth=8000e9, interconnect_bandwidth=900e9,
                       cpu_launch_per_layer=1.137e-3)

LLAMA2_7B = ModelSpec(name="llama2-7b", num_layers=32, hidden_size=4096, elem_bytes=2,
                      weight_bytes=13.476e9, flops_per_prompt_token=1.3476e10,
                      flops_per_decode_token_nonattn=1.3476e10,
                      bytes_per_decode_step_nonattn=13.476e9)
LLAMA2_13B = ModelSpec(name="llama2-13b", num_layers=40, hidden_size=5120, elem_bytes=2,
                       weight_bytes=26.032e9, flops_per_prompt_token=2.6032e10,
                       flops_per_decode_token_nonattn=2.6032e10,
                       bytes_per_decode_step_nonattn=26.032e9)
LLAMA3_8B = ModelSpec(name="llama3-8b", num_layers=32, hidden_size=4096, elem_bytes=2,
                      weight_bytes=16.06e9, flops_per_prompt_token=1.606e10,
                      flops_per_decode_token_nonattn=1.606e10,
                      bytes_per_decode_step_nonattn=16.06e9,
                      num_q_heads=32, num_kv_heads=8, head_dim=128)
LLAMA3_70B = ModelSpec(name="llama3-70b", num_layers=80, hidden_size=8192, elem_bytes=2,
                       weight_bytes=141.1e9, flops_per_prompt_token=1.411e11,
                       flops_per_decode_token_nonattn=1.411e11,
                       bytes_per_decode_step_nonattn=141.1e9,
                       num_q_heads=64, num_kv_heads=8, head_dim=128)

GPU_PRESETS = {g.name: g for g in (A100_80G, B200, B200_NOMINAL)}
MODEL_PRESETS = {m.name: m for m in (LLAMA2_7B, LLAMA2_13B, LLAMA3_8B, LLAMA3_70B)}
