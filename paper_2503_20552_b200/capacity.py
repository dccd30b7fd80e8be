"""Capacity-bound decode batches with and without attention offloading.

The paper's headline (BASELINE.json target "offloaded decoding
raising decode batch size and tokens/s by at least 1.5x over the no-offload
configuration") is a CAPACITY claim: a decode GPU's batch is bounded by its KV
pool (config.py:93-106 ``pool_bytes``), and offloading part of the attention
to the idle HBM of prefill GPUs lets the batch grow. ``plan_capacity`` builds
the steady-state batch of one decoder both ways, with the reference's own
admission rules (engine.py:326-355 ``_admit``; Algorithm 1, scheduling.py:
176-221, through the O(1) ``OffloadLedger``):

  * requests are drawn from a workload preset (workload.synth_requests), each
    caught at a seeded point of its decode (resident KV = prompt + generated
    tokens + the reserved next one);
  * no offload: requests join the decoder's pool while their KV fits;
  * offload: Algorithm 1 at the planner bound places each request locally or on
    the decoder's executor; a request whose chosen home is full blocks the
    queue (never falls back: engine.py:332-335).

``bench.py --capacity`` runs both batches for real (full decode layers on the
decode GPU, offloaded attention on the executor GPU's SM partition beside a
prefill GEMM load) and reports batch, tokens/s and NVLink traffic.
"""
from __future__ import annotations

import dataclasses
import random
from dataclasses import dataclass, field

from . import specs, workload
from .config import SimConfig
from .scheduling import OffloadLedger, Request

__all__ = ["CapacityPlan", "CapacityCase", "CAPACITY_CASES", "LLAMA3_70B_TP8W", "LONGCTX",
           "plan_capacity", "snapshot_requests", "case_requests"]

# C5 (BASELINE.json configs[4]): Llama-3-70B attention shapes (64q/8kv x 128,
# 80 layers) with the weights sharded 8 ways (17.6 GB per GPU): whole 70B
# weights leave no KV room on one 180 GB GPU under the reference memory policy
# (config.py:80-86 raises), and the non-attention work is outside the offload
# path anyway.
LLAMA3_70B_TP8W = dataclasses.replace(specs.LLAMA3_70B, name="llama3-70b-tp8-weights",
                                      weight_bytes=141.1e9 / 8,
                                      flops_per_prompt_token=1.411e11 / 8,
                                      flops_per_decode_token_nonattn=1.411e11 / 8,
                                      bytes_per_decode_step_nonattn=141.1e9 / 8)
# long-context mix for the C5 shape (prompts ~16k, up to 32k tokens)
LONGCTX = (workload.LogNormal(16000.0, 0.5, 1024, 32768), workload.LogNormal(800.0, 0.6, 16, 4096))


@dataclass(frozen=True)
class CapacityCase:
    """One capacity-bound decode comparison (bench.py --capacity --capacity-config)."""

    name: str
    model: specs.ModelSpec    # memory policy / Algorithm 1 model
    dims: str                 # decoder.MODEL_DIMS key (attention and layer shapes)
    preset: str               # workload preset, or "longctx"
    nonattn: bool             # run the non-attention GEMMs (else attention-only layers)
    offload_ratio: float | None  # SimConfig.offload_ratio (None: the planner's Eq. 1-3 bound)
    note: str


CAPACITY_CASES = {
    "C4": CapacityCase("C4", specs.LLAMA2_13B, "llama2-13b", "sharegpt_like", True, None,
                       "Llama-2-13B, ShareGPT-like lengths, 40 full layers (cuBLAS GEMMs with "
                       "synthetic weights around our attention)"),
    "C5": CapacityCase("C5", LLAMA3_70B_TP8W, "llama3-70b", "longctx", False, 0.7,
                       "Llama-3-70B attention shapes (64q/8kv, 80 layers), long-context mix "
                       "(prompts ~16k, <= 32k), memory policy with 8-way sharded weights, "
                       "offload bound 0.7 (the planner's Eq. 1-3 bound is 0 here); "
                       "attention-only layers (the 70B GEMMs are not on the offload path)"),
}


def case_requests(case: CapacityCase, seed: int, n: int = 4000) -> list[Request]:
    """Mid-decode snapshots of ``n`` requests of the case's length mix."""
    if case.preset == "longctx":
        spec = workload.WorkloadSpec(rate=10.0, num_requests=n, prompt_dist=LONGCTX[0],
                                     output_dist=LONGCTX[1], name="longctx")
    else:
        spec = workload.preset(case.preset, 10.0, n)
    return snapshot_requests(workload.synth_requests(spec, 17 + seed), seed)


@dataclass
class CapacityPlan:
    """Steady-state batch of ONE decoder (and the executor it offloads to)."""

    bound: float                      # Algorithm 1 offload bound used
    pool_bytes: float                 # decoder KV pool (config.py pool_bytes)
    exec_budget_bytes: float          # executor KV budget available to this decoder
    kv_bytes_per_token: int
    no_offload: list[int] = field(default_factory=list)   # resident tokens per request
    local: list[int] = field(default_factory=list)
    offloaded: list[int] = field(default_factory=list)
    rules: dict = field(default_factory=dict)              # Algorithm 1 rule counts
    blocked_by: str = ""                                   # what stopped the offload fill

    @property
    def batch_no_offload(self) -> int:
        return len(self.no_offload)

    @property
    def batch_offload(self) -> int:
        return len(self.local) + len(self.offloaded)

    @property
    def batch_gain(self) -> float:
        return self.batch_offload / max(1, self.batch_no_offload)

    def bytes(self, which: str) -> int:
        return sum(getattr(self, which)) * self.kv_bytes_per_token

    def summary(self) -> dict:
        return {"bound": self.bound, "pool_GB": self.pool_bytes / 1e9,
                "exec_budget_GB": self.exec_budget_bytes / 1e9,
                "batch_no_offload": self.batch_no_offload,
                "batch_offload": self.batch_offload, "n_local": len(self.local),
                "n_offloaded": len(self.offloaded), "batch_gain": self.batch_gain,
                "kv_GB_no_offload": self.bytes("no_offload") / 1e9,
                "kv_GB_local": self.bytes("local") / 1e9,
                "kv_GB_offloaded": self.bytes("offloaded") / 1e9,
                "rules": dict(self.rules), "offload_fill_stopped_by": self.blocked_by}


def snapshot_requests(requests, seed: int = 0) -> list[Request]:
    """Each request caught mid-decode: used_token = prompt + U{0..output-1}
    generated tokens (the engine's used_token after that many steps)."""
    rng = random.Random(seed)
    out = []
    for r in requests:
        q = Request(r.req_id, r.arrival_time, r.prompt_tokens, r.output_tokens)
        q.used_token = r.prompt_tokens + rng.randrange(r.output_tokens)
        out.append(q)
    return out


def plan_capacity(cfg: SimConfig, requests, exec_budget_bytes: float | None = None,
                  bound: float | None = None, scale: float = 1.0) -> CapacityPlan:
    """Fill one decoder's pool from ``requests`` (mid-decode snapshots, in
    order) without and with offloading. ``exec_budget_bytes`` defaults to one
    prefill GPU's executor budget shared by the decoders that map to it
    (``num_prefill / num_decode`` of it per decoder, as the engine's
    least-loaded executor choice balances it). ``scale`` shrinks both budgets
    (the 1-GPU degenerate run, where decoder and executor share one GPU)."""
    kv_tok = cfg.model.kv_bytes_per_token
    pool = cfg.pool_bytes * scale
    if exec_budget_bytes is None:
        exec_budget_bytes = cfg.executor_budget_bytes * cfg.num_prefill / max(1, cfg.num_decode)
    exec_budget = exec_budget_bytes * scale
    b = cfg.effective_bound() if bound is None else bound
    plan = CapacityPlan(b, pool, exec_budget, kv_tok)
    # no offload: the pool alone (engine.py:341-344; need = resident + the next token)
    used = 0
    for r in requests:
        need = (r.used_token + 1) * kv_tok
        if used + need > pool:
            break
        used += need
        plan.no_offload.append(r.used_token + 1)
    # offload: Algorithm 1 against this decoder's sets, budgets on both homes
    led = OffloadLedger()
    used_l = used_x = 0
    for r in requests:
        dec = led.decide(r, b, c1_uses_max_tokens=cfg.c1_uses_max_tokens)
        need = (r.used_token + 1) * kv_tok
        plan.rules[dec.rule] = plan.rules.get(dec.rule, 0) + 1
        if dec.offload:
            if used_x + need > exec_budget:
                plan.blocked_by = "executor budget"
                break
            used_x += need
            led.add(r, offloaded=True)
            plan.offloaded.append(r.used_token + 1)
        else:
            if used_l + need > pool:
                plan.blocked_by = "decoder pool"
                break
            used_l += need
            led.add(r, offloaded=False)
            plan.local.append(r.used_token + 1)
    return plan
