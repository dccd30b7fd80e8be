"""The closed loop's measured step prices (runtime.MeasuredPricer): every
StepRecord (engine.py:40-64) is filled from the CUDA-event timings of a real
offloaded decode step, with the executor on a green-context partition beside a
running prefill GEMM load."""
import math

import pytest
import torch

from paper_2503_20552_b200 import coloc, config, engine, specs, workload
from paper_2503_20552_b200.kvcache import PagedKVMirror
from paper_2503_20552_b200.runtime import MeasuredPricer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("zero_copy", [True, False])
def test_measured_pricer_records_are_the_event_timings(cuda, zero_copy):
    cfg = config.SimConfig(gpu=specs.B200, model=specs.LLAMA3_8B, num_prefill=1, num_decode=1,
                           offload_ratio=0.5, avg_context_tokens=4096)
    mirror = PagedKVMirror.for_config(cfg, slack_pages=256, keep_log=False)
    chain = 2
    pricer = MeasuredPricer(cfg, mirror, chain=chain, zero_copy=zero_copy, keep_records=1 << 20)
    reqs = workload.synth_requests(workload.preset("sharegpt_like", 12.0, 24), 0)
    res = engine.simulate(cfg, reqs, pricer=pricer, observer=mirror)
    assert all(math.isfinite(r.finish_time) for r in res.requests)
    assert len(pricer.records) == len(res.steps)
    m = cfg.model
    L = m.num_layers
    per_row = (m.q_heads + 2 * m.kv_heads) * m.dim_per_head * 2 + m.q_heads * m.dim_per_head * 2
    k = L / chain
    offloaded = 0
    for rec, runs in pricer.records:
        mean_local = sum(t.local_attn for t in runs) / len(runs)
        assert rec.local_attn == pytest.approx(mean_local * k, rel=1e-12)
        assert rec.stall == pytest.approx(max(t.stall for t in runs) * k, rel=1e-12)
        assert rec.stall >= 0.0
        assert rec.link_bytes == pytest.approx(per_row * rec.batch_offload * L, rel=1e-12)
        if rec.batch_local:
            assert rec.local_attn > 0
        assert set(rec.exec_attn) == set(rec.exec_kv_bytes)
        for e, v in rec.exec_attn.items():
            assert v > 0
        assert rec.duration == pytest.approx(rec.launch + rec.nonattn + rec.local_attn + rec.stall,
                                             rel=1e-9)
        offloaded += rec.batch_offload
    assert offloaded > 0  # Algorithm 1 offloaded some requests and they were priced by running them
    if pricer.prefill is not None:
        assert pricer.uncovered_steps == 0  # every offloaded step ran beside a busy prefill partition


@pytest.mark.skipif(not coloc.green_contexts_supported(), reason="no green contexts")
def test_executor_attention_under_concurrent_prefill_matches_oracle(cuda):
    """Executor attention on a 64-SM green context while prefill GEMMs keep the
    other partition busy through the whole attention window: outputs match the
    oracle and are bit-identical call to call."""
    import numpy as np
    import oracle as orc
    from paper_2503_20552_b200 import ops
    from paper_2503_20552_b200.synthetic import DecodeShape, make_layer
    part = coloc.SmPartition(0, 64)
    pre = coloc.PrefillLoad(2048, 4096, 11008, cuda)
    shape = DecodeShape("co", 16, 32, 8, 128, 1, (4096, 17, 2000, 3000, 1, 999, 4096, 64,
                                                 2500, 3333, 16, 1024, 4000, 700, 128, 2049))
    x = make_layer(shape, cuda)
    ws = ops.DecodeWorkspace(16, 32, 8, 128, cuda, max_blocks_per_seq=shape.max_pages)
    outs = [torch.empty(16, 32, 128, dtype=torch.float32, device=cuda) for _ in range(6)]
    it = iter(outs)
    fa = lambda: ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                       x["seq_lens"], out=next(it), out_dtype=torch.float32,
                                       workspace=ws, stream=part.attn_stream,
                                       num_sms=part.attn_sms, pdl=True)
    ov = coloc.run_under_prefill(part.attn_stream, fa, 6, part.prefill_stream, pre, 16)
    assert ov.covered
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                   x["seq_lens"], 1.0 / math.sqrt(128))
    for o in outs:
        g = o.cpu().numpy()
        assert np.abs(g - ref).max() <= 2e-2
        assert np.abs(g - ref).sum() / np.abs(ref).sum() <= 1e-3
        assert torch.equal(o, outs[0])
