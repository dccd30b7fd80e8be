"""Shapes of the synthetic full decode layers (decoder.py) on CPU."""
from paper_2503_20552_b200.decoder import MODEL_DIMS


def test_model_dims_match_decode_shapes():
    from paper_2503_20552_b200.synthetic import CONFIGS
    for cfg, model in (("C2", "llama2-7b"), ("C3", "llama3-8b"), ("C5", "llama3-70b")):
        d, s = MODEL_DIMS[model], CONFIGS[cfg]
        assert (d.num_q_heads, d.num_kv_heads, d.head_dim) == (s.num_q_heads, s.num_kv_heads,
                                                               s.head_dim)
    # 7B: 202M parameters per layer -> 0.40 GB bf16 (32 layers: 12.9 GB of the 13.5 GB model)
    assert MODEL_DIMS["llama2-7b"].weight_bytes_per_layer() == 2 * (
        3 * 4096 * 4096 + 4096 * 4096 + 3 * 4096 * 11008 + 2 * 4096)
