import math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
import numpy as np, torch
import oracle as orc
from paper_2503_20552_b200 import ops
from paper_2503_20552_b200.synthetic import DecodeShape, make_layer
dev = torch.device("cuda:0")
def run(shape, lse_on, workers=0, dtype=torch.float32, ws=None):
    x = make_layer(shape, dev)
    sc = 1 / math.sqrt(shape.head_dim)
    ws = ws or ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, dev, num_workers=workers)
    lse = torch.empty(shape.batch, shape.num_q_heads, device=dev) if lse_on else None
    out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"], lse=lse, scale=sc, out_dtype=dtype, workspace=ws)
    torch.cuda.synchronize()
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"], sc)
    err = np.abs(out.float().cpu().numpy() - ref).max(axis=2)
    bad = np.argwhere(err > 2e-2)
    print(shape.name, "lse" if lse_on else "nolse", workers, dtype, "maxerr", err.max(), "bad rows", len(bad), bad[:10].tolist(), flush=True)
s = DecodeShape("C3-b8", 8, 32, 8, 128, 1, 4096)
run(s, True); run(s, False); run(s, True, dtype=torch.bfloat16); run(s, False, dtype=torch.bfloat16)
run(s, False, workers=37); run(s, True, workers=37)
a = DecodeShape("a", 3, 32, 8, 128, 1, (900, 33, 2000))
run(a, True, workers=37); run(a, False, workers=37); run(a, False)
