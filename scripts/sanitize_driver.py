"""Small decode-attention workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every code path of decode_attn_kernel at sizes the
sanitizers finish in minutes, each result checked against the oracle.

  dynamic grid (split pairs + merge phase), static grid (last-arriver merge),
  split-pair CTA kernel (shared-memory combine, last-arriving CTA merges),
  fused append, PDL chain of layers, two concurrent persistent grids on two
  streams, row maps (zero-copy offload), the standalone byte kernels, and a
  call on bad tables (the kernel must stay inside the cache).

Usage: compute-sanitizer --tool memcheck python scripts/sanitize_driver.py
"""
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as orc  # noqa: E402
from paper_2503_20552_b200 import ops  # noqa: E402
from paper_2503_20552_b200.synthetic import DecodeShape, make_layer  # noqa: E402

dev = torch.device("cuda:0")


def check(out, x, scale, kc=None, vc=None):
    ref, _ = orc.paged_decode_attn(x["q"], x["k_cache"] if kc is None else kc,
                                   x["v_cache"] if vc is None else vc, x["block_table"],
                                   x["seq_lens"], scale)
    g = out.float().cpu().numpy()
    err = float(np.abs(g - ref).max())
    assert err <= 2e-2, err
    return err


def main():
    scale = 1.0 / math.sqrt(128)
    cases = [DecodeShape("mha", 3, 8, 8, 128, 1, (700, 64, 1500)),
             DecodeShape("gqa4", 5, 16, 4, 128, 1, (33, 1, 0, 900, 257)),
             DecodeShape("gqa8-d64", 2, 16, 2, 64, 1, (2049, 16)),
             DecodeShape("gqa8", 2, 64, 8, 128, 1, (3000, 65))]  # split kernel's 4x2 variant
    n = 0
    for shape in cases:
        x = make_layer(shape, dev)
        s = 1.0 / math.sqrt(shape.head_dim)
        for grid in ("dynamic", "static", "split"):
            for workers in ((0, 96) if grid != "split" else (0,)):
                ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads,
                                         shape.head_dim, dev, num_workers=workers)
                lse = torch.empty(shape.batch, shape.num_q_heads, dtype=torch.float32, device=dev)
                out = ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                            x["seq_lens"], lse=lse, scale=s,
                                            out_dtype=torch.float32, workspace=ws, grid=grid)
                torch.cuda.synchronize()
                check(out, x, s)
                n += 1
        # fused append + PDL chain of 3 layers (bf16 out)
        ws = ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads,
                                 shape.head_dim, dev, max_blocks_per_seq=shape.max_pages)
        kc, vc = x["k_cache"].clone(), x["v_cache"].clone()
        for grid in ("auto", "auto", "split", "split", "auto"):
            ops.paged_decode_attn(x["q"], kc, vc, x["block_table"], x["seq_lens"], scale=s,
                                  workspace=ws, k_new=x["k_new"], v_new=x["v_new"], pdl=True,
                                  grid=grid)
            n += 1
        torch.cuda.synchronize()
    # two concurrent persistent grids
    shapes = [DecodeShape("c0", 4, 32, 8, 128, 1, 2048), DecodeShape("c1", 2, 32, 32, 128, 1, 1024)]
    xs = [make_layer(sh, dev, seed=i) for i, sh in enumerate(shapes)]
    wss = [ops.DecodeWorkspace(sh.batch, sh.num_q_heads, sh.num_kv_heads, 128, dev) for sh in shapes]
    sts = [torch.cuda.Stream(dev) for _ in shapes]
    torch.cuda.synchronize()
    outs = []
    for x, w, st, grid in zip(xs, wss, sts, ("auto", "split")):
        outs.append(ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"],
                                          x["seq_lens"], scale=scale, out_dtype=torch.float32,
                                          workspace=w, stream=st, grid=grid))
        n += 1
    torch.cuda.synchronize()
    for o, x in zip(outs, xs):
        check(o, x, scale)
    # row maps (zero-copy offload on one device)
    sh = DecodeShape("rows", 3, 32, 8, 128, 1, (300, 16, 1000))
    x = make_layer(sh, dev)
    ws = ops.DecodeWorkspace(3, 32, 8, 128, dev)
    q_src = torch.randn(6, 32, 128, device=dev).to(torch.bfloat16)
    rows = torch.tensor([5, 0, 3], dtype=torch.int32, device=dev)
    out = torch.zeros(6, 32, 128, dtype=torch.float32, device=dev)
    ops.paged_decode_attn(q_src, x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"],
                          out=out, scale=scale, out_dtype=torch.float32, workspace=ws,
                          in_rows=rows, out_rows=rows)
    torch.cuda.synchronize()
    n += 1
    # byte kernels
    slots = ops.slot_mapping(x["block_table"], x["seq_lens"].long() - 1)
    ops.kv_append(x["k_new"], x["v_new"], x["k_cache"], x["v_cache"], slots)
    msg = ops.pack_qkv(x["q"], x["k_new"], x["v_new"], rows.clamp(max=2))
    q2, k2, v2 = ops.unpack_qkv(msg, 3, 32, 8, 128)
    o2 = torch.zeros(3, 32, 128, dtype=torch.bfloat16, device=dev)
    ops.scatter_out(q2, torch.tensor([2, 0, 1], dtype=torch.int32, device=dev), o2)
    pages = torch.tensor([0, 1], dtype=torch.int32, device=dev)
    ops.kv_transfer(x["k_cache"], x["v_cache"], pages, x["k_cache"], x["v_cache"], pages + 2)
    torch.cuda.synchronize()
    # bad tables: page out of range and seq_len past the row — no OOB access
    sh = DecodeShape("bad", 4, 8, 2, 128, 1, (40, 100, 16, 70))
    x = make_layer(sh, dev)
    ws = ops.DecodeWorkspace(4, 8, 2, 128, dev)
    bt = x["block_table"].clone()
    bt[1, 6] = x["k_cache"].shape[0] + 1000
    sl = x["seq_lens"].clone()
    sl[3] = bt.shape[1] * 16 + 5
    for grid in ("auto", "split"):
        ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], bt, sl, workspace=ws,
                              k_new=x["k_new"], v_new=x["v_new"], grid=grid)
        assert ops.decode_status(ws) == 3
        n += 1
    print(f"sanitize_driver: {n} decode calls checked")


if __name__ == "__main__":
    main()
