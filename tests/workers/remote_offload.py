"""Worker of tests/test_gpu_ipc.py: full decode layers with the offloaded rows'
attention in ANOTHER process (decoder.RemoteOffloadedDecoder + OffloadServer) —
rank 0 decoder, rank 1 executor, sharing one GPU (CUDA IPC works within a
device). The decoder checks that two steps of the two-process split give the
same bits as the one-process loopback (decoder.OffloadedDecoder) on identical
weights, caches and tables.

    python tests/workers/remote_offload.py RANK PORT DEVICE MHA
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import torch
import torch.distributed as dist

from paper_2503_20552_b200.decoder import (LayerDims, OffloadedDecoder, OffloadServer,
                                           RemoteOffloadedDecoder)
from paper_2503_20552_b200.synthetic import DecodeShape, make_block_table, make_layer

L = 2
CTX_LOCAL = (300, 17, 1024, 1, 64)
CTX_OFF = (900, 33, 2000)


def caches(shape, dev, base_seed):
    bt = make_block_table(shape)
    layers = [make_layer(shape, dev, seed=base_seed + l, block_table=bt) for l in range(L)]
    return [(x["k_cache"], x["v_cache"]) for x in layers], layers[0]["block_table"], layers[0]["seq_lens"]


def main() -> None:
    rank, port, device, mha = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1"
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    dims = LayerDims(256, 512, 8, 8 if mha else 2, 64)
    Hq, Hkv, D = dims.num_q_heads, dims.num_kv_heads, dims.head_dim
    sh_l = DecodeShape("loc", len(CTX_LOCAL), Hq, Hkv, D, L, CTX_LOCAL, spare_pages=3)
    sh_x = DecodeShape("off", len(CTX_OFF), Hq, Hkv, D, L, CTX_OFF, spare_pages=5)
    nl, B = len(CTX_LOCAL), len(CTX_LOCAL) + len(CTX_OFF)
    if rank == 1:
        box = [None]
        dist.recv_object_list(box, src=0)
        exec_kv, xbt, xseq = caches(sh_x, dev, 100)
        srv = OffloadServer(box[0], exec_kv, dev)
        for s in (1, 2):
            srv.step(s, xbt, xseq)
        torch.cuda.synchronize(dev)
        dist.barrier()
        srv.close()
        dist.destroy_process_group()
        print("executor ok")
        return
    kv, bt, seq = caches(sh_l, dev, 0)
    kv_ref = [(k.clone(), v.clone()) for k, v in kv]
    dec = RemoteOffloadedDecoder(dims, kv, B, nl, dev, seed=5)
    dist.send_object_list([dec.export()], dst=1)
    g = torch.Generator(device=dev).manual_seed(9)
    x0 = torch.randn(B, dims.hidden, generator=g, device=dev).to(torch.bfloat16)
    x = x0.clone()
    for _ in range(2):
        dec.step(x, bt, seq)
    torch.cuda.synchronize(dev)
    # one-process loopback reference: same weights (seed), caches (seeds), tables
    exec_kv, xbt, xseq = caches(sh_x, dev, 100)
    ref = OffloadedDecoder(dims, kv_ref, exec_kv, B, nl, dev, seed=5)
    y = x0.clone()
    for _ in range(2):
        ref.step(y, bt, seq, xbt, xseq)
    torch.cuda.synchronize(dev)
    assert bool(torch.isfinite(x).all()), "non-finite activations"
    assert torch.equal(x, y), f"two-process step differs from loopback: {(x.float() - y.float()).abs().max()}"
    for (k, v), (kr, vr) in zip(kv, kv_ref):
        assert torch.equal(k, kr) and torch.equal(v, vr), "local caches differ"
    dist.barrier()
    dist.destroy_process_group()
    print("decoder ok")


if __name__ == "__main__":
    main()
