"""World-size-2 gloo run of the decode<->executor message exchange
(exchange.DistTransport): per layer the decoder ships one packed q/k/v message
and receives one output message; the executor side answers in layer order.
CPU tensors only — this covers the host-side protocol, framing and ordering that
the NCCL path uses on GPUs."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_20552_b200.exchange import DistTransport, TAG_OUT, TAG_QKV, out_message_bytes, qkv_message_bytes

L, N_OFF, HQ, HKV, D = 4, 5, 8, 2, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        t = DistTransport(peer_rank=1 - rank)
        width = (HQ + 2 * HKV) * D
        if rank == 0:  # decoder
            got = []
            for l in range(L):
                msg = torch.full((N_OFF, width), float(l), dtype=torch.bfloat16)
                msg[:, 0] = torch.arange(N_OFF, dtype=torch.bfloat16)
                t.send(TAG_QKV, l, msg)
                out = torch.empty((N_OFF, HQ, D), dtype=torch.bfloat16)
                t.recv(TAG_OUT, l, out)
                got.append(out)
            t.flush()
            ok = all(torch.equal(got[l][:, 0, 0], torch.arange(N_OFF, dtype=torch.bfloat16) + l)
                     and torch.all(got[l][:, 1:, :] == l) for l in range(L))
            q.put(("decoder", ok, t.bytes_moved))
        else:  # executor: "attention" = echo q rows shifted by the layer id
            for l in range(L):
                msg = torch.empty((N_OFF, width), dtype=torch.bfloat16)
                t.recv(TAG_QKV, l, msg)
                out = msg[:, : HQ * D].reshape(N_OFF, HQ, D).clone()
                out[:, 0, 0] += l
                t.send(TAG_OUT, l, out)
            t.flush()
            q.put(("executor", True, t.bytes_moved))
    finally:
        dist.destroy_process_group()


def test_dist_transport_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        role, ok, nbytes = q.get(timeout=120)
        res[role] = (ok, nbytes)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["decoder"][0] and res["executor"][0]
    assert res["decoder"][1] == L * qkv_message_bytes(N_OFF, HQ, HKV, D)
    assert res["executor"][1] == L * out_message_bytes(N_OFF, HQ, D)
