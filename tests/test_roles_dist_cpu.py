"""World-size-2 gloo run of runtime.RoleSplitStep: rank 0 is the decoder, rank 1
the executor of a prefill-role GPU. The attention callable is a float64 CPU
stand-in (test-only) so the message protocol, row packing and output
placement are checked end to end: every output row must be the attention of
its own request over the right rank's cache."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_2503_20552_b200.exchange import DistTransport
from paper_2503_20552_b200.runtime import RoleSplitStep

L, B, N_LOCAL, HQ, HKV, D, T = 3, 6, 4, 4, 2, 16, 9


def _cache(seed, rows):
    g = torch.Generator().manual_seed(seed)
    return [(torch.randn(rows, T, HKV, D, generator=g), torch.randn(rows, T, HKV, D, generator=g))
            for _ in range(L)]


def _attend_factory(cache):
    def attend(l, q, k_new, v_new, out):
        kc, vc = cache[l]
        for i in range(q.shape[0]):
            kk = torch.cat([kc[i, :-1], k_new[i:i + 1]]).double()   # token T-1 is the appended one
            vv = torch.cat([vc[i, :-1], v_new[i:i + 1]]).double()
            out[i] = torch.from_numpy(orc.dense_attention_fp64(q[i].double().numpy(), kk.numpy(),
                                                               vv.numpy(), D ** -0.5)).to(out.dtype)
    return attend


def _pack(q, k, v, rows):
    r = rows.long()
    return torch.cat([q[r].reshape(len(r), -1), k[r].reshape(len(r), -1), v[r].reshape(len(r), -1)], 1)


def _unpack(msg, n):
    q = msg[:, :HQ * D].reshape(n, HQ, D)
    k = msg[:, HQ * D:(HQ + HKV) * D].reshape(n, HKV, D)
    v = msg[:, (HQ + HKV) * D:].reshape(n, HKV, D)
    return q.contiguous(), k.contiguous(), v.contiguous()


def _scatter(src, rows, out):
    out[rows.long()] = src


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        t = DistTransport(peer_rank=1 - rank)
        if rank == 0:
            cache = _cache(1, N_LOCAL)
            step = RoleSplitStep("decoder", HQ, HKV, D, t, attend=_attend_factory(cache),
                                 pack=_pack, unpack=_unpack, scatter=_scatter)
            g = torch.Generator().manual_seed(7)
            qs = [torch.randn(B, HQ, D, generator=g) for _ in range(L)]
            ks = [torch.randn(B, HKV, D, generator=g) for _ in range(L)]
            vs = [torch.randn(B, HKV, D, generator=g) for _ in range(L)]
            outs = [torch.zeros(B, HQ, D) for _ in range(L)]
            link = step.run_decoder(qs, ks, vs, N_LOCAL, outs)
            # expected: local rows over the decoder cache, offloaded rows over the executor cache
            exec_cache = _cache(2, B - N_LOCAL)
            ok = True
            for l in range(L):
                exp = torch.zeros(B, HQ, D)
                _attend_factory(cache)(l, qs[l][:N_LOCAL], ks[l][:N_LOCAL], vs[l][:N_LOCAL], exp[:N_LOCAL])
                _attend_factory(exec_cache)(l, qs[l][N_LOCAL:], ks[l][N_LOCAL:], vs[l][N_LOCAL:], exp[N_LOCAL:])
                ok &= bool(torch.allclose(outs[l], exp, atol=1e-6))
            q.put(("decoder", ok, link))
        else:
            cache = _cache(2, B - N_LOCAL)
            step = RoleSplitStep("executor", HQ, HKV, D, t, attend=_attend_factory(cache),
                                 pack=_pack, unpack=_unpack, scatter=_scatter)
            step.run_executor(L, B - N_LOCAL, torch.float32, torch.device("cpu"))
            q.put(("executor", True, 0))
    finally:
        dist.destroy_process_group()


def test_role_split_step_two_ranks_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((role, (ok, link)) for role, ok, link in (q.get(timeout=180) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["decoder"][0] and res["executor"][0]
    n_off = B - N_LOCAL
    assert res["decoder"][1] == L * (n_off * (HQ + 2 * HKV) * D + n_off * HQ * D) * 4
