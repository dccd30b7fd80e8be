"""Zero-copy decode/executor role split across two processes (CUDA IPC +
stream-ordered flags + adr_paged_decode_attn_rows), run as two ranks on one
GPU: the executor process's kernel reads the decoder process's q/k/v rows and
writes the decoder's output rows; the decoder checks its outputs (local and
offloaded rows) against the oracle."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

WORKER = Path(__file__).resolve().parent / "workers" / "ipc_roles.py"


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_zero_copy_roles_two_processes_one_gpu(cuda):
    port = free_port()
    env = dict(os.environ)
    procs = [subprocess.Popen([sys.executable, str(WORKER), str(r), str(port), "0"],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env)
             for r in (0, 1)]
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=240)
            outs.append(out)
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{out[-3000:]}"
    assert "decoder ok" in outs[0] and "executor ok" in outs[1]


@pytest.mark.parametrize("mha", [True, False])
def test_remote_offloaded_decoder_two_processes_one_gpu(cuda, mha):
    """Full decode layers, offloaded rows attended in another process
    (RemoteOffloadedDecoder + OffloadServer over CUDA IPC and stream flags):
    bit-identical to the one-process loopback OffloadedDecoder."""
    worker = Path(__file__).resolve().parent / "workers" / "remote_offload.py"
    port = free_port()
    procs = [subprocess.Popen([sys.executable, str(worker), str(r), str(port), "0", "1" if mha else "0"],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                              env=dict(os.environ))
             for r in (0, 1)]
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=240)
            outs.append(out)
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{out[-3000:]}"
    assert "decoder ok" in outs[0] and "executor ok" in outs[1]
