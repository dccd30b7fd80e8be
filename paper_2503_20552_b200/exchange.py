"""Decode <-> executor message transport for offloaded attention.

Per layer the decode GPU sends ONE message with the offloaded rows' q/k/v
(``adr_pack_qkv`` layout, PAPER.md:371 step 2) and receives ONE message with
their attention outputs (PAPER.md:371 step 3). The reference prices these as
``qkv = 1.5 * kv_tok * n / ic`` and ``recv = 0.5 * kv_tok * n / ic``
(engine.py:436-438); here they are real transfers:

  LoopbackTransport  executor on the same GPU (1-GPU testing / colocated
                     partition): device copy + CUDA events, stream-ordered
  PeerTransport      one process driving two GPUs: cudaMemcpyPeerAsync over
                     NVLink (adr_copy_peer) + cross-device events
  DistTransport      one process per GPU: torch.distributed isend/irecv
                     (NCCL over NVLink on GPUs; gloo on CPU for tests)

Every transport moves opaque byte tensors and is stream-ordered (no host
sync); message sizes are fixed per layer by the offloaded batch, so the same
calls are CUDA-graph capturable for the loopback / peer transports.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _ffi

__all__ = ["qkv_message_bytes", "out_message_bytes", "LoopbackTransport", "PeerTransport",
           "DistTransport", "TAG_QKV", "TAG_OUT", "DevicePtr", "ipc_export", "ipc_import"]

TAG_QKV = 1
TAG_OUT = 2


def qkv_message_bytes(n_rows: int, Hq: int, Hkv: int, D: int, elem: int = 2) -> int:
    """Bytes of one layer's q/k/v message for n offloaded rows."""
    return n_rows * (Hq + 2 * Hkv) * D * elem


def out_message_bytes(n_rows: int, Hq: int, D: int, elem: int = 2) -> int:
    return n_rows * Hq * D * elem


def _stream(s):
    return s if s is not None else torch.cuda.current_stream()


@dataclass
class _Mailbox:
    buf: torch.Tensor
    ready: torch.cuda.Event


class LoopbackTransport:
    """Both ends on one device. send() copies into the receiver's buffer on the
    sender's stream and records an event; recv() makes the receiver's stream
    wait for it. The copy is what an NVLink transfer would be on two GPUs."""

    def __init__(self, device: torch.device) -> None:
        self.device = device
        self.boxes: dict[tuple[int, int], _Mailbox] = {}
        self.bytes_moved = 0

    def _box(self, key, like: torch.Tensor) -> _Mailbox:
        box = self.boxes.get(key)
        if box is None or box.buf.numel() < like.numel():
            box = _Mailbox(torch.empty(like.numel(), dtype=like.dtype, device=self.device),
                           torch.cuda.Event())
            self.boxes[key] = box
        return box

    def send(self, tag: int, layer: int, msg: torch.Tensor, stream=None) -> None:
        s = _stream(stream)
        box = self._box((tag, layer), msg)
        with torch.cuda.stream(s):
            box.buf[:msg.numel()].copy_(msg.reshape(-1), non_blocking=True)
        box.ready.record(s)
        self.bytes_moved += msg.numel() * msg.element_size()

    def recv(self, tag: int, layer: int, out: torch.Tensor, stream=None) -> torch.Tensor:
        s = _stream(stream)
        box = self.boxes[(tag, layer)]
        s.wait_event(box.ready)
        with torch.cuda.stream(s):
            out.reshape(-1).copy_(box.buf[:out.numel()], non_blocking=True)
        return out


class PeerTransport(LoopbackTransport):
    """Sender and receiver on different GPUs of one process: the copy is
    cudaMemcpyPeerAsync (NVLink P2P when peer access is enabled)."""

    def __init__(self, src_device: torch.device, dst_device: torch.device) -> None:
        super().__init__(dst_device)
        self.src_device = src_device
        if src_device.index != dst_device.index:
            _ffi.call("adr_peer_open", src_device.index, dst_device.index)

    def send(self, tag: int, layer: int, msg: torch.Tensor, stream=None) -> None:
        s = _stream(stream)
        box = self._box((tag, layer), msg)
        nbytes = msg.numel() * msg.element_size()
        _ffi.call("adr_copy_peer", box.buf.data_ptr(), self.device.index, msg.data_ptr(),
                  msg.device.index, nbytes, s.cuda_stream)
        box.ready.record(s)
        self.bytes_moved += nbytes


class DistTransport:
    """One process per GPU: the peer is another rank of the default group.
    Uses torch.distributed isend/irecv (NCCL on GPUs, gloo on CPU tensors)."""

    def __init__(self, peer_rank: int, group=None) -> None:
        import torch.distributed as dist
        self.dist = dist
        self.peer = peer_rank
        self.group = group
        self.pending: list = []
        self.bytes_moved = 0

    def send(self, tag: int, layer: int, msg: torch.Tensor, stream=None) -> None:
        self.pending.append(self.dist.isend(msg.contiguous(), self.peer, group=self.group))
        self.bytes_moved += msg.numel() * msg.element_size()

    def recv(self, tag: int, layer: int, out: torch.Tensor, stream=None) -> torch.Tensor:
        work = self.dist.irecv(out, self.peer, group=self.group)
        work.wait()
        return out

    def flush(self) -> None:
        for w in self.pending:
            w.wait()
        self.pending.clear()


# ---- zero-copy offload across processes (CUDA IPC) ---------------------------

class DevicePtr:
    """A contiguous device array mapped from another process (or any raw device
    pointer): the attributes ``ops`` checks and passes to the C-ABI, nothing
    more. ``base`` is the mapped allocation (for adr_ipc_close)."""

    is_cuda = True

    def __init__(self, ptr: int, shape, dtype: torch.dtype, device: torch.device,
                 base: int | None = None) -> None:
        self.ptr, self.shape, self.dtype, self.device, self.base = ptr, torch.Size(shape), dtype, device, base

    def data_ptr(self) -> int:
        return self.ptr

    def dim(self) -> int:
        return len(self.shape)

    def is_contiguous(self) -> bool:
        return True

    def numel(self) -> int:
        return self.shape.numel()

    def element_size(self) -> int:
        return torch.empty((), dtype=self.dtype).element_size()

    def row(self, i: int) -> "DevicePtr":
        """Sub-array [i] along the first dimension."""
        stride = self.shape[1:].numel() * self.element_size()
        return DevicePtr(self.ptr + i * stride, self.shape[1:], self.dtype, self.device)

    def close(self) -> None:
        if self.base is not None:
            _ffi.call("adr_ipc_close", self.base)
            self.base = None


def ipc_export(t: torch.Tensor) -> dict:
    """Picklable description of a contiguous CUDA tensor for another process."""
    import ctypes
    if not (t.is_cuda and t.is_contiguous()):
        raise ValueError("ipc_export needs a contiguous CUDA tensor")
    h = (ctypes.c_uint8 * _ffi.ADR_IPC_HANDLE_BYTES)()
    off = ctypes.c_uint64()
    _ffi.call("adr_ipc_export", t.data_ptr(), ctypes.cast(h, ctypes.c_void_p), ctypes.byref(off))
    return {"handle": bytes(h), "offset": off.value, "shape": tuple(t.shape),
            "dtype": str(t.dtype).replace("torch.", "")}


def ipc_import(desc: dict, device: torch.device) -> DevicePtr:
    """Map an ipc_export()ed tensor of another process (peer access enabled)."""
    import ctypes
    h = (ctypes.c_uint8 * _ffi.ADR_IPC_HANDLE_BYTES).from_buffer_copy(desc["handle"])
    ptr, base = ctypes.c_void_p(), ctypes.c_void_p()
    with torch.cuda.device(device):
        _ffi.call("adr_ipc_import", ctypes.cast(h, ctypes.c_void_p), desc["offset"],
                  ctypes.byref(ptr), ctypes.byref(base))
    return DevicePtr(ptr.value, desc["shape"], getattr(torch, desc["dtype"]), device, base.value)
