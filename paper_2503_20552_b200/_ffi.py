"""ctypes binding of libadrenaline.so (declared in include/adrenaline.h).

This is the same binding a maintainer of the reference would add (see
INTEGRATION.md): plain pointers, sizes and a stream handle. There is no CPU
fallback — if the library is missing or a call fails, an ``AdrError`` is raised.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libadrenaline.so"

ADR_OK = 0
ADR_ERR_INVALID = -1
ADR_ERR_UNSUPPORTED = -2
ADR_ERR_CUDA = -3
ADR_ERR_WORKSPACE = -4
ADR_DTYPE_BF16 = 0
ADR_DTYPE_F32 = 1
ADR_DECODE_PDL = 1
ADR_DECODE_GRID_DYNAMIC = 2
ADR_DECODE_GRID_STATIC = 4
ADR_DECODE_GRID_SPLIT = 8
ADR_IPC_HANDLE_BYTES = 64
ADR_STATUS_BAD_SEQ_LEN = 1
ADR_STATUS_BAD_PAGE = 2

_c_void_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_size = ctypes.c_size_t
_f32 = ctypes.c_float

# name -> (restype, argtypes); mirrors include/adrenaline.h one to one.
SIGNATURES: dict[str, tuple] = {
    "adr_version": (_i32, []),
    "adr_last_error": (ctypes.c_char_p, []),
    "adr_device_info": (_i32, [_i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "adr_decode_workspace_bytes": (_size, [_i32, _i32, _i32, _i32, _i32]),
    "adr_decode_workspace_size": (_size, [_i32, _i32, _i32, _i32, _i32, _i32]),
    "adr_decode_status": (_i32, [_c_void_p, _size, _i32, ctypes.POINTER(_i32), _c_void_p]),
    "adr_check_decode_tables": (_i32, [_c_void_p, _c_void_p, _i32, _i32, _i64, _c_void_p, _size,
                                       _c_void_p]),
    "adr_decode_warps_per_sm": (_i32, [_i32]),
    "adr_paged_decode_attn": (_i32, [
        _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
        _c_void_p, _i32, _i32, _i32, _i32, _i32, _i32, _i64, _f32, _i32, _i32, _i32, _u32,
        _c_void_p, _size, _c_void_p]),
    "adr_paged_decode_attn_rows": (_i32, [
        _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
        _c_void_p, _c_void_p, _c_void_p, _i32, _i32, _i32, _i32, _i32, _i32, _i64, _f32, _i32,
        _i32, _i32, _u32, _c_void_p, _size, _c_void_p]),
    "adr_kv_append": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                             _i32, _i32, _i32, _i32, _i64, _c_void_p]),
    "adr_pack_qkv": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i32, _i32, _i32, _i32,
                            _c_void_p, _c_void_p]),
    "adr_unpack_qkv": (_i32, [_c_void_p, _i32, _i32, _i32, _i32, _c_void_p, _c_void_p, _c_void_p,
                              _c_void_p]),
    "adr_scatter_out": (_i32, [_c_void_p, _c_void_p, _i32, _i32, _i32, _c_void_p, _c_void_p]),
    "adr_kv_transfer": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                               _i32, _i32, _i32, _i32, _c_void_p]),
    "adr_peer_open": (_i32, [_i32, _i32]),
    "adr_sm_partition_create": (_i32, [_i32, _i32, _i32, _i32, ctypes.POINTER(_c_void_p),
                                       ctypes.POINTER(_c_void_p), ctypes.POINTER(_i32),
                                       ctypes.POINTER(_i32), ctypes.POINTER(_c_void_p)]),
    "adr_sm_partition_destroy": (_i32, [_c_void_p]),
    "adr_copy_peer": (_i32, [_c_void_p, _i32, _c_void_p, _i32, _size, _c_void_p]),
    "adr_ipc_export": (_i32, [_c_void_p, _c_void_p, ctypes.POINTER(ctypes.c_uint64)]),
    "adr_ipc_import": (_i32, [_c_void_p, ctypes.c_uint64, ctypes.POINTER(_c_void_p),
                              ctypes.POINTER(_c_void_p)]),
    "adr_ipc_close": (_i32, [_c_void_p]),
    "adr_signal": (_i32, [_c_void_p, _u32, _c_void_p]),
    "adr_wait": (_i32, [_c_void_p, _u32, _c_void_p]),
}


class AdrError(RuntimeError):
    """A libadrenaline call returned a non-zero status."""

    def __init__(self, fn: str, code: int, message: str) -> None:
        super().__init__(f"{fn} failed ({code}): {message}")
        self.code = code


_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raises if it was never built."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("ADRENALINE_LIB", LIB_PATH))
        if not path.exists():
            raise AdrError("load", ADR_ERR_CUDA,
                           f"{path} missing: run __graft_entry__.build() (no CPU fallback)")
        handle = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def call(name: str, *args) -> int:
    """Invoke an entry point, raising ``AdrError`` on a negative status."""
    rc = getattr(lib(), name)(*args)
    if rc != ADR_OK:
        msg = lib().adr_last_error().decode(errors="replace")
        raise AdrError(name, rc, msg)
    return rc


def last_error() -> str:
    return lib().adr_last_error().decode(errors="replace")
