"""CPU-side checks of the C-ABI boundary: the library builds, loads, exports
every symbol include/adrenaline.h declares, and the Python front end refuses
CPU tensors (no fallback). No compute calls — there is no GPU here."""
import re
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "adrenaline.h").read_text()
    return sorted(set(re.findall(r"ADR_API\s+[\w\s\*]+?\b(adr_\w+)\s*\(", text)))


def test_header_declares_expected_surface():
    syms = declared_symbols()
    for name in ["adr_paged_decode_attn", "adr_kv_append", "adr_pack_qkv", "adr_unpack_qkv",
                 "adr_scatter_out", "adr_decode_workspace_bytes", "adr_last_error",
                 "adr_peer_open", "adr_copy_peer", "adr_signal", "adr_wait"]:
        assert name in syms


def test_library_exports_every_declared_symbol(built):
    from paper_2503_20552_b200 import _ffi
    lib = _ffi.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # the Python binding covers exactly the header
    assert set(_ffi.SIGNATURES) == set(declared_symbols())


def test_version_and_error_string(built):
    from paper_2503_20552_b200 import _ffi
    assert _ffi.lib().adr_version() >= 1
    assert isinstance(_ffi.last_error(), str)


def test_invalid_arguments_are_rejected_before_any_device_work(built):
    from paper_2503_20552_b200 import _ffi
    lib = _ffi.lib()
    # GQA group 16 > 8 is unsupported; null pointers are invalid. Both fail fast.
    rc = lib.adr_paged_decode_attn(None, None, None, None, None, None, None, None, None, 1, 32, 2,
                                   128, 16, 1, 1, 1.0, 0, 0, 0, 0, None, 0, None)
    assert rc == _ffi.ADR_ERR_INVALID
    assert "null" in _ffi.last_error()
    rc = lib.adr_kv_append(None, None, None, None, None, 1, 8, 128, 16, 4, None)
    assert rc == _ffi.ADR_ERR_INVALID
    rc = lib.adr_pack_qkv(None, None, None, None, 2, 32, 8, 100, None, None)
    assert rc == _ffi.ADR_ERR_INVALID  # D % 8 != 0


def test_ops_refuse_cpu_tensors(built):
    from paper_2503_20552_b200 import ops
    q = torch.zeros(1, 2, 64, dtype=torch.bfloat16)
    kc = torch.zeros(1, 2, 16, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        ops.paged_decode_attn(q, kc, kc, torch.zeros(1, 1, dtype=torch.int32),
                              torch.ones(1, dtype=torch.int32))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2503_20552_b200 import _ffi
    monkeypatch.setattr(_ffi, "_lib", None)
    monkeypatch.setenv("ADRENALINE_LIB", str(tmp_path / "nope.so"))
    with pytest.raises(_ffi.AdrError, match="no CPU fallback"):
        _ffi.lib()


def test_header_constants_match_binding():
    """Every #define ADR_* value in include/adrenaline.h equals the ctypes binding's."""
    import re
    from pathlib import Path
    from paper_2503_20552_b200 import _ffi
    text = (Path(__file__).resolve().parent.parent / "include" / "adrenaline.h").read_text()
    found = dict(re.findall(r"#define\s+(ADR_\w+)\s+\(?(-?\d+)u?\)?", text))
    assert "ADR_DECODE_GRID_STATIC" in found and "ADR_ERR_WORKSPACE" in found
    for name, value in found.items():
        if hasattr(_ffi, name):
            assert getattr(_ffi, name) == int(value), name
