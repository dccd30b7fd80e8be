"""Build libadrenaline.so (sm_100a) and the C oracle in-tree.

Invoked by ``__graft_entry__.build()``; also runnable as
``python -m paper_2503_20552_b200._build``. nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libadrenaline.so"
SOURCES = ["abi.cu", "paged_decode_attn.cu", "decode_split.cu", "kv_and_exchange.cu"]
HEADERS = ["adr_device.cuh", "adr_internal.h", "decode_common.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "adrenaline.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    build_dir = PKG / "_obj"
    build_dir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):  # the translation units compile in parallel
        obj = build_dir / (Path(src).stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        for src, obj, res in pool.map(compile_one, SOURCES):
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
            if verbose:
                sys.stderr.write(res.stderr)
            (build_dir / (Path(src).stem + ".ptxas.txt")).write_text(res.stderr)
            objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           *objs, "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_oracle(force: bool = False) -> Path:
    """Compile oracle/attn_oracle.c (the CPU checker; test infrastructure only)."""
    src = ROOT / "oracle" / "attn_oracle.c"
    out = ROOT / "oracle" / "liboracle.so"
    if not force and not _stale(out, [src]):
        return out
    cc = os.environ.get("CC", "gcc")
    cmd = [cc, "-O3", "-march=x86-64-v2", "-pthread", "-fPIC", "-shared", "-std=c11",
           str(src), "-o", str(out), "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stderr}")
    return out


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build_cuda(force=force, verbose=True))
    print(build_oracle(force=force))
