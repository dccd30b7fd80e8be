#!/usr/bin/env python
"""Where does a decode-attention call spend its time? Builds a diagnostic copy
of libadrenaline.so with -DADR_TIMELINE (per-warp globaltimer stamps), runs a
PDL chain of calls on a BASELINE shape and prints, for the last call, the
distribution of entry / dependency-wait / first page / stream end / merge end
relative to the first warp's entry.   python scripts/timeline.py [C2|C3|C5]"""
import ctypes, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
OUT = ROOT / "scripts" / "probe" / "libadrenaline_tl.so"
from paper_2503_20552_b200 import _build
objs = []
deps = [_build.CSRC / f for f in _build.SOURCES + _build.HEADERS]
fresh = OUT.exists() and all(d.stat().st_mtime < OUT.stat().st_mtime for d in deps)
for src in ([] if fresh else _build.SOURCES):
    o = ROOT / "scripts" / "probe" / (Path(src).stem + "_tl.o")
    subprocess.run([_build._nvcc(), *_build.NVCC_FLAGS, "-DADR_TIMELINE", "-I", str(ROOT / "include"),
                    "-c", str(_build.CSRC / src), "-o", str(o)], check=True, capture_output=True)
    objs.append(str(o))
if not fresh:
    subprocess.run([_build._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-cudart", "static", *objs, "-o", str(OUT)], check=True)
if len(sys.argv) > 2 and sys.argv[2] == "--build-only":
    sys.exit(0)
os.environ["ADRENALINE_LIB"] = str(OUT)
import numpy as np
import torch
from paper_2503_20552_b200 import _ffi, ops
from paper_2503_20552_b200.synthetic import CONFIGS, make_block_table, make_layer

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
GRID = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--grid=")), "auto")
GRAPH = "--graph" in sys.argv  # chain captured in a CUDA graph (no host gaps between calls)
import re
from paper_2503_20552_b200.synthetic import DecodeShape
m = re.fullmatch(r"B(\d+)c(\d+)k(\d+)", name)  # ad-hoc shape, e.g. B8c1024k8 (Hq 32, D 128)
shape = CONFIGS[name] if m is None else DecodeShape(name, int(m[1]), 32, int(m[3]), 128, 4, int(m[2]))
dev = torch.device("cuda:0")
bt = make_block_table(shape)
layers = [make_layer(shape, dev, seed=l, block_table=bt) for l in range(4)]
ws = [ops.DecodeWorkspace(shape.batch, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, dev) for _ in range(2)]
out = torch.empty(shape.batch, shape.num_q_heads, shape.head_dim, dtype=torch.bfloat16, device=dev)
def call(i):
    x = layers[i % 4]
    ops.paged_decode_attn(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["seq_lens"], out=out,
                          workspace=ws[i % 2], k_new=x["k_new"], v_new=x["v_new"], pdl=True, grid=GRID)
for i in range(12):
    call(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if GRAPH:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(8):
            call(i)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
else:
    e0.record()
    for i in range(8):
        call(i)
    e1.record()
torch.cuda.synchronize()
print(f"{name} grid={GRID} graph={GRAPH}: {e0.elapsed_time(e1) / 8 * 1e3:.1f} us per call in the chain")
tl = np.zeros((4096, 12), dtype=np.uint64)
getattr(_ffi.lib(), "adr_debug_timeline_split" if GRID == "split" else "adr_debug_timeline")(
    ctypes.c_void_p(tl.ctypes.data), ctypes.c_size_t(tl.nbytes))
tl = tl[tl[:, 0] > 0].astype(np.float64)
ntask = tl[:, 8] / 20.0  # accumulated over the 20 calls of this script
tl[:, 8] = tl[:, 0]
t0 = tl[:, 0].min()
rel = (tl - t0) / 1e3
labels = ["entry", "pre-wait done", "wait done", "first page", "stream end", "merge end",
          "last task claimed", "its pieces in", "-", "rows merged", "next task known", "retired"]
if GRID == "split":  # prologue stamps of decode_split_kernel
    labels[6:11] = ["pages scanned", "candidates", "-", "items laid out", "first item set"]
for k, lab in enumerate(labels):
    if lab == "-":
        continue
    v = rel[:, k][rel[:, k] > -1e6]
    if v.size == 0:
        continue
    print(f"{lab:14s} min {v.min():8.1f} p10 {np.percentile(v, 10):8.1f} p50 {np.percentile(v, 50):8.1f} "
          f"p90 {np.percentile(v, 90):8.1f} max {v.max():8.1f} us")
last = np.argsort(rel[:, 5])[-8:]
if GRID in ("static", "split"):
    ret = rel[:, 11][rel[:, 11] > -1e6]
    per = e0.elapsed_time(e1) / 8 * 1e3
    print(f"call span (dependency released -> last warp retired): {ret.max() - rel[:, 2].min():.1f} us; "
          f"boundary (last retire -> next release): {per - (ret.max() - rel[:, 2].min()):.1f} us")
    sys.exit(0)
print("latest-finishing warps: stream end / task claimed / pieces in / rows merged / next known / merge end (us), tasks")
for i in last:
    print(f"  {rel[i, 4]:8.1f} {rel[i, 6]:8.1f} {rel[i, 7]:8.1f} {rel[i, 9]:8.1f} {rel[i, 10]:8.1f} {rel[i, 5]:8.1f}  {ntask[i]:.1f}")
print(f"tasks merged per warp per call: max {ntask.max():.1f}, total {ntask.sum():.0f}")
ret = rel[:, 11][rel[:, 11] > -1e6]
if ret.size == 0:
    sys.exit(0)
per = e0.elapsed_time(e1) / 8 * 1e3
print(f"call span (dependency released -> last warp retired): {ret.max() - rel[:, 2].min():.1f} us; "
      f"boundary (last retire -> next release, from the chain period): "
      f"{per - (ret.max() - rel[:, 2].min()):.1f} us")
