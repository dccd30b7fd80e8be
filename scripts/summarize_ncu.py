#!/usr/bin/env python
"""Summarise an ncu capture + launch list into profiles/ (committed evidence).

    python scripts/summarize_ncu.py r01b
reads gpurun_out/prof_<tag>.ncu-rep and gpurun_out/launches_<tag>.csv, writes
profiles/ncu_<tag>.md, profiles/launches_<tag>.csv (per-kernel shares) and
updates profiles/ncu_summary.json (dram bytes per launch, read by bench.py).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw_table(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stall_table(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[0], rows[2:]
    res = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
                (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
            try:
                res.append((h, float(data[0][i].replace(",", ""))))
            except (ValueError, IndexError):
                pass
    res.sort(key=lambda x: -x[1])
    return res[:12]


def launch_shares(path: Path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].split("::")[-1]
            d[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    return [(k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in sorted(d.items(), key=lambda x: -sum(x[1]))]


def main():
    tag = sys.argv[1]
    rep = ROOT / "gpurun_out" / f"prof_{tag}.ncu-rep"
    hdr, units, data = raw_table(rep)
    lines = [f"# ncu capture `{tag}` — decode_attn_kernel (bench.py C2 workload)", "",
             "`ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel` "
             "(cold cache, serialised replay; see scripts/profile_ncu.sh). One column per captured launch.",
             "", "| metric | unit | " + " | ".join(f"launch {i}" for i in range(len(data))) + " |",
             "|---|---|" + "---|" * len(data)]
    summary = {}
    for key, label in METRICS:
        if key in hdr:
            i = hdr.index(key)
            vals = [d[i] for d in data]
            lines.append(f"| {label} (`{key}`) | {units[i]} | " + " | ".join(vals) + " |")
            summary[key] = {"unit": units[i], "values": vals}
    try:
        st = stall_table(rep)
        if st:
            lines += ["", "Top warp-stall metrics (launch 0):", ""]
            lines += [f"- `{k}`: {v}" for k, v in st]
    except subprocess.CalledProcessError:
        pass
    lp = ROOT / "gpurun_out" / f"launches_{tag}.csv"
    if lp.exists():
        shares = launch_shares(lp)
        lines += ["", "## Launch list (all our kernels in `bench.py --steps 2 --warmup 3`)", "",
                  "| kernel | launches | avg ns | share of device time |", "|---|---|---|---|"]
        lines += [f"| {k} | {n} | {a:.0f} | {s * 100:.2f}% |" for k, n, a, s in shares]
        (ROOT / "profiles" / f"launches_{tag}.csv").write_text(
            "kernel,launches,avg_ns,share\n" + "".join(f"{k},{n},{a:.1f},{s:.5f}\n" for k, n, a, s in shares))
    (ROOT / "profiles" / f"ncu_{tag}.md").write_text("\n".join(lines) + "\n")

    def num(key, scale):
        i = hdr.index(key)
        return [float(d[i].replace(",", "")) * scale for d in data]
    unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = num("dram__bytes_read.sum", unit_scale[units[hdr.index("dram__bytes_read.sum")]])
    wr = num("dram__bytes_write.sum", unit_scale[units[hdr.index("dram__bytes_write.sum")]])
    traffic = sum(r + w for r, w in zip(rd, wr)) / len(rd)
    js = {"tag": tag, "kernel": "decode_attn_kernel", "dram_bytes_per_launch": traffic,
          "metrics": summary}
    (ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(js, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
