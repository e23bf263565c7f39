"""Summarise ncu reports into committed text under profiles/.

    python tools/ncu_summary.py OUT.md REP1.ncu-rep [REP2.ncu-rep ...]
    python tools/ncu_summary.py --launches OUT.md launches.csv

Per kernel launch: duration, DRAM read/write bytes, occupancy, pipe
utilisation, issue activity, and the top source lines by warp-stall samples
(needs -lineinfo). Also merges per-kernel DRAM bytes per launch into
profiles/ncu_traffic.json (read by bench.py for the roofline "traffic" key).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__occupancy_limit_registers", "occ limit regs"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]
TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TO_US = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, label in METRICS:
            if m in hdr:
                k = hdr.index(m)
                try:
                    v = float(r[k].replace(",", ""))
                except ValueError:
                    continue
                u = units[k]
                if u in TO_BYTES:
                    v, u = v * TO_BYTES[u], "B"
                elif u in TO_US:
                    v, u = v * TO_US[u], "us"
                d[label] = (v, u)
        res.append(d)
    return res


def hot_lines(rep: str, top: int = 12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    try:
        hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    except StopIteration:
        return []
    hdr = rows[hi]
    if "Warp Stall Sampling (All Samples)" not in hdr:
        return []
    si = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    tot = sum(f(r[si]) for r in data) or 1.0
    data.sort(key=lambda r: -f(r[si]))
    return [(f(r[si]) / tot, r[0], r[1].strip()[:100]) for r in data[:top] if f(r[si]) > 0]


def fmt(v):
    x, u = v
    if u == "B":
        return f"{x / 1e6:.3f} MB"
    if u == "us":
        return f"{x:.2f} us"
    return f"{x:g} {u}".strip()


def summarise(out: Path, reps: list[str]):
    lines = []
    traffic_p = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_p.read_text()) if traffic_p.exists() else {}
    for rep in reps:
        name = Path(rep).stem
        lines.append(f"## {name} (`ncu --set full --clock-control none --import-source on`)\n")
        launches = raw(rep)
        for d in launches:
            lines.append(f"### {d['kernel'][:120]}")
            for _, label in METRICS:
                if label in d:
                    lines.append(f"- {label}: {fmt(d[label])}")
            lines.append("")
        by = collections.defaultdict(list)
        for d in launches:
            if "dram read" in d and "dram write" in d:
                kname = d["kernel"].split("(")[0].split("<")[0].replace("void ", "").strip()
                kname = kname.replace("unnamed>::", "").replace("(anonymous namespace)::", "")
                by[kname].append(d["dram read"][0] + d["dram write"][0])
        for k, v in by.items():
            traffic[f"{k}@{name}"] = {"bytes_per_launch": sum(v) / len(v), "launches": len(v), "report": name}
        hl = hot_lines(rep)
        if hl:
            lines.append("Top source lines by warp-stall samples (all kernels in the report):\n")
            for frac, ln, src in hl:
                lines.append(f"- {frac:6.1%}  L{ln}: `{src}`")
            lines.append("")
    out.write_text("\n".join(lines) + "\n")
    traffic_p.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")


def launches(out: Path, csv_path: str):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", "")) * TO_US.get(r[ui], 1e-3)
        a = agg.setdefault(r[ki][:110], [0.0, 0])
        a[0] += v
        a[1] += 1
    lines = ["| launches | avg us | total us | kernel |", "|---:|---:|---:|---|"]
    for k, (t, n) in agg.items():
        lines.append(f"| {n} | {t / n:.2f} | {t:.1f} | `{k}` |")
    out.write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(Path(sys.argv[2]), sys.argv[3])
    else:
        summarise(Path(sys.argv[1]), sys.argv[2:])
