"""Summarise ncu output into profiles/ (run here, on the CPU side).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_c2.ncu-rep --out profiles/r01_c2_ncu.md --title "..."

* launches: per-kernel totals / counts / share of device time from the
  `--metrics gpu__time_duration.sum` launch list (cold, serialised).
* rep: the key counters of one `ncu --set full` capture (DRAM bytes per
  launch = the roofline `traffic`, L1/L2 hit rates, occupancy, issue rate).
"""

from __future__ import annotations

import argparse
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth achieved"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput % of peak (max unit)"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors from L1"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global store requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_atom.sum", "global atom sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "global atom requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "global red sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "global red requests"),
]
RATIOS = [("ld", "global loads"), ("st", "global stores"), ("atom", "global atomics (returning)"),
          ("red", "global reductions (red.*)")]


def launches(path: str):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    unit = None
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        unit = r[ui]
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0][:90]
        tot[name] += v
        cnt[name] += 1
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    allt = sum(tot.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
        out.append(f"| `{k}` | {cnt[k]} | {v * scale:.1f} | {v * scale / cnt[k]:.1f} | {100 * v / allt:.1f}% |")
    return out


def rep(path: str):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"**{name[:100]}**")
        out.append("")
        out.append("| counter | value | unit |")
        out.append("|---|---:|---|")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"| {label} (`{k}`) | {row[i]} | {u[i]} |")
        for op, label in RATIOS:
            ks = f"l1tex__t_sectors_pipe_lsu_mem_global_op_{op}.sum"
            kr = f"l1tex__t_requests_pipe_lsu_mem_global_op_{op}.sum"
            if ks in h and kr in h:
                sec = float(row[h.index(ks)].replace(",", "") or 0)
                req = float(row[h.index(kr)].replace(",", "") or 0)
                if req:
                    out.append(f"| **sectors / request, {label}** | {sec / req:.2f} | sector/request |")
        out.append("")
    return out


def stalls(path: str, top: int = 15):
    """Top source lines by sampled warp stalls (needs -lineinfo + --import-source on)."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hi = next((i for i, r in enumerate(rows) if any("Warp Stall Sampling (All" in c for c in r)), None)
    if hi is None:
        return ["(no source page)"]
    h = rows[hi]
    si = next(i for i, c in enumerate(h) if "Warp Stall Sampling (All" in c)
    li = h.index("# Address") if "# Address" in h else (h.index("Line") if "Line" in h else 0)
    ci = h.index("Source") if "Source" in h else len(h) - 1
    body = []
    for r in rows[hi + 1:]:
        if len(r) <= max(si, ci):
            continue
        try:
            body.append((float(r[si].replace(",", "") or 0), r[li], r[ci].strip()[:110]))
        except ValueError:
            continue
    allv = sum(b[0] for b in body) or 1.0
    out = ["| share | line | source |", "|---:|---:|---|"]
    for v, ln, src in sorted(body, key=lambda b: -b[0])[:top]:
        out.append(f"| {100 * v / allv:.1f}% | {ln} | `{src.replace('|', '/')}` |")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.note:
        lines += [a.note, ""]
    if a.launches:
        lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
                  "Cold-cache and serialised: compare shares, not absolutes.", ""]
        lines += launches(a.launches) + [""]
    if a.rep:
        lines += ["## `ncu --set full` capture", ""] + rep(a.rep)
        lines += ["## Warp-stall samples by source line (top 15)", ""] + stalls(a.rep) + [""]
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
