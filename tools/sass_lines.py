"""Map ncu source-page SASS stall samples back to CUDA source lines.

    python tools/sass_lines.py --so paper_2306_07872_b200/libdawn.so --kernel dawn_batch_persistentIfjLb1 \
        --source gpurun_out/r02_c3_source.csv.gz [--top 25]

ncu's source page (CSV) lists SASS instructions with absolute addresses; the
first row is the function entry.  nvdisasm -g on the same cubin gives each
instruction offset its file:line (the library is built with -lineinfo).  The
samples are summed per CUDA line.
"""
import argparse
import collections
import csv
import gzip
import re
import subprocess
import tempfile
from pathlib import Path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", required=True)
    ap.add_argument("--kernel", required=True, help="substring of the mangled kernel name")
    ap.add_argument("--source", required=True)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(a.so).resolve())], cwd=tmp, capture_output=True)
    cubin = max(tmp.glob("*.cubin"), key=lambda p: p.stat().st_size)
    elf = subprocess.run(["cuobjdump", "-elf", str(cubin)], capture_output=True, text=True).stdout
    idx = None
    for ln in elf.splitlines():
        f = ln.split()
        if len(f) >= 7 and f[-1].startswith("_ZN") and a.kernel in f[-1] and f[3] == "0x12":
            idx = int(f[0], 16)
            break
    if idx is None:
        raise SystemExit(f"kernel {a.kernel} not found")
    dis = subprocess.run(["nvdisasm", "-g", "-c", "-fun", str(idx), str(cubin)], capture_output=True, text=True).stdout
    where = {}
    cur = "?"
    for ln in dis.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{Path(m.group(1)).name}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m:
            where[int(m.group(1), 16)] = cur
    op = gzip.open if a.source.endswith(".gz") else open
    rows = list(csv.reader(op(a.source, "rt")))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]
    ai, si = h.index("Address"), next(i for i, c in enumerate(h) if "Warp Stall Sampling (All" in c)
    body = [r for r in rows[hi + 1:] if len(r) > si and r[ai].startswith("0x")]
    base = int(body[0][ai], 16)
    per = collections.Counter()
    for r in body:
        per[where.get(int(r[ai], 16) - base, "?")] += float(r[si] or 0)
    tot = sum(per.values()) or 1
    src_cache = {}
    print(f"| share | line | code |\n|---:|---|---|")
    for loc, v in per.most_common(a.top):
        code = ""
        if ":" in loc:
            fn, no = loc.split(":")
            p = next(Path(a.so).resolve().parent.glob(f"csrc/{fn}"), None)
            if p:
                lines = src_cache.setdefault(fn, p.read_text().splitlines())
                code = lines[int(no) - 1].strip()[:100].replace("|", "/")
        print(f"| {100 * v / tot:.1f}% | {loc} | `{code}` |")


if __name__ == "__main__":
    main()
