"""Write profiles/traffic.json from ncu --set full captures of the C2 solve.

    python tools/traffic_stamp.py --rep gpurun_out/r02_c2.ncu-rep --rep gpurun_out/r02_wl.ncu-rep \
        --key c2_async_fp32 --out gpurun_out/traffic.json --capture r02

DRAM bytes per solve = the sum over the given captures (one launch each: the
persistent kernel and its worklist tail) of dram__bytes_read.sum +
dram__bytes_write.sum.  The file carries the sha256 of the CUDA sources it was
captured on; bench.py drops the figure when the sources differ (stale).
"""
import argparse
import csv
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def dram_bytes(rep: str) -> tuple[float, str]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    tot, names = 0.0, []
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for row in rows[2:]:
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(k)
            tot += float(row[i].replace(",", "")) * scale.get(u[i], 1)
        names.append(row[h.index("Kernel Name")][:60])
    return tot, ";".join(names)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", required=True)
    ap.add_argument("--key", default="c2_async_fp32")
    ap.add_argument("--out", required=True)
    ap.add_argument("--capture", default="")
    a = ap.parse_args()
    import bench

    out = Path(a.out)
    t = json.loads(out.read_text()) if out.exists() else {}
    sha = bench.kernel_source_sha()
    if t.get("src_sha256") != sha:
        t = {"src_sha256": sha, "kernels": {}}
    t["capture"] = a.capture
    total, kernels = 0.0, []
    for r in a.rep:
        b, k = dram_bytes(r)
        total += b
        kernels.append({"rep": Path(r).name, "kernels": k, "dram_bytes": b})
    t["kernels"][a.key] = {"dram_bytes_per_solve": int(total), "parts": kernels}
    out.write_text(json.dumps(t, indent=1))
    print(json.dumps(t, indent=1))


if __name__ == "__main__":
    main()
