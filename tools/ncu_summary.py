"""Summarise an `ncu --csv --page raw` metrics dump (per-kernel: launches, time, DRAM bytes, fmaheavy %).

    python tools/ncu_summary.py gpurun_out/ncu_metrics.csv [steps] > profiles/rNN_ncu_summary.json
"""
import collections
import csv
import json
import re
import sys


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = []
    for r in rows:
        if "Kernel Name" in r and "ID" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            recs.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in recs:
        name = re.sub(r"^void ", "", d["Kernel Name"]).split("(")[0]
        name = name.replace("zkl::", "")
        name = re.sub(r"<.*", "", name)   # template instances aggregate under the kernel name
        a = agg.setdefault(name, {"launches": 0, "time_ms": 0.0, "dram_bytes": 0.0, "fmaheavy_pct_wsum": 0.0})
        a["launches"] += 1
        t = num(d.get("gpu__time_duration.sum")) or 0.0
        # ncu reports time in the unit of its column header row; raw pages use ns or us (units row skipped)
        a["time_ms"] += t / 1e6   # raw page: ns
        a["dram_bytes"] += (num(d.get("dram__bytes_read.sum")) or 0) + (num(d.get("dram__bytes_write.sum")) or 0)
        f = num(d.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"))
        if f is not None:
            a["fmaheavy_pct_wsum"] += f * t / 1e6
    out = {}
    for k, a in agg.items():
        out[k] = {"launches_per_step": a["launches"] / steps, "time_per_step": a["time_ms"] / steps,
                  "dram_bytes_per_step": a["dram_bytes"] / steps,
                  "fmaheavy_pct": (a["fmaheavy_pct_wsum"] / a["time_ms"]) if a["time_ms"] else None}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
