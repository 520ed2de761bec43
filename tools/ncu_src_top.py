"""Top stall lines of an ncu --page source --csv --print-source sass dump (read here, no GPU)."""
import collections
import csv
import sys


def main(path, n=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Warp Stall Sampling (All Samples)" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            try:
                float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except ValueError:
                continue
            data.append(dict(zip(hdr, r)))
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[key] or 0) for d in data) or 1
    print("instructions", len(data), "samples", tot)
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:n]:
        print(f"{float(d[key]) / tot * 100:5.1f}% {d['Address']} {d['Source'][:100]}")
    c = collections.Counter()
    for d in data:
        toks = d["Source"].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        c[op.split(".")[0]] += float(d[key] or 0)
    print("by opcode:", [(k, round(v / tot * 100, 1)) for k, v in c.most_common(14)])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
