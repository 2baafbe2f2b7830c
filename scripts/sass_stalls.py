"""Summarise an ncu source-page CSV (--page source --print-source sass):
top instructions by warp-stall samples, and the stall reasons per opcode."""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    data = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        try:
            s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        data.append((s, r))
    tot = sum(s for s, _ in data)
    print("%s: %d instructions, %d stall samples" % (path, len(data), tot))
    by_op = defaultdict(lambda: defaultdict(int))
    for s, r in data:
        op = r[idx["Source"]].strip().split()[0] if r[idx["Source"]].strip() else "?"
        if op.startswith("@"):
            op = r[idx["Source"]].strip().split()[1]
        op = op.split(".")[0]
        for k in stalls:
            by_op[op][k] += int(r[idx[k]] or 0)
    print("\nsamples by opcode (top reasons):")
    for op, d in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
        t = sum(d.values())
        rs = ", ".join("%s %d" % (k[6:], v) for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:4] if v)
        print("  %-10s %6d (%4.1f%%)  %s" % (op, t, 100.0 * t / max(1, tot), rs))
    print("\ntop instructions:")
    for s, r in sorted(data, key=lambda x: -x[0])[:top]:
        rs = ", ".join("%s %s" % (k[6:], r[idx[k]]) for k in stalls if r[idx[k]] not in ("0", ""))
        print("  %6d %-60s %s" % (s, r[idx["Source"]].strip()[:60], rs))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
