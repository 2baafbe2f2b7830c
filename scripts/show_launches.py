import csv, sys
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
    out = [(r[ki], float(r[vi]) / 1e6) for r in rows[1:]]
    n = len(out) // 2
    print(f, ' '.join(f"{k[3:9]}:{v:.2f}" for k, v in out[n:] if v > 0.05))
