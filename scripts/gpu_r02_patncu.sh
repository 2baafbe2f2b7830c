# ncu --set full of the address-pattern probe: fast (position 3 in the chunk) vs slow pattern
cd $GRAFT_REPO_ROOT
B=scripts/dev/pattern_bw
for tag in slow:0,1,2,17,18,19,20,21,22,23,24,25 fast:0,1,2,3,17,18,19,20,21,22,23,24; do
  name=${tag%%:*}; pos=${tag#*:}
  timeout 600 ncu --set full --clock-control none -s 1 -c 1 -o /tmp/pat_$name $B 30 $pos > gpurun_out/patncu_$name.log 2>&1
  ncu -i /tmp/pat_$name.ncu-rep --page raw --csv > /tmp/pat_${name}_raw.csv 2>/dev/null
  python3 - "$name" <<'PY'
import csv, sys
name = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/pat_{name}_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
keep = [i for i, h in enumerate(hdr) if any(k in h for k in ("dram__", "lts__t_sectors", "lts__t_requests", "lts__d_", "fbpa", "ltc__", "gpu__time_duration", "lts__throughput", "lts__average", "l1tex__m_xbar2l1tex", "lts__xbar"))]
with open(f"gpurun_out/patncu_{name}_metrics.csv", "w") as f:
    w = csv.writer(f)
    for i in keep:
        w.writerow([hdr[i], units[i], vals[i]])
PY
done
