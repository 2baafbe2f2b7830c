"""Summarise an ncu report (.ncu-rep) or an ncu launch-list CSV into text
for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/r01_k1.txt
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/r01_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_bytes.sum",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no data")
        return
    h, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(h)}
    name_i = idx.get("Kernel Name")
    print("ncu --set full summary of", path)
    for r in rows[2:]:
        print("-" * 78)
        print("kernel:", r[name_i] if name_i is not None else "?")
        for m in METRICS:
            if m in idx:
                print("  %-72s %s %s" % (m, r[idx[m]], units[idx[m]]))
        try:
            rd = float(r[idx["dram__bytes_read.sum"]])
            wr = float(r[idx["dram__bytes_write.sum"]])
            t = float(r[idx["gpu__time_duration.sum"]])
            ur, ut = units[idx["dram__bytes_read.sum"]], units[idx["gpu__time_duration.sum"]]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[ur]
            tsc = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}[ut]
            print("  traffic (read+write) = %.3f GB; achieved DRAM = %.1f GB/s"
                  % ((rd + wr) * scale / 1e9, (rd + wr) * scale / (t * tsc) / 1e9))
        except Exception:
            pass


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    idx = {k: i for i, k in enumerate(h)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print("ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)")
    print("%-44s %8s %12s %8s" % ("kernel", "launches", "total ms", "share"))
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-44s %8d %12.3f %7.1f%%" % (k[:44], n, ms, 100 * ms / tot))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
