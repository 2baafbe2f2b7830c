"""One line per profiled launch from an ncu --page raw --csv export:
time, DRAM bytes and rate (vs the measured copy peak), FP64 pipe, warps
active, issue active, registers, grid x block, top stall reasons."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = {
    "t": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread", "grid": "launch__grid_size", "block": "launch__block_size",
}
STALLS = ["long_scoreboard", "short_scoreboard", "mio_throttle", "barrier", "lg_throttle", "math_pipe_throttle",
          "wait", "not_selected"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(h)}

    def val(r, key):
        i = idx[key]
        v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else float("nan")
        return v * SCALE.get(units[i], 1.0)
    print("%3s %8s %8s %7s %6s %6s %6s %5s %9s  %s" % ("#", "ms", "GB", "frac", "fp64%", "warp%", "iss%", "regs",
                                                     "grid*blk", "stalls per issue (top 4)"))
    for n, r in enumerate(rows[2:]):
        if len(r) < len(h):
            continue
        t = val(r, COLS["t"])
        b = val(r, COLS["rd"]) + val(r, COLS["wr"])
        st = []
        for s in STALLS:
            k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
            if k in idx:
                st.append((float(r[idx[k]] or 0), s))
        st.sort(reverse=True)
        print("%3d %8.3f %8.2f %7.3f %6.1f %6.1f %6.1f %5d %4d*%-4d  %s" % (
            n, t * 1e3, b / 1e9, b / t / 1e9 / peak, val(r, COLS["fp64"]), val(r, COLS["warps"]),
            val(r, COLS["issue"]), int(val(r, COLS["regs"])), int(val(r, COLS["grid"])), int(val(r, COLS["block"])),
            ", ".join("%s %.2f" % (s, v) for v, s in st[:4])))


if __name__ == "__main__":
    main(sys.argv[1])
