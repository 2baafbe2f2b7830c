"""Kernel micro-benchmark: read+write passes with growing op counts on a
30-qubit state (16 GiB), to calibrate the chunk-kernel memory ceiling against
the per-op compute cost.  Prints one JSON line per case (device ms per pass,
effective GB/s, fraction of MEASURED_PEAKS hbm_gbs)."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_12256_b200 as qs  # noqa: E402
import workloads as W  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    G = W.Gate
    cases = {
        "rx1": [G("RX", (0,), (), (0.3,))],
        "rx_low4": [G("RX", (q,), (), (0.3,)) for q in range(4)],
        "rx_high4": [G("RX", (q,), (), (0.3,)) for q in range(20, 24)],
        "h8": [G("H", (q,), ()) for q in list(range(4)) + list(range(20, 24))],
        "h12": [G("H", (q,), ()) for q in list(range(5)) + list(range(20, 27))],
        "rx12": [G("RX", (q,), (), (0.1 * q,)) for q in list(range(5)) + list(range(20, 27))],
        "qft_low11": W.qft(11, swaps=False),
        "cz_chain": [G("CZ", (q + 1,), (q,)) for q in range(n - 1)],
        "rzz_all": W.rzz_full(n, 3, h_layer=False),
        "u3_12": [G("U3", (q,), (), (0.1, 0.2, 0.3)) for q in list(range(5)) + list(range(20, 27))],
        # QAOA mixer-like passes: RX on k mid qubits (l = 3 low positions + k)
        "rx9_mid": [G("RX", (q,), (), (0.1 * q,)) for q in range(9, 18)],
        "rx8_mid": [G("RX", (q,), (), (0.1 * q,)) for q in range(9, 17)],
        "rx7_mid": [G("RX", (q,), (), (0.1 * q,)) for q in range(9, 16)],
        "rx4_mid": [G("RX", (q,), (), (0.1 * q,)) for q in range(9, 13)],
        "h9_mid": [G("H", (q,), ()) for q in range(9, 18)],
    }
    sim = qs.Simulator(n)
    sim.apply([G("H", (q,)) for q in range(n)])  # materialise a dense state
    for name, gates in cases.items():
        for _ in range(2):
            sim.apply(gates)  # warm (JIT compile + cache)
        tot = 0.0
        reps = 3
        for _ in range(reps):
            sim.apply(gates)
            tot += sim.stats()["t_device_ms"]
        st = sim.stats()
        ms = tot / reps
        gbs = st["bytes_hbm"] / (ms * 1e-3) / 1e9
        print(json.dumps({"case": name, "gates": len(gates), "passes": st["n_passes"],
                          "kernels": {k: sim.kernel_timing(k)["launches"] for k in ("K1_chunk", "K2_dense", "K3_diag")},
                          "ms": round(ms, 3), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3)}), flush=True)
    sim.close()


if __name__ == "__main__":
    main()
