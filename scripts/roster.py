"""PAPER.md Table 2 / Table 3 mirrors on B200.

Table 2 (L777-806): per-gate time of the roster circuits (BV, HS, QAOA, QFT,
QV, SC, VC) at n qubits on one GPU, with the optimisations switched on in the
paper's order: none (one dense gate per pass; diagonals still batched),
fusion only, blocking + fusion + detector ("Ours"), and everything incl. the
merge booster ("Ours_b").
Table 3 (L811-858): the 5-level fully connected QAOA with each optimisation
flag on/off.

    python scripts/roster.py [--n 31] [--table 2|3|both] [--precompile]

--precompile only plans (detail=2: compiles every specialised kernel into the
on-disk cache, no GPU needed).  Prints one JSON line per (circuit, mode).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_12256_b200 as qs  # noqa: E402
import workloads as W  # noqa: E402

MODES2 = {
    "none": qs.QS_OPT_BLOCK * 0,
    "fuse": qs.QS_OPT_FUSE,
    "ours": qs.QS_OPT_BLOCK | qs.QS_OPT_FUSE | qs.QS_OPT_DIAG,
    "ours_b": qs.QS_OPT_ALL,
}
MODES3 = {
    "none": 0,
    "cache": qs.QS_OPT_BLOCK,
    "fusion": qs.QS_OPT_FUSE | qs.QS_OPT_DIAG,
    "boost": qs.QS_OPT_BOOST,
    "cache+fusion": qs.QS_OPT_BLOCK | qs.QS_OPT_FUSE | qs.QS_OPT_DIAG,
    "all": qs.QS_OPT_ALL,
}


def cases(table, n):
    out = []
    if table in ("2", "both"):
        for name, f in W.ROSTER.items():
            nn = n if not (name == "hs" and n % 2) else n - 1
            out += [("table2", name, nn, f(nn), mode, fl) for mode, fl in MODES2.items()]
    if table in ("3", "both"):
        nq = 30
        g = W.qaoa_complete(nq, 5)
        out += [("table3", "qaoa_complete_p5", nq, g, mode, fl) for mode, fl in MODES3.items()]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=31)
    ap.add_argument("--table", default="both")
    ap.add_argument("--precompile", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    for table, name, n, gates, mode, flags in cases(a.table, a.n):
        cfg = qs.make_config(flags=flags)
        if a.precompile:
            t0 = time.time()
            p = qs.plan_json(n, gates, config=cfg, basis=0, detail=2)
            print(json.dumps({"table": table, "circuit": name, "mode": mode, "n": n,
                              "passes": p["stats"]["n_passes"], "compile_s": round(time.time() - t0, 1)}), flush=True)
            continue
        sim = qs.Simulator(n)
        sim.set_config(cfg)
        best = None
        for rep in range(a.reps + 1):  # first repetition warms the kernels
            sim.set_basis_state(0)
            sim.apply(gates)
            st = sim.stats()
            if rep and (best is None or st["t_device_ms"] < best["t_device_ms"]):
                best = st
        sim.close()
        ms = best["t_device_ms"] + best["t_plan_ms"]
        print(json.dumps({"table": table, "circuit": name, "mode": mode, "n": n, "gates": len(gates),
                          "passes": best["n_passes"], "swaps": best["n_swaps"],
                          "circuit_ms": round(ms, 3), "device_ms": round(best["t_device_ms"], 3),
                          "plan_ms": round(best["t_plan_ms"], 3),
                          "per_gate_ms": round(ms / len(gates), 4)}), flush=True)


if __name__ == "__main__":
    main()
