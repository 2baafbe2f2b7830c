"""Committed GPU records (-m "not gpu"): the full-state N = 30 oracle
comparison of the five bench workloads (scripts/full_parity.py on a B200;
north_star: "matching the CPU oracle to 1e-10 at every tested size")."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_full_state_parity_n30_record():
    path = os.path.join(ROOT, "profiles", "r02_full_parity_n30.jsonl")
    rows = [json.loads(l) for l in open(path) if l.strip()]
    seen = {r["workload"] for r in rows}
    assert {"qft30", "rzz30", "diag30", "qaoa30", "rand30"} <= seen
    for r in rows:
        assert r["max_abs_diff"] <= 1e-10 and r["pass"], r["workload"]
        assert abs(r["gpu_norm"] - 1.0) < 1e-10
        assert r["jit"]["jit_errors"] == 0 and r["jit"]["jit_launches"] >= 1
