"""bench.py contract pieces that run without a GPU (-m "not gpu")."""
import json
import os
import subprocess
import sys

import pytest

import bench
import paper_2604_12256_b200 as qs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("key", sorted(bench.PLAN_BYTES))
def test_plan_bytes_table_matches_planner(key):
    """bench.PLAN_BYTES (the bytes both arms divide by) is this build's plan:
    whole-job algorithmic bytes = per-GPU plan bytes x ranks."""
    w = key.rstrip("0123456789")
    n = int(key[len(w):])
    ranks = 1 << (n - 30)
    g = bench.make_circuit(w, n)
    p = qs.plan_json(n, g, n_ranks=ranks, basis=bench.BASIS_X % (1 << n))
    assert p["stats"]["bytes_hbm"] * ranks == bench.PLAN_BYTES[key]


def test_reference_arm_never_loads_the_product():
    """--impl reference runs the CPU oracle only (the tier's reference arm):
    libqs is never imported; the JSON line carries impl/cpu_baseline/e2e."""
    code = (
        "import sys, argparse, json; sys.path.insert(0, %r); import bench;"
        "bench.PLAN_BYTES['qft14'] = 14 * 2 ** 20;"
        "a = argparse.Namespace(gpus=1, steps=2, warmup=1, n=14, workload='qft');"
        "bench.run_reference(a);"
        "assert 'paper_2604_12256_b200' not in sys.modules, 'product imported'" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["workload"] == "qft14"
