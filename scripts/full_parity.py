"""Full-state oracle parity of the bench workloads at their bench size
(N = 30, 16 GiB; VERDICT r1 "Next round" item 1, north_star "matching the
CPU oracle to 1e-10 at every tested size").

For each workload: the GPU path runs the circuit exactly as bench.py does
(default configuration, qs_set_basis_state(x) + qs_apply_circuit); the
oracle (Alg. 1) runs the same gate list on the host from
|x> in place; every one of the 2^N amplitudes is compared, streamed in
slices.  One JSON line per workload (max |d|, ||d||_2, times, host).

    python scripts/full_parity.py [--n 30] [--workloads qft,rzz,diag,qaoa,rand] [--out F]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2604_12256_b200 as qs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--workloads", default="qft,rzz,diag,qaoa,rand")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n = args.n
    x = bench.BASIS_X % (1 << n)
    out = open(args.out, "a") if args.out else None
    oracle.build()
    host = bench.host_info()
    for wl in args.workloads.split(","):
        gates = bench.make_circuit(wl, n)
        sim = qs.Simulator(n)
        t0 = time.perf_counter()
        sim.set_basis_state(x)
        sim.apply(gates)
        t_gpu = time.perf_counter() - t0
        st = sim.stats()
        info = qs.jit_info(sim)
        t0 = time.perf_counter()
        psi = oracle.apply_circuit(n, gates, x=x)
        t_or = time.perf_counter() - t0
        slab = 1 << 24
        buf = np.empty(slab, dtype=np.complex128)
        dmax, l2, norm = 0.0, 0.0, 0.0
        for off in range(0, 1 << n, slab):
            got = sim.state(off, slab, out=buf)
            d = np.abs(got - psi[off:off + slab])
            dmax = max(dmax, float(d.max()))
            l2 += float(np.dot(d, d))
            norm += float(np.vdot(got, got).real)
        sim.close()
        del psi
        line = {"workload": "%s%d" % (wl, n), "gates": len(gates), "basis": x, "max_abs_diff": dmax,
                "l2_diff": l2 ** 0.5, "gpu_norm": norm, "bar": 1e-10, "pass": dmax <= 1e-10,
                "gpu_first_call_s": t_gpu, "oracle_s": t_or, "oracle_threads": oracle.num_threads(),
                "plan": {k: st[k] for k in ("n_passes", "n_swaps", "bytes_hbm")},
                "jit": {k: info[k] for k in ("jit_launches", "jit_errors", "variants")}, "host": host}
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")
            out.flush()


if __name__ == "__main__":
    main()
