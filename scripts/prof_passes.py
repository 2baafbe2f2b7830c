"""Profile one application of a bench workload's circuit (after a warm-up
call that compiles every specialised pass) between cudaProfilerStart/Stop,
so `ncu --profile-from-start off` captures exactly one circuit's launches.

    ncu --profile-from-start off --set full ... python scripts/prof_passes.py qaoa 30
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_12256_b200 as qs  # noqa: E402


def main():
    wl = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    gates = bench.make_circuit(wl, n)
    cuda = ctypes.CDLL("libcuda.so.1")  # cuProfilerStart/Stop act on the current (primary) context
    s = qs.Simulator(n)
    s.set_basis_state(bench.BASIS_X % (1 << n))
    s.apply(gates)
    s.set_basis_state(bench.BASIS_X % (1 << n))
    cuda.cuProfilerStart()
    s.apply(gates)
    cuda.cuProfilerStop()
    st = s.stats()
    kt = {k: s.kernel_timing(k) for k in qs.KERNELS}
    print(json.dumps({"workload": wl, "n": n, "stats": st, "kernels": kt, "jit": qs.jit_info(s)}))
    s.close()


if __name__ == "__main__":
    main()
