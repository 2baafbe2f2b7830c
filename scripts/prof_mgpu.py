"""One process driving `world` GPUs (qs_create(n, world): NVLink peer access,
fused swaps by peer stores) applying a bench workload once between
cuProfilerStart/Stop, for an ncu capture with NVLink counters.

    ncu --profile-from-start off --metrics ...,nvltx__bytes.sum,nvlrx__bytes.sum \
        python scripts/prof_mgpu.py qaoa 2
"""
import ctypes
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_12256_b200 as qs  # noqa: E402


def main():
    wl = sys.argv[1]
    world = int(sys.argv[2])
    n = 30 + int(math.log2(world))
    gates = bench.make_circuit(wl, n)
    s = qs.Simulator(n, n_gpus=world)
    s.set_basis_state(bench.BASIS_X % (1 << n))
    s.apply(gates)
    s.set_basis_state(bench.BASIS_X % (1 << n))
    cuda = ctypes.CDLL("libcuda.so.1")
    cuda.cuProfilerStart()
    s.apply(gates)
    cuda.cuProfilerStop()
    st = s.stats()
    print(json.dumps({"workload": wl, "n": n, "world": world, "stats": st,
                      "fused": s.kernel_timing("fused_swap_pass"), "swap": s.kernel_timing("K4_swap")}))
    s.close()


if __name__ == "__main__":
    main()
