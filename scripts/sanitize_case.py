"""Small steady-state cases for compute-sanitizer (racecheck / synccheck /
memcheck) over the specialised kernels: n = 21-22 at the default
configuration (>= 4 chunks per CTA), checked against the oracle.

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2604_12256_b200 as qs  # noqa: E402
import workloads as W  # noqa: E402

cases = [
    (21, W.random_circuit(21, 120, 77, diag_bias=0.4, max_generic=3), 5),
    (22, W.qaoa_maxcut(22, 2, 3), 0),
    (21, W.qft(21), 12345),
    (22, W.supremacy(4, 5, 6, 2, dense=True) + [W.Gate("UNITARY", (0, 4, 9, 13, 17), (), (),
                                                       W.haar_unitary(32, np.random.default_rng(1)))], 0),
]
worst = 0.0
for n, gates, x in cases:
    nn = max(n, max(max(g.support) for g in gates) + 1)
    s = qs.Simulator(nn)
    s.set_basis_state(x)
    s.apply(gates)
    psi = s.state()
    info = qs.jit_info(s)
    s.close()
    d = float(np.max(np.abs(psi - oracle.apply_circuit(nn, gates, x=x))))
    worst = max(worst, d)
    print("n=%d gates=%d max|d|=%.2e jit=%s" % (nn, len(gates), d, info), flush=True)
assert worst < 1e-12, worst
print("sanitize cases ok")
