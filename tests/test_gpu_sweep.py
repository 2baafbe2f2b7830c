"""Seeded parity sweep (-m gpu): many random circuits at n = 21-22 through
the default configuration and the flag / fusion / rank variants that change
the plan ("plan replay = oracle on >= 200 seeded random
circuits ... for each flag combination" -- here on the GPU path itself, at
sizes where the specialised kernels run with several chunks per CTA)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.conftest import cuda_available

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def qs():
    if not cuda_available():
        pytest.skip("no CUDA device")
    import paper_2604_12256_b200 as qs
    qs.load_library()
    return qs


VARIANTS = [
    # (ranks, flags, fuse_cap)
    (1, 15, 4), (1, 15, 2), (1, 7, 4), (1, 11, 4), (1, 3, 4), (1, 1, 4),
    (2, 15, 4), (4, 15, 4), (8, 15, 4),
]


@pytest.mark.parametrize("i", range(len(VARIANTS)))
def test_random_sweep(qs, i):
    ranks, flags, fuse = VARIANTS[i]
    rng = np.random.default_rng(1000 + i)
    for rep in range(3):
        n = int(rng.integers(21, 23))
        seed = int(rng.integers(1 << 30))
        gates = W.random_circuit(n, 140, seed, diag_bias=float(rng.uniform(0.1, 0.7)), max_generic=3)
        if rep == 1:   # a wide unitary and a QAOA / supremacy tail
            tg = tuple(int(q) for q in rng.permutation(n)[:5])
            gates.append(W.Gate("UNITARY", tg, (), (), W.haar_unitary(32, rng)))
            gates += W.qaoa_maxcut(n, 1, seed, degree=3 if n % 2 == 0 else 4)[n:]
        if rep == 2:
            gates += W.supremacy_n(n, 4, seed)
        x = int(rng.integers(1 << n))
        kw = {"loopback_ranks": ranks} if ranks > 1 else {}
        s = qs.Simulator(n, **kw)
        s.set_config(qs.make_config(flags=flags, fuse_cap=fuse))
        s.set_basis_state(x)
        s.apply(gates)
        psi = s.state()
        info = qs.jit_info(s)
        s.close()
        assert info["jit_errors"] == 0, info["last_error"]
        d = float(np.max(np.abs(psi - oracle.apply_circuit(n, gates, x=x))))
        assert d < TOL, (n, ranks, flags, fuse, rep, d)
