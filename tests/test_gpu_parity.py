"""GPU parity tests (-m gpu): libqs (through the C-ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): max |delta amp| <= 1e-10 in fp64; the test
asserts the tighter 1e-12 tripwire of SURVEY 8(c) where the oracle runs
(rounding-only differences are ~1e-16), bit-exact index ordering for
permutation circuits, and closed forms at sizes the oracle cannot reach.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W
from tests import pins
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


def sim_run(qs, n, gates, basis=0, ranks=1, flags=None, **cfgkw):
    kw = {"loopback_ranks": ranks} if ranks > 1 else {}
    s = qs.Simulator(n, **kw)
    if flags is not None or cfgkw:
        s.set_config(qs.make_config(flags=qs.QS_OPT_ALL if flags is None else flags, **cfgkw))
    s.set_basis_state(basis)
    s.apply(gates)
    psi = s.state()
    st = s.stats()
    s.close()
    return psi, st


def maxdiff(a, b):
    return float(np.max(np.abs(a - b)))


# ------------------------------------------------------------ small / SMALL kernel

@pytest.mark.parametrize("seed", range(6))
def test_random_small(qs, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 12))
    gates = W.random_circuit(n, 120, seed, diag_bias=0.3)
    x = int(rng.integers(1 << n))
    psi, _ = sim_run(qs, n, gates, basis=x)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=x)) < TOL


# ------------------------------------------------------------ chunk kernels

@pytest.mark.parametrize("n,seed", [(13, 0), (14, 1), (16, 2), (18, 3), (20, 4)])
def test_random_chunked(qs, n, seed):
    gates = W.random_circuit(n, 200, seed, diag_bias=0.4, max_generic=3)
    psi, st = sim_run(qs, n, gates, basis=7)
    assert st["n_passes"] >= 1
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=7)) < TOL


@pytest.mark.parametrize("jit", [0, 99])
@pytest.mark.parametrize("n", [16, 20])
def test_store_relabel(qs, jit, n):
    """QFT's chunk pass stores through the output relabel (opos != cpos) on
    both kernel paths; compared with the oracle element by element."""
    gates = W.qft(n)
    plan = qs.plan_json(n, gates, basis=9, detail=True)
    assert any(s["opos"] != s["cpos"] for s in plan["steps"] if s["type"] == "pass" and "opos" in s)
    psi, _ = sim_run(qs, n, gates, basis=9, jit_min_qubits=jit)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=9)) < TOL


@pytest.mark.parametrize("mode", ["QS_JIT_NOTAB", "QS_JIT_CTATAB"])
def test_specialised_table_modes(qs, mode, monkeypatch):
    """The specialised kernels' level-1 shape sums: in-kernel (no per-chunk
    table) and the CTA-wide table row, on chunk/dense/diag passes with
    chunk-dependent diagonals (the default per-warp rows run everywhere else)."""
    monkeypatch.setenv(mode, "1")
    n = 20
    gates = W.random_circuit(n, 260, 21, diag_bias=0.7, max_generic=3) + W.qft(n)[:60] + W.diag_chain(n, 2, 2)
    psi, _ = sim_run(qs, n, gates, basis=6, jit_min_qubits=0)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=6)) < TOL


@pytest.mark.parametrize("jit", [0, 99])
@pytest.mark.parametrize("n,seed", [(13, 10), (15, 11), (17, 12)])
def test_specialised_vs_interpreter_kernels(qs, jit, n, seed):
    """Both kernel paths (NVRTC-specialised per pass: jit_min_qubits=0;
    interpreter: 99) against the oracle, incl. every op type."""
    gates = W.random_circuit(n, 220, seed, diag_bias=0.4, max_generic=3)
    gates += W.qft(n)[:40] + W.supremacy(3, n // 3, 3, seed)
    psi, _ = sim_run(qs, n, gates, basis=5, jit_min_qubits=jit)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=5)) < TOL


@pytest.mark.parametrize("jit", [0, 99])
def test_specialised_sharded_expand(qs, jit):
    n = 16
    gates = W.qaoa_maxcut(n, 2, 4) + W.rzz_full(n, 2, h_layer=False)
    psi, _ = sim_run(qs, n, gates, ranks=2, jit_min_qubits=jit)
    assert maxdiff(psi, oracle.apply_circuit(n, gates)) < TOL


@pytest.mark.parametrize("flags", [0, 1, 3, 5, 9, 15])
def test_flag_combinations(qs, flags):
    n = 17
    gates = W.random_circuit(n, 150, 100 + flags, diag_bias=0.5)
    psi, _ = sim_run(qs, n, gates, basis=11, flags=flags)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=11)) < TOL


def test_tensor_tma_load_pass(qs):
    """A read pass with a 128 B low run and few position runs (positions
    0-2 + 9-17): loaded with one cp.async.bulk.tensor per chunk."""
    n = 20
    g1 = W.random_circuit(n, 60, 4)
    g2 = [W.Gate("RX", (q,), (), (0.1 * q,)) for q in range(9, 18)] + [W.Gate("CZ", (13,), (4,))]
    s = qs.Simulator(n)
    s.set_config(qs.make_config(jit_min_qubits=0))
    s.apply(g1)
    s.apply(g2)
    psi = s.state()
    assert qs.jit_info(s)["jit_errors"] == 0
    s.close()
    want = oracle.apply_circuit(n, g2, state=oracle.apply_circuit(n, g1))
    assert maxdiff(psi, want) < TOL


def test_not_product_state_second_circuit(qs):
    """Second apply on a non-product state: plain loads (no booster)."""
    n = 16
    g1 = W.random_circuit(n, 80, 1)
    g2 = W.random_circuit(n, 80, 2, diag_bias=0.5)
    s = qs.Simulator(n)
    s.apply(g1)
    s.apply(g2)
    psi = s.state()
    s.close()
    want = oracle.apply_circuit(n, g2, state=oracle.apply_circuit(n, g1))
    assert maxdiff(psi, want) < TOL


@pytest.mark.parametrize("n", [10, 16, 20, 24])
def test_qft_closed_form(qs, n):
    for x in (0, 12345 % (1 << n)):
        psi, _ = sim_run(qs, n, W.qft(n), basis=x)
        assert maxdiff(psi, pins.qft_closed_form(n, x)) < TOL


@pytest.mark.parametrize("name", sorted(W.ROSTER))
def test_roster_gpu(qs, name):
    """PAPER.md Table 2 roster (BV, HS, QAOA, QFT, QV, SC, VC) at 18 qubits
    (specialised kernels) against the oracle."""
    n = 18
    gates = W.ROSTER[name](n)
    psi, _ = sim_run(qs, n, gates)
    assert maxdiff(psi, oracle.apply_circuit(n, gates)) < TOL


@pytest.mark.parametrize("n", [3, 13, 22])
def test_ghz(qs, n):
    psi, _ = sim_run(qs, n, W.ghz(n))
    assert maxdiff(psi, pins.ghz_closed_form(n)) < 1e-15


@pytest.mark.parametrize("n", [14, 20])
def test_benchmark_families(qs, n):
    fams = [W.rzz_full(n, 3), W.diag_chain(n, 4), W.qaoa_maxcut(n, 2, 5),
            W.supremacy(4, n // 4, 6, 6), W.supremacy(4, n // 4, 4, 7, dense=True)]
    for gates in fams:
        nn = max(max(g.support) for g in gates) + 1
        psi, _ = sim_run(qs, nn, gates)
        assert maxdiff(psi, oracle.apply_circuit(nn, gates)) < TOL


def test_permutation_circuit_bit_exact(qs):
    """Classical reversible circuits on |x>: exactly one amplitude 1.0 at f(x)
    (0/1 matrices: no rounding), through relabels and shards."""
    rng = np.random.default_rng(9)
    for n, ranks in [(12, 1), (18, 1), (18, 4), (16, 8)]:
        gates = []
        for _ in range(60):
            k = int(rng.integers(3))
            a, b, c = (int(v) for v in rng.permutation(n)[:3])
            if k == 0:
                gates.append(W.Gate("X", (a,)))
            elif k == 1:
                gates.append(W.Gate("CX", (a,), (b,)))
            else:
                gates.append(W.Gate("SWAP", (a, b)) if rng.uniform() < .5 else W.Gate("X", (a,), (b, c)))
        x = int(rng.integers(1 << n))
        y = x
        for g in gates:   # classical evaluation
            if g.kind == "SWAP":
                a, b = g.targets
                ba, bb = (y >> a) & 1, (y >> b) & 1
                y = (y & ~((1 << a) | (1 << b))) | (ba << b) | (bb << a)
            elif all((y >> c) & 1 for c in g.controls):
                y ^= 1 << g.targets[0]
        psi, _ = sim_run(qs, n, gates, basis=x, ranks=ranks)
        want = np.zeros(1 << n, dtype=complex)
        want[y] = 1
        assert np.array_equal(psi, want)


# ------------------------------------------------------------ sharded (loopback)

@pytest.mark.parametrize("ranks", [2, 4, 8])
@pytest.mark.parametrize("n", [8, 15, 18])
def test_loopback_sharded(qs, ranks, n):
    gates = W.random_circuit(n, 150, 7 * n + ranks, diag_bias=0.3)
    psi, st = sim_run(qs, n, gates, basis=3, ranks=ranks)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=3)) < TOL


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_loopback_fused_swaps(qs, ranks):
    """SURVEY 8(f) f1 on one GPU: with specialised kernels everywhere the pass
    before each fusable swap stores the exported pieces straight into the
    other shards' receive buffers; parity with the oracle and the swaps are
    reported as fused."""
    n = 18
    gates = W.qaoa_maxcut(n, 3, 2)
    psi, st = sim_run(qs, n, gates, ranks=ranks, jit_min_qubits=0)
    assert st["n_swaps"] >= 2 and st["n_fused_swaps"] >= 1
    assert maxdiff(psi, oracle.apply_circuit(n, gates)) < TOL
    psi2, st2 = sim_run(qs, n, W.random_circuit(n, 160, 5 + ranks, diag_bias=0.3), basis=3,
                        ranks=ranks, jit_min_qubits=0)
    assert maxdiff(psi2, oracle.apply_circuit(n, W.random_circuit(n, 160, 5 + ranks, diag_bias=0.3), x=3)) < TOL


@pytest.mark.parametrize("ranks", [2, 4])
def test_loopback_direct_swaps_unfused(qs, ranks, monkeypatch):
    """Swaps planned against the victims' own positions (for fusion) but run
    without peer stores: transpose, swap the top positions, transpose back."""
    monkeypatch.setenv("QS_NO_FUSED_SWAP", "1")
    n = 18
    nl = n - (ranks.bit_length() - 1)
    for seed in range(3, 40):   # a circuit whose plan has a direct swap off the top positions
        gates = W.supremacy_n(n, 8, seed)
        plan = qs.plan_json(n, gates, n_ranks=ranks, config=qs.make_config(jit_min_qubits=0), detail=True)
        if any(s["type"] == "swap" and s["lpos"] != list(range(nl - s["j"], nl)) for s in plan["steps"]):
            break
    else:
        pytest.fail("no direct swap off the top positions in 37 seeded circuits")
    psi, st = sim_run(qs, n, gates, ranks=ranks, jit_min_qubits=0)
    assert st["n_fused_swaps"] == 0 and st["n_swaps"] >= 1
    assert maxdiff(psi, oracle.apply_circuit(n, gates)) < TOL


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_loopback_fused_direct_swaps(qs, ranks):
    """Supremacy-style circuits: every swap fused, exchanging the globals
    directly with the victims' positions (no permute passes)."""
    n = 18
    gates = W.supremacy_n(n, 10, 5)
    psi, st = sim_run(qs, n, gates, ranks=ranks, jit_min_qubits=0)
    assert st["n_swaps"] >= 1 and st["n_fused_swaps"] == st["n_swaps"]
    assert maxdiff(psi, oracle.apply_circuit(n, gates)) < TOL
    # the counters are per call
    s = qs.Simulator(n, loopback_ranks=ranks)
    s.set_config(qs.make_config(jit_min_qubits=0))
    for _ in range(2):
        s.set_basis_state(0)
        s.apply(gates)
        st2 = s.stats()
        assert st2["n_fused_swaps"] == st2["n_swaps"] == st["n_swaps"]
    s.close()


def test_loopback_qaoa_swaps(qs):
    n = 18
    gates = W.qaoa_maxcut(n, 3, 2)
    psi, st = sim_run(qs, n, gates, ranks=4)
    assert st["n_swaps"] >= 1
    assert maxdiff(psi, oracle.apply_circuit(n, gates)) < TOL


# ------------------------------------------------------------ readout / API

def test_probabilities_and_slices(qs):
    n = 15
    gates = W.random_circuit(n, 100, 3)
    s = qs.Simulator(n, loopback_ranks=2)
    s.apply(gates)
    psi = s.state()
    assert np.array_equal(s.state(100, 1000), psi[100:1100])
    pr = s.probabilities()
    assert np.allclose(pr, np.abs(psi) ** 2, atol=1e-15)
    s.close()


def test_invalid_gate_leaves_state(qs):
    n = 14
    s = qs.Simulator(n)
    s.apply(W.random_circuit(n, 50, 1))
    before = s.state()
    with pytest.raises(qs.QSError) as e:
        s.apply([W.Gate("H", (0,)), W.Gate("H", (14,))])
    assert e.value.code == qs.QS_EINVAL
    assert np.array_equal(s.state(), before)
    s.close()


def test_empty_circuit_and_basis(qs):
    for n in (1, 5, 13, 21):
        x = (1 << n) - 1
        psi, _ = sim_run(qs, n, [], basis=x)
        want = np.zeros(1 << n, dtype=complex)
        want[x] = 1
        assert np.array_equal(psi, want)


def test_launch_count_and_timing(qs):
    n = 20
    s = qs.Simulator(n)
    s.apply(W.qft(n))
    assert s.launches() >= 1
    t = s.kernel_timing("K1_chunk")
    assert t["launches"] >= 1 and t["ms"] > 0
    s.close()


def test_wide_gates_small_state(qs):
    """5- and 6-target unitaries / diagonals (QS_MAX_TARGETS) on <= 12-qubit
    shards (SMALL kernel) vs the oracle."""
    rng = np.random.default_rng(21)
    n = 11
    gates = [W.Gate("UNITARY", tuple(int(q) for q in rng.permutation(n)[:6]), (), (), W.haar_unitary(64, rng)),
             W.Gate("DIAGONAL", tuple(int(q) for q in rng.permutation(n)[:6]), (), (), W.random_phases(64, rng)),
             W.Gate("UNITARY", (1, 3, 5, 7, 9), (0,), (), W.haar_unitary(32, rng))]
    gates = W.random_circuit(n, 40, 3) + gates + W.random_circuit(n, 40, 4)
    psi, _ = sim_run(qs, n, gates, basis=9)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=9)) < TOL


def test_wide_gate_large_state(qs):
    """4-6-target unitaries on a 16-qubit state (formerly QS_EUNSUPPORTED)
    run as the shared-memory op (OP_DW) on both kernel paths; the full-size
    cases are in test_gpu_fullsize.py."""
    rng = np.random.default_rng(2)
    n = 16
    for jit in (0, 99):
        gates = [W.Gate("UNITARY", (0, 3, 7, 11), (), (), W.haar_unitary(16, rng)),
                 W.Gate("UNITARY", (1, 2, 5, 9, 14), (4,), (), W.haar_unitary(32, rng)),
                 W.Gate("UNITARY", (0, 6, 8, 10, 12, 15), (), (), W.haar_unitary(64, rng))]
        gates = W.random_circuit(n, 30, 5) + gates + W.random_circuit(n, 30, 6)
        psi, _ = sim_run(qs, n, gates, basis=5, jit_min_qubits=jit)
        assert maxdiff(psi, oracle.apply_circuit(n, gates, x=5)) < TOL


@pytest.mark.parametrize("n", [12, 13])
def test_small_kernel_boundary(qs, n):
    """nl = 12 runs the SMALL kernel, nl = 13 the chunk kernels."""
    gates = W.random_circuit(n, 150, 30 + n, diag_bias=0.3)
    psi, st = sim_run(qs, n, gates, basis=1)
    assert maxdiff(psi, oracle.apply_circuit(n, gates, x=1)) < TOL


def test_empty_circuit_sharded(qs):
    psi, _ = sim_run(qs, 10, [], basis=1000, ranks=4)
    want = np.zeros(1 << 10, dtype=complex)
    want[1000] = 1
    assert np.array_equal(psi, want)


def test_qft33_single_gpu_max_size(qs):
    """Largest single-B200 size (128 GiB state): QFT-33 closed form, sampled."""
    n = 33
    x = 0x1F2E3D4C5 % (1 << n)
    s = qs.Simulator(n)
    s.set_basis_state(x)
    s.apply(W.qft(n))
    for off in (0, (1 << n) // 2 + 12345, (1 << n) - 2048):
        got = s.state(int(off), 2048)
        k = np.arange(int(off), int(off) + 2048, dtype=np.int64)
        want = np.exp(2j * math.pi * ((x * k) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        assert maxdiff(got, want) < 1e-12
    s.close()


# ------------------------------------------------------------ bench configuration

def test_qft30_sampled_closed_form(qs):
    """configs[1] at full size in the launch configuration bench.py times:
    sampled amplitudes vs the closed form (SURVEY 8(c) pins)."""
    n = 30
    x = 987654321 % (1 << n)
    s = qs.Simulator(n)
    s.set_basis_state(x)
    s.apply(W.qft(n))
    rng = np.random.default_rng(0)
    for off in list(rng.integers(0, (1 << n) - 4096, size=8)) + [0, (1 << n) - 4096]:
        got = s.state(int(off), 4096)
        k = np.arange(int(off), int(off) + 4096, dtype=np.int64)
        want = np.exp(2j * math.pi * ((x * k) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        assert maxdiff(got, want) < 1e-12
    s.close()


def _norm(sim, n, slab=1 << 24):
    buf = np.empty(slab, dtype=np.float64)
    tot = 0.0
    for off in range(0, 1 << n, slab):
        tot += float(sim.probabilities(off, slab, out=buf).sum())
    return tot


@pytest.mark.parametrize("workload", ["rzz", "diag", "qaoa", "rand"])
def test_bench_workloads_30_properties(qs, workload):
    """The other bench workloads at their full size (30 qubits, the launch
    configuration bench.py times), checked through properties that hold at
    any size: norm 1 (all 2^30 probabilities summed); RZZ after H^n is a pure
    phase pattern, |a| = 2^-15 everywhere sampled; MaxCut QAOA is symmetric
    under flipping every qubit, a(x) = a(~x)."""
    import bench
    n = 30
    gates = bench.make_circuit(workload, n)
    s = qs.Simulator(n)
    s.apply(gates)
    assert qs.jit_info(s)["jit_errors"] == 0   # the specialised kernels ran
    assert abs(_norm(s, n) - 1.0) < 1e-10
    rng = np.random.default_rng(3)
    offs = [int(o) for o in rng.integers(0, (1 << n) - 4096, size=6)]
    if workload == "rzz":
        for off in offs:
            got = s.state(off, 4096)
            assert np.max(np.abs(np.abs(got) - 2.0 ** (-n / 2))) < 1e-12
    if workload == "qaoa":
        full = (1 << n) - 1
        for off in offs:
            a = s.state(off, 4096)
            b = s.state(full - off - 4095, 4096)[::-1]   # indices full - x
            assert maxdiff(a, b) < 1e-12
    s.close()
