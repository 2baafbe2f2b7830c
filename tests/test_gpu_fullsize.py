"""GPU parity at sizes where the specialised kernels run in steady state
(-m gpu; VERDICT r1 "Next round" item 1).

Every test here uses the DEFAULT configuration (passes over >= 13 local
qubits run as NVRTC-specialised kernels) at n = 23-26, i.e. 2^11-2^14
chunks per pass: with the 148-296 CTA grids each CTA processes 7-55 chunks,
so the refill ring (mbarrier phases >= 1, the two-group "issued" wait), the
per-warp table-row double buffer and the hoisted expand gathers all run
past their first use -- the paths the bench runs.  The result is compared
with the CPU oracle (Alg. 1) element by element at the
1e-12 tripwire (north_star bar: 1e-10), and each test asserts which chunk
refill engines its passes used (qs_jit_info "variants").
"""
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


def run(qs, n, gates, basis=0, ranks=1):
    kw = {"loopback_ranks": ranks} if ranks > 1 else {}
    s = qs.Simulator(n, **kw)
    s.set_basis_state(basis)
    s.apply(gates)
    psi = s.state()
    info = qs.jit_info(s)
    st = s.stats()
    s.close()
    assert info["jit_errors"] == 0, info["last_error"]
    assert info["jit_launches"] >= 1
    return psi, st, info


def check(psi, n, gates, basis=0):
    want = oracle.apply_circuit(n, gates, x=basis)
    d = float(np.max(np.abs(psi - want)))
    assert d < TOL, d


def test_random_3q_unitaries_controls_n24(qs):
    """Every gate kind, generic 3-target unitaries/diagonals, <= 2 controls."""
    n = 24
    gates = W.random_circuit(n, 260, 2401, diag_bias=0.4, max_generic=3)
    psi, st, info = run(qs, n, gates, basis=0x5A5A5A)
    check(psi, n, gates, basis=0x5A5A5A)
    v = info["variants"]
    assert st["n_passes"] >= 3
    assert v["bulk_tma"] + v["tensor_tma"] + v["cp_async"] >= 1   # read passes ran a refill ring


def test_qaoa_n24(qs):
    n = 24
    gates = W.qaoa_maxcut(n, 4, 24)
    psi, st, info = run(qs, n, gates)
    check(psi, n, gates)
    v = info["variants"]
    assert v["write_only"] >= 1 and v["bulk_tma"] + v["tensor_tma"] + v["cp_async"] >= 3


@pytest.mark.parametrize("dense", [False, True])
def test_supremacy_n24(qs, dense):
    """Google-2019-style circuit on a 4x6 grid: CZ couplers, or a Haar 4x4
    unitary per coupler (K2-heavy)."""
    gates = W.supremacy(4, 6, 10, 31, dense=dense)
    n = 24
    psi, st, info = run(qs, n, gates)
    check(psi, n, gates)
    assert st["n_passes"] >= 3


def test_diag_chain_n24(qs):
    n = 24
    gates = W.diag_chain(n, 5)
    psi, _, info = run(qs, n, gates)
    check(psi, n, gates)
    assert info["variants"]["write_only"] >= 1


def test_rzz_full_n24(qs):
    """PAPER.md L715 gate-level benchmark (H^n + RZZ on every pair): one
    write-only diagonal pass fused with the booster's expansion."""
    n = 24
    gates = W.rzz_full(n, 7)
    psi, st, info = run(qs, n, gates)
    check(psi, n, gates)
    assert st["n_passes"] == 1 and info["variants"]["write_only"] == 1


def test_qft_n26_oracle(qs):
    """QFT-26 from a basis state: element by element against the oracle
    (not only the closed form)."""
    n = 26
    x = 0x2A5F3C71 % (1 << n)
    gates = W.qft(n)
    psi, st, info = run(qs, n, gates, basis=x)
    check(psi, n, gates, basis=x)


def test_second_circuit_read_passes_n23(qs):
    """A second circuit on a non-product state: every pass loads (no booster
    source), random circuit with controls, steady-state refill ring."""
    n = 23
    g1 = W.random_circuit(n, 120, 231, diag_bias=0.3, max_generic=2)
    g2 = W.random_circuit(n, 200, 232, diag_bias=0.5, max_generic=3)
    s = qs.Simulator(n)
    s.apply(g1)
    s.apply(g2)
    psi = s.state()
    info = qs.jit_info(s)
    s.close()
    assert info["jit_errors"] == 0
    want = oracle.apply_circuit(n, g2, state=oracle.apply_circuit(n, g1))
    assert float(np.max(np.abs(psi - want))) < TOL


@pytest.mark.parametrize("k", [4, 5, 6])
def test_wide_unitaries_n22(qs, k):
    """a8 at F = 4 and 4-6-target generic unitaries on a 22-qubit shard
    (Eq. 3 generalised): a shared-memory op at a layout
    exchange (OP_DW); with and without a control."""
    rng = np.random.default_rng(220 + k)
    n = 22
    gates = W.random_circuit(n, 30, k, diag_bias=0.3)
    for i in range(4):
        tg = tuple(int(q) for q in rng.permutation(n)[:k])
        ctl = (int(rng.choice([q for q in range(n) if q not in tg])),) if i % 2 else ()
        gates.append(W.Gate("UNITARY", tg, ctl, (), W.haar_unitary(1 << k, rng)))
        gates += W.random_circuit(n, 12, int(rng.integers(1 << 30)), diag_bias=0.5)
    psi, st, info = run(qs, n, gates, basis=77)
    check(psi, n, gates, basis=77)


def test_fused_four_qubit_unitary_n22(qs):
    """fuse_cap = 4 effective: many two-qubit gates on 4 qubits fuse into one
    16x16 unitary (shared-memory op); parity with the oracle."""
    rng = np.random.default_rng(5)
    n = 22
    qb = [1, 9, 14, 20]
    gates = W.random_circuit(n, 20, 3)
    for _ in range(20):
        a, b = (int(x) for x in rng.choice(qb, 2, replace=False))
        gates.append(W.Gate("UNITARY", (a, b), (), (), W.haar_unitary(4, rng)))
    psi, _, _ = run(qs, n, gates, basis=3)
    check(psi, n, gates, basis=3)


@pytest.mark.parametrize("ranks", [2, 4])
@pytest.mark.parametrize("fused", [True, False])
def test_loopback_sharded_n24(qs, ranks, fused, monkeypatch):
    """Sharded plans at n = 24 (22-23 local qubits): QAOA and a
    supremacy-style circuit, with the exchanges fused into the preceding
    pass's stores (f1) or run as separate copies."""
    if not fused:
        monkeypatch.setenv("QS_NO_FUSED_SWAP", "1")
    n = 24
    for gates in (W.qaoa_maxcut(n, 3, 40 + ranks), W.supremacy_n(n, 8, 41 + ranks)):
        psi, st, info = run(qs, n, gates, ranks=ranks)
        assert st["n_swaps"] >= 1
        if fused:
            assert st["n_fused_swaps"] >= 1
        else:
            assert st["n_fused_swaps"] == 0
        check(psi, n, gates)


def test_loopback_16_ranks_unfusable_swaps(qs):
    """16 shards: swaps of 4 global qubits exceed the fused-swap peer table
    (8 destinations) and run unfused; swaps of <= 3 still fuse."""
    n = 22
    gates = W.qaoa_maxcut(n, 2, 16)
    psi, st, info = run(qs, n, gates, ranks=16)
    assert st["n_swaps"] >= 1
    check(psi, n, gates)


@pytest.mark.parametrize("jit", [0, 99])
def test_unit_scaled_ops_and_pass_scales(qs, jit):
    """Uncontrolled unit-scaled gates (r9: SX, SY, e^{ia} X, e^{ia} (X+iY)-type
    Paulis) with their scalars folded into the pass scale: products that are
    real, pure imaginary, an eighth turn and a general phase; controlled
    copies keep their matrices.  Both kernel paths, against the oracle."""
    rng = np.random.default_rng(77)
    n = 20
    ph = np.exp(1j * 0.7345)
    gx = np.array([[0, ph], [ph, 0]])                 # e^{ia} X
    gy = np.array([[0, -1j * ph], [1j * ph, 0]])      # e^{ia} Y
    circ = []
    for layer in range(6):
        for q in range(n):
            k = int(rng.integers(5))
            if k == 0:
                circ.append(W.Gate("SX", (q,)))
            elif k == 1:
                circ.append(W.Gate("SY", (q,)))
            elif k == 2:
                circ.append(W.Gate("UNITARY", (q,), (), (), gx))
            elif k == 3:
                circ.append(W.Gate("UNITARY", (q,), (), (), gy))
            else:
                circ.append(W.Gate("SX", (q,), ((q + 3) % n,)))     # controlled: no extraction
        circ += [W.Gate("CZ", ((q + 1) % n,), (q,)) for q in range(0, n, 2)]
        circ += [W.Gate("S", (int(rng.integers(n)),)), W.Gate("T", (int(rng.integers(n)),))]
    s = qs.Simulator(n)
    s.set_config(qs.make_config(jit_min_qubits=jit))
    s.set_basis_state(5)
    s.apply(circ)
    psi = s.state()
    s.close()
    check(psi, n, circ, basis=5)


@pytest.mark.parametrize("wbits", [15, 18, 21])
def test_l2_blocked_runs_n24(qs, wbits):
    """Two-level blocking: runs of passes whose positions
    lie below W execute wave by wave over 2^W-amplitude blocks (2^(24-W)
    waves, each launch covering a chunk range).  QFT-24 from a basis state
    (both passes grouped) and a random circuit whose dense gates act below W
    (every pass grouped), against the oracle."""
    n = 24
    low = ([W.Gate("H", (q,)) for q in range(n)] +
           W.random_circuit(wbits, 200, 2411 + wbits, diag_bias=0.4, max_generic=2) +
           W.random_circuit(n, 40, 7, diag_bias=0.9))   # dense work below W, phases anywhere
    cases = [(W.qft(n), 0x9E3779 % (1 << n)), (low, 12345)]
    for gates, basis in cases:
        cfg = qs.make_config(l2_block_qubits=wbits)
        plan = qs.plan_json(n, gates, config=cfg, basis=basis)
        assert plan["stats"]["n_l2_groups"] >= 1
        s = qs.Simulator(n)
        s.set_config(cfg)
        s.set_basis_state(basis)
        s.apply(gates)
        psi = s.state()
        info = qs.jit_info(s)
        s.close()
        assert info["jit_errors"] == 0 and info["l2_groups"] >= 1
        check(psi, n, gates, basis=basis)


def test_accumulating_mode_back_to_back_circuits(qs):
    """qs_set_timing(2): a call returns once its launches are enqueued and the
    next call's planning overlaps them; results, device time and per-kernel
    counts are taken at the next call or query.  Three back-to-back QFT-22
    circuits from different basis states: the last state matches the oracle
    and the accumulated launch counts are three times one call's."""
    n = 22
    gates = W.qft(n)
    s = qs.Simulator(n)
    s.set_basis_state(1)
    s.apply(gates)
    s.set_timing(1)
    s.set_basis_state(2)
    s.apply(gates)
    one = {k: s.kernel_timing(k)["launches"] for k in ("K1_chunk", "K2_dense", "K3_diag")}
    s.set_timing(2)
    for x in (0x15, 0x2A5, 0x3FF0F):
        s.set_basis_state(x)
        s.apply(gates)
    acc = {k: s.kernel_timing(k)["launches"] for k in ("K1_chunk", "K2_dense", "K3_diag")}
    st = s.stats()
    psi = s.state()
    s.set_timing(0)
    s.close()
    assert acc == {k: 3 * v for k, v in one.items()}
    assert st["t_device_ms"] > 0
    check(psi, n, gates, basis=0x3FF0F)


def test_l2_runs_not_used_on_loopback_shards(qs):
    """Loopback shards share one device, so marked runs execute pass by pass
    there (two cooperative launches would compete for the same SMs)."""
    n = 24
    gates = W.qft(n)
    cfg = qs.make_config(l2_block_qubits=18)
    s = qs.Simulator(n, loopback_ranks=2)
    s.set_config(cfg)
    s.set_basis_state(77)
    s.apply(gates)
    psi = s.state()
    info = qs.jit_info(s)
    s.close()
    assert info["l2_groups"] == 0
    check(psi, n, gates, basis=77)


@pytest.mark.parametrize("jit", [0, 99])
def test_row_scaled_one_qubit_gates_special_angles(qs, jit):
    """r9b: uncontrolled RX/RY/U3 applied as lam [[1, b/lam], [c/lam, 1]] with
    lam in the pass scale -- at the angles where an entry vanishes or the
    larger entry switches (0, pi/2, pi, -pi, 3pi/2) and at random angles,
    controlled copies unscaled; both kernel paths, against the oracle."""
    rng = np.random.default_rng(909)
    n = 20
    angles = [0.0, np.pi / 2, np.pi, -np.pi, 1.5 * np.pi, 1e-9, np.pi - 1e-9]
    circ = [W.Gate("H", (q,)) for q in range(n)]
    for layer in range(4):
        for q in range(n):
            th = float(angles[(q + layer) % len(angles)]) if q % 3 else float(rng.uniform(-4, 4))
            kind = ("RX", "RY")[(q + layer) % 2]
            circ.append(W.Gate(kind, (q,), (), (th,)))
        circ.append(W.Gate("U3", (layer,), (), tuple(float(x) for x in rng.uniform(-3, 3, 3))))
        circ.append(W.Gate("RX", (layer + 5,), (layer + 9,), (float(rng.uniform(-3, 3)),)))
        circ += [W.Gate("CZ", ((q + 1) % n,), (q,)) for q in range(layer % 2, n, 2)]
    s = qs.Simulator(n)
    s.set_config(qs.make_config(jit_min_qubits=jit))
    s.set_basis_state(11)
    s.apply(circ)
    psi = s.state()
    s.close()
    check(psi, n, circ, basis=11)
