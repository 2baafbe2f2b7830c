"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: the paper's
Kronecker formula (Eq. 3), a tensor-contraction
application, matrix exponentials of Pauli generators, algebraic identities,
QFT / GHZ closed forms, SPEC.md worked examples and norm
preservation.  A dropped term, wrong sign, wrong index order or transposed
operand in oracle.c fails at least one of them.
"""
import math

import numpy as np
import pytest
from scipy.linalg import expm

import oracle
import workloads as W
from tests import pins

RNG = np.random.default_rng(12345)


def M(kind, t=1, params=(), matrix=None):
    return oracle.gate_matrix(kind, t, params, matrix)


# --------------------------------------------------------------------------
# Gate table (reading c3), pinned by identities / exponentials
# --------------------------------------------------------------------------

def test_pauli_algebra():
    X, Y, Z = M("X"), M("Y"), M("Z")
    I = np.eye(2)
    for P in (X, Y, Z):
        assert np.allclose(P @ P, I)
    assert np.allclose(X @ Y, 1j * Z)
    assert np.allclose(Y @ Z, 1j * X)
    # Z|0> = |0>, X|0> = |1> fixes the basis convention
    assert np.allclose(Z @ [1, 0], [1, 0])
    assert np.allclose(X @ [1, 0], [0, 1])
    assert np.allclose(Y, pins.PY)


def test_clifford_t_relations():
    H, S, T, Z, X = M("H"), M("S"), M("T"), M("Z"), M("X")
    assert np.allclose(H, (X + Z) / math.sqrt(2))
    assert np.allclose(H @ H, np.eye(2))
    assert np.allclose(S @ S, Z)
    assert np.allclose(T @ T, S)
    assert np.allclose(M("SDG"), S.conj().T)
    assert np.allclose(M("TDG"), T.conj().T)
    assert np.allclose(H @ X @ H, Z)


@pytest.mark.parametrize("th", [0.0, 0.3, 1.7, math.pi, 5.9])
def test_rotations_are_pauli_exponentials(th):
    assert np.allclose(M("RX", 1, (th,)), expm(-1j * th / 2 * pins.PX), atol=1e-14)
    assert np.allclose(M("RY", 1, (th,)), expm(-1j * th / 2 * pins.PY), atol=1e-14)
    assert np.allclose(M("RZ", 1, (th,)), expm(-1j * th / 2 * pins.PZ), atol=1e-14)
    # U1(l) = e^{i l/2} RZ(l); CP is U1 with a control
    assert np.allclose(M("U1", 1, (th,)), np.exp(1j * th / 2) * pins.rz(th), atol=1e-14)
    assert np.allclose(M("CP", 1, (th,)), M("U1", 1, (th,)))
    # RZZ(th) = exp(-i th/2 Z(x)Z)
    assert np.allclose(M("RZZ", 2, (th,)), expm(-1j * th / 2 * np.kron(pins.PZ, pins.PZ)), atol=1e-14)


@pytest.mark.parametrize("seed", range(5))
def test_u2_u3_euler(seed):
    rng = np.random.default_rng(seed)
    th, ph, la = rng.uniform(0, 2 * math.pi, 3)
    u3 = np.exp(1j * (ph + la) / 2) * pins.rz(ph) @ pins.ry(th) @ pins.rz(la)
    assert np.allclose(M("U3", 1, (th, ph, la)), u3, atol=1e-14)
    assert np.allclose(M("U2", 1, (ph, la)), M("U3", 1, (math.pi / 2, ph, la)), atol=1e-14)


def test_sqrt_gates():
    W_ = (pins.PX + pins.PY) / math.sqrt(2)
    for kind, P in (("SX", pins.PX), ("SY", pins.PY), ("SW", W_)):
        R = M(kind)
        assert np.allclose(R @ R, P, atol=1e-15)
        assert np.allclose(R @ R.conj().T, np.eye(2), atol=1e-15)
        # branch: e^{i pi/4} exp(-i pi/4 P)
        assert np.allclose(R, np.exp(1j * math.pi / 4) * expm(-1j * math.pi / 4 * P), atol=1e-15)


def test_swap_and_cx_cz():
    S = M("SWAP", 2)
    XX, YY, ZZ = (np.kron(P, P) for P in (pins.PX, pins.PY, pins.PZ))
    assert np.allclose(S, (np.eye(4) + XX + YY + ZZ) / 2)
    assert np.allclose(M("CX"), M("X"))
    assert np.allclose(M("CZ"), M("Z"))


def test_generic_passthrough():
    u = W.haar_unitary(8, RNG)
    assert np.allclose(M("UNITARY", 3, (), u), u)
    d = W.random_phases(4, RNG)
    assert np.allclose(M("DIAGONAL", 2, (), d), np.diag(d))


# --------------------------------------------------------------------------
# Index semantics: Eq. 2 / Eq. 3 and the generalisation, by brute force
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 5, 6])
def test_single_qubit_matches_paper_kron(n):
    for j in range(n):
        u = W.haar_unitary(2, RNG)
        psi = pins.random_state(n, RNG)
        got = oracle.apply_circuit(n, [W.Gate("UNITARY", (j,), (), (), u)], state=psi)
        want = pins.paper_single_qubit_operator(n, j, u) @ psi
        assert np.allclose(got, want, atol=1e-14)


@pytest.mark.parametrize("n", [2, 4, 6])
def test_two_qubit_matches_eq3_row_order(n):
    for k in range(n - 1):
        v = W.haar_unitary(4, RNG)
        psi = pins.random_state(n, RNG)
        got = oracle.apply_circuit(n, [W.Gate("UNITARY", (k, k + 1), (), (), v)], state=psi)
        want = pins.paper_adjacent_two_qubit_operator(n, k, v) @ psi
        assert np.allclose(got, want, atol=1e-14)


@pytest.mark.parametrize("seed", range(30))
def test_random_gate_matches_full_operator(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 7))
    (g,) = W.random_circuit(n, 1, seed=seed + 77, max_controls=2) or [W.Gate("H", (0,))]
    u = oracle.gate_matrix(g.kind, len(g.targets), g.params, g.matrix)
    full = pins.full_operator(n, u, g.targets, g.controls)
    assert np.allclose(full @ full.conj().T, np.eye(1 << n), atol=1e-12)
    psi = pins.random_state(n, rng)
    got = oracle.apply_circuit(n, [g], state=psi)
    assert np.allclose(got, full @ psi, atol=1e-13)


@pytest.mark.parametrize("seed", range(6))
def test_random_circuit_matches_tensor_contraction(seed):
    n = 7
    gates = W.random_circuit(n, 60, seed=seed)
    psi = pins.random_state(n, np.random.default_rng(seed))
    want = psi.copy()
    for g in gates:
        u = oracle.gate_matrix(g.kind, len(g.targets), g.params, g.matrix)
        want = pins.tensor_apply(want, n, u, g.targets, g.controls)
    got = oracle.apply_circuit(n, gates, state=psi)
    assert np.allclose(got, want, atol=1e-12)
    assert abs(np.linalg.norm(got) - 1) < 1e-12


# --------------------------------------------------------------------------
# Closed forms
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n,x", [(3, 5), (5, 0), (6, 37), (8, 201), (10, 0), (10, 777), (12, 4001)])
def test_qft_closed_form(n, x):
    got = oracle.apply_circuit(n, W.qft(n), x=x)
    assert np.max(np.abs(got - pins.qft_closed_form(n, x))) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 5, 11])
def test_ghz_closed_form(n):
    got = oracle.apply_circuit(n, W.ghz(n))
    assert np.max(np.abs(got - pins.ghz_closed_form(n))) < 1e-15


def test_norm_preserved_large_random():
    n = 14
    gates = W.random_circuit(n, 200, seed=5)
    got = oracle.apply_circuit(n, gates, x=123)
    assert abs(np.linalg.norm(got) - 1) < 1e-12


# --------------------------------------------------------------------------
# SPEC.md worked examples
# --------------------------------------------------------------------------

def test_spec_examples():
    r = 1 / math.sqrt(2)
    assert np.allclose(oracle.apply_circuit(2, [W.Gate("H", (0,))]), [r, r, 0, 0])
    th = 0.77
    psi = oracle.apply_circuit(2, [W.Gate("CP", (0,), (1,), (th,))], x=3)
    assert np.allclose(psi, [0, 0, 0, np.exp(1j * th)])
    uni = np.full(4, 0.5, dtype=complex)
    assert np.allclose(oracle.apply_circuit(2, [W.Gate("Z", (1,))], state=uni), [.5, .5, -.5, -.5])
    d = np.array([1, 1j, 1j, -1])
    assert np.allclose(oracle.apply_circuit(2, [W.Gate("DIAGONAL", (0, 1), (), (), d)], x=2),
                       [0, 0, 1j, 0])
    assert np.allclose(oracle.apply_circuit(2, [W.Gate("SWAP", (0, 1))], x=1), [0, 0, 1, 0])
    assert np.allclose(oracle.apply_circuit(2, [W.Gate("H", (0,)), W.Gate("CX", (1,), (0,))]),
                       [r, 0, 0, r])


def test_rejects_bad_gates():
    with pytest.raises(ValueError):
        oracle.apply_circuit(2, [W.Gate("H", (2,))])
    with pytest.raises(ValueError):
        oracle.apply_circuit(3, [W.Gate("CX", (1,), (1,))])


def test_generator_counts():
    # SPEC.md L451-453 and SURVEY 8(a) a1 gate counts
    assert len(W.qft(3)) == 7 and len(W.qft(10)) == 60 and len(W.qft(30)) == 480
    assert len(W.rzz_full(8, h_layer=False)) == 28
    assert len(W.diag_chain(30)) == 750
    assert len(W.qaoa_maxcut(32, 4, 1)) == 352
    f23 = W.fixture_f23()
    assert len(f23) == 40 and sum(1 for g in f23 if g.controls) == 14
