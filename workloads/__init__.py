"""Seeded synthetic circuit generators -- shared INPUT module.

This module is the only code shared by the CPU oracle (``oracle/``) and the
product path (``paper_2604_12256_b200``).  It holds none of the method's
arithmetic: it emits gate *lists* (kind name, targets, controls, angles and,
for GENERIC gates, a caller-drawn matrix).  Each side turns a kind name into a
matrix with its own independent code.

Constructions:
  qft            reading c18: for j = N-1..0: H(j); for
                 k = j-1..0: CP(pi/2^(j-k)) on (k, j); then SWAP(i, N-1-i).
  ghz            H(0), CX(i-1 -> i).
  rzz_full       PAPER.md L715 gate-level benchmark: H on every qubit, then
                 RZZ(theta_jk) on every pair j<k in lexicographic order.
  diag_chain     diagonal-heavy RZ/CZ/CP chains with one RX barrier per layer.
  qaoa_maxcut    MaxCut QAOA on a seeded random d-regular graph.
  supremacy      Google-2019-like random circuit on a rows x cols grid.
  bernstein_vazirani, hidden_shift, quantum_volume, variational,
  supremacy_n    PAPER.md Table 2 roster (BV, HS, QV, VC, SC; L777-806).
  qaoa_complete  PAPER.md Table 3 "5-level fully connected" QAOA (L715).
  random_circuit seeded mix of every supported kind (parity tests).
  fixture_f4     PAPER.md Fig. 4 (L652-682), reconstructed.
  fixture_f23    PAPER.md Fig. 2/3 (L336, L468-474), reconstructed (F23).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Gate", "qft", "ghz", "rzz_full", "diag_chain", "qaoa_maxcut",
    "random_regular_graph", "supremacy", "random_circuit", "fixture_f4",
    "fixture_f23", "haar_unitary", "random_phases", "KIND_ARITY",
    "DIAGONAL_KINDS", "splitmix64", "bernstein_vazirani", "hidden_shift",
    "quantum_volume", "variational", "supremacy_n", "qaoa_complete", "ROSTER",
]

# Number of targets per kind (None: taken from the matrix).
KIND_ARITY = {
    "H": 1, "X": 1, "Y": 1, "Z": 1, "S": 1, "SDG": 1, "T": 1, "TDG": 1,
    "RX": 1, "RY": 1, "RZ": 1, "U1": 1, "U2": 1, "U3": 1, "CX": 1, "CZ": 1,
    "CP": 1, "RZZ": 2, "SWAP": 2, "SX": 1, "SY": 1, "SW": 1,
    "UNITARY": None, "DIAGONAL": None,
}
# Kinds whose matrix is diagonal by definition (a structural fact of the
# input, used by generators and tests for labelling only).
DIAGONAL_KINDS = {"Z", "S", "SDG", "T", "TDG", "RZ", "U1", "CZ", "CP", "RZZ", "DIAGONAL"}
_NPARAMS = {"RX": 1, "RY": 1, "RZ": 1, "U1": 1, "CP": 1, "RZZ": 1, "U2": 2, "U3": 3}


@dataclass
class Gate:
    kind: str
    targets: Tuple[int, ...]
    controls: Tuple[int, ...] = ()
    params: Tuple[float, ...] = ()
    matrix: Optional[np.ndarray] = field(default=None, repr=False)

    def __post_init__(self):
        self.targets = tuple(int(q) for q in self.targets)
        self.controls = tuple(int(q) for q in self.controls)
        self.params = tuple(float(p) for p in self.params)

    @property
    def support(self) -> Tuple[int, ...]:
        return self.targets + self.controls


def splitmix64(x: int) -> int:
    """SplitMix64 step (seed -> basis-state index recipe)."""
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


# --------------------------------------------------------------------------
# Benchmark circuits
# --------------------------------------------------------------------------

def qft(n: int, swaps: bool = True) -> List[Gate]:
    """QFT, reading c18.  Gate count: n + n(n-1)/2 + floor(n/2)."""
    g: List[Gate] = []
    for j in range(n - 1, -1, -1):
        g.append(Gate("H", (j,)))
        for k in range(j - 1, -1, -1):
            g.append(Gate("CP", (j,), (k,), (math.pi / (1 << (j - k)),)))
    if swaps:
        for i in range(n // 2):
            g.append(Gate("SWAP", (i, n - 1 - i)))
    return g


def ghz(n: int) -> List[Gate]:
    g = [Gate("H", (0,))]
    for i in range(1, n):
        g.append(Gate("CX", (i,), (i - 1,)))
    return g


def rzz_full(n: int, seed: int = 1, h_layer: bool = True) -> List[Gate]:
    """RZZ with full connectivity (N(N-1)/2 gates), after an
    H layer (SURVEY 8(d) diag30 (a))."""
    rng = np.random.default_rng(seed)
    g: List[Gate] = [Gate("H", (q,)) for q in range(n)] if h_layer else []
    for j in range(n):
        for k in range(j + 1, n):
            g.append(Gate("RZZ", (j, k), (), (float(rng.uniform(0, 2 * math.pi)),)))
    return g


def diag_chain(n: int, seed: int = 1, layers: int = 8) -> List[Gate]:
    """SURVEY 8(d) diag30 (b): H^n, then per layer: RZ on all q; CZ(q, q+1);
    CP(q, (q+3) mod n); one RX on qubit 7l mod n (a detector barrier)."""
    rng = np.random.default_rng(seed)
    g: List[Gate] = [Gate("H", (q,)) for q in range(n)]
    for l in range(layers):
        for q in range(n):
            g.append(Gate("RZ", (q,), (), (float(rng.uniform(0, 2 * math.pi)),)))
        for q in range(n - 1):
            g.append(Gate("CZ", (q + 1,), (q,)))
        for q in range(n):
            p = (q + 3) % n
            if p == q:
                continue
            g.append(Gate("CP", (p,), (q,), (float(rng.uniform(0, 2 * math.pi)),)))
        g.append(Gate("RX", ((7 * l) % n,), (), (float(rng.uniform(0, 2 * math.pi)),)))
    return g


def random_regular_graph(n: int, d: int, seed: int) -> List[Tuple[int, int]]:
    """Pairing model with rejection (no loops, no multi-edges); edges sorted."""
    if (n * d) % 2:
        raise ValueError("n*d must be even")
    rng = np.random.default_rng(seed)
    while True:
        stubs = np.repeat(np.arange(n), d)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        edges = set()
        ok = True
        for a, b in pairs:
            a, b = int(a), int(b)
            if a == b:
                ok = False
                break
            e = (min(a, b), max(a, b))
            if e in edges:
                ok = False
                break
            edges.add(e)
        if ok:
            return sorted(edges)


def qaoa_maxcut(n: int, p: int = 4, seed: int = 1, degree: int = 3) -> List[Gate]:
    """MaxCut QAOA (SURVEY 8(d) qaoa32): H^n, then per layer l: RZZ(gamma_l)
    on each edge and RX(2 beta_l) on each qubit; gamma ~ U[0, pi),
    beta ~ U[0, pi/2)."""
    edges = random_regular_graph(n, degree, seed)
    rng = np.random.default_rng(seed + 7919)
    g: List[Gate] = [Gate("H", (q,)) for q in range(n)]
    for _ in range(p):
        gamma = float(rng.uniform(0, math.pi))
        beta = float(rng.uniform(0, math.pi / 2))
        for a, b in edges:
            g.append(Gate("RZZ", (a, b), (), (gamma,)))
        for q in range(n):
            g.append(Gate("RX", (q,), (), (2 * beta,)))
    return g


def haar_unitary(dim: int, rng: np.random.Generator) -> np.ndarray:
    """QR of a complex Gaussian matrix with the phase fix (Mezzadri)."""
    z = (rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))) / math.sqrt(2)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))


def random_phases(dim: int, rng: np.random.Generator) -> np.ndarray:
    return np.exp(1j * rng.uniform(0, 2 * math.pi, size=dim))


def supremacy(rows: int = 5, cols: int = 7, depth: int = 20, seed: int = 1,
              dense: bool = False) -> List[Gate]:
    """SURVEY 8(d) rand35: qubit q = cols*row + col.  Each cycle: one of
    {SX, SY, SW} on every qubit (never the previous one for that qubit), then
    CZ (or a seeded Haar 4x4 when ``dense``) on the couplers of pattern
    A B C D C D A B ...; a final layer of 1-qubit gates."""
    rng = np.random.default_rng(seed)
    n = rows * cols
    q = lambda r, c: cols * r + c
    pats = {
        "A": [(q(r, c), q(r, c + 1)) for r in range(rows) for c in range(0, cols - 1, 2)],
        "B": [(q(r, c), q(r, c + 1)) for r in range(rows) for c in range(1, cols - 1, 2)],
        "C": [(q(r, c), q(r + 1, c)) for r in range(0, rows - 1, 2) for c in range(cols)],
        "D": [(q(r, c), q(r + 1, c)) for r in range(1, rows - 1, 2) for c in range(cols)],
    }
    order = "ABCDCDAB"
    prev = [None] * n
    g: List[Gate] = []

    def one_qubit_layer():
        for i in range(n):
            choices = [k for k in ("SX", "SY", "SW") if k != prev[i]]
            k = choices[int(rng.integers(len(choices)))]
            prev[i] = k
            g.append(Gate(k, (i,)))

    for cyc in range(depth):
        one_qubit_layer()
        for a, b in pats[order[cyc % len(order)]]:
            if dense:
                g.append(Gate("UNITARY", (a, b), (), (), haar_unitary(4, rng)))
            else:
                g.append(Gate("CZ", (b,), (a,)))
    one_qubit_layer()
    return g


# --------------------------------------------------------------------------
# PAPER.md Table 2 roster (L777-806; "benchmark circuits drawn from various
# application domains", cited to the qibojit benchmark suite).  The paper
# gives names only; the constructions below are the textbook circuits in the
# shape that suite uses (reading r6).
# --------------------------------------------------------------------------

def bernstein_vazirani(n: int, seed: int = 1) -> List[Gate]:
    """BV: n-1 data qubits + ancilla n-1.  X(anc), H on all, CX(i -> anc)
    for every set bit of a seeded secret, H on the data qubits."""
    rng = np.random.default_rng(seed)
    secret = [int(b) for b in rng.integers(0, 2, size=n - 1)]
    anc = n - 1
    g: List[Gate] = [Gate("X", (anc,))] + [Gate("H", (q,)) for q in range(n)]
    g += [Gate("CX", (anc,), (i,)) for i in range(n - 1) if secret[i]]
    g += [Gate("H", (q,)) for q in range(n - 1)]
    return g


def hidden_shift(n: int, seed: int = 1) -> List[Gate]:
    """HS (bent-function hidden shift, n even): H all; X on the shift's set
    bits; CZ(2i, 2i+1); X on the shift; H all; CZ(2i, 2i+1); H all."""
    assert n % 2 == 0, "hidden shift needs an even qubit count"
    rng = np.random.default_rng(seed)
    shift = [int(b) for b in rng.integers(0, 2, size=n)]
    H = [Gate("H", (q,)) for q in range(n)]
    X = [Gate("X", (q,)) for q in range(n) if shift[q]]
    CZ = [Gate("CZ", (2 * i + 1,), (2 * i,)) for i in range(n // 2)]
    return H + X + CZ + X + H + list(CZ) + H


def quantum_volume(n: int, depth: Optional[int] = None, seed: int = 1) -> List[Gate]:
    """QV: `depth` (default n) layers; each pairs the qubits of a seeded
    random permutation and applies a Haar-random 4x4 unitary per pair."""
    rng = np.random.default_rng(seed)
    g: List[Gate] = []
    for _ in range(depth if depth is not None else n):
        perm = [int(q) for q in rng.permutation(n)]
        for i in range(0, n - 1, 2):
            a, b = perm[i], perm[i + 1]
            g.append(Gate("UNITARY", (a, b), (), (), haar_unitary(4, rng)))
    return g


def variational(n: int, layers: int = 5, seed: int = 1) -> List[Gate]:
    """VC (hardware-efficient ansatz): per layer RY(theta) on every qubit,
    CZ on the even pairs (0,1),(2,3)..., RY on every qubit, CZ on the odd
    pairs (1,2),(3,4)...; a final RY layer.  theta ~ U[0, 2 pi)."""
    rng = np.random.default_rng(seed)
    ry = lambda: [Gate("RY", (q,), (), (float(rng.uniform(0, 2 * math.pi)),)) for q in range(n)]
    g: List[Gate] = []
    for _ in range(layers):
        g += ry() + [Gate("CZ", (q + 1,), (q,)) for q in range(0, n - 1, 2)]
        g += ry() + [Gate("CZ", (q + 1,), (q,)) for q in range(1, n - 1, 2)]
    return g + ry()


def supremacy_n(n: int, depth: int = 20, seed: int = 1) -> List[Gate]:
    """SC on n qubits: the `supremacy` construction on the smallest grid of
    width ceil(sqrt(n)) holding n qubits, couplers to absent sites dropped."""
    cols = int(math.ceil(math.sqrt(n)))
    rows = (n + cols - 1) // cols
    full = supremacy(rows, cols, depth, seed)
    return [x for x in full if max(x.support) < n]


def qaoa_complete(n: int, p: int = 5, seed: int = 1) -> List[Gate]:
    """PAPER.md L715/L811-858 Table 3 workload: "5-level fully connected"
    QAOA -- H^n, then per level RZZ(gamma) on every pair j<k and RX(2 beta)
    on every qubit."""
    rng = np.random.default_rng(seed + 104729)
    g: List[Gate] = [Gate("H", (q,)) for q in range(n)]
    for _ in range(p):
        gamma = float(rng.uniform(0, math.pi))
        beta = float(rng.uniform(0, math.pi / 2))
        g += [Gate("RZZ", (a, b), (), (gamma,)) for a in range(n) for b in range(a + 1, n)]
        g += [Gate("RX", (q,), (), (2 * beta,)) for q in range(n)]
    return g


ROSTER = {
    "bv": bernstein_vazirani, "hs": hidden_shift, "qaoa": lambda n: qaoa_maxcut(n, 4, 1, 3 if n % 2 == 0 else 4),
    "qft": qft, "qv": quantum_volume, "sc": supremacy_n, "vc": variational,
}


# --------------------------------------------------------------------------
# Test circuits
# --------------------------------------------------------------------------

ALL_KINDS = ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "U1",
             "U2", "U3", "CX", "CZ", "CP", "RZZ", "SWAP", "SX", "SY", "SW",
             "UNITARY", "DIAGONAL"]


def random_circuit(n: int, n_gates: int, seed: int, kinds: Sequence[str] = ALL_KINDS,
                   max_controls: int = 2, max_generic: int = 3,
                   diag_bias: float = 0.0) -> List[Gate]:
    """Seeded mix over ``kinds``; random extra controls on any kind; generic
    unitaries/diagonals on up to ``max_generic`` targets (Haar / random
    phases).  ``diag_bias`` in [0,1) raises the share of diagonal kinds."""
    rng = np.random.default_rng(seed)
    kinds = list(kinds)
    diag = [k for k in kinds if k in DIAGONAL_KINDS]
    g: List[Gate] = []
    for _ in range(n_gates):
        if diag and rng.uniform() < diag_bias:
            kind = diag[int(rng.integers(len(diag)))]
        else:
            kind = kinds[int(rng.integers(len(kinds)))]
        arity = KIND_ARITY[kind]
        if arity is None:
            arity = int(rng.integers(1, min(max_generic, n) + 1))
        if arity > n:
            continue
        base_ctrl = 1 if kind in ("CX", "CZ", "CP") else 0
        nc_max = min(max_controls, n - arity)
        if base_ctrl > nc_max:
            continue
        nc = int(rng.integers(base_ctrl, nc_max + 1)) if nc_max > base_ctrl else base_ctrl
        qs = rng.permutation(n)[: arity + nc]
        targets = tuple(int(x) for x in qs[:arity])
        controls = tuple(int(x) for x in qs[arity:])
        params = tuple(float(x) for x in rng.uniform(0, 2 * math.pi, size=_NPARAMS.get(kind, 0)))
        matrix = None
        if kind == "UNITARY":
            matrix = haar_unitary(1 << arity, rng)
        elif kind == "DIAGONAL":
            matrix = random_phases(1 << arity, rng)
        g.append(Gate(kind, targets, controls, params, matrix))
    return g


def fixture_f4() -> List[Gate]:
    """PAPER.md Fig. 4 (L652-682) as reconstructed in SURVEY 8(c) F4.
    Gate i (1-based) of the paper's labelling is element i-1."""
    a = [0.3, 0.5, 0.7, 1.1, 1.3, 1.7, 1.9, 2.3, 2.9, 3.1, 0.2]
    return [
        Gate("H", (0,)),                       # 1  H
        Gate("RZZ", (0, 1), (), (a[1],)),      # 2  RZZ
        Gate("H", (2,)),                       # 3  H
        Gate("RY", (3,), (), (a[3],)),         # 4  RY
        Gate("RZZ", (1, 2), (), (a[4],)),      # 5  RZZ
        Gate("CP", (3,), (2,), (a[5],)),       # 6  CP
        Gate("RX", (0,), (), (a[6],)),         # 7  RX  (barrier)
        Gate("RZZ", (1, 3), (), (a[7],)),      # 8  RZZ
        Gate("CP", (3,), (2,), (a[8],)),       # 9  CP
        Gate("RY", (0,), (), (a[9],)),         # 10 RY
        Gate("RZZ", (0, 4), (), (a[10],)),     # 11 RZZ (stopped)
    ]


def fixture_f23() -> List[Gate]:
    """PAPER.md Fig. 2/3 (L336, L468-474): 8 qubits, 40 gates = 26 single +
    14 controlled, reconstructed in SURVEY 8(c) F23."""
    th = iter(np.linspace(0.25, 2.75, 40))
    t = lambda: (float(next(th)),)
    CX = lambda c, x: Gate("CX", (x,), (c,))
    CZ = lambda a, b: Gate("CZ", (b,), (a,))
    CP = lambda a, b: Gate("CP", (b,), (a,), t())
    H = lambda q: Gate("H", (q,))
    RX = lambda q: Gate("RX", (q,), (), t())
    RY = lambda q: Gate("RY", (q,), (), t())
    RZ = lambda q: Gate("RZ", (q,), (), t())
    return [
        # round 1, group {0,1}
        H(0), H(1), CX(0, 1), RZ(0), RX(1), CZ(0, 1),
        # group {2,3}
        H(2), RY(3), CX(2, 3), RZ(2), H(3), CP(2, 3),
        # group {4,5}
        H(4), H(5), CX(4, 5), RX(4), RZ(5), CX(5, 4), RY(5),
        # group {6,7}
        RY(6), H(7), CX(6, 7), RZ(6), RX(7), CZ(6, 7), H(6),
        # round 2, {0..3}
        CX(1, 2), RZ(1), H(2), CX(0, 3), RX(0), CP(1, 3), RY(3),
        # round 2, {4..7}
        CX(5, 6), H(5), RY(6), RZ(6),
        # round 3
        CX(3, 4), CX(0, 7), RX(4),
    ]
