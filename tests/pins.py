"""Independent mathematical constructions used to PIN the oracle.

Nothing here is the oracle's formula retyped: each helper reaches the same
object by a different route (Kronecker products from PAPER.md L125, numpy
tensor contraction over a [2]*N tensor, matrix exponentials of Pauli
generators, closed forms).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.linalg import expm

# Pauli algebra: defined by their action on the computational basis.
I2 = np.eye(2, dtype=np.complex128)
PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
PZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)
PY = 1j * PX @ PZ  # Y = i X Z


def kron_all(*ms):
    out = np.eye(1, dtype=np.complex128)
    for m in ms:
        out = np.kron(out, m)
    return out


def paper_single_qubit_operator(n: int, j: int, u: np.ndarray) -> np.ndarray:
    """U_j = I^{(x) N-j-1} (x) U (x) I^{(x) j}."""
    return kron_all(np.eye(1 << (n - j - 1)), u, np.eye(1 << j))


def paper_adjacent_two_qubit_operator(n: int, k: int, v: np.ndarray) -> np.ndarray:
    """Eq. 3 for adjacent j = k+1: rows ordered
    0_j0_k, 0_j1_k, 1_j0_k, 1_j1_k, i.e. I (x) V (x) I."""
    return kron_all(np.eye(1 << (n - k - 2)), v, np.eye(1 << k))


def tensor_apply(psi: np.ndarray, n: int, u: np.ndarray, targets, controls=()) -> np.ndarray:
    """Apply u (matrix index bit i <-> targets[i]) by contracting a [2]*n
    tensor (axis a <-> qubit n-1-a), restricted to the slice where every
    control axis is 1."""
    t = len(targets)
    psi_t = psi.reshape([2] * n).copy()
    ax = lambda q: n - 1 - q
    # u as tensor: out bits (t-1..0), in bits (t-1..0) -- matrix index is
    # big-endian over reversed targets.
    ut = u.reshape([2] * (2 * t))
    # axes of ut: [out_{t-1},...,out_0, in_{t-1},...,in_0]
    sl = [slice(None)] * n
    for c in controls:
        sl[ax(c)] = 1
    sub = psi_t[tuple(sl)]
    # axes in sub: remaining axes in order (controls removed)
    remaining = [a for a in range(n) if a not in {ax(c) for c in controls}]
    pos = {a: i for i, a in enumerate(remaining)}
    in_axes = [pos[ax(targets[i])] for i in range(t - 1, -1, -1)]
    res = np.tensordot(ut, sub, axes=(list(range(t, 2 * t)), in_axes))
    # res axes: out_{t-1..0} then the remaining non-target axes of sub in order
    rest = [i for i in range(sub.ndim) if i not in in_axes]
    # res axis k<t is the output for in_axes[k]; the others follow in order.
    res = np.moveaxis(res, list(range(sub.ndim)), in_axes + rest)
    psi_t[tuple(sl)] = res
    return psi_t.reshape(-1)


def full_operator(n: int, u: np.ndarray, targets, controls=()) -> np.ndarray:
    """2^n x 2^n operator by applying tensor_apply to every basis vector."""
    dim = 1 << n
    m = np.zeros((dim, dim), dtype=np.complex128)
    for b in range(dim):
        e = np.zeros(dim, dtype=np.complex128)
        e[b] = 1
        m[:, b] = tensor_apply(e, n, u, targets, controls)
    return m


def rx(th):
    return expm(-1j * th / 2 * PX)


def ry(th):
    return expm(-1j * th / 2 * PY)


def rz(th):
    return expm(-1j * th / 2 * PZ)


def qft_closed_form(n: int, x: int) -> np.ndarray:
    """QFT|x> = 2^{-N/2} sum_k e^{2 pi i x k / 2^N} |k>  (reading c18);
    x*k reduced mod 2^N exactly in integers before the fp64 angle."""
    k = np.arange(1 << n, dtype=np.int64)
    ph = (x * k) % (1 << n)
    return np.exp(2j * math.pi * ph / (1 << n)) / math.sqrt(1 << n)


def ghz_closed_form(n: int) -> np.ndarray:
    v = np.zeros(1 << n, dtype=np.complex128)
    v[0] = v[-1] = 1 / math.sqrt(2)
    return v


def random_state(n: int, rng: np.random.Generator) -> np.ndarray:
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)
