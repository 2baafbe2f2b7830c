"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A plain gate-by-gate state-vector simulator (Alg. 1, with
Eq. 2/3 generalised to t targets and c controls), written in C
(``oracle/oracle.c``) and loaded here with ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2604_12256_b200``) never imports it and shares no code
with it; the only shared module is ``workloads`` (seeded input generators,
which hold none of the method's arithmetic).

Parity pins for this oracle live in ``tests/test_oracle.py`` (-m "not gpu").
Every function here is pinned; see DESIGN.md "Oracle and its pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MAX_T = 10

# Oracle's own kind numbering (mirrors the enum in oracle.c, not the product's).
KINDS = {
    "H": 0, "X": 1, "Y": 2, "Z": 3, "S": 4, "T": 5, "RX": 6, "RY": 7,
    "RZ": 8, "U1": 9, "U2": 10, "U3": 11, "CX": 12, "CZ": 13, "CP": 14,
    "RZZ": 15, "SWAP": 16, "SX": 17, "SY": 18, "SW": 19, "UNITARY": 20,
    "DIAGONAL": 21, "SDG": 22, "TDG": 23,
}


class _Gate(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("t", ctypes.c_int32), ("nc", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("targets", ctypes.c_int32 * MAX_T), ("controls", ctypes.c_int32 * MAX_T),
        ("params", ctypes.c_double * 3), ("matrix", ctypes.c_void_p),
    ]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -fopenmp).  Building the checker is not
    using it; __graft_entry__.build() calls this."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fcx-limited-range", "-fopenmp", "-fPIC", "-shared", "-std=gnu11",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_apply_circuit.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                             ctypes.POINTER(_Gate), ctypes.c_int64]
        lib.oracle_apply_circuit.restype = ctypes.c_int
        lib.oracle_gate_matrix.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_gate_matrix.restype = ctypes.c_int
        lib.oracle_basis_state.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(k: int) -> None:
    """OpenMP thread count of the oracle's loop (libgomp's process-wide
    setting; the CPU-baseline single-thread leg)."""
    _load()
    ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(k))


def _marshal(gates):
    arr = (_Gate * max(1, len(gates)))()
    keep = []
    for i, g in enumerate(gates):
        rec = arr[i]
        rec.kind = KINDS[g.kind]
        rec.t = len(g.targets)
        rec.nc = len(g.controls)
        if rec.t > MAX_T or rec.nc > MAX_T:
            raise ValueError("oracle supports at most %d targets/controls" % MAX_T)
        for j, q in enumerate(g.targets):
            rec.targets[j] = q
        for j, q in enumerate(g.controls):
            rec.controls[j] = q
        for j, p in enumerate(g.params[:3]):
            rec.params[j] = p
        if g.matrix is not None:
            m = np.ascontiguousarray(np.asarray(g.matrix, dtype=np.complex128))
            keep.append(m)
            rec.matrix = m.ctypes.data
        else:
            rec.matrix = None
    return arr, keep


def gate_matrix(kind: str, n_targets: int, params=(), matrix=None) -> np.ndarray:
    """The oracle's 2^t x 2^t matrix for a gate kind (reading c3)."""
    lib = _load()
    dim = 1 << n_targets
    out = np.zeros((dim, dim), dtype=np.complex128)
    p = np.zeros(3, dtype=np.float64)
    p[:len(params)] = params
    user = None
    if matrix is not None:
        user = np.ascontiguousarray(np.asarray(matrix, dtype=np.complex128))
    rc = lib.oracle_gate_matrix(KINDS[kind], n_targets, p.ctypes.data,
                                None if user is None else user.ctypes.data,
                                out.ctypes.data)
    if rc != 0:
        raise ValueError("bad gate %s/%d" % (kind, n_targets))
    return out


def basis_state(n: int, x: int = 0) -> np.ndarray:
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[x] = 1.0
    return psi


def apply_circuit(n: int, gates, state: np.ndarray | None = None, x: int = 0,
                  inplace: bool = False) -> np.ndarray:
    """Alg. 1 over ``gates`` starting from ``state`` (copied, or updated in
    place with ``inplace=True`` -- large states) or |x>."""
    lib = _load()
    if state is None:
        psi = basis_state(n, x)
    elif inplace:
        psi = state
        assert psi.dtype == np.complex128 and psi.shape == (1 << n,) and psi.flags.c_contiguous
    else:
        psi = np.array(state, dtype=np.complex128, copy=True)
        assert psi.shape == (1 << n,)
    arr, keep = _marshal(gates)
    rc = lib.oracle_apply_circuit(psi.ctypes.data, n, arr, len(gates))
    if rc != 0:
        raise ValueError("oracle rejected gate %d" % (-rc - 1))
    return psi
