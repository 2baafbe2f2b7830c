"""B200-native state-vector hot path of arxiv 2604.12256.

Thin ctypes binding of ``include/qs.h`` (argument marshalling only: every step
of the path runs in ``libqs.so``'s CUDA kernels / NCCL).  The binding fails
loudly if the library cannot be loaded; there is no CPU fallback.

    import paper_2604_12256_b200 as qs
    sim = qs.Simulator(n_qubits=20)          # qs_create
    sim.apply(gates)                         # qs_apply_circuit
    psi = sim.state()                        # qs_get_state

Gate lists are sequences of objects with ``kind`` (name), ``targets``,
``controls``, ``params`` and ``matrix`` attributes (e.g. ``workloads.Gate``).
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqs.so")

QS_OK, QS_EINVAL, QS_ENOMEM, QS_ECUDA, QS_ENCCL, QS_EPOISONED, QS_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
QS_OPT_BLOCK, QS_OPT_FUSE, QS_OPT_DIAG, QS_OPT_BOOST, QS_OPT_ALL = 1, 2, 4, 8, 15
MAX_TARGETS = 6
MAX_CONTROLS = 6

# qs_kind (include/qs.h)
KINDS = {
    "H": 0, "X": 1, "Y": 2, "Z": 3, "S": 4, "SDG": 5, "T": 6, "TDG": 7,
    "RX": 8, "RY": 9, "RZ": 10, "U1": 11, "U2": 12, "U3": 13,
    "CX": 14, "CZ": 15, "CP": 16, "RZZ": 17, "SWAP": 18,
    "SX": 19, "SY": 20, "SW": 21, "UNITARY": 22, "DIAGONAL": 23,
}
KERNELS = {"K1_chunk": 0, "K2_dense": 1, "K3_diag": 2, "small": 3, "K5_expand": 4,
           "K5_merge": 5, "init": 6, "K4_swap": 7, "K6_read": 8, "substate": 9,
           "fused_swap_pass": 10, "pull_pass": 11, "l2_group": 12}


class QSError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("qs error %d: %s" % (code, msg))
        self.code = code


class qs_gate_t(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("n_targets", ctypes.c_int32),
        ("targets", ctypes.c_int32 * MAX_TARGETS), ("n_controls", ctypes.c_int32),
        ("controls", ctypes.c_int32 * MAX_CONTROLS), ("params", ctypes.c_double * 3),
        ("matrix", ctypes.c_void_p),
    ]


class qs_config_t(ctypes.Structure):
    _fields_ = [("chunk_qubits", ctypes.c_int32), ("fuse_cap", ctypes.c_int32),
                ("diag_cap", ctypes.c_int32), ("boost_div", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("jit_min_qubits", ctypes.c_int32),
                ("l2_block_qubits", ctypes.c_int32)]


class qs_stats_t(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in (
        "n_gates_in", "n_passes", "n_chunk_passes", "n_dense_passes", "n_diag_passes",
        "n_small_passes", "n_expand", "n_swaps", "n_substate_gates", "n_fused_diag",
        "bytes_hbm", "bytes_nvlink", "paper_updates", "naive_updates")] + [
        ("t_plan_ms", ctypes.c_double), ("t_device_ms", ctypes.c_double),
        ("t_swap_ms", ctypes.c_double), ("n_fused_swaps", ctypes.c_uint64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libqs.so (raises if missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libqs.so not built (run __graft_entry__.build() or "
                          "python paper_2604_12256_b200/build.py)")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.c_void_p
    sig = {
        "qs_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]),
        "qs_create_loopback": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]),
        "qs_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
        "qs_create_rank": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_char_p, ctypes.POINTER(P)]),
        "qs_destroy": (None, [P]),
        "qs_set_config": (ctypes.c_int, [P, ctypes.POINTER(qs_config_t)]),
        "qs_get_config": (ctypes.c_int, [P, ctypes.POINTER(qs_config_t)]),
        "qs_default_config": (None, [ctypes.POINTER(qs_config_t)]),
        "qs_set_basis_state": (ctypes.c_int, [P, ctypes.c_uint64]),
        "qs_apply_circuit": (ctypes.c_int, [P, ctypes.POINTER(qs_gate_t), ctypes.c_size_t]),
        "qs_get_state": (ctypes.c_int, [P, P, ctypes.c_uint64, ctypes.c_uint64]),
        "qs_probabilities": (ctypes.c_int, [P, P, ctypes.c_uint64, ctypes.c_uint64]),
        "qs_get_stats": (ctypes.c_int, [P, ctypes.POINTER(qs_stats_t)]),
        "qs_last_error": (ctypes.c_char_p, [P]),
        "qs_plan_json": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(qs_config_t),
                                          ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(qs_gate_t),
                                          ctypes.c_size_t, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]),
        "qs_divider": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
        "qs_last_launches": (ctypes.c_uint64, [P]),
        "qs_set_timing": (ctypes.c_int, [P, ctypes.c_int]),
        "qs_get_stream": (ctypes.c_void_p, [P, ctypes.c_int]),
        "qs_jit_info": (ctypes.c_int64, [P, ctypes.c_char_p, ctypes.c_size_t]),
        "qs_get_kernel_timing": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                                ctypes.POINTER(ctypes.c_double),
                                                ctypes.POINTER(ctypes.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


EXPORTED_SYMBOLS = [
    "qs_create", "qs_create_loopback", "qs_nccl_unique_id", "qs_create_rank", "qs_destroy",
    "qs_set_config", "qs_get_config", "qs_default_config", "qs_set_basis_state",
    "qs_apply_circuit", "qs_get_state", "qs_probabilities", "qs_get_stats", "qs_last_error",
    "qs_plan_json", "qs_divider", "qs_last_launches", "qs_set_timing", "qs_get_kernel_timing",
    "qs_get_stream", "qs_jit_info",
]


def jit_info(sim=None) -> dict:
    buf = ctypes.create_string_buffer(1024)
    load_library().qs_jit_info(sim.h if sim is not None else None, buf, 1024)
    return json.loads(buf.value.decode())


_GATE_DTYPE = np.dtype({
    "names": ["kind", "n_targets", "targets", "n_controls", "controls", "params", "matrix"],
    "formats": [np.int32, np.int32, (np.int32, MAX_TARGETS), np.int32, (np.int32, MAX_CONTROLS),
                (np.float64, 3), np.uint64],
    "offsets": [getattr(qs_gate_t, f).offset for f in
                ("kind", "n_targets", "targets", "n_controls", "controls", "params", "matrix")],
    "itemsize": ctypes.sizeof(qs_gate_t),
})


def marshal_gates(gates: Sequence) -> tuple:
    """Gate objects -> (qs_gate_t array, keep-alive list): filled column-wise
    through a numpy view of the records (argument marshalling only)."""
    n = len(gates)
    arr = (qs_gate_t * max(1, n))()
    keep = []
    if not n:
        return arr, keep
    v = np.frombuffer(arr, dtype=_GATE_DTYPE)
    nt = [len(g.targets) for g in gates]
    nc = [len(g.controls) for g in gates]
    if max(nt) > MAX_TARGETS or max(nc) > MAX_CONTROLS:
        raise ValueError("too many targets/controls")
    v["kind"] = [KINDS[g.kind] for g in gates]
    v["n_targets"] = nt
    v["n_controls"] = nc
    zt, zc, zp = (0,) * MAX_TARGETS, (0,) * MAX_CONTROLS, (0.0, 0.0, 0.0)
    v["targets"] = [(tuple(g.targets) + zt)[:MAX_TARGETS] for g in gates]
    v["controls"] = [(tuple(g.controls) + zc)[:MAX_CONTROLS] for g in gates]
    v["params"] = [(tuple(g.params) + zp)[:3] for g in gates]
    for i, g in enumerate(gates):
        if getattr(g, "matrix", None) is not None:
            m = np.ascontiguousarray(np.asarray(g.matrix, dtype=np.complex128))
            keep.append(m)
            v["matrix"][i] = m.ctypes.data
    return arr, keep


def default_config() -> qs_config_t:
    c = qs_config_t()
    load_library().qs_default_config(ctypes.byref(c))
    return c


def make_config(flags: int = QS_OPT_ALL, fuse_cap: int = 4, diag_cap: int = 0,
                boost_div: int = 2, chunk_qubits: int = 12,
                jit_min_qubits: Optional[int] = None,
                l2_block_qubits: Optional[int] = None) -> qs_config_t:
    d = default_config()
    if jit_min_qubits is None:
        jit_min_qubits = d.jit_min_qubits
    if l2_block_qubits is None:
        l2_block_qubits = d.l2_block_qubits
    return qs_config_t(chunk_qubits, fuse_cap, diag_cap, boost_div, flags, jit_min_qubits,
                       l2_block_qubits)


def plan_json(n_qubits: int, gates: Sequence, n_ranks: int = 1, config: Optional[qs_config_t] = None,
              product_state: bool = True, basis: int = 0, detail: bool = False) -> dict:
    """Host-only optimiser output (qs_plan_json): no GPU needed."""
    lib = load_library()
    arr, keep = marshal_gates(gates)
    cfg = ctypes.byref(config) if config is not None else None
    ebuf = ctypes.create_string_buffer(512)
    n = lib.qs_plan_json(n_qubits, n_ranks, cfg, int(product_state), basis, arr, len(gates),
                         int(detail), ebuf, 512)
    if n < 0:
        raise QSError(int(n), "qs_plan_json: " + ebuf.value.decode())
    buf = ctypes.create_string_buffer(int(n) + 1)
    lib.qs_plan_json(n_qubits, n_ranks, cfg, int(product_state), basis, arr, len(gates),
                     int(detail), buf, n + 1)
    return json.loads(buf.value.decode())


def divider(n: int, div_size: int) -> list:
    out = (ctypes.c_int * 64)()
    k = load_library().qs_divider(n, div_size, out, 64)
    if k < 0:
        raise QSError(k, "qs_divider")
    return list(out[:k])


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load_library().qs_nccl_unique_id(buf)
    if rc:
        raise QSError(rc, "qs_nccl_unique_id")
    return buf.raw


class Simulator:
    """Owning wrapper of one qs_ctx handle."""

    def __init__(self, n_qubits: int, n_gpus: int = 1, *, loopback_ranks: int = 0,
                 device: int = 0, rank: Optional[int] = None, world_size: int = 1,
                 nccl_id: Optional[bytes] = None, config: Optional[qs_config_t] = None):
        self.lib = load_library()
        self.n = n_qubits
        h = ctypes.c_void_p()
        if rank is not None:
            rc = self.lib.qs_create_rank(n_qubits, world_size, rank, device, nccl_id, ctypes.byref(h))
            self.n_ranks = world_size
        elif loopback_ranks:
            rc = self.lib.qs_create_loopback(n_qubits, loopback_ranks, device, ctypes.byref(h))
            self.n_ranks = loopback_ranks
        else:
            rc = self.lib.qs_create(n_qubits, n_gpus, ctypes.byref(h))
            self.n_ranks = n_gpus
        self.h = h
        if rc != QS_OK:
            msg = self.lib.qs_last_error(h).decode() if h.value else ""
            if h.value:
                self.lib.qs_destroy(h)
                self.h = ctypes.c_void_p()
            raise QSError(rc, msg or "create failed")
        if config is not None:
            self.set_config(config)

    def _check(self, rc: int):
        if rc != QS_OK:
            raise QSError(rc, self.lib.qs_last_error(self.h).decode())

    def set_config(self, cfg: qs_config_t):
        self._check(self.lib.qs_set_config(self.h, ctypes.byref(cfg)))

    def set_basis_state(self, x: int = 0):
        self._check(self.lib.qs_set_basis_state(self.h, x))

    def apply(self, gates: Sequence, marshalled=None):
        arr, keep = marshalled if marshalled is not None else marshal_gates(gates)
        self._check(self.lib.qs_apply_circuit(self.h, arr, len(gates)))

    @staticmethod
    def _out(out, count, dtype):
        if out is None:
            return np.empty(count, dtype=dtype)
        if out.dtype != dtype or out.size < count or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous {np.dtype(dtype).name} array of >= {count} elements")
        return out

    def state(self, offset: int = 0, count: Optional[int] = None,
              out: Optional[np.ndarray] = None) -> np.ndarray:
        """Amplitudes [offset, offset+count) in logical order.  `out` (e.g. a
        view of pinned host memory) is filled in place and returned."""
        if count is None:
            count = (1 << self.n) - offset
        out = self._out(out, count, np.complex128)
        self._check(self.lib.qs_get_state(self.h, out.ctypes.data, offset, count))
        return out

    def probabilities(self, offset: int = 0, count: Optional[int] = None,
                      out: Optional[np.ndarray] = None) -> np.ndarray:
        if count is None:
            count = (1 << self.n) - offset
        out = self._out(out, count, np.float64)
        self._check(self.lib.qs_probabilities(self.h, out.ctypes.data, offset, count))
        return out

    def stats(self) -> dict:
        s = qs_stats_t()
        self._check(self.lib.qs_get_stats(self.h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in qs_stats_t._fields_}

    def kernel_timing(self, kernel: str) -> dict:
        n = ctypes.c_uint64()
        ms = ctypes.c_double()
        b = ctypes.c_uint64()
        self._check(self.lib.qs_get_kernel_timing(self.h, KERNELS[kernel], ctypes.byref(n),
                                                  ctypes.byref(ms), ctypes.byref(b)))
        return {"launches": n.value, "ms": ms.value, "bytes": b.value}

    def launches(self) -> int:
        return int(self.lib.qs_last_launches(self.h))

    def set_timing(self, mode: int):
        """0 off, 1 per call (default), 2 accumulate over calls (qs_set_timing)."""
        self._check(self.lib.qs_set_timing(self.h, int(mode)))

    def close(self):
        if self.h and self.h.value:
            self.lib.qs_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _stream_of(sim: "Simulator", i: int = 0) -> int:
    """cudaStream_t (int) the handle launches shard i on (qs_get_stream)."""
    return int(sim.lib.qs_get_stream(sim.h, i) or 0)


Simulator.stream = _stream_of
