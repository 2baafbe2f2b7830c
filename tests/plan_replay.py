"""TEST-ONLY numpy interpreter of the optimiser's plan (qs_plan_json detail).

It replays the host plan -- passes as ordered physical-position ops, global
<->local swaps, booster sub-states, tensor-product merges/expansion and the
final virtual qubit map -- on CPU arrays, so the planner (detector, booster,
blocking, fusion, relabels, swap piece routing) can be checked against the
oracle without a GPU.  It does NOT exercise the kernels' register/phase
encoding; the -m gpu parity tests do.  Nothing in the product imports this.
"""
from __future__ import annotations

import math

import numpy as np

U64 = np.uint64


def _apply_dense(arr, nl, rank, mat, tpos, cmask):
    t = len(tpos)
    d = 1 << t
    m = np.array(mat[0::2]) + 1j * np.array(mat[1::2])
    m = m.reshape(d, d)
    # global controls: must be set in the rank bits
    gmask = cmask >> nl
    if (rank & gmask) != gmask:
        return arr
    lmask = cmask & ((1 << nl) - 1)
    idx = np.arange(1 << nl, dtype=np.int64)
    tm = 0
    for p in tpos:
        tm |= 1 << p
    base = idx[((idx & tm) == 0) & ((idx & lmask) == lmask)]
    offs = []
    for r in range(d):
        o = 0
        for i, p in enumerate(tpos):
            if r >> i & 1:
                o |= 1 << p
        offs.append(o)
    v = np.stack([arr[base | o] for o in offs])          # d x B
    w = m @ v
    out = arr.copy()
    for r, o in enumerate(offs):
        out[base | o] = w[r]
    return out


def _apply_diag(arr, nl, rank, mono):
    phys = (np.arange(1 << nl, dtype=np.uint64) | (U64(rank) << U64(nl)))
    ang = np.zeros(1 << nl, dtype=np.uint64)
    for mask_s, coeff_s in mono:
        m = U64(int(mask_s))
        c = U64(int(coeff_s))
        sel = (phys & m) == m
        ang[sel] += c  # wraps mod 2^64
    # exact split into two 32-bit halves before the float conversion
    hi = (ang >> U64(32)).astype(np.float64)
    lo = (ang & U64(0xFFFFFFFF)).astype(np.float64)
    turns = (hi + lo / 2.0 ** 32) / 2.0 ** 32
    return arr * np.exp(2j * math.pi * turns)


def _relabel(arr, cpos, opos):
    if list(cpos) == list(opos):
        return arr
    n = int(math.log2(arr.size))
    idx = np.arange(arr.size, dtype=np.int64)
    dst = idx.copy()
    cm = 0
    for c in cpos:
        cm |= 1 << c
    dst &= ~cm
    for c, o in zip(cpos, opos):
        dst |= ((idx >> c) & 1) << o
    out = np.empty_like(arr)
    out[dst] = arr
    return out


def replay(plan: dict, n: int, n_ranks: int) -> np.ndarray:
    shards = replay_shards(plan, n, n_ranks)
    mp = plan["map_out"]
    L = np.arange(1 << n, dtype=np.int64)
    phys = np.zeros_like(L)
    for q in range(n):
        phys |= ((L >> q) & 1) << mp[q]
    full = np.concatenate(shards)
    return full[phys]


_SUBS = {}


def replay_shards(plan: dict, n: int, n_ranks: int, shards=None, subs=None) -> list:
    """Run the plan's steps on per-rank shards (physical order); returns the
    shards.  `subs` (booster sub-states) persists across calls if given."""
    g = int(round(math.log2(n_ranks)))
    nl = n - g
    if shards is None:
        shards = [np.zeros(1 << nl, dtype=np.complex128) for _ in range(n_ranks)]
    shards = list(shards)
    if subs is None:
        subs = _SUBS
    sub_nq = {i + 1: s["nq"] for i, s in enumerate(plan["subs"])}
    local = np.arange(1 << nl, dtype=np.uint64)

    def expand(bufs, los, lens, rank):
        phys = local | (U64(rank) << U64(nl))
        v = np.ones(1 << nl, dtype=np.complex128)
        for b, lo, ln in zip(bufs, los, lens):
            v = v * subs[b][((phys >> U64(lo)) & U64((1 << ln) - 1)).astype(np.int64)]
        return v

    for st in plan["steps"]:
        ty = st["type"]
        if ty == "init_basis":
            b = int(st["basis"])
            for r in range(n_ranks):
                shards[r][:] = 0
                if b >> nl == r:
                    shards[r][b & ((1 << nl) - 1)] = 1
        elif ty == "sub_init":
            v = np.zeros(1 << sub_nq[st["buf"]], dtype=np.complex128)
            v[int(st["basis"])] = 1
            subs[st["buf"]] = v
        elif ty == "sub_merge":
            subs[st["buf"]] = np.kron(subs[st["b"]], subs[st["a"]])
        elif ty == "expand":
            for r in range(n_ranks):
                shards[r] = expand(st["bufs"], st["exp_lo"], st["exp_len"], r)
        elif ty == "permute":
            idx = np.arange(1 << nl, dtype=np.int64)
            dst = idx.copy()
            for a, b in zip(st["gpos"], st["lpos"]):
                x = ((idx >> a) ^ (idx >> b)) & 1
                dst ^= (x << a) | (x << b)
            for r in range(n_ranks):
                out = np.empty_like(shards[r])
                out[dst] = shards[r]
                shards[r] = out
        elif ty == "swap":
            j = st["j"]
            bits = [p - nl for p in st["gpos"]]
            top = list(range(nl - j, nl))
            # a swap with non-top local positions (fused swaps, reading r8)
            # = local transpositions lpos[i] <-> top[i], the top swap, and
            # the same transpositions again
            tr = [(a, b) for a, b in zip(st["lpos"], top) if a != b]
            assert all(a < nl - j for a, _ in tr), "non-top victims pair with free top slots"

            def transpose(shards):
                if not tr:
                    return shards
                idx = np.arange(1 << nl, dtype=np.int64)
                dst = idx.copy()
                for a, b in tr:
                    x = ((idx >> a) ^ (idx >> b)) & 1
                    dst ^= (x << a) | (x << b)
                out = []
                for sh in shards:
                    o = np.empty_like(sh)
                    o[dst] = sh
                    out.append(o)
                return out
            shards = transpose(shards)
            piece = 1 << (nl - j)
            new = [np.empty_like(s) for s in shards]
            for r in range(n_ranks):
                ur = sum(((r >> b) & 1) << i for i, b in enumerate(bits))
                for s in range(1 << j):
                    d = r
                    for i, b in enumerate(bits):
                        d = (d & ~(1 << b)) | (((s >> i) & 1) << b)
                    new[d][ur * piece:(ur + 1) * piece] = shards[r][s * piece:(s + 1) * piece]
            shards = transpose(new)
        elif ty == "pass":
            buf = st["buf"]
            ranks = range(n_ranks) if buf == 0 else [0]
            for r in ranks:
                if buf == 0:
                    pnl = nl
                    if st["src_mode"] == 1:
                        arr = expand(st["exp_bufs"], st["exp_lo"], st["exp_len"], r)
                    elif st["src_mode"] == 2:
                        arr = np.zeros(1 << nl, dtype=np.complex128)
                        b = int(st["basis"])
                        if b >> nl == r:
                            arr[b & ((1 << nl) - 1)] = 1
                    else:
                        arr = shards[r]
                else:
                    pnl = sub_nq[buf]
                    arr = subs[buf]
                for op in st["ops"]:
                    if op["t"] == "dense":
                        arr = _apply_dense(arr, pnl, r if buf == 0 else 0, op["mat"], op["tpos"],
                                           int(op["cmask"]))
                    else:
                        arr = _apply_diag(arr, pnl, r if buf == 0 else 0, op["mono"])
                if st["cpos"]:
                    arr = _relabel(arr, st["cpos"], st["opos"])
                if buf == 0:
                    shards[r] = arr
                else:
                    subs[buf] = arr
        else:
            raise ValueError(ty)
    return shards


def check_structure(plan: dict, n: int, n_ranks: int):
    """Invariants every plan must satisfy (locality of non-diagonal targets)."""
    g = int(round(math.log2(n_ranks)))
    nl = n - g
    for st in plan["steps"]:
        if st["type"] != "pass":
            continue
        pnl = nl if st["buf"] == 0 else plan["subs"][st["buf"] - 1]["nq"]
        if st["kernel"] == "small":
            assert pnl <= 12
            continue
        assert pnl > 12
        cpos = st["cpos"]
        assert len(cpos) == 12 and cpos == sorted(cpos) and set(range(3)) <= set(cpos)
        assert 1 <= len(st["phase_regs"]) <= 8
        for op in st["ops"]:
            if op["t"] == "dense":
                assert set(op["tpos"]) <= set(cpos), (op["tpos"], cpos)
                assert all(p < pnl for p in op["tpos"])
