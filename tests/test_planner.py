"""Host optimiser tests (-m "not gpu"): the plan produced by libqs's planner
(qs_plan_json, no GPU) is replayed by tests/plan_replay.py and compared with
the CPU oracle, and its structure is checked against the paper's pins
(Alg. 6 traces, Fig. 2/3 update counts, Fig. 4 grouping)."""
import itertools

import numpy as np
import pytest

import oracle
import paper_2604_12256_b200 as qs
import workloads as W
from tests import pins
from tests.plan_replay import check_structure, replay

ALL = qs.QS_OPT_ALL


def cfg(flags=ALL, fuse=4, diag=0, boost=2):
    return qs.make_config(flags=flags, fuse_cap=fuse, diag_cap=diag, boost_div=boost)


def run(n, gates, ranks=1, c=None, basis=0):
    plan = qs.plan_json(n, gates, n_ranks=ranks, config=c, product_state=True, basis=basis,
                        detail=True)
    check_structure(plan, n, ranks)
    return plan, replay(plan, n, ranks)


# ------------------------------------------------------------------ Alg. 6

def test_divider_traces():
    # SPEC.md L293-295 / SURVEY App. A
    assert qs.divider(8, 2) == [2, 2, 2, 2]
    assert qs.divider(4, 4) == [4]
    assert qs.divider(5, 2) == [2, 1, 2]
    assert qs.divider(32, 16) == [16, 16]        # P:L484 two 2^16 sub-states
    assert qs.divider(30, 8) == [7, 8, 7, 8]
    assert qs.divider(35, 9) == [8, 9, 9, 9]
    for n in range(1, 41):
        for d in range(1, n + 1):
            assert sum(qs.divider(n, d)) == n


# ------------------------------------------------------------------ Fig. 2/3

def test_booster_paper_update_count_f23():
    """40 * 2^8 = 10,240 naive -> 1,336 with the merge booster
    (B = 4 -> divSize 2 -> [2,2,2,2]); rounds [[6,6,7,7],[7,4],[3]]."""
    gates = W.fixture_f23()
    c = cfg(flags=qs.QS_OPT_BOOST | qs.QS_OPT_BLOCK, boost=4)
    plan, psi = run(8, gates, c=c)
    st = plan["stats"]
    assert st["naive_updates"] == 10240
    assert st["booster_rounds"] == [[6, 6, 7, 7], [7, 4]]
    assert st["paper_updates"] == 1336
    want = oracle.apply_circuit(8, gates)
    assert np.max(np.abs(psi - want)) < 1e-12


# ------------------------------------------------------------------ Fig. 4

def test_detector_fig4_grouping():
    """RZZ2, RZZ5, CP6, RZZ8, CP9 fuse into one 4-qubit diagonal; H3,
    RY4 bypassed, RX7 deferred, RZZ11 stopped."""
    gates = W.fixture_f4()
    c = cfg(flags=qs.QS_OPT_DIAG | qs.QS_OPT_BLOCK)
    plan, psi = run(5, gates, c=c)
    assert plan["stats"]["n_fused_diag"] == 1
    (p,) = [s for s in plan["steps"] if s["type"] == "pass"]
    kinds = [(o["t"], o.get("tpos"), o["n_src"]) for o in p["ops"]]
    # H1, H3, RY4 | D{2,5,6,8,9} | RX7, RY10 | RZZ11
    assert kinds[0] == ("dense", [0], 1)
    assert kinds[1] == ("dense", [2], 1)
    assert kinds[2] == ("dense", [3], 1)
    assert kinds[3][0] == "diag" and kinds[3][2] == 5
    assert kinds[4] == ("dense", [0], 1) and kinds[5] == ("dense", [0], 1)
    assert kinds[6][0] == "diag" and kinds[6][2] == 1
    want = oracle.apply_circuit(5, gates)
    assert np.max(np.abs(psi - want)) < 1e-12


def test_detector_ablation_random():
    """with the corrections c4-c7, 0/200 random 4-qubit
    RZZ/CP/RZ/RX/CX circuits differ from the oracle."""
    c = cfg(flags=qs.QS_OPT_DIAG | qs.QS_OPT_BLOCK)
    for seed in range(200):
        gates = W.random_circuit(4, 14, seed, kinds=["RZZ", "CP", "RZ", "RX", "CX"], max_controls=0)
        _, psi = run(4, gates, c=c)
        want = oracle.apply_circuit(4, gates)
        assert np.max(np.abs(psi - want)) < 1e-12, seed


# ------------------------------------------------------------------ replay

FLAGS = [0, qs.QS_OPT_BLOCK, qs.QS_OPT_BLOCK | qs.QS_OPT_FUSE, qs.QS_OPT_DIAG | qs.QS_OPT_BLOCK,
         qs.QS_OPT_BOOST | qs.QS_OPT_BLOCK, ALL]


@pytest.mark.parametrize("flags", FLAGS)
@pytest.mark.parametrize("seed", range(8))
def test_replay_random_small(flags, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 11))
    gates = W.random_circuit(n, 80, seed, diag_bias=0.4)
    basis = int(rng.integers(1 << n))
    _, psi = run(n, gates, c=cfg(flags=flags), basis=basis)
    want = oracle.apply_circuit(n, gates, x=basis)
    assert np.max(np.abs(psi - want)) < 1e-11


@pytest.mark.parametrize("n,seed", [(13, 0), (14, 1), (15, 2)])
def test_replay_random_chunked(n, seed):
    gates = W.random_circuit(n, 150, seed, diag_bias=0.4, max_generic=3)
    _, psi = run(n, gates, basis=3)
    want = oracle.apply_circuit(n, gates, x=3)
    assert np.max(np.abs(psi - want)) < 1e-11


@pytest.mark.parametrize("ranks", [2, 4, 8])
@pytest.mark.parametrize("n", [6, 9, 14])
def test_replay_sharded(ranks, n):
    gates = W.random_circuit(n, 120, 10 * n + ranks, diag_bias=0.3)
    plan, psi = run(n, gates, ranks=ranks, basis=5)
    want = oracle.apply_circuit(n, gates, x=5)
    assert np.max(np.abs(psi - want)) < 1e-11


@pytest.mark.parametrize("n", [10, 13, 14])
def test_replay_qft_closed_form(n):
    for x in (0, 5):
        plan, psi = run(n, W.qft(n), basis=x)
        assert np.max(np.abs(psi - pins.qft_closed_form(n, x))) < 1e-12


@pytest.mark.parametrize("n", [14, 16])
def test_store_relabel_replay(n):
    """The last layout of QFT's chunk pass holds the lowest chunk bits: the
    pass stores with its chunk bits permuted (opos != cpos) and the map
    records it (reading r2); the replayed result is still the closed form."""
    plan, psi = run(n, W.qft(n), basis=3)
    passes = [s for s in plan["steps"] if s["type"] == "pass" and "opos" in s]
    assert any(s["opos"] != s["cpos"] for s in passes)
    assert np.max(np.abs(psi - pins.qft_closed_form(n, 3))) < 1e-12


def test_replay_qaoa_sharded():
    n = 14
    gates = W.qaoa_maxcut(n, 2, 3)
    for ranks in (1, 2, 4):
        plan, psi = run(n, gates, ranks=ranks)
        want = oracle.apply_circuit(n, gates)
        assert np.max(np.abs(psi - want)) < 1e-11
        if ranks > 1:
            assert plan["stats"]["n_swaps"] >= 1


def test_plan_shapes_large():
    """Plan shape of the benchmark configs (no replay at this size)."""
    p = qs.plan_json(30, W.qft(30))
    assert p["stats"]["n_passes"] <= 4
    p = qs.plan_json(30, W.rzz_full(30))
    assert p["stats"]["n_passes"] == 1 and p["stats"]["n_diag"] == 1
    p = qs.plan_json(30, W.diag_chain(30))
    assert p["stats"]["n_passes"] <= 3
    p = qs.plan_json(33, W.qft(33), n_ranks=8)
    assert p["stats"]["n_swaps"] <= 2
    p = qs.plan_json(35, W.supremacy(5, 7, 20), n_ranks=8)
    assert p["stats"]["n_passes"] >= 1


@pytest.mark.parametrize("n", [1, 2, 12, 13])
def test_replay_size_boundaries(n):
    gates = W.random_circuit(n, 60, 100 + n, diag_bias=0.3)
    _, psi = run(n, gates, basis=(1 << n) - 1)
    assert np.max(np.abs(psi - oracle.apply_circuit(n, gates, x=(1 << n) - 1))) < 1e-11


def test_replay_wide_gates_small():
    rng = np.random.default_rng(4)
    n = 9
    gates = [W.Gate("UNITARY", (0, 2, 4, 6, 8, 1), (), (), W.haar_unitary(64, rng)),
             W.Gate("DIAGONAL", (3, 5, 7, 0, 1), (2,), (), W.random_phases(32, rng))]
    _, psi = run(n, W.random_circuit(n, 20, 1) + gates)
    want = oracle.apply_circuit(n, W.random_circuit(n, 20, 1) + gates)
    assert np.max(np.abs(psi - want)) < 1e-11


def test_plan_dims_rejected():
    with pytest.raises(qs.QSError):
        qs.plan_json(41, [])
    with pytest.raises(qs.QSError):
        qs.plan_json(4, [], n_ranks=3)
    with pytest.raises(qs.QSError):
        qs.plan_json(3, [], n_ranks=8)


def test_invalid_gates_rejected():
    with pytest.raises(qs.QSError):
        qs.plan_json(3, [W.Gate("H", (3,))])
    with pytest.raises(qs.QSError):
        qs.plan_json(3, [W.Gate("CX", (1,), (1,))])
    bad = np.eye(2) * 1.1
    with pytest.raises(qs.QSError):
        qs.plan_json(3, [W.Gate("UNITARY", (0,), (), (), bad)])
    with pytest.raises(qs.QSError):
        qs.plan_json(3, [W.Gate("DIAGONAL", (0,), (), (), np.array([1, 2]))])


@pytest.mark.parametrize("name", sorted(W.ROSTER))
@pytest.mark.parametrize("flags", [qs.QS_OPT_ALL, qs.QS_OPT_FUSE, 0])
def test_roster_replay(name, flags):
    """PAPER.md Table 2 roster circuits (L799-805) under the ablation modes:
    plan replay equals the oracle."""
    n = 12
    gates = W.ROSTER[name](n)
    plan = qs.plan_json(n, gates, config=qs.make_config(flags=flags), detail=True)
    psi = replay(plan, n, 1)
    assert np.max(np.abs(psi - oracle.apply_circuit(n, gates))) < 1e-11


def test_nofusion_nonblocking_is_one_gate_per_pass():
    """Without blocking or fusion every dense gate costs one state sweep; with
    fusion only, gates whose targets fuse into <= F qubits share one."""
    n = 14
    gates = [W.Gate("RX", (q,), (), (0.1 * q,)) for q in range(n)]
    p0 = qs.plan_json(n, gates, config=qs.make_config(flags=0), detail=True)
    pf = qs.plan_json(n, gates, config=qs.make_config(flags=qs.QS_OPT_FUSE, fuse_cap=4), detail=True)
    assert p0["stats"]["n_passes"] == n
    assert pf["stats"]["n_passes"] == -(-n // 4)


def test_fusable_swaps_marked():
    """a swap right after a specialised pass is marked fusable
    and that pass exports the swap's j top local bits."""
    n, ranks = 18, 4
    gates = W.qaoa_maxcut(n, 3, 2)
    plan = qs.plan_json(n, gates, n_ranks=ranks, config=qs.make_config(jit_min_qubits=0), detail=True)
    steps = plan["steps"]
    fused = [i for i, s in enumerate(steps) if s["type"] == "swap" and s["fusable"]]
    assert fused and plan["stats"]["n_fusable_swaps"] == len(fused)
    nl = n - 2
    for i in fused:
        p = steps[i - 1]
        assert p["type"] == "pass" and p["x_j"] == steps[i]["j"]
    # replay (the fused exchange has the swap's semantics) still matches
    psi = replay(plan, n, ranks)
    assert np.max(np.abs(psi - oracle.apply_circuit(n, gates))) < 1e-11


def test_specialised_kernels_compile(tmp_path, monkeypatch):
    """Every pass shape of the bench workloads compiles as a specialised
    sm_100a kernel (NVRTC runs without a GPU): a generator bug must fail
    here, not silently fall back to the interpreter kernels on the GPU."""
    monkeypatch.setenv("QS_JIT_CACHE", str(tmp_path))
    import bench
    cfg = qs.make_config(jit_min_qubits=0)
    n = 20
    for w in ("qft", "rzz", "diag", "qaoa", "rand"):
        gates = bench.make_circuit(w, n)
        for ranks in (1, 4):
            qs.plan_json(n, gates, n_ranks=ranks, config=cfg, basis=5, detail=2)
    assert any(p.suffix == ".cubin" for p in tmp_path.iterdir())


# ------------------------------------------------------------ round-2 limits

def test_fused_swaps_capped_at_three_exported_bits():
    """A fused swap's pass stores to at most 2^3 destinations (the kernel's
    peer table): with 16 and 32 ranks, swaps of j > 3 qubits stay unfused,
    and the replay still equals the oracle."""
    n = 14
    gates = W.qaoa_maxcut(n, 2, 4)
    for ranks in (16, 32):
        nl = n - (ranks.bit_length() - 1)
        if nl < ranks.bit_length() - 1:
            continue
        plan = qs.plan_json(n, gates, n_ranks=ranks, config=qs.make_config(jit_min_qubits=0), detail=True)
        for i, s in enumerate(plan["steps"]):
            if s["type"] == "swap" and s["fusable"]:
                assert s["j"] <= 3
            if s["type"] == "pass":
                assert s["x_j"] <= 3
        psi = replay(plan, n, ranks)
        assert np.max(np.abs(psi - oracle.apply_circuit(n, gates))) < 1e-11
    plan = qs.plan_json(24, W.qaoa_maxcut(24, 2, 4), n_ranks=16, config=qs.make_config(jit_min_qubits=0))
    assert all(s["j"] <= 3 for s in plan["steps"] if s["type"] == "swap" and s["fusable"])


def test_many_wide_diagonals_plan_within_encoder_limits():
    """600 random 6-target DIAGONAL gates on 16 qubits (up to 63 monomials
    each): the scheduler closes passes before the encoder's shape limit, so
    the plan encodes, compiles and replays to the oracle."""
    rng = np.random.default_rng(600)
    n = 16
    gates = [W.Gate("DIAGONAL", tuple(int(q) for q in rng.permutation(n)[:6]), (), (),
                    W.random_phases(64, rng)) for _ in range(600)]
    plan, psi = run(n, gates, basis=0)
    assert plan["stats"]["n_passes"] >= 2
    want = oracle.apply_circuit(n, gates)
    assert np.max(np.abs(psi - want)) < 1e-11


@pytest.mark.parametrize("k", [4, 5, 6])
def test_wide_unitaries_large_state_plan(k, tmp_path, monkeypatch):
    """k-target unitaries (Eq. 3 generalised) on a 20-qubit
    shard: 4-6 targets run as a shared-memory op (OP_DW)
    at a layout exchange; the plan replays to the oracle and every
    pass compiles as a specialised kernel."""
    monkeypatch.setenv("QS_JIT_CACHE", str(tmp_path))
    rng = np.random.default_rng(40 + k)
    n = 20
    gates = W.random_circuit(n, 40, k, diag_bias=0.3, max_generic=3)
    for _ in range(3):
        tg = tuple(int(q) for q in rng.permutation(n)[:k])
        ctl = (int(rng.choice([q for q in range(n) if q not in tg])),) if rng.uniform() < 0.5 else ()
        gates.append(W.Gate("UNITARY", tg, ctl, (), W.haar_unitary(1 << k, rng)))
        gates += W.random_circuit(n, 10, int(rng.integers(1000)), diag_bias=0.5)
    plan = qs.plan_json(n, gates, config=qs.make_config(jit_min_qubits=0), product_state=True, basis=3,
                        detail=2)
    check_structure(plan, n, 1)
    psi = replay(plan, n, 1)
    assert np.max(np.abs(psi - oracle.apply_circuit(n, gates, x=3))) < 1e-11
    tks = [len(o["tpos"]) for s in plan["steps"] if s["type"] == "pass" for o in s["ops"] if o["t"] == "dense"]
    assert max(tks) == k


def test_fusion_reaches_four_targets():
    """fuse_cap = 4 is effective: enough 1-/2-qubit gates on 4 qubits fuse
    into one 16x16 unitary when the FP64 cost model says it saves work."""
    rng = np.random.default_rng(7)
    n = 16
    qb = [3, 5, 8, 12]
    gates = []
    for _ in range(20):
        a, b = (int(x) for x in rng.choice(qb, 2, replace=False))
        gates.append(W.Gate("UNITARY", (a, b), (), (), W.haar_unitary(4, rng)))
    plan, psi = run(n, gates, basis=1)
    tks = [len(o["tpos"]) for s in plan["steps"] if s["type"] == "pass" for o in s["ops"] if o["t"] == "dense"]
    assert 4 in tks
    assert np.max(np.abs(psi - oracle.apply_circuit(n, gates, x=1))) < 1e-11


def test_write_only_budget_candidates():
    """The optimiser tries FP64 budgets 40/48/64 for the write-only first pass
    and keeps the plan with the fewest full-state passes: QAOA-30 p=4 takes
    11 (12 at the balanced 40), QFT stays at 2 at every bench size."""
    import bench
    p = qs.plan_json(30, bench.make_circuit("qaoa", 30), basis=5)
    assert p["stats"]["n_passes"] <= 11
    for n, r in ((30, 1), (31, 2), (32, 4), (33, 8)):
        p = qs.plan_json(n, bench.make_circuit("qft", n), n_ranks=r, basis=5)
        assert p["stats"]["n_passes"] == 2, (n, r)


@pytest.mark.parametrize("name", ["SX", "SY"])
def test_unit_scaled_gates_replay(name):
    """SX / SY (unit-scaled: +-lam, +-i lam entries) on a 14-qubit state with
    other gates around: the plan replays to the oracle (the kernels' scalar
    extraction is covered by the GPU tests)."""
    n = 14
    gates = []
    for q in range(n):
        gates.append(W.Gate(name, (q,)))
        gates.append(W.Gate("CZ", ((q + 1) % n,), (q,)))
    gates += W.random_circuit(n, 40, 3)
    _, psi = run(n, gates, basis=9)
    assert np.max(np.abs(psi - oracle.apply_circuit(n, gates, x=9))) < 1e-11


def test_l2_groups_marked_by_position_bound():
    """Two-level blocking: runs of >= 2
    consecutive full-state passes whose chunk and output positions all lie
    below W are marked as one group; off (0) by default; the HBM bytes of a
    group are its first pass's."""
    n = 26
    gates = W.qft(n)
    assert qs.plan_json(n, gates)["stats"]["n_l2_groups"] == 0
    for wb in (15, 18, 22):
        p = qs.plan_json(n, gates, config=qs.make_config(l2_block_qubits=wb), basis=5)
        full = [s for s in p["steps"] if s["type"] == "pass" and s["nl"] == n]
        grouped = [s for s in full if s["l2_grp"] >= 0]
        assert p["stats"]["n_l2_groups"] >= 1 and len(grouped) >= 2
        for s in grouped:
            assert max(s["cpos"] + s["opos"]) < wb
            assert s["x_j"] == 0 and s["pull_j"] == 0
        saved = 0
        for g in set(s["l2_grp"] for s in grouped):
            saved += (sum(1 for s in grouped if s["l2_grp"] == g) - 1) * (32 << n)
        assert p["stats"]["bytes_hbm_l2"] == p["stats"]["bytes_hbm"] - saved
    # a bound below the passes' positions: nothing grouped
    p = qs.plan_json(n, gates, config=qs.make_config(l2_block_qubits=14), basis=5)
    assert all(max(s["cpos"] + s["opos"]) < 14 for s in p["steps"]
               if s["type"] == "pass" and s.get("l2_grp", -1) >= 0)

