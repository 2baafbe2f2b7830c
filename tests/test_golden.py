"""Paper / SPEC worked-example values stored under tests/golden/ (each file
carries its citation), checked against the oracle, the planner and (gpu) the
CUDA path."""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2604_12256_b200 as qs
import workloads as W
from tests.conftest import cuda_available
from tests.plan_replay import replay

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return json.load(open(os.path.join(GOLD, name)))


def spec_cases():
    d = load("spec_examples.json")
    for c in d["cases"]:
        gates = [W.Gate(k, t, cs, p) for k, t, cs, p in c["gates"]]
        want = np.array([complex(re, im) for re, im in c["state"]])
        yield c["name"], c["n"], c["basis"], gates, want


def test_spec_examples_oracle():
    for name, n, basis, gates, want in spec_cases():
        got = oracle.apply_circuit(n, gates, x=basis)
        assert np.max(np.abs(got - want)) < 1e-15, name


def test_spec_examples_plan_replay():
    for name, n, basis, gates, want in spec_cases():
        plan = qs.plan_json(n, gates, basis=basis, detail=True)
        assert np.max(np.abs(replay(plan, n, 1) - want)) < 1e-15, name


def test_divider_traces_golden():
    for t in load("divider_traces.json")["traces"]:
        assert qs.divider(t["n"], t["div_size"]) == t["groups"]


def test_f23_update_counts_golden():
    g = load("f23_update_counts.json")
    gates = W.fixture_f23()
    assert len(gates) == g["n_gates"]
    assert sum(1 for x in gates if x.controls) == g["n_controlled"]
    cfg = qs.make_config(flags=qs.QS_OPT_BOOST | qs.QS_OPT_BLOCK, boost_div=g["boost_div"])
    plan = qs.plan_json(g["n_qubits"], gates, config=cfg, detail=True)
    st = plan["stats"]
    assert st["naive_updates"] == g["naive_updates"]
    assert st["booster_rounds"] == g["booster_rounds_group_gates"]
    assert st["paper_updates"] == g["paper_updates"]


def test_f4_grouping_golden():
    g = load("f4_detector_grouping.json")
    gates = W.fixture_f4()
    cfg = qs.make_config(flags=qs.QS_OPT_DIAG | qs.QS_OPT_BLOCK)
    plan = qs.plan_json(5, gates, config=cfg, detail=True)
    (p,) = [s for s in plan["steps"] if s["type"] == "pass"]
    ops = p["ops"]
    # position of the fused diagonal (1-based) among the emitted ops
    pos = [i for i, o in enumerate(ops) if o["t"] == "diag" and o["n_src"] == len(g["fused_gate_indices_1based"])]
    assert pos and pos[0] + 1 == g["fused_position_1based"]
    fused = ops[pos[0]]
    support = 0
    for m, _ in fused["mono"]:
        support |= int(m)
    assert bin(support).count("1") == g["fused_support_size"]
    # bypassed gates before it, deferred after it, the stopped RZZ last
    assert [o["tpos"] for o in ops[:pos[0]]] == [list(gates[i - 1].targets) for i in g["bypassed_before_fusion_1based"]]
    after = ops[pos[0] + 1:]
    assert [o["tpos"] for o in after[:2]] == [list(gates[i - 1].targets) for i in g["deferred_after_fusion_1based"]]
    assert after[-1]["t"] == "diag" and after[-1]["n_src"] == 1


@pytest.mark.gpu
def test_spec_examples_gpu():
    if not cuda_available():
        pytest.skip("no CUDA device")
    for name, n, basis, gates, want in spec_cases():
        with qs.Simulator(n) as s:
            s.set_basis_state(basis)
            s.apply(gates)
            assert np.max(np.abs(s.state() - want)) < 1e-15, name
