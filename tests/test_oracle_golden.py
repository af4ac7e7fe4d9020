"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  If these pass, the oracle reproduces the
reference and can be trusted as the checker for the GPU path at sizes the
fixtures do not cover.  CPU only.
"""

import os

import numpy as np
import pytest

from oracle import c_oracle, qsim_oracle as orc
from golden_util import load_circuits, load_gate_cases, load_haar, load_observables, \
    record_from_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_haar_bit_exact():
    for key, vec in load_haar().items():
        n, seed = key[1:].split("_s")
        got = orc.haar_state(int(n), int(seed))
        assert np.array_equal(got.view(np.uint64), vec.view(np.uint64)), key


def test_gate_cases_match_reference():
    cases, outs = load_gate_cases()
    worst = 0.0
    for case in cases:
        n = case["n"]
        amps = orc.haar_state(n, case["seed"])
        orc.apply_record(amps, n, record_from_json(case["record"]))
        worst = max(worst, float(np.max(np.abs(amps - outs[case["id"]]))))
    assert worst <= 1e-15, worst


def test_generator_circuits_match_reference():
    meta, outs = load_circuits()
    for e in meta["circuits"]:
        if "opt" in e:
            continue
        n = e["n"]
        if e["name"] == "cnot-ring":
            recs = orc.cnot_ring_records(n, e["seed"])
        else:
            recs = orc.cz_ladder_records(n, e["depth"], e["seed"],
                                         commuting=e["name"].endswith("commuting"))
        assert len(recs) == e["gate_count"]
        amps = orc.zero_state(n) if e["start_seed"] is None else orc.haar_state(n, e["start_seed"])
        orc.run_records(amps, n, recs)
        assert np.max(np.abs(amps - outs[e["id"]])) <= 1e-13, e


def test_observables_match_reference():
    data = load_observables()
    for case in data["random"]:
        n = case["n"]
        terms = [(complex(*t["coef"]), [tuple(o) for o in t["ops"]]) for t in case["terms"]]
        psi = orc.haar_state(n, case["seed"])
        bra = orc.haar_state(n, case["seed"] + 1)
        v = orc.expectation(psi, psi, n, terms)
        tr = orc.expectation(bra, psi, n, terms)
        assert abs(v - complex(*case["value"])) <= 1e-13
        assert abs(tr - complex(*case["transition"])) <= 1e-13


def test_c_oracle_matches_numpy_oracle():
    rng = np.random.default_rng(5)
    for n in (9, 17):
        for trial in range(40):
            psi = orc.haar_state(n, trial)
            ref = psi.copy()
            k = int(rng.integers(1, 4))
            qs = [int(v) for v in rng.permutation(n)]
            t, rest = qs[:k], qs[k:]
            nc = int(rng.integers(0, 3))
            ctl = tuple((rest[i], int(rng.integers(2))) for i in range(nc))
            kind = trial % 4
            if kind == 0:
                rec = ("dense", t, orc.pauli_matrix([1] * k) * 0.3 + np.eye(1 << k), ctl)
            elif kind == 1:
                rec = ("diag", t, np.exp(1j * rng.uniform(0, 6, 1 << k)), ctl)
            elif kind == 2:
                rec = ("pauli_rot", t, [int(v) for v in rng.integers(1, 4, k)],
                       float(rng.uniform(-7, 7)), ctl)
            else:
                rec = ("pauli", t, [int(v) for v in rng.integers(1, 4, k)], ctl)
            c_oracle.apply_record(psi, n, rec)
            orc.apply_record(ref, n, rec)
            assert np.max(np.abs(psi - ref)) <= 1e-14, trial
    # rotations and Paulis are bit-identical by construction
    n = 9
    psi = orc.haar_state(n, 99)
    ref = psi.copy()
    c_oracle.apply_record(psi, n, ("pauli_rot", (3,), (1,), 0.37, ()))
    orc.apply_pauli_rotation(ref, n, [3], [1], 0.37)
    assert np.array_equal(psi, ref)
    got = c_oracle.pauli_term(psi, psi, n, [(0, 1), (4, 2)])
    v = orc.expectation(psi, psi, n, [(1.0, [(0, 1), (4, 2)])])
    assert abs(got - v) <= 1e-14
    assert abs(c_oracle.norm2(psi, n) - orc.squared_norm(psi)) <= 1e-14


def test_cfg3_reference_value_recorded():
    vqe = {e["n"]: e for e in load_observables()["vqe"]}
    # <H> = -0.201996915076406 for the 24-qubit instance
    if 24 in vqe:
        assert vqe[24]["value"] == pytest.approx(-0.201996915076406, abs=1e-14)
    assert vqe[8]["gates"] == 92 and vqe[12]["params"] == 96


def test_cfg1_oracle_matches_reference():
    """The numpy oracle reproduces the reference's cfg1 digests (cnot-ring(16)
    seeds 0..4, from |0> and Haar starts; tests/golden/cfg1.*)."""
    from paper_2011_13524_b200 import workloads
    from paper_2011_13524_b200._circuit import circuit_records
    from golden_util import cfg1_digest, load_cfg1
    meta, outs = load_cfg1()
    assert len(meta["cases"]) == 10
    for e in meta["cases"]:
        n = 16
        recs = circuit_records(workloads.generate_cnot_ring(n, seed=e["seed"]))
        start = orc.zero_state(n) if e["start_seed"] is None else orc.haar_state(n, e["start_seed"])
        dg = cfg1_digest(orc.run_records(start, n, recs))
        key = e["id"]
        assert np.max(np.abs(dg["amps"] - outs[f"{key}/amps"])) <= 1e-15, key
        assert np.max(np.abs(dg["proj"] - outs[f"{key}/proj"])) <= 1e-13, key
        assert np.max(np.abs(dg["z"] - outs[f"{key}/z"])) <= 1e-15, key
