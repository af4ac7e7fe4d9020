"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  If these pass, the oracle reproduces the
reference and can be trusted as the checker for the GPU path at sizes the
fixtures do not cover.  CPU only.
"""

import ctypes as C
import os

import numpy as np
import pytest

from oracle import qsim_oracle as orc
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
    lib = C.CDLL(os.path.join(ROOT, "oracle", "liboracle_c.so"))
    rng = np.random.default_rng(5)
    n = 9
    ip = lambda v: (C.c_int * max(1, len(v)))(*v)  # noqa: E731
    for trial in range(40):
        psi = orc.haar_state(n, trial)
        ref = psi.copy()
        k = int(rng.integers(1, 4))
        qs = [int(v) for v in rng.permutation(n)]
        t, rest = qs[:k], qs[k:]
        nc = int(rng.integers(0, 3))
        ctl = [(rest[i], int(rng.integers(2))) for i in range(nc)]
        kind = trial % 4
        if kind == 0:
            mat = orc.pauli_matrix([1] * k) * 0.3 + np.eye(1 << k)
            lib.oracle_apply_dense(psi.ctypes.data, n, ip(t), k, mat.ctypes.data,
                                   ip([q for q, _ in ctl]), ip([v for _, v in ctl]), nc)
            orc.apply_dense(ref, n, t, mat, ctl)
        elif kind == 1:
            d = np.exp(1j * rng.uniform(0, 6, 1 << k))
            lib.oracle_apply_diag(psi.ctypes.data, n, ip(t), k, d.ctypes.data,
                                  ip([q for q, _ in ctl]), ip([v for _, v in ctl]), nc)
            orc.apply_diagonal(ref, n, t, d, ctl)
        elif kind == 2:
            ids = [int(v) for v in rng.integers(1, 4, k)]
            ang = float(rng.uniform(-7, 7))
            lib.oracle_apply_pauli_rot(psi.ctypes.data, n, ip(t), ip(ids), k, C.c_double(ang))
            orc.apply_pauli_rotation(ref, n, t, ids, ang)
        else:
            ids = [int(v) for v in rng.integers(1, 4, k)]
            lib.oracle_apply_pauli(psi.ctypes.data, n, ip(t), ip(ids), k)
            orc.apply_pauli(ref, n, t, ids)
        assert np.max(np.abs(psi - ref)) <= 1e-14, trial
    # rotations and Paulis are bit-identical by construction
    psi = orc.haar_state(n, 99)
    ref = psi.copy()
    lib.oracle_apply_pauli_rot(psi.ctypes.data, n, ip([3]), ip([1]), 1, C.c_double(0.37))
    orc.apply_pauli_rotation(ref, n, [3], [1], 0.37)
    assert np.array_equal(psi, ref)
    out = (C.c_double * 2)()
    lib.oracle_pauli_term(psi.ctypes.data, psi.ctypes.data, n, ip([0, 4]), ip([1, 2]), 2, out)
    v = orc.expectation(psi, psi, n, [(1.0, [(0, 1), (4, 2)])])
    assert abs(complex(out[0], out[1]) - v) <= 1e-14


def test_cfg3_reference_value_recorded():
    vqe = {e["n"]: e for e in load_observables()["vqe"]}
    # <H> = -0.201996915076406 for the 24-qubit instance
    if 24 in vqe:
        assert vqe[24]["value"] == pytest.approx(-0.201996915076406, abs=1e-14)
    assert vqe[8]["gates"] == 92 and vqe[12]["params"] == 96
