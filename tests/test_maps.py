"""Quantum maps: CPTP channels, instruments,
probabilistic / adaptive gates, noise channels and measurement on the GPU
state.

Golden fixtures (tests/golden/maps.*) are the reference bindings' own
outputs for seeded noise circuits (tests/golden/make_golden.py).  The CPU
tests pin the oracle's map restatement (oracle/qsim_oracle.py) to them; the
GPU tests check that the engine picks the same branches (same numpy draws)
and reaches the same states (<= 1e-12) and classical registers.
"""

import numpy as np
import pytest

from oracle import qsim_oracle as orc
from golden_util import build_map_circuit, load_maps, map_circuit_specs


def _ours():
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import gate as qg
    return qs, qg


def _spec(name):
    for nm, n, hseed, seeds, spec in map_circuit_specs():
        if nm == name:
            return n, hseed, spec
    raise KeyError(name)


def test_oracle_maps_match_reference():
    from paper_2011_13524_b200._circuit import circuit_records
    qs, qg = _ours()
    meta, outs = load_maps()
    for case in meta:
        n, hseed, spec = _spec(case["name"])
        circ = build_map_circuit(n, spec, qs.QuantumCircuit, qg)
        amps, cregs = orc.run_records_rng(orc.haar_state(n, hseed), n, circuit_records(circ),
                                          case["seed"])
        assert np.max(np.abs(amps - outs[case["key"]])) <= 1e-14, case["key"]
        assert (cregs + [0] * 6)[:6] == case["cregs"], case["key"]


def test_map_validation_errors():
    qs, qg = _ours()
    with pytest.raises(ValueError):
        qg.CPTP([qg.DenseMatrix([0], [[1, 0], [0, 0.5]])])  # not trace preserving
    with pytest.raises(ValueError):
        qg.Probabilistic([0.7, 0.6], [qg.X(0), qg.Z(0)])
    with pytest.raises(ValueError):
        qg.Probabilistic([0.5], [qg.X(0), qg.Z(0)])
    with pytest.raises(ValueError):
        qg.AmplitudeDampingNoise(0, 1.5)
    with pytest.raises(ValueError):
        qg.Instrument([qg.P0(0), qg.P1(0)], -1)
    # maps are fences for the optimizer and count in the depth
    c = qs.QuantumCircuit(2)
    c.add_gate(qg.H(0))
    c.add_gate(qg.Measurement(0, 0))
    c.add_gate(qg.H(0))
    assert c.calculate_depth() == 3
    from paper_2011_13524_b200.circuit import QuantumCircuitOptimizer
    QuantumCircuitOptimizer().optimize_light(c)
    assert c.get_gate_count() == 3


@pytest.mark.gpu
def test_gpu_maps_match_reference():
    qs, qg = _ours()
    meta, outs = load_maps()
    for case in meta:
        n, hseed, spec = _spec(case["name"])
        circ = build_map_circuit(n, spec, qs.QuantumCircuit, qg)
        st = qs.QuantumState(n)
        st.set_Haar_random_state(hseed)
        circ.update_quantum_state(st, seed=case["seed"])
        assert np.max(np.abs(st.get_vector() - outs[case["key"]])) <= 1e-12, case["key"]
        assert [st.get_classical_value(i) for i in range(6)] == case["cregs"], case["key"]


@pytest.mark.gpu
def test_gpu_maps_vs_oracle_larger():
    """Noise between random layers at n=14 (the branch norm kernel runs on a
    real sweep), every map kind, 5 seeds, against the oracle."""
    from paper_2011_13524_b200._circuit import circuit_records
    qs, qg = _ours()
    n = 14
    rng = np.random.default_rng(0)
    c = qs.QuantumCircuit(n)
    for layer in range(4):
        for q in range(n):
            c.add_gate(qg.RandomUnitary([q], seed=int(rng.integers(1 << 30))))
        for q in range(layer % 2, n - 1, 2):
            c.add_gate(qg.CNOT(q, q + 1))
        c.add_gate(qg.AmplitudeDampingNoise(int(rng.integers(n)), 0.4))
        c.add_gate(qg.DepolarizingNoise(int(rng.integers(n)), 0.5))
        c.add_gate(qg.TwoQubitDepolarizingNoise(3, 11, 0.7))
        c.add_gate(qg.Measurement(int(rng.integers(n)), layer))
        c.add_gate(qg.Adaptive(qg.X(5), lambda regs, k=layer: regs[k] == 1))
    wide = [qg.DenseMatrix([0, 1, 2, 3, 4, 5], np.eye(64) * np.sqrt(0.5)),
            qg.DenseMatrix([0, 1, 2, 3, 4, 5], np.diag(np.exp(1j * np.arange(64))) * np.sqrt(0.5))]
    c.add_gate(qg.CPTP(wide))  # 6-qubit Kraus: copy-apply-norm path
    for seed in range(5):
        st = qs.QuantumState(n)
        st.set_Haar_random_state(seed)
        c.update_quantum_state(st, seed=100 + seed)
        ref, cregs = orc.run_records_rng(orc.haar_state(n, seed), n, circuit_records(c),
                                         100 + seed)
        assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12, seed
        assert [st.get_classical_value(i) for i in range(4)] == (cregs + [0] * 4)[:4]
        assert abs(st.get_squared_norm() - 1.0) <= 1e-12


@pytest.mark.gpu
def test_gpu_amplitude_damping_statistics():
    """Branch frequencies follow |K_i psi|^2: decay of |1> with gamma = 0.3
    over 2000 seeds within 4 sigma (test_maps.py style 3-4 sigma checks)."""
    qs, qg = _ours()
    c = qs.QuantumCircuit(3)
    c.add_gate(qg.AmplitudeDampingNoise(1, 0.3))
    c.add_gate(qg.Measurement(1, 0))
    st = qs.QuantumState(3)
    ones = 0
    trials = 2000
    for seed in range(trials):
        st.set_computational_basis(2)
        c.update_quantum_state(st, seed=seed)
        ones += st.get_classical_value(0)
    p = 0.7
    sigma = np.sqrt(trials * p * (1 - p))
    assert abs(ones - trials * p) <= 4 * sigma, ones
