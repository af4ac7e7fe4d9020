"""Tile-pass engine (several gates per HBM sweep) against the per-gate path
and the C oracle on random circuits mixing every gate kind."""

import numpy as np
import pytest

import paper_2011_13524_b200 as qs
from paper_2011_13524_b200 import gate as qg
from paper_2011_13524_b200._circuit import circuit_records

from oracle import c_oracle, qsim_oracle as orc

pytestmark = pytest.mark.gpu


def random_circuit(n, ngates, seed, max_k=4):
    rng = np.random.default_rng(seed)
    c = qs.QuantumCircuit(n)
    for _ in range(ngates):
        kind = int(rng.integers(0, 10))
        perm = [int(v) for v in rng.permutation(n)]
        if kind == 0:
            g = qg.RandomUnitary([perm[0]], seed=int(rng.integers(1 << 30)))
        elif kind == 1:
            k = int(rng.integers(2, max_k + 1))
            g = qg.RandomUnitary(perm[:k], seed=int(rng.integers(1 << 30)))
        elif kind == 2:
            g = qg.CNOT(perm[0], perm[1])
        elif kind == 3:
            g = qg.CZ(perm[0], perm[1])
        elif kind == 4:
            g = qg.RZ(perm[0], float(rng.uniform(-7, 7)))
        elif kind == 5:
            g = qg.RX(perm[0], float(rng.uniform(-7, 7)))
        elif kind == 6:
            k = int(rng.integers(1, 4))
            g = qg.DiagonalMatrix(perm[:k], np.exp(1j * rng.uniform(0, 6, 1 << k)))
        elif kind == 7:
            k = int(rng.integers(1, 5))
            ids = [int(v) for v in rng.integers(1, 4, k)]
            g = qg.PauliRotation(perm[:k], ids, float(rng.uniform(-7, 7)))
        elif kind == 8:
            k = int(rng.integers(1, 4))
            g = qg.Pauli(perm[:k], [int(v) for v in rng.integers(1, 4, k)])
        else:
            g = qg.RandomUnitary([perm[0]], seed=int(rng.integers(1 << 30)))
            g.add_control_qubit(perm[1], int(rng.integers(2)))
            if rng.integers(2):
                g.add_control_qubit(perm[2], int(rng.integers(2)))
        c.add_gate(g)
    return c


@pytest.mark.parametrize("rf", [0, 1])
@pytest.mark.parametrize("n,L,seed", [(6, 6, 0), (9, 8, 1), (13, 12, 2), (14, 8, 3),
                                      (16, 12, 4), (18, 10, 5), (20, 12, 6)])
def test_tiles_match_oracle(n, L, seed, rf):
    circ = random_circuit(n, 160, seed)
    circ.set_plan_options(use_tiles=1, tile_qubits=L, real_frames=rf)
    stats = circ.program_stats()
    assert stats["num_tile_passes"] >= 1, stats
    st = qs.QuantumState(n)
    st.set_Haar_random_state(seed)
    circ.update_quantum_state(st)
    ref = orc.haar_state(n, seed)
    c_oracle.run_records(ref, n, circuit_records(circ))
    err = np.max(np.abs(st.get_vector() - ref))
    assert err <= 1e-12, (err, stats)


@pytest.mark.parametrize("fuse", [0, 1])
def test_tiles_equal_per_gate_path(fuse):
    n = 15
    circ = random_circuit(n, 300, 42)
    a, b = qs.QuantumState(n), qs.QuantumState(n)
    a.set_Haar_random_state(1)
    b.set_Haar_random_state(1)
    circ.set_plan_options(use_tiles=0, fuse=0)
    circ.update_quantum_state(a)
    circ.set_plan_options(use_tiles=1, fuse=fuse)
    circ.update_quantum_state(b)
    assert np.max(np.abs(a.get_vector() - b.get_vector())) <= 1e-12


def test_tiles_cz_ladder_pass_count_and_parity():
    """cz-ladder: diagonal gates (RZ, CZ) never force a tile qubit, so a
    20-qubit, depth-8 ladder needs only a handful of passes."""
    from paper_2011_13524_b200 import workloads
    n = 20
    circ = workloads.generate_cz_ladder(n, 8, seed=1)
    stats = circ.program_stats()
    assert stats["num_tile_passes"] <= 12, stats
    st = qs.QuantumState(n)
    st.set_Haar_random_state(3)
    circ.update_quantum_state(st)
    ref = orc.haar_state(n, 3)
    c_oracle.run_records(ref, n, circuit_records(circ))
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def layered_circuit(n, layers, seed):
    """Random-circuit shape the real-frame planner targets: layers of random
    1-qubit unitaries / rotations, then CZ / CNOT / controlled-phase ladders."""
    rng = np.random.default_rng(seed)
    c = qs.QuantumCircuit(n)
    for layer in range(layers):
        for q in range(n):
            r = int(rng.integers(4))
            if r == 0:
                c.add_gate(qg.RandomUnitary([q], seed=int(rng.integers(1 << 30))))
            elif r == 1:
                c.add_gate(qg.RZ(q, float(rng.uniform(-7, 7))))
                c.add_gate(qg.RX(q, float(rng.uniform(-7, 7))))
                c.add_gate(qg.RZ(q, float(rng.uniform(-7, 7))))
            elif r == 2:
                c.add_gate(qg.H(q))
                c.add_gate(qg.T(q))
            else:
                c.add_gate(qg.RX(q, float(rng.uniform(-7, 7))))
        for q in range(layer % 2, n - 1, 2):
            r = int(rng.integers(4))
            a, b = (q, q + 1) if rng.integers(2) else (q + 1, q)
            if r == 0:
                c.add_gate(qg.CNOT(a, b))
            elif r == 1:
                g = qg.DiagonalMatrix([b], [1, np.exp(1j * rng.uniform(0, 6))])
                g.add_control_qubit(a, 1)
                c.add_gate(g)
            else:
                c.add_gate(qg.CZ(a, b))
        if layer % 3 == 2:
            c.add_gate(qg.Z(int(rng.integers(n))))
            c.add_gate(qg.S(int(rng.integers(n))))
    return c


@pytest.mark.parametrize("n,L,layers,seed", [(7, 6, 6, 0), (12, 8, 8, 1), (16, 12, 10, 2),
                                             (20, 12, 12, 3), (22, 11, 6, 4)])
def test_real_frames_layered_circuits(n, L, layers, seed):
    circ = layered_circuit(n, layers, seed)
    ref = orc.haar_state(n, seed)
    c_oracle.run_records(ref, n, circuit_records(circ))
    for rf in (1, 0):
        circ.set_plan_options(use_tiles=1, tile_qubits=L, real_frames=rf)
        st = qs.QuantumState(n)
        st.set_Haar_random_state(seed)
        circ.update_quantum_state(st)
        err = np.max(np.abs(st.get_vector() - ref))
        assert err <= 1e-12, (rf, err, circ.program_stats())


def test_real_frames_benchmark_circuits():
    from paper_2011_13524_b200 import workloads
    n = 20
    for circ in (workloads.generate_cz_ladder(n, 6, seed=2), workloads.generate_cnot_ring(n, seed=2)):
        ref = orc.haar_state(n, 9)
        c_oracle.run_records(ref, n, circuit_records(circ))
        for rf in (1, 0):
            circ.set_plan_options(real_frames=rf)
            st = qs.QuantumState(n)
            st.set_Haar_random_state(9)
            circ.update_quantum_state(st)
            assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12, rf


@pytest.mark.parametrize("variant", ["4", "5"])
def test_both_kernel_variants(variant, monkeypatch):
    """The planner picks the 16- or 32-amplitude tile kernel per program;
    force each and check parity on circuits that exercise every op kind."""
    monkeypatch.setenv("QSV_TILE_VARIANT", variant)
    for n, L, seed in ((12, 10, 7), (17, 12, 8)):
        for circ in (layered_circuit(n, 5, seed), random_circuit(n, 120, seed)):
            circ.set_plan_options(tile_qubits=L)
            st = qs.QuantumState(n)
            st.set_Haar_random_state(seed)
            circ.update_quantum_state(st)
            ref = orc.haar_state(n, seed)
            c_oracle.run_records(ref, n, circuit_records(circ))
            assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12, (variant, n)


def qft_circuit(n, inverse_bits=0):
    import math
    c = qs.QuantumCircuit(n)
    for i in range(n - 1, -1, -1):
        c.add_gate(qg.H(i))
        for j in range(i - 1, -1, -1):
            g = qg.DiagonalMatrix([i], [1, np.exp(1j * math.pi / (1 << (i - j)))])
            g.add_control_qubit(j, 1 if (j + inverse_bits) % 3 else 0)
            c.add_gate(g)
    return c


@pytest.mark.parametrize("n,L", [(14, 12), (18, 10), (21, 12)])
def test_qft_controlled_phases_merge(n, L):
    """Controlled phases between register, thread and tile bits merge into
    per-thread scalar / per-slot phase rules (T_PHASES); control value 0
    included."""
    circ = qft_circuit(n, inverse_bits=1)
    circ.set_plan_options(tile_qubits=L)
    st = qs.QuantumState(n)
    st.set_Haar_random_state(n)
    circ.update_quantum_state(st)
    ref = orc.haar_state(n, n)
    c_oracle.run_records(ref, n, circuit_records(circ))
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_planner_fuzz():
    """Random circuits (every gate kind, random widths) under random plan
    options and forced kernel variants, against the C oracle."""
    import os
    rng = np.random.default_rng(int(os.environ.get("QSV_FUZZ_SEED", "2024")))
    for case in range(int(os.environ.get("QSV_FUZZ_CASES", "40"))):
        n = int(rng.integers(6, 19))
        L = int(rng.integers(6, 13))
        ng = int(rng.integers(20, 200))
        seed = int(rng.integers(1 << 30))
        circ = random_circuit(n, ng, seed, max_k=int(rng.integers(2, 5))) if case % 2 \
            else layered_circuit(n, int(rng.integers(2, 8)), seed)
        if case % 5 == 4:
            L = 0  # the planner's own choice (n = 12..18: 8-amplitude kernel)
        opts = dict(tile_qubits=L, real_frames=int(rng.integers(2)), fuse=int(rng.integers(2)),
                    use_graph=int(rng.integers(2)))
        variant = ("", "3", "4", "5")[int(rng.integers(4))]  # r3 caps tiles at 11 qubits
        if variant:
            os.environ["QSV_TILE_VARIANT"] = variant
        try:
            circ.set_plan_options(**opts)
            st = qs.QuantumState(n)
            st.set_Haar_random_state(seed % 1000)
            circ.update_quantum_state(st)
            circ.update_quantum_state(st)  # second run: CUDA graph replay
        finally:
            os.environ.pop("QSV_TILE_VARIANT", None)
        ref = orc.haar_state(n, seed % 1000)
        recs = circuit_records(circ)
        c_oracle.run_records(ref, n, recs)
        c_oracle.run_records(ref, n, recs)
        err = np.max(np.abs(st.get_vector() - ref))
        assert err <= 1e-12, (case, n, L, ng, opts, variant, err)
