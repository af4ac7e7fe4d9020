"""Generated tile-pass kernels (qsv_tile_jit.cuh, compiled by NVRTC in
qsv_jit.cu) against the C oracle: random circuits mixing every gate kind,
both register variants, every tile size, controls on register / thread /
tile bits, shared-memory phases; plus the compile cache (a VQE parameter
update reuses the compiled kernels) and the auto mode (interpreter on the
first run, generated kernels from the second)."""

import numpy as np
import pytest

import paper_2011_13524_b200 as qs
from paper_2011_13524_b200 import workloads
from paper_2011_13524_b200._circuit import circuit_records
from paper_2011_13524_b200._lib import jit_stats

from oracle import c_oracle, qsim_oracle as orc
from test_gpu_tiles import layered_circuit, qft_circuit, random_circuit

pytestmark = pytest.mark.gpu


def _run_vs_oracle(circ, n, seed, runs=1):
    st = qs.QuantumState(n)
    st.set_Haar_random_state(seed)
    for _ in range(runs):
        circ.update_quantum_state(st)
    ref = orc.haar_state(n, seed)
    recs = circuit_records(circ)
    for _ in range(runs):
        c_oracle.run_records(ref, n, recs)
    return float(np.max(np.abs(st.get_vector() - ref)))


@pytest.mark.parametrize("variant", ["4", "5"])
@pytest.mark.parametrize("n,L,seed", [(7, 6, 0), (10, 8, 1), (13, 12, 2), (16, 10, 3),
                                      (18, 12, 4), (20, 11, 5)])
def test_jit_random_circuits_match_oracle(n, L, seed, variant, monkeypatch):
    monkeypatch.setenv("QSV_TILE_VARIANT", variant)
    for circ in (random_circuit(n, 150, seed), layered_circuit(n, 6, seed)):
        circ.set_plan_options(tile_qubits=L, jit=2)
        stats = circ.program_stats()
        assert stats["num_tile_passes"] >= 1
        assert stats["num_jit_passes"] == stats["num_tile_passes"], stats
        err = _run_vs_oracle(circ, n, seed, runs=2)
        assert err <= 1e-12, (err, stats)


@pytest.mark.parametrize("n,L", [(14, 12), (19, 10)])
def test_jit_controlled_phases(n, L):
    circ = qft_circuit(n, inverse_bits=1)
    circ.set_plan_options(tile_qubits=L, jit=2)
    assert circ.program_stats()["num_jit_passes"] >= 1
    assert _run_vs_oracle(circ, n, n) <= 1e-12


def test_jit_benchmark_circuits():
    """cz-ladder (real frames, merged flushes) and cnot-ring (complex 2x2,
    controlled swaps) at n=22 through generated kernels."""
    for circ, n in ((workloads.generate_cz_ladder(22, 8, seed=1), 22),
                    (workloads.generate_cnot_ring(20, seed=2), 20)):
        circ.set_plan_options(jit=2)
        st = circ.program_stats()
        assert st["num_jit_passes"] == st["num_tile_passes"] >= 1, st
        assert _run_vs_oracle(circ, n, 3) <= 1e-12


def test_jit_auto_mode_and_cache():
    """Default jit=1: the first run uses the interpreter, the second the
    generated kernels (same result); a parameter update with new angles
    keeps the structure, so the recompiled program finds every pass kernel
    in the in-process cache (no new NVRTC compile)."""
    n = 16
    circ = workloads.vqe_ansatz(n)
    st = qs.QuantumState(n)
    circ.update_quantum_state(st)
    assert circ.program_stats()["num_jit_passes"] == 0
    first = st.get_vector()
    st.set_zero_state()
    circ.update_quantum_state(st)
    stats = circ.program_stats()
    assert stats["num_jit_passes"] == stats["num_tile_passes"] >= 1
    assert np.max(np.abs(st.get_vector() - first)) <= 1e-13
    before = jit_stats()
    rng = np.random.default_rng(3)
    for k in range(circ.get_parameter_count()):
        circ.set_parameter(k, float(rng.uniform(0, 2 * np.pi)))
    st.set_zero_state()
    circ.update_quantum_state(st)
    after = jit_stats()
    assert after["compiles"] == before["compiles"]
    assert circ.program_stats()["num_jit_passes"] == stats["num_tile_passes"]
    ref = c_oracle.run_records(orc.zero_state(n), n, circuit_records(circ))
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_jit_off_keeps_interpreter():
    circ = workloads.generate_cz_ladder(14, 4, seed=2)
    circ.set_plan_options(jit=0)
    st = qs.QuantumState(14)
    circ.update_quantum_state(st)
    circ.update_quantum_state(st)
    assert circ.program_stats()["num_jit_passes"] == 0
