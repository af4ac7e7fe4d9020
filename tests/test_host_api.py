"""CPU-only checks of the boundary and the host logic (no GPU calls)."""

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2011_13524_b200 import _lib, _optimizer
from paper_2011_13524_b200 import _gates as G
from paper_2011_13524_b200 import workloads
from paper_2011_13524_b200._circuit import circuit_records
from paper_2011_13524_b200._observable import parse_openfermion_text, parse_pauli_string

from oracle import qsim_oracle as orc
from golden_util import load_circuits, load_observables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qsv.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(qsv_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(qsv_op), offsetof(qsv_op, angle),
         offsetof(qsv_op, data), offsetof(qsv_op, nc), sizeof(qsv_plan_opts),
         sizeof(qsv_program_stats));
  return 0;
}}''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(_lib.QsvOp), _lib.QsvOp.angle.offset, _lib.QsvOp.data.offset,
            _lib.QsvOp.nc.offset, C.sizeof(_lib.QsvPlanOpts), C.sizeof(_lib.QsvProgramStats)]
    assert got == want


def test_state_creation_fails_loudly_without_gpu():
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    import paper_2011_13524_b200 as qs
    with pytest.raises(RuntimeError):
        qs.QuantumState(3)


def test_generators_match_oracle_generators():
    for n, d, s in ((5, 3, 1), (9, 2, 7)):
        ours = circuit_records(workloads.generate_cz_ladder(n, d, seed=s))
        ref = orc.cz_ladder_records(n, d, s)
        assert len(ours) == len(ref)
        for a, b in zip(ours, ref):
            assert a[0] == b[0] and tuple(a[1]) == tuple(b[1])
            if a[0] == "pauli_rot":
                assert a[3] == b[3]
    ours = circuit_records(workloads.generate_cnot_ring(7, seed=3))
    ref = orc.cnot_ring_records(7, 3)
    assert [(r[0], tuple(r[1])) for r in ours] == [(r[0], tuple(r[1])) for r in ref]
    assert all(workloads.generate_cnot_ring(n, seed=0).get_gate_count() == 41 * n
               for n in range(2, 12))


def test_optimizer_gate_counts_match_reference():
    meta, _ = load_circuits()
    for key, count in meta["optimizer_counts"].items():
        _, n, d, s, strat = key.split("/")
        c = workloads.generate_cz_ladder(int(n), int(d), seed=int(s))
        if strat == "light":
            _optimizer.optimize_light(c._core)
        else:
            _optimizer.optimize_heavy(c._core, int(strat))
        assert c.get_gate_count() == count, key


def test_optimized_circuits_match_reference_on_oracle():
    """Host optimizer output, executed by the oracle, equals the reference's
    optimized-circuit output."""
    meta, outs = load_circuits()
    for e in meta["circuits"]:
        if "opt" not in e:
            continue
        c = workloads.generate_cz_ladder(e["n"], e["depth"], seed=e["seed"])
        if e["opt"] == "light":
            _optimizer.optimize_light(c._core)
        else:
            _optimizer.optimize_heavy(c._core, e["opt"])
        assert c.get_gate_count() == e["gate_count"]
        amps = orc.haar_state(e["n"], e["start_seed"])
        orc.run_records(amps, e["n"], circuit_records(c))
        assert np.max(np.abs(amps - outs[e["id"]])) <= 1e-12


def test_merge_and_expanded_matrix():
    m = G.merge(G.H(0), G.CNOT(0, 1)).gate_matrix()
    state = np.zeros(4, complex)
    state[0] = 1
    np.testing.assert_allclose(m @ state, np.array([1, 0, 0, 1]) / np.sqrt(2), atol=1e-15)
    a = G.merge(G.X(0), G.Z(0)).gate_matrix()
    np.testing.assert_allclose(a, G.Z(0).gate_matrix() @ G.X(0).gate_matrix(), atol=1e-15)
    assert G.merge(G.CNOT(0, 1), G.RZ(1, 0.3)).controls == ()
    with pytest.raises(ValueError):
        G.merge(G.ParametricRX(0, 0.1), G.H(0))


def test_validation_errors():
    with pytest.raises(ValueError):
        G.DenseGate([0, 1], [[0, 1], [1, 0]])
    with pytest.raises(ValueError):
        G.X(0).with_control(0, 1)
    with pytest.raises(ValueError):
        G.X(0).with_control(1, 1).with_control(1, 0)
    with pytest.raises(ValueError):
        G.PauliGate([0], [4])
    with pytest.raises(ValueError):
        G.PauliRotationGate([0], [1], float("nan"))
    with pytest.raises(ValueError):
        G.DiagonalGate([0, 1], [1, -1])
    with pytest.raises(ValueError):
        G.PermutationGate([0, 1], [0, 0, 1, 2])
    with pytest.raises(ValueError):
        G.SparseGate([0], [(0, 0, 1.0), (0, 0, 2.0)])
    assert G.DenseGate(3, np.eye(2)).targets == (3,)   # int target accepted


def test_pauli_parsing_and_openfermion():
    t = parse_pauli_string("X 0 Y 2 Z 4", 0.5)
    assert t.ops == ((0, 1), (2, 2), (4, 3))
    with pytest.raises(ValueError):
        parse_pauli_string("X")
    with pytest.raises(ValueError):
        parse_pauli_string("Q 0")
    text = load_observables()["hamiltonian_text"]
    op = parse_openfermion_text(text)
    assert op.num_qubits == 4 and op.get_term_count() == 15
    assert op.get_term(1).ops == ((0, 1), (1, 3), (2, 1))
    for bad in ("", "(1.0) [X0] junk (2.0) [Z0]", "(abc) [X0]", "(1.0) [W0]", "(1.0) [X0 X0]"):
        with pytest.raises(ValueError):
            parse_openfermion_text(bad)


def test_commutation_labels():
    assert _optimizer.commutation_check(G.RZ(0, 0.1), G.CZ(0, 1))
    assert not _optimizer.commutation_check(G.RX(0, 0.1), G.CZ(0, 1))
    assert _optimizer.commutation_check(G.CNOT(0, 1), G.RZ(0, 0.3))
    assert _optimizer.commutation_check(G.Identity(0), G.H(0))


def test_core_module_exports_reference_core_names():
    """paper_2011_13524_b200.core carries the reference's qsimcore names
    (pkg/src/qsimcore/__init__.py) for scripts written against the core."""
    import paper_2011_13524_b200.core as core
    names = ["AdaptiveGate", "AmplitudeDampingNoise", "BasicGate", "BitFlipNoise", "CNOT", "CZ",
             "Circuit", "CircuitFormatError", "CptpMap", "DenseGate", "DensityMatrix",
             "DephasingNoise", "DepolarizingNoise", "DiagonalGate", "FREDKIN", "GeneralOperator",
             "H", "Identity", "Instrument", "Measurement", "Observable", "P0", "P1",
             "ParametricCircuit", "ParametricPauliRotation", "ParametricRX", "ParametricRY",
             "ParametricRZ", "PauliGate", "PauliProduct", "PauliRotationGate", "PermutationGate",
             "ProbabilisticMap", "QuantumGate", "RX", "RY", "RZ", "RandomUnitary", "S", "SWAP",
             "Sdag", "SparseGate", "StateVector", "T", "TOFFOLI", "Tdag",
             "TwoQubitDepolarizingNoise", "U1", "U2", "U3", "WILDCARD", "X", "Y", "Z",
             "add_observable_rotation", "circuit_from_dict", "circuit_to_dict",
             "commutation_check", "density_from_pure", "drop_qubit", "dump_circuit",
             "gate_from_dict", "gate_to_dict", "inner_product", "load_circuit", "merge",
             "merge_all", "optimize_heavy", "optimize_light", "parse_openfermion_text",
             "parse_pauli_string", "permutate_qubit", "sqrtX", "sqrtXdag", "sqrtY", "sqrtYdag",
             "tensor_product"]
    missing = [n for n in names if not hasattr(core, n)]
    assert not missing, missing


def _core(circ):
    return circ._core if hasattr(circ, "_core") else circ


def test_small_state_tile_size_choice(monkeypatch):
    """n <= 20: the planner keeps the cheapest of the L = 10/11/12 plans
    (qsv_tile_select.cu); under generated kernels n = 12..18 take the
    8-amplitude kernel with 10-qubit (n <= 16) or 11-qubit tiles; larger
    states and explicit tile sizes are unchanged."""
    for n, expect_l in ((16, 11), (20, 12)):
        c = _core(workloads.generate_cnot_ring(n, seed=1))
        auto = c.plan_stats(use_tiles=1, jit=0)
        per_l = {L: c.plan_stats(use_tiles=1, tile_qubits=L, jit=0) for L in (10, 11, 12)}
        assert auto == per_l[expect_l], (n, auto, per_l)
    assert (_core(workloads.generate_cnot_ring(20, seed=1)).plan_stats(use_tiles=1, jit=1)
            ["num_steps"] == 21)
    for n, l3 in ((14, 10), (16, 10), (18, 11)):
        c = _core(workloads.generate_cnot_ring(n, seed=1))
        auto = c.plan_stats(use_tiles=1, jit=1)
        monkeypatch.setenv("QSV_TILE_VARIANT", "3")
        forced = c.plan_stats(use_tiles=1, tile_qubits=l3, jit=1)
        monkeypatch.delenv("QSV_TILE_VARIANT")
        assert auto == forced, (n, auto, forced)
    c = _core(workloads.generate_cz_ladder(24, 4, seed=1))
    assert c.plan_stats(use_tiles=1) == c.plan_stats(use_tiles=1, tile_qubits=12)


def test_tile_set_search_pass_counts():
    """The planner's tile-set search (multi-start + one pass of lookahead,
    the fewer-pass plan kept; qsv_tile_impl.cuh select_pass / qsv_tile_select.cu)
    packs the benchmark circuits into at most these many HBM sweeps (greedy:
    cz-ladder(30) 22, VQE(24) 8)."""
    for circ, most in ((workloads.generate_cz_ladder(30, 20, seed=1), 18),
                       (workloads.generate_cz_ladder(28, 20, seed=1), 16),
                       (workloads.vqe_ansatz(24), 5)):
        st = _core(circ).plan_stats()
        assert st["num_tile_passes"] <= most, st


def test_parametric_replan_replays_the_same_plan():
    """New angles keep the pass structure: the recorded pass selections are
    replayed (structure-keyed cache) and give the plan a fresh search gives."""
    import numpy as np
    circ = workloads.vqe_ansatz(20)
    first = _core(circ).plan_stats()
    rng = np.random.default_rng(4)
    for _ in range(3):
        for k in range(circ.get_parameter_count()):
            circ.set_parameter(k, float(rng.uniform(0, 2 * np.pi)))
        again = _core(circ).plan_stats()
        assert again["num_tile_passes"] == first["num_tile_passes"]
        assert again["num_steps"] == first["num_steps"]
        assert again["hbm_bytes"] == first["hbm_bytes"]
