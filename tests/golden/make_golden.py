"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is mounted read-only there):

    PYTHONDONTWRITEBYTECODE=1 \
    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/bindings/src \
    python tests/golden/make_golden.py [--with-cfg3]

It imports ``qsimcore`` / ``qsimbind`` from /root/reference and writes small
fixtures next to this script:

* ``gates.json`` + ``gates.npz`` -- one case per (gate factory, qubits):
  factory name and args (to rebuild the gate through our API), the
  reference gate's kernel record (to drive the oracle), the Haar seed of the
  input state and the reference output state.
* ``circuits.json`` + ``circuits.npz`` -- benchmark-generator circuits
  (cnot-ring, cz-ladder), reference optimizer gate counts and final states.
* ``observables.json`` -- expectation values computed by the reference.
* ``haar.npz`` -- set_haar_random outputs (bit-exact pin of the PCG64 path).
* ``analysis.json`` + ``analysis.npz`` -- marginal probabilities, sampling
  results, tensor_product / permutate_qubit / drop_qubit outputs.
* ``cfg1.json`` + ``cfg1.npz`` -- cnot-ring(16) seeds 0..4 from |0> and from
  Haar starts (digests: sampled amplitudes, random projections, <Z_q>).

Nothing on the GPU box reads /root/reference; only these files travel.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

import qsimcore as core  # noqa: E402  (reference, from /root/reference)
from qsimcore import bench as rbench  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cpl(z):
    return [float(np.real(z)), float(np.imag(z))]


def record_of(gate):
    """Kernel record of a reference gate (which kernel it dispatches to)."""
    ctl = [[int(q), int(v)] for q, v in gate.controls]
    if isinstance(gate, core.PauliRotationGate):
        return {"kind": "pauli_rot", "targets": list(gate.targets),
                "ids": list(gate.pauli_ids), "angle": gate.angle, "controls": ctl}
    if isinstance(gate, core.PauliGate):
        return {"kind": "pauli", "targets": list(gate.targets),
                "ids": list(gate.pauli_ids), "controls": ctl}
    if isinstance(gate, core.DiagonalGate):
        return {"kind": "diag", "targets": list(gate.targets),
                "diag": [cpl(v) for v in gate.diag], "controls": ctl}
    # Dense, Sparse and Permutation kinds: the oracle applies the matrix
    return {"kind": "dense", "targets": list(gate.targets),
            "matrix": [[cpl(v) for v in row] for row in gate.gate_matrix()],
            "controls": ctl}


def gate_cases():
    rng = np.random.default_rng(20260101)
    cases = []

    def add(factory, args, n, controls=()):
        cases.append({"factory": factory, "args": args, "n": n,
                      "controls": [list(c) for c in controls],
                      "seed": int(rng.integers(1 << 30))})

    n = 6
    for t in range(n):
        for f in ("X", "Y", "Z", "H", "S", "Sdag", "T", "Tdag", "sqrtX", "sqrtXdag",
                  "sqrtY", "sqrtYdag", "P0", "P1", "Identity"):
            add(f, [t], n)
        for f in ("RX", "RY", "RZ", "U1"):
            add(f, [t, float(rng.uniform(-7, 7))], n)
        add("U2", [t, float(rng.uniform(-7, 7)), float(rng.uniform(-7, 7))], n)
        add("U3", [t] + [float(v) for v in rng.uniform(-7, 7, 3)], n)
        for c in range(n):
            if c != t:
                add("CNOT", [c, t], n)
                add("CZ", [c, t], n)
                add("SWAP", [c, t], n)
    for (a, b, c) in ((0, 1, 2), (5, 0, 3), (2, 4, 1), (1, 5, 0)):
        add("TOFFOLI", [a, b, c], n)
        add("FREDKIN", [a, b, c], n)
    # dense k-qubit gates, controlled variants, diagonal, Pauli products
    for k in (1, 2, 3, 4, 5):
        for _ in range(4):
            tg = [int(v) for v in rng.permutation(8)[:k]]
            add("RandomUnitary", [tg, int(rng.integers(1 << 20))], 8)
    for _ in range(6):
        perm = [int(v) for v in rng.permutation(8)]
        k = int(rng.integers(1, 3))
        tg, rest = perm[:k], perm[k:]
        nc = int(rng.integers(1, 3))
        ctl = [(rest[i], int(rng.integers(2))) for i in range(nc)]
        add("RandomUnitary", [tg, int(rng.integers(1 << 20))], 8, ctl)
    for _ in range(6):
        k = int(rng.integers(1, 4))
        tg = [int(v) for v in rng.permutation(7)[:k]]
        d = [cpl(np.exp(1j * v)) for v in rng.uniform(0, 2 * np.pi, 1 << k)]
        add("DiagonalMatrix", [tg, d], 7)
    for _ in range(8):
        k = int(rng.integers(1, 5))
        tg = [int(v) for v in rng.permutation(7)[:k]]
        ids = [int(v) for v in rng.integers(1, 4, k)]
        add("Pauli", [tg, ids], 7)
        add("PauliRotation", [tg, ids, float(rng.uniform(-7, 7))], 7)
    # controlled rotation (goes through the reference's dense path)
    add("RX", [2, 0.77], 6, [(4, 1)])
    add("RZ", [0, -1.3], 6, [(5, 0), (3, 1)])
    add("PauliRotation", [[1, 3], [1, 2], 0.41], 6, [(0, 1)])
    return cases


def build_ref_gate(case):
    f, a = case["factory"], case["args"]
    if f == "RandomUnitary":
        g = core.RandomUnitary(a[0], a[1])
    elif f == "DiagonalMatrix":
        g = core.DiagonalGate(a[0], [complex(*v) for v in a[1]])
    elif f == "Pauli":
        g = core.PauliGate(a[0], a[1])
    elif f == "PauliRotation":
        g = core.PauliRotationGate(a[0], a[1], a[2])
    else:
        g = getattr(core, f)(*a)
    for q, v in case["controls"]:
        g = g.with_control(q, v)
    return g


def make_gates():
    cases = gate_cases()
    outs = {}
    for i, case in enumerate(cases):
        g = build_ref_gate(case)
        st = core.StateVector(case["n"])
        st.set_haar_random(case["seed"])
        g.apply(st)
        case["id"] = f"g{i:04d}"
        case["record"] = record_of(g)
        outs[case["id"]] = st.get_vector()
    with open(os.path.join(HERE, "gates.json"), "w") as fh:
        json.dump(cases, fh)
    np.savez_compressed(os.path.join(HERE, "gates.npz"), **outs)
    print(f"gates: {len(cases)} cases")


def circuit_records(circ):
    return [record_of(g) for g in circ.gates]


def make_circuits():
    entries = []
    outs = {}

    def add(name, circ, start_seed, extra=None):
        st = core.StateVector(circ.num_qubits)
        if start_seed is not None:
            st.set_haar_random(start_seed)
        circ.update_state(st)
        key = f"c{len(entries):03d}"
        e = {"id": key, "name": name, "n": circ.num_qubits, "start_seed": start_seed,
             "gate_count": circ.get_gate_count(), "depth": circ.calculate_depth()}
        if extra:
            e.update(extra)
        entries.append(e)
        outs[key] = st.get_vector()

    for s in range(5):
        add("cnot-ring", rbench.generate_cnot_ring(10, seed=s), None, {"seed": s})
    add("cnot-ring", rbench.generate_cnot_ring(16, seed=0), None, {"seed": 0})
    add("cnot-ring", rbench.generate_cnot_ring(12, seed=3), 5, {"seed": 3})
    for (n, d, s) in ((8, 4, 1), (12, 6, 2), (14, 10, 1)):
        add("cz-ladder", rbench.generate_cz_ladder(n, d, seed=s), 11, {"depth": d, "seed": s})
        for strat in ("light", 2, 3, 4, 5):
            c = rbench.generate_cz_ladder(n, d, seed=s)
            if strat == "light":
                core.optimize_light(c)
            else:
                core.optimize_heavy(c, strat)
            add("cz-ladder", c, 11, {"depth": d, "seed": s, "opt": strat})
    add("cz-ladder-commuting", rbench.generate_cz_ladder(9, 5, seed=3, commuting=True), 2,
        {"depth": 5, "seed": 3})
    # optimizer gate counts at benchmark sizes (host-only, fast)
    counts = {}
    for (n, d, s) in ((30, 20, 1), (16, 10, 1)):
        for strat in ("light", 2, 4, 5):
            c = rbench.generate_cz_ladder(n, d, seed=s)
            if strat == "light":
                core.optimize_light(c)
            else:
                core.optimize_heavy(c, strat)
            counts[f"cz-ladder/{n}/{d}/{s}/{strat}"] = c.get_gate_count()
    with open(os.path.join(HERE, "circuits.json"), "w") as fh:
        json.dump({"circuits": entries, "optimizer_counts": counts}, fh)
    np.savez_compressed(os.path.join(HERE, "circuits.npz"), **outs)
    print(f"circuits: {len(entries)} cases; counts {counts}")


HAM_TEXT = """(-0.8126100000000005+0j) [] +
(0.04532175+0j) [X0 Z1 X2] +
(0.04532175+0j) [X0 Z1 X2 Z3] +
(0.04532175+0j) [Y0 Z1 Y2] +
(0.04532175+0j) [Y0 Z1 Y2 Z3] +
(0.17120100000000002+0j) [Z0] +
(0.17120100000000002+0j) [Z0 Z1] +
(0.165868+0j) [Z0 Z1 Z2] +
(0.165868+0j) [Z0 Z1 Z2 Z3] +
(0.12054625+0j) [Z0 Z2] +
(0.12054625+0j) [Z0 Z2 Z3] +
(0.16862325+0j) [Z1] +
(-0.22279649999999998+0j) [Z1 Z2 Z3] +
(0.17434925+0j) [Z1 Z3] +
(-0.22279649999999998+0j) [Z2]"""


def vqe_ansatz(n, layers=4, seed=0):
    """cfg3 ansatz: per layer ParametricRY/RZ on every qubit
    with rng.uniform(0, 2pi) angles, then CNOT(i, i+1)."""
    rng = np.random.default_rng(seed)
    c = core.ParametricCircuit(n)
    for _ in range(layers):
        for i in range(n):
            c.add_parametric_gate(core.ParametricRY(i, rng.uniform(0, 2 * np.pi)))
            c.add_parametric_gate(core.ParametricRZ(i, rng.uniform(0, 2 * np.pi)))
        for i in range(n - 1):
            c.add_gate(core.CNOT(i, i + 1))
    return c


def tfim(n):
    obs = core.Observable(n)
    for i in range(n - 1):
        obs.add_operator(-1.0, f"Z {i} Z {i + 1}")
    for i in range(n):
        obs.add_operator(-0.5, f"X {i}")
    return obs


def make_observables(with_cfg3):
    rng = np.random.default_rng(77)
    out = {"random": [], "tfim": [], "vqe": []}
    for trial in range(12):
        n = int(rng.integers(2, 9))
        terms = []
        obs = core.GeneralOperator(n)
        for _ in range(int(rng.integers(1, 8))):
            k = int(rng.integers(0, n + 1))
            qs = [int(v) for v in rng.permutation(n)[:k]]
            ops = [(q, int(rng.integers(1, 4))) for q in qs]
            coef = complex(rng.standard_normal(), rng.standard_normal() if trial % 2 else 0.0)
            obs.add_operator(core.PauliProduct(ops, coef))
            terms.append({"coef": cpl(coef), "ops": ops})
        seed = int(rng.integers(1 << 20))
        st = core.StateVector(n)
        st.set_haar_random(seed)
        bra = core.StateVector(n)
        bra.set_haar_random(seed + 1)
        out["random"].append({"n": n, "seed": seed, "terms": terms,
                              "value": cpl(obs.get_expectation_value(st)),
                              "transition": cpl(obs.get_transition_amplitude(bra, st))})
    for n, seed in ((6, 0), (10, 3), (12, 9)):
        st = core.StateVector(n)
        st.set_haar_random(seed)
        out["tfim"].append({"n": n, "seed": seed,
                            "value": tfim(n).get_expectation_value(st)})
    op = core.parse_openfermion_text(HAM_TEXT)
    out["hamiltonian_zero"] = cpl(op.get_expectation_value(core.StateVector(4)))
    st = core.StateVector(4)
    st.set_haar_random(5)
    out["hamiltonian_haar5"] = cpl(op.get_expectation_value(st))
    out["hamiltonian_text"] = HAM_TEXT
    sizes = [8, 12] + ([24] if with_cfg3 else [])
    for n in sizes:
        c = vqe_ansatz(n)
        st = core.StateVector(n)
        c.update_state(st)
        out["vqe"].append({"n": n, "gates": c.get_gate_count(),
                           "params": c.get_parameter_count(),
                           "value": tfim(n).get_expectation_value(st),
                           "norm": st.get_squared_norm()})
        print(f"vqe n={n}: {out['vqe'][-1]['value']!r}", flush=True)
    with open(os.path.join(HERE, "observables.json"), "w") as fh:
        json.dump(out, fh)


def make_haar():
    outs = {}
    for n, seed in ((1, 0), (4, 42), (10, 7), (13, 123)):
        st = core.StateVector(n)
        st.set_haar_random(seed)
        outs[f"n{n}_s{seed}"] = st.get_vector()
    np.savez_compressed(os.path.join(HERE, "haar.npz"), **outs)


def analysis_cases():
    """Inputs of the state-analysis fixtures (also rebuilt by the tests)."""
    marg = [(5, 3, [0, 1, 2, 2, 1]), (5, 3, [2, 2, 2, 2, 2]), (8, 11, [1, 0, 2, 2, 0, 1, 2, 2]),
            (12, 4, [2] * 6 + [1, 0, 1, 0, 2, 2]), (12, 4, [0] * 12), (13, 9, [2, 1] * 6 + [0])]
    samp = [(4, 1, 10, 0), (9, 2, 1000, 5), (13, 3, 4096, 77), (16, 8, 20000, 1), (16, 8, 0, 1)]
    kron = [(3, 1, 4, 2), (1, 5, 6, 6), (7, 3, 5, 4)]
    perm = [(4, 2, [3, 2, 1, 0]), (6, 5, [1, 4, 0, 5, 2, 3]), (11, 6, [10, 0, 9, 1, 8, 2, 7, 3, 6, 4, 5])]
    drop = [(4, 2, [1], [1]), (6, 3, [5, 0], [0, 1]), (10, 8, [2, 7, 4], [1, 1, 0]),
            (9, 1, [0, 1, 2, 3, 4, 5, 6, 7], [1, 0, 1, 1, 0, 0, 1, 0])]
    return {"marginal": marg, "sampling": samp, "tensor": kron, "permutate": perm, "drop": drop}


def make_analysis():
    cases = analysis_cases()
    meta = {"marginal": [], "sampling": [], "tensor": [], "permutate": [], "drop": []}
    outs = {}

    def haar(n, seed):
        st = core.StateVector(n)
        st.set_haar_random(seed)
        return st

    for i, (n, seed, pat) in enumerate(cases["marginal"]):
        meta["marginal"].append({"n": n, "seed": seed, "pattern": pat,
                                 "value": haar(n, seed).get_marginal_probability(pat)})
    for i, (n, seed, count, sseed) in enumerate(cases["sampling"]):
        meta["sampling"].append({"n": n, "seed": seed, "count": count, "sample_seed": sseed,
                                 "samples": haar(n, seed).sampling(count, seed=sseed)})
    for i, (n1, s1, n2, s2) in enumerate(cases["tensor"]):
        outs[f"tensor{i}"] = core.tensor_product(haar(n1, s1), haar(n2, s2)).get_vector()
        meta["tensor"].append({"n1": n1, "s1": s1, "n2": n2, "s2": s2, "key": f"tensor{i}"})
    for i, (n, seed, order) in enumerate(cases["permutate"]):
        outs[f"perm{i}"] = core.permutate_qubit(haar(n, seed), order).get_vector()
        meta["permutate"].append({"n": n, "seed": seed, "order": order, "key": f"perm{i}"})
    for i, (n, seed, tg, vals) in enumerate(cases["drop"]):
        outs[f"drop{i}"] = core.drop_qubit(haar(n, seed), tg, vals).get_vector()
        meta["drop"].append({"n": n, "seed": seed, "targets": tg, "values": vals,
                             "key": f"drop{i}"})
    with open(os.path.join(HERE, "analysis.json"), "w") as fh:
        json.dump(meta, fh)
    np.savez_compressed(os.path.join(HERE, "analysis.npz"), **outs)


def make_maps():
    """Noise / measurement circuits run by the reference bindings with a
    seed: final states and classical registers."""
    sys.path.insert(0, os.path.dirname(HERE))
    import qsimbind as qb
    from qsimbind import gate as qbg
    from golden_util import build_map_circuit, map_circuit_specs
    meta, outs = [], {}
    for name, n, hseed, seeds, spec in map_circuit_specs():
        for rs in seeds:
            c = build_map_circuit(n, spec, qb.QuantumCircuit, qbg)
            st = qb.StateVector(n)
            st.set_Haar_random_state(hseed)
            c.update_quantum_state(st, seed=rs)
            key = f"{name}_r{rs}"
            outs[key] = st.get_vector()
            meta.append({"name": name, "seed": rs, "key": key,
                         "cregs": [st.get_classical_value(i) for i in range(6)]})
    with open(os.path.join(HERE, "maps.json"), "w") as fh:
        json.dump(meta, fh)
    np.savez_compressed(os.path.join(HERE, "maps.npz"), **outs)


def make_density():
    """Density-matrix evolution through apply_density (reference core)."""
    sys.path.insert(0, os.path.dirname(HERE))
    from golden_util import core_factory, density_specs
    meta, outs = [], {}
    for name, n, hseed, ops in density_specs():
        if hseed is None:
            rho = core.DensityMatrix(n)
        else:
            st = core.StateVector(n)
            st.set_haar_random(hseed)
            rho = core.density_from_pure(st)
        for fac, args in ops:
            core_factory(fac, core)(*args).apply_density(rho)
        outs[name] = rho.elements
        tr = rho.get_trace()
        meta.append({"name": name, "trace": [tr.real, tr.imag]})
    with open(os.path.join(HERE, "density.json"), "w") as fh:
        json.dump(meta, fh)
    np.savez_compressed(os.path.join(HERE, "density.npz"), **outs)


def make_serialize():
    """A circuit touching every serialisable kind, written by the reference
    serializer, plus its run result (zero state, default_rng(7)) and the
    optimizer gate counts of the reference CLI passes."""
    from qsimcore import maps as M
    from qsimcore import serialize as S
    from qsimcore.optimizer import optimize_heavy, optimize_light
    c = core.Circuit(5)
    c.add_gate(core.H(0))
    c.add_gate(core.RX(1, 0.3))
    c.add_gate(core.U3(2, 0.1, 0.2, 0.3))
    c.add_gate(core.CNOT(0, 1))
    c.add_gate(core.TOFFOLI(0, 1, 3))
    c.add_gate(core.FREDKIN(4, 2, 3))
    c.add_gate(core.DenseGate([1, 3], np.linalg.qr(np.arange(16).reshape(4, 4) + 1j)[0],
                              [(0, 1)]))
    c.add_gate(core.SparseGate([2], [(0, 1, 1.0), (1, 0, 1j)]))
    c.add_gate(core.DiagonalGate([3, 4], [1, 1j, -1, -1j]))
    c.add_gate(core.PermutationGate([0, 2], [3, 0, 1, 2]))
    c.add_gate(core.PauliGate([1, 4], [2, 3]))
    c.add_gate(core.PauliRotationGate([0, 2, 3], [1, 2, 3], 0.77))
    c.add_gate(M.AmplitudeDampingNoise(2, 0.4))
    c.add_gate(M.Measurement(3, 1))
    c.add_gate(M.DepolarizingNoise(0, 0.3))
    c.add_gate(M.CptpMap([core.DenseGate([4], [[np.sqrt(0.5), 0], [0, np.sqrt(0.5)]]),
                          core.DenseGate([4], [[0, np.sqrt(0.5)], [np.sqrt(0.5), 0]])]))
    c.add_gate(core.RZ(4, -0.4))
    for q in range(5):
        c.add_gate(core.H(q))
    S.dump_circuit(c, os.path.join(HERE, "circuit_doc.json"))
    st = core.StateVector(5)
    c.update_state(st, rng=np.random.default_rng(7))
    counts = {}
    for label in ("light", "heavy2", "heavy3"):
        d = S.load_circuit(os.path.join(HERE, "circuit_doc.json"))
        if label == "light":
            optimize_light(d)
        else:
            optimize_heavy(d, int(label[-1]))
        counts[label] = d.get_gate_count()
    np.savez_compressed(os.path.join(HERE, "serialize.npz"), amplitudes=st.get_vector())
    with open(os.path.join(HERE, "serialize.json"), "w") as fh:
        json.dump({"cregs": list(st.classical_registers), "optimizer_counts": counts}, fh)


def make_cfg1():
    """cfg1: cnot-ring(16) seeds 0..4 from |0> and from a Haar
    start (seed 10 + s), run by the reference.  A 16-qubit state is 1 MiB,
    so each case keeps a digest instead of the full vector: the amplitudes at
    CFG1_SAMPLES fixed indices, CFG1_PROJ projections <w_k|psi> onto fixed
    PCG64 Gaussian vectors (every amplitude moves them), the squared norm
    and <Z_q> of every qubit (golden_util.cfg1_digest recomputes the same
    digest from any candidate state)."""
    sys.path.insert(0, os.path.dirname(HERE))
    from golden_util import cfg1_digest
    entries, outs = [], {}
    for s in range(5):
        for start in (None, 10 + s):
            circ = rbench.generate_cnot_ring(16, seed=s)
            st = core.StateVector(16)
            if start is not None:
                st.set_haar_random(start)
            circ.update_state(st)
            key = f"cfg1_s{s}_" + ("zero" if start is None else f"haar{start}")
            entries.append({"id": key, "seed": s, "start_seed": start,
                            "gate_count": circ.get_gate_count()})
            for k, v in cfg1_digest(st.get_vector()).items():
                outs[f"{key}/{k}"] = v
    with open(os.path.join(HERE, "cfg1.json"), "w") as fh:
        json.dump({"cases": entries}, fh)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **outs)
    print(f"cfg1: {len(entries)} cases")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-cfg3", action="store_true",
                    help="also run the 24-qubit VQE instance (~3 min)")
    ap.add_argument("--only", default=None, help="regenerate one fixture set (e.g. analysis)")
    args = ap.parse_args()
    if not core.__file__.startswith("/root/reference"):
        sys.exit("qsimcore must be imported from /root/reference")
    if args.only == "analysis":
        make_analysis()
        return
    if args.only == "maps":
        make_maps()
        return
    if args.only == "density":
        make_density()
        return
    if args.only == "serialize":
        make_serialize()
        return
    if args.only == "cfg1":
        make_cfg1()
        return
    make_haar()
    make_analysis()
    make_maps()
    make_density()
    make_serialize()
    make_gates()
    make_circuits()
    make_observables(args.with_cfg3)
    make_cfg1()


if __name__ == "__main__":
    main()
