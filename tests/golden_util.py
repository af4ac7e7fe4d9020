"""Helpers to read the golden fixtures produced by tests/golden/make_golden.py."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cx(v):
    return complex(v[0], v[1])


def load_gate_cases():
    with open(os.path.join(GOLDEN, "gates.json")) as fh:
        cases = json.load(fh)
    outs = np.load(os.path.join(GOLDEN, "gates.npz"))
    return cases, outs


def record_from_json(rec):
    """Golden kernel record -> oracle record tuple."""
    ctl = tuple((int(q), int(v)) for q, v in rec["controls"])
    t = tuple(rec["targets"])
    kind = rec["kind"]
    if kind == "dense":
        mat = np.array([[_cx(v) for v in row] for row in rec["matrix"]], dtype=np.complex128)
        return ("dense", t, mat, ctl)
    if kind == "diag":
        return ("diag", t, np.array([_cx(v) for v in rec["diag"]], dtype=np.complex128), ctl)
    if kind == "pauli":
        return ("pauli", t, tuple(rec["ids"]), ctl)
    if kind == "pauli_rot":
        return ("pauli_rot", t, tuple(rec["ids"]), float(rec["angle"]), ctl)
    raise ValueError(kind)


def build_gate(case, gate_mod):
    """Rebuild a golden case through a Qulacs-style gate module (ours)."""
    f, a = case["factory"], case["args"]
    if f == "DiagonalMatrix":
        g = gate_mod.DiagonalMatrix(a[0], [_cx(v) for v in a[1]])
    else:
        g = getattr(gate_mod, f)(*a)
    for q, v in case["controls"]:
        g.add_control_qubit(q, v)
    return g


def load_circuits():
    with open(os.path.join(GOLDEN, "circuits.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLDEN, "circuits.npz"))


def load_observables():
    with open(os.path.join(GOLDEN, "observables.json")) as fh:
        return json.load(fh)


def load_haar():
    return np.load(os.path.join(GOLDEN, "haar.npz"))


# ------------------------------------------------------------ quantum maps
def map_circuit_specs():
    """Noise / measurement circuits (shared by make_golden.py, which builds
    them with the reference bindings, and the tests, which build them with
    ours): (name, n, haar_seed, run_seeds, spec).  A spec item is
    (factory, args); "Adaptive" args are (inner_item, register, value)."""
    import math
    s = math.sqrt
    kraus_bitflip = [("DenseMatrix", [[1], [[s(0.7), 0], [0, s(0.7)]]]),
                     ("DenseMatrix", [[1], [[0, s(0.3)], [s(0.3), 0]]])]
    kraus_ctl = [("DenseMatrix", [[0, 2], [[1, 0, 0, 0], [0, s(0.5), 0, 0],
                                           [0, 0, 1, 0], [0, 0, 0, s(0.5)]]]),
                 ("DenseMatrix", [[0, 2], [[0, s(0.5), 0, 0], [0, 0, 0, 0],
                                           [0, 0, 0, s(0.5)], [0, 0, 0, 0]]])]
    noisy = [("H", [0]), ("RX", [1, 0.7]), ("CNOT", [0, 2]),
             ("AmplitudeDampingNoise", [0, 0.35]), ("DepolarizingNoise", [1, 0.4]),
             ("Measurement", [2, 0]), ("BitFlipNoise", [3, 0.5]), ("DephasingNoise", [0, 0.5]),
             ("Adaptive", [("X", [1]), 0, 1]), ("TwoQubitDepolarizingNoise", [1, 3, 0.6]),
             ("CPTP", [kraus_bitflip]), ("Instrument", [kraus_ctl, 1]), ("RY", [2, 1.1]),
             ("Measurement", [0, 2]), ("Probabilistic", [[0.2, 0.5], [("Y", [3]), ("S", [1])]]),
             ("Adaptive", [("Z", [3]), 2, 0])]
    meas = [("H", [q]) for q in range(5)] + [("CZ", [0, 1]), ("CZ", [2, 3])] + \
           [("Measurement", [q, q]) for q in range(5)]
    return [("noisy4", 4, 3, [0, 1, 2, 3, 11, 12, 13, 14], noisy),
            ("measure5", 5, 8, [0, 5, 6, 7], meas)]


def build_map_gate(item, gm):
    fac, args = item
    if fac == "Adaptive":
        inner, reg, val = args
        return gm.Adaptive(build_map_gate(inner, gm),
                           lambda regs, r=reg, v=val: len(regs) > r and regs[r] == v)
    if fac in ("CPTP",):
        return gm.CPTP([build_map_gate(k, gm) for k in args[0]])
    if fac == "Instrument":
        return gm.Instrument([build_map_gate(k, gm) for k in args[0]], args[1])
    if fac == "Probabilistic":
        return gm.Probabilistic(args[0], [build_map_gate(k, gm) for k in args[1]])
    return getattr(gm, fac)(*args)


def build_map_circuit(n, spec, circuit_cls, gm):
    c = circuit_cls(n)
    for item in spec:
        c.add_gate(build_map_gate(item, gm))
    return c


def load_maps():
    with open(os.path.join(GOLDEN, "maps.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLDEN, "maps.npz"))


# ---------------------------------------------------------- density matrices
def density_specs():
    """(name, n, haar_seed or None, [(core factory, args), ...]) applied with
    ``apply_density``; None starts from DensityMatrix(n) = |0><0|."""
    ops = [("H", [0]), ("CNOT", [0, 2]), ("RX", [1, 0.4]), ("AmplitudeDampingNoise", [0, 0.3]),
           ("DepolarizingNoise", [1, 0.2]), ("TwoQubitDepolarizingNoise", [0, 2, 0.1]),
           ("RZ", [2, -1.3]), ("BitFlipNoise", [2, 0.25]), ("T", [1]), ("DephasingNoise", [0, 0.4])]
    return [("mixed3", 3, 5, ops),
            ("zero2", 2, None, [("X", [1]), ("H", [0]), ("AmplitudeDampingNoise", [1, 0.6])]),
            ("mixed5", 5, 9, ops + [("CZ", [3, 4]), ("DepolarizingNoise", [4, 0.5])])]


def core_factory(name, gates_mod, maps_mod=None):
    f = getattr(gates_mod, name, None)
    if f is None and maps_mod is not None:
        f = getattr(maps_mod, name)
    return f


def load_density():
    with open(os.path.join(GOLDEN, "density.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLDEN, "density.npz"))


CFG1_SAMPLES = 4096
CFG1_PROJ = 16


def cfg1_digest(psi):
    """Size-independent digest of a 16-qubit state (see make_golden.make_cfg1):
    amplitudes at fixed indices, projections onto fixed Gaussian vectors,
    squared norm, <Z_q> for every qubit."""
    psi = np.asarray(psi, dtype=np.complex128)
    n = psi.size.bit_length() - 1
    rng = np.random.default_rng(1601)
    idx = np.sort(rng.choice(psi.size, CFG1_SAMPLES, replace=False))
    w = rng.standard_normal((CFG1_PROJ, psi.size)) + 1j * rng.standard_normal((CFG1_PROJ, psi.size))
    p = np.abs(psi) ** 2
    x = np.arange(psi.size)
    z = np.array([np.sum(p * (1 - 2 * ((x >> q) & 1))) for q in range(n)])
    return {"idx": idx, "amps": psi[idx], "proj": w.conj() @ psi,
            "norm2": np.array([np.sum(p)]), "z": z}


def load_cfg1():
    with open(os.path.join(GOLDEN, "cfg1.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLDEN, "cfg1.npz"))
