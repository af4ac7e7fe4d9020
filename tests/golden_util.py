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
