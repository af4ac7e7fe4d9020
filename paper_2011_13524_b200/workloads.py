"""Benchmark circuit generators (reference ``bench.py:28-81``).

Same gate sequence and the same PCG64 angle stream
(``default_rng(seed).random() * 2 pi`` in gate order) as the reference
generators, so a seed reproduces the reference circuit exactly.
"""

from __future__ import annotations

import numpy as np

from . import _gates as G
from ._circuit import Circuit, ParametricCircuit, QuantumCircuit, ParametricQuantumCircuit
from ._observable import HermitianOperator, Observable


def _wrap_circuit(core, cls=QuantumCircuit):
    out = cls.__new__(cls)
    out._core = core
    return out


def generate_cz_ladder(num_qubits: int, depth: int, seed=None, commuting=False):
    """depth+1 rotation layers (RZ RX RZ per qubit, or a single RZ when
    commuting) separated by CZ(q, q+1) for q = layer parity, step 2."""
    if num_qubits < 2:
        raise ValueError("the CZ ladder needs at least 2 qubits")
    if depth < 0:
        raise ValueError("depth must be non-negative")
    rng = np.random.default_rng(seed)
    c = Circuit(num_qubits)
    two_pi = 2 * np.pi
    for layer in range(depth + 1):
        for q in range(num_qubits):
            c.add_gate(G.RZ(q, rng.random() * two_pi))
            if not commuting:
                c.add_gate(G.RX(q, rng.random() * two_pi))
                c.add_gate(G.RZ(q, rng.random() * two_pi))
        if layer < depth:
            for q in range(layer % 2, num_qubits - 1, 2):
                c.add_gate(G.CZ(q, q + 1))
    return _wrap_circuit(c)


def generate_cnot_ring(num_qubits: int, seed=None):
    """Eleven rotation layers (the first without its leading RZ, the last
    without its trailing RZ) with CNOT((q+1) % n, q) rings between them."""
    if num_qubits < 2:
        raise ValueError("the CNOT ring needs at least 2 qubits")
    rng = np.random.default_rng(seed)
    c = Circuit(num_qubits)
    two_pi = 2 * np.pi
    for layer in range(11):
        for q in range(num_qubits):
            if layer:
                c.add_gate(G.RZ(q, rng.random() * two_pi))
            c.add_gate(G.RX(q, rng.random() * two_pi))
            if layer != 10:
                c.add_gate(G.RZ(q, rng.random() * two_pi))
        if layer != 10:
            for q in range(num_qubits):
                c.add_gate(G.CNOT((q + 1) % num_qubits, q))
    return _wrap_circuit(c)


def vqe_ansatz(num_qubits: int, layers: int = 4, seed=0):
    """cfg3 ansatz: per layer ParametricRY then ParametricRZ
    on every qubit with rng.uniform(0, 2 pi) angles, then CNOT(i, i+1)."""
    rng = np.random.default_rng(seed)
    c = ParametricCircuit(num_qubits)
    for _ in range(layers):
        for i in range(num_qubits):
            c.add_parametric_gate(G.ParametricRY(i, rng.uniform(0, 2 * np.pi)))
            c.add_parametric_gate(G.ParametricRZ(i, rng.uniform(0, 2 * np.pi)))
        for i in range(num_qubits - 1):
            c.add_gate(G.CNOT(i, i + 1))
    return _wrap_circuit(c, ParametricQuantumCircuit)


def tfim_observable(num_qubits: int, j: float = 1.0, h: float = 0.5):
    """Transverse-field Ising: -J sum Z_i Z_{i+1} - h sum X_i (cfg3)."""
    obs = Observable.__new__(Observable)
    obs._core = HermitianOperator(num_qubits)
    for i in range(num_qubits - 1):
        obs._core.add_operator(-j, f"Z {i} Z {i + 1}")
    for i in range(num_qubits):
        obs._core.add_operator(-h, f"X {i}")
    return obs
