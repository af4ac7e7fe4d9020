"""B200-native state-vector engine with the Qulacs-style API of the
reference package (arXiv 2011.13524 hot path).

Drop-in names (reference ``qsimbind``): ``QuantumState`` (= ``StateVector``),
``QuantumCircuit``, ``ParametricQuantumCircuit``, ``Observable``,
``GeneralQuantumOperator``, ``PauliOperator``, ``QuantumGateBase`` and the
submodules ``gate``, ``circuit``, ``state``, ``quantum_operator``.  All
amplitudes live in GPU memory and every operation runs through libqsv.so
(hand-written sm_100a CUDA behind the C ABI in include/qsv.h); there is no
CPU fallback.
"""

from __future__ import annotations

from ._lib import device_count  # noqa: F401  (fails loudly if libqsv.so is missing)
from ._handles import QuantumGateBase, unwrap
from ._state import QuantumState, StateVector
from ._circuit import ParametricQuantumCircuit, QuantumCircuit
from ._observable import GeneralQuantumOperator, Observable, PauliOperator
from ._density import DensityMatrix, density_from_pure
from . import circuit, gate, quantum_operator, state  # noqa: F401

__all__ = [
    "QuantumState", "StateVector", "QuantumCircuit", "ParametricQuantumCircuit",
    "Observable", "PauliOperator", "GeneralQuantumOperator", "QuantumGateBase",
    "unwrap", "gate", "circuit", "state", "quantum_operator", "device_count",
    "DensityMatrix", "density_from_pure",
]

__version__ = "0.1.0"
