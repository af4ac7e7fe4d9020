"""The reference's core-level names (``qsimcore``, pkg/src/qsimcore/__init__.py)
on the GPU engine, for scripts written against the core package rather than
the Qulacs-named bindings:

    import paper_2011_13524_b200.core as qsimcore

Gates, maps, circuits, the optimizer passes, observables, serialization,
state utilities and the benchmark generators keep the core names and
signatures.  Differences: ``StateVector.amplitudes`` is a host copy of the
device buffer (assign to it, or ``load``, to change the state); the thread
knobs of ``qsimcore.config`` have no GPU equivalent.
"""

from __future__ import annotations

from ._circuit import Circuit, ParametricCircuit
from ._density import DensityMatrix, density_from_pure
from ._gates import (CNOT, CZ, FREDKIN, P0, P1, SWAP, TOFFOLI, BasicGate, DenseGate,  # noqa: F401
                     DiagonalGate, H, Identity, ParametricPauliRotation, ParametricRX,
                     ParametricRY, ParametricRZ, PauliGate, PauliRotationGate, PermutationGate,
                     QuantumGate, RandomUnitary, RX, RY, RZ, S, Sdag, SparseGate, T, Tdag, U1,
                     U2, U3, X, Y, Z, expanded_matrix, merge, sqrtX, sqrtXdag, sqrtY, sqrtYdag)
from ._maps import (AdaptiveGate, AmplitudeDampingNoise, BitFlipNoise, CptpMap,  # noqa: F401
                    DephasingNoise, DepolarizingNoise, Instrument, Measurement,
                    ProbabilisticMap, TwoQubitDepolarizingNoise)
from ._observable import (GeneralOperator, HermitianOperator, Observable,  # noqa: F401
                          PauliProduct, add_observable_rotation, parse_openfermion_text,
                          parse_pauli_string)
from ._optimizer import commutation_check, merge_all, optimize_heavy, optimize_light  # noqa: F401
from ._state import (WILDCARD, StateVector, drop_qubit, inner_product,  # noqa: F401
                     permutate_qubit, tensor_product)
from .serialize import (CircuitFormatError, circuit_from_dict, circuit_to_dict,  # noqa: F401
                        dump_circuit, gate_from_dict, gate_to_dict, load_circuit)
