"""Density matrices on the GPU (reference ``DensityMatrix`` /
``density_from_pure``, state.py:195-222, and every ``apply_density``:
gates.py:102-106, maps.py:79-86, 149-158, 180-182).

A 2^h x 2^h matrix rho is held as a 2h-qubit device vector with element
(r, c) at index (r << h) | c.  Then

    U rho U^dag  =  (U on the row qubits h + t) (conj(U) on the column qubits t)

so a basic gate costs two ordinary gate launches of the state-vector
engine, and channels are sums of such terms (device copies, adds, scales).
The reference builds a sparse 4^h full-space operator per gate instead
(kernels.py:246-269).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, int_array, lib
from ._state import StateVector, tensor_product


class DensityMatrix:
    """Mixed state of ``num_qubits`` qubits, initialised to |0><0|."""

    __slots__ = ("num_qubits", "_sv", "__weakref__")

    def __init__(self, num_qubits: int, device: int = 0):
        if isinstance(num_qubits, bool) or not isinstance(num_qubits, (int, np.integer)) \
                or num_qubits < 1:
            raise ValueError(f"qubit count must be a positive integer, got {num_qubits!r}")
        self.num_qubits = int(num_qubits)
        self._sv = StateVector(2 * self.num_qubits, device)  # |0..0> = |0><0|

    @property
    def dim(self) -> int:
        return 1 << self.num_qubits

    def copy(self) -> "DensityMatrix":
        out = DensityMatrix.__new__(DensityMatrix)
        out.num_qubits = self.num_qubits
        out._sv = self._sv.copy()
        return out

    def get_trace(self) -> complex:
        out = (C.c_double * 2)()
        check(lib.qsv_trace_pairs(self._sv._handle(), out))
        return complex(out[0], out[1])

    @property
    def elements(self) -> np.ndarray:
        """Host copy of the 2^h x 2^h matrix."""
        return self._sv.get_vector().reshape(self.dim, self.dim)

    @elements.setter
    def elements(self, value) -> None:
        mat = np.asarray(value, dtype=np.complex128)
        if mat.shape != (self.dim, self.dim):
            raise ValueError(f"expected a {self.dim}x{self.dim} matrix, got {mat.shape}")
        self._sv.load(mat.reshape(-1))

    # -- helpers used by apply_density -----------------------------------
    def _accumulate(self, terms) -> None:
        """rho <- sum_k w_k * rho_k for (weight, DensityMatrix) terms."""
        acc = None
        for w, rho in terms:
            if w != 1.0:
                rho._sv.multiply_coef(w)
            if acc is None:
                acc = rho
            else:
                acc._sv.add_state(rho._sv)
        if acc is None:
            self._sv.multiply_coef(0.0)
        else:
            self._sv = acc._sv

    def __repr__(self) -> str:
        return f"DensityMatrix(qubits={self.num_qubits})"


def density_from_pure(state: StateVector) -> DensityMatrix:
    """|psi><psi| (state.py:219-222): kron(psi, conj(psi)) on the device."""
    n = state.get_qubit_count()
    conj = state.copy()
    check(lib.qsv_conj(conj._handle()))
    out = DensityMatrix.__new__(DensityMatrix)
    out.num_qubits = n
    out._sv = tensor_product(conj, state)  # conj(psi) on the column (low) qubits
    return out


def apply_basic_density(gate, rho: DensityMatrix) -> None:
    """U rho U^dag for a basic gate (gates.py:102-106): U on the row qubits,
    conj(U) on the column qubits, controls shifted / kept alike."""
    gate._check_width(rho.num_qubits)
    h = rho.num_qubits
    mat = np.ascontiguousarray(gate.gate_matrix(), dtype=np.complex128)
    cmat = np.ascontiguousarray(mat.conj())
    m = len(gate.targets)
    cq = [q for q, _ in gate.controls]
    cv = [v for _, v in gate.controls]
    handle = rho._sv._handle()
    check(lib.qsv_apply_dense(handle, int_array(t + h for t in gate.targets), m, mat.ctypes.data,
                              int_array(q + h for q in cq), int_array(cv), len(cq)))
    check(lib.qsv_apply_dense(handle, int_array(gate.targets), m, cmat.ctypes.data,
                              int_array(cq), int_array(cv), len(cq)))
