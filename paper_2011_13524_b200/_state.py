"""Device-resident state vector (``QuantumState`` / ``StateVector``).

Mirrors the reference container (``qsimcore.StateVector``, state.py:22-133)
and its Qulacs-named handle (``qsimbind.StateVector``, _handles.py:55-112),
but the 2^n complex128 amplitudes live in HBM, owned by a libqsv handle that
is released deterministically with the Python object.  Host copies happen
only in ``load`` / ``get_vector`` / ``set_Haar_random_state``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, int_array, lib

WILDCARD = 2


def _check_count(n) -> int:
    if isinstance(n, bool) or not isinstance(n, (int, np.integer)) or n < 1:
        raise ValueError(f"qubit count must be a positive integer, got {n!r}")
    return int(n)


def haar_vector(num_qubits: int, seed=None) -> np.ndarray:
    """Host draw of the reference's Haar state: real block, then imaginary
    block of PCG64 normals, divided by the norm (state.py:46-54)."""
    dim = 1 << int(num_qubits)
    gen = np.random.default_rng(seed)
    raw = gen.standard_normal(dim) + 1j * gen.standard_normal(dim)
    raw /= np.linalg.norm(raw)
    return raw


class StateVector:
    """2^n amplitudes on a GPU plus the classical register list."""

    __slots__ = ("_h", "_n", "_device", "_cregs", "_parent", "__weakref__")

    def __init__(self, qubit_count: int, device: int = 0, shared: bool = False):
        n = _check_count(qubit_count)
        self._h = None
        self._n = n
        self._device = int(device)
        self._cregs: list[int] = []
        self._parent = None
        h = C.c_void_p()
        create = lib.qsv_state_create_shared if shared else lib.qsv_state_create
        check(create(n, self._device, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.qsv_state_destroy(h)
            self._h = None

    def _handle(self):
        return self._h

    def _view(self, offset: int, qubit_count: int) -> "StateVector":
        """Non-owning state over amplitudes [offset, offset + 2^qubit_count)
        (qsv_state_view); keeps this state alive while it exists."""
        v = StateVector.__new__(StateVector)
        v._h = None
        v._n = int(qubit_count)
        v._device = self._device
        v._cregs = []
        v._parent = self
        h = C.c_void_p()
        check(lib.qsv_state_view(self._h, int(offset), v._n, C.byref(h)))
        v._h = h
        return v

    def _set_sm_limit(self, sms: int) -> None:
        check(lib.qsv_set_sm_limit(self._h, int(sms)))

    # -- shape -------------------------------------------------------------
    def get_qubit_count(self) -> int:
        return self._n

    @property
    def num_qubits(self) -> int:
        return self._n

    @property
    def dim(self) -> int:
        return 1 << self._n

    def get_device(self) -> int:
        return self._device

    # -- initialisation (state.py:32-54) ------------------------------------
    def set_zero_state(self) -> None:
        check(lib.qsv_set_zero(self._h))

    def set_computational_basis(self, index: int) -> None:
        index = int(index)
        if not 0 <= index < self.dim:
            raise ValueError(f"basis index {index} out of range for {self._n} qubits")
        check(lib.qsv_set_basis(self._h, index))

    def set_Haar_random_state(self, seed=None) -> None:
        """Complex Gaussian (real block, then imaginary block, PCG64) divided
        by its norm -- drawn on the host with numpy so that a seed gives the
        bit-identical state of the reference (state.py:46-54)."""
        self._upload(haar_vector(self._n, seed))

    set_haar_random = set_Haar_random_state

    def set_random_state_device(self, seed: int = 0) -> None:
        """Benchmark-only initialiser: Gaussian amplitudes generated on the
        GPU from a counter hash, normalised.  NOT bit-compatible with
        ``set_Haar_random_state``; used where only the timing matters."""
        check(lib.qsv_set_random_device(self._h, int(seed) & ((1 << 64) - 1)))

    # -- transfer (state.py:56-73) -----------------------------------------
    def _upload(self, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr, dtype=np.complex128)
        check(lib.qsv_load(self._h, arr.ctypes.data, arr.size))

    def load(self, state) -> None:
        if isinstance(state, StateVector):
            if state._n != self._n:
                raise ValueError(f"expected {self.dim} amplitudes, got {state.dim}")
            check(lib.qsv_copy(state._h, self._h))
            self._cregs = list(state._cregs)
            return
        data = np.asarray(state, dtype=np.complex128)
        if data.shape != (self.dim,):
            raise ValueError(f"expected {self.dim} amplitudes, got shape {data.shape}")
        self._upload(data)

    def get_vector(self, out: np.ndarray | None = None, blocking: bool = True) -> np.ndarray:
        """A host copy (mutating it never touches the device state).  ``out``
        may supply a contiguous complex128 buffer, e.g. pinned memory; with
        ``blocking=False`` the copy is only enqueued on the state's stream
        (read ``out`` after ``synchronize()``)."""
        if out is None:
            if not blocking:
                raise ValueError("a non-blocking copy needs an output buffer")
            out = np.empty(self.dim, dtype=np.complex128)
        elif out.dtype != np.complex128 or out.shape != (self.dim,) or \
                not out.flags.c_contiguous:
            raise ValueError(f"out must be a contiguous complex128 array of {self.dim}")
        check((lib.qsv_get if blocking else lib.qsv_get_async)(self._h, out.ctypes.data, out.size))
        return out

    def copy(self) -> "StateVector":
        out = StateVector(self._n, self._device)
        check(lib.qsv_copy(self._h, out._h))
        out._cregs = list(self._cregs)
        return out

    # -- algebra (state.py:75-81, 108-114) --------------------------------
    def get_squared_norm(self) -> float:
        out = C.c_double()
        check(lib.qsv_norm2(self._h, C.byref(out)))
        return float(out.value)

    def normalize(self, squared_norm: float) -> None:
        if squared_norm <= 0:
            raise ValueError("squared norm must be positive")
        check(lib.qsv_scale(self._h, 1.0 / float(np.sqrt(squared_norm)), 0.0))

    def multiply_coef(self, coef) -> None:
        c = complex(coef)
        check(lib.qsv_scale(self._h, c.real, c.imag))

    def add_state(self, other: "StateVector") -> None:
        if other._n != self._n:
            raise ValueError("qubit counts differ")
        check(lib.qsv_add(self._h, other._h))

    def multiply_elementwise_function(self, func) -> None:
        """amps[i] *= func(i) (state.py:116-119).  ``func`` is arbitrary
        Python, so it is evaluated on the host exactly as the reference does
        (one call per index, in index order); the multiply runs on the GPU."""
        coefs = np.fromiter((func(i) for i in range(self.dim)), dtype=np.complex128,
                            count=self.dim)
        check(lib.qsv_mul_elementwise(self._h, coefs.ctypes.data, coefs.size))

    # -- measurement statistics (state.py:83-106) --------------------------
    def get_marginal_probability(self, measured_value) -> float:
        """Sum of |psi_x|^2 over the x matching a pattern of 0 / 1 / WILDCARD
        (=2) per qubit (state.py:83-95), as one masked GPU reduction."""
        pattern = list(measured_value)
        if len(pattern) != self._n:
            raise ValueError("pattern length must equal the qubit count")
        mask = value = 0
        for q, want in enumerate(pattern):
            if want == WILDCARD:
                continue
            if want not in (0, 1):
                raise ValueError(f"pattern entry must be 0, 1 or WILDCARD, got {want!r}")
            mask |= 1 << q
            value |= int(want) << q
        out = C.c_double()
        check(lib.qsv_marginal_prob(self._h, mask, value, C.byref(out)))
        return float(out.value)

    def sampling(self, count: int, seed=None) -> list[int]:
        """Z-basis samples (state.py:97-106): draws ``rng.random(count)`` on
        the host (numpy PCG64, so a seed gives the reference's draws) and
        inverts the cumulative distribution of |psi|^2 on the GPU."""
        if count == 0:
            return []
        if count < 0:
            raise ValueError("sample count must be non-negative")
        u = np.random.default_rng(seed).random(count)
        out = np.empty(count, dtype=np.uint64)
        check(lib.qsv_sampling(self._h, u.ctypes.data, int(count), out.ctypes.data))
        return out.astype(np.int64).tolist()

    # -- classical registers (state.py:116-127) ----------------------------
    def get_classical_value(self, index: int) -> int:
        if index < 0:
            raise ValueError("register address must be non-negative")
        return self._cregs[index] if index < len(self._cregs) else 0

    def set_classical_value(self, index: int, value: int) -> None:
        if index < 0:
            raise ValueError("register address must be non-negative")
        if index >= len(self._cregs):
            self._cregs.extend([0] * (index + 1 - len(self._cregs)))
        self._cregs[index] = int(value)

    # -- qsimcore attribute names (state.py:22-31) ----------------------------
    @property
    def amplitudes(self) -> np.ndarray:
        """Host copy of the amplitudes (qsimcore exposes its numpy buffer;
        here the buffer is in HBM, so in-place edits of the returned array do
        not reach the state -- assign to ``amplitudes`` or call ``load``)."""
        return self.get_vector()

    @amplitudes.setter
    def amplitudes(self, value) -> None:
        self.load(value)

    @property
    def classical_registers(self) -> list:
        return self._cregs

    def synchronize(self) -> None:
        check(lib.qsv_sync(self._h))

    def set_stream(self, cuda_stream_ptr: int) -> None:
        """Enqueue this state's work on an external CUDA stream (e.g.
        ``torch.cuda.current_stream().cuda_stream``)."""
        check(lib.qsv_set_stream(self._h, C.c_void_p(int(cuda_stream_ptr))))

    def __repr__(self) -> str:
        return f"QuantumState(qubits={self._n}, device={self._device})"


QuantumState = StateVector


def inner_product(bra: StateVector, ket: StateVector) -> complex:
    """<bra|ket> (state.py:136-139)."""
    if bra.get_qubit_count() != ket.get_qubit_count():
        raise ValueError("qubit counts differ")
    out = (C.c_double * 2)()
    check(lib.qsv_inner(bra._h, ket._h, out))
    return complex(out[0], out[1])


def tensor_product(first: StateVector, second: StateVector) -> StateVector:
    """kron(second, first): ``first`` on the low qubits (state.py:142-146)."""
    out = StateVector(first._n + second._n, first._device)
    check(lib.qsv_tensor_product(first._h, second._h, out._h))
    return out


def permutate_qubit(state: StateVector, order) -> StateVector:
    """New qubit i carries the role of old qubit order[i] (state.py:149-161)."""
    n = state._n
    order = [int(q) for q in order]
    if sorted(order) != list(range(n)):
        raise ValueError(f"order must be a permutation of 0..{n - 1}")
    out = StateVector(n, state._device)
    check(lib.qsv_permutate_qubit(state._h, int_array(order), n, out._h))
    return out


def drop_qubit(state: StateVector, targets, values) -> StateVector:
    """Project ``targets`` onto ``values`` and remove them, without
    renormalising (state.py:164-192)."""
    n = state._n
    targets = [int(t) for t in targets]
    values = list(values)
    if len(targets) != len(values):
        raise ValueError("targets and projection values must pair up")
    if len(set(targets)) != len(targets):
        raise ValueError("target qubits must be distinct")
    if len(targets) >= n:
        raise ValueError("cannot drop every qubit")
    for t, v in zip(targets, values):
        if not 0 <= t < n:
            raise ValueError(f"target {t} out of range")
        if v not in (0, 1):
            raise ValueError("projection values must be 0 or 1")
    out = StateVector(n - len(targets), state._device)
    check(lib.qsv_drop_qubit(state._h, int_array(targets), int_array([int(v) for v in values]),
                             len(targets), out._h))
    return out
