"""Circuits: ordered gate lists compiled into libqsv programs.

Core semantics follow the reference ``Circuit`` / ``ParametricCircuit``
(circuit.py:11-125) and the Qulacs-named handles ``QuantumCircuit`` /
``ParametricQuantumCircuit`` (bindings __init__.py:91-149).  The reference
runs ``for gate in gates: gate.apply(state)`` (circuit.py:54-55); here the
gate list is lowered once into a ``qsv_program`` (fused + tiled + replayed as
a CUDA graph by the native planner) and re-lowered only when the list or a
rotation angle changes.
"""

from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _lib
from ._gates import BasicGate, PauliRotationGate, QuantumGate
from ._handles import QuantumGateBase, unwrap
from ._lib import check, lib


_OP_SIZE = C.sizeof(_lib.QsvOp)
_ANGLE_OFF = _lib.QsvOp.angle.offset
_put_angle = struct.Struct("<d").pack_into  # angle field of a packed qsv_op


class _OpsCache:
    """qsv_op array of one gate list, kept with the arrays it points to;
    a recompile after ParametricCircuit.set_parameter copies it and patches
    only the rotation angles."""

    __slots__ = ("ids", "gates", "blob", "rot")

    def __init__(self, gates):
        self.gates = list(gates)  # keeps the gates (and their cached arrays) alive
        self.ids = tuple(id(g) for g in gates)
        self.blob = bytes(_fill_ops_uncached(gates))
        self.rot = [(i, g) for i, g in enumerate(gates) if isinstance(g, PauliRotationGate)]

    def ops(self):
        blob = bytearray(self.blob)
        for i, g in self.rot:
            _put_angle(blob, i * _OP_SIZE + _ANGLE_OFF, g.angle)
        return (_lib.QsvOp * max(1, len(self.gates))).from_buffer(blob)


def fill_ops(gates, cache_owner=None):
    """qsv_op array for a gate list (cached on ``cache_owner`` when given)."""
    if cache_owner is None:
        return _fill_ops_uncached(gates)
    c = getattr(cache_owner, "_ops_cache", None)
    if c is None or c.ids != tuple(id(g) for g in gates):
        c = _OpsCache(gates)
        cache_owner._ops_cache = c
    return c.ops()


def _fill_ops_uncached(gates):
    """qsv_op array for a gate list.  Each gate's op is built once and cached
    on the gate (with the arrays it points to); only angles are re-read."""
    # packed into one buffer (slice copies + struct stores: a ctypes element
    # proxy per gate cost several microseconds each on 600-gate circuits)
    parts = []
    rot = []
    for i, g in enumerate(gates):
        cached = getattr(g, "_op_cache", None)
        if cached is None:
            tmp = _lib.QsvOp()
            keep = []
            g.fill_op(tmp, keep)
            cached = (bytes(tmp), keep)
            g._op_cache = cached
        parts.append(cached[0])
        if isinstance(g, PauliRotationGate):
            rot.append((i, g.angle))
    blob = bytearray(b"".join(parts) if parts else bytes(_OP_SIZE))
    for i, angle in rot:
        _put_angle(blob, i * _OP_SIZE + _ANGLE_OFF, angle)
    return (_lib.QsvOp * max(1, len(gates))).from_buffer(blob)


class _Program:
    """Owner of one native program handle."""

    __slots__ = ("h",)

    def __init__(self, n, gates, opts, cache_owner=None):
        ops = fill_ops(gates, cache_owner)
        h = C.c_void_p()
        check(lib.qsv_program_create(n, ops, len(gates), C.byref(opts), C.byref(h)))
        self.h = h

    @property
    def stats(self) -> dict:
        st = _lib.QsvProgramStats()
        check(lib.qsv_program_stats_get(self.h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in _lib.QsvProgramStats._fields_ if f != "reserved"}

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib.qsv_program_destroy(h)
            self.h = None

    def run(self, state):
        check(lib.qsv_program_run(self.h, state._handle()))


def default_plan_opts(**kw) -> _lib.QsvPlanOpts:
    o = _lib.QsvPlanOpts()
    o.use_tiles = int(kw.get("use_tiles", 1))
    o.tile_qubits = int(kw.get("tile_qubits", 0))
    o.fuse = int(kw.get("fuse", 1))
    o.use_graph = int(kw.get("use_graph", 1))
    o.real_frames = int(kw.get("real_frames", 1))
    o.jit = int(kw.get("jit", 1))
    return o


class Circuit:
    """Ordered gate list over a fixed qubit count (circuit.py:11-72)."""

    def __init__(self, num_qubits: int):
        if num_qubits < 1:
            raise ValueError("qubit count must be positive")
        self.num_qubits = int(num_qubits)
        self.gates: list[QuantumGate] = []
        self._prog = None
        self._prog_key = None
        self._ops_cache = None
        self._plan = default_plan_opts()

    # -- editing -------------------------------------------------------------
    def _check_gate(self, gate) -> None:
        if not isinstance(gate, QuantumGate):
            raise TypeError(f"expected a gate, got {type(gate).__name__}")
        top = max(gate.touched_qubits(), default=-1)
        if top >= self.num_qubits:
            raise ValueError(f"gate touches qubit {top} but the circuit has "
                             f"{self.num_qubits} qubits")

    def add_gate(self, gate, position=None) -> None:
        self._check_gate(gate)
        if position is None:
            self.gates.append(gate)
            return
        if not 0 <= position <= len(self.gates):
            raise ValueError(f"insert position {position} out of range")
        self.gates.insert(position, gate)

    def remove_gate(self, position: int) -> None:
        if not 0 <= position < len(self.gates):
            raise ValueError(f"position {position} out of range")
        del self.gates[position]

    def get_gate(self, position: int):
        if not 0 <= position < len(self.gates):
            raise ValueError(f"position {position} out of range")
        return self.gates[position].copy()

    def get_gate_count(self) -> int:
        return len(self.gates)

    def calculate_depth(self) -> int:
        """ASAP layering over touched qubits (circuit.py:57-67)."""
        level = [0] * self.num_qubits
        depth = 0
        for g in self.gates:
            qs = g.touched_qubits()
            layer = max((level[q] for q in qs), default=0) + 1
            for q in qs:
                level[q] = layer
            depth = max(depth, layer)
        return depth

    def copy(self):
        out = type(self).__new__(type(self))
        Circuit.__init__(out, self.num_qubits)
        out.gates = [g.copy() for g in self.gates]
        out._plan = self._plan
        return out

    # -- execution -------------------------------------------------------------
    def set_plan_options(self, **kw) -> None:
        """Engine knobs: use_tiles, tile_qubits, fuse, use_graph, real_frames,
        jit (0 interpreter only, 1 generated pass kernels from the second
        run, 2 compiled at program creation)."""
        self._plan = default_plan_opts(**kw)
        self._prog = None

    def _key(self):
        # the gate objects themselves (identity compare, keeps ids alive)
        return (tuple(self.gates),
                tuple(g.angle for g in self.gates if isinstance(g, PauliRotationGate)),
                bytes(self._plan))

    def compile(self):
        """Lower the gate list: runs of basic gates become native programs,
        quantum maps (maps.py) stay host-driven steps between them.  Returns
        the program of an all-basic circuit, else the list of steps."""
        key = self._key()
        if self._prog is None or self._prog_key != key:
            if all(isinstance(g, BasicGate) for g in self.gates):
                self._prog = _Program(self.num_qubits, self.gates, self._plan, self)
            else:
                steps, run = [], []
                for g in self.gates:
                    if isinstance(g, BasicGate):
                        run.append(g)
                        continue
                    if run:
                        steps.append(_Program(self.num_qubits, run, self._plan))
                        run = []
                    steps.append(g)
                if run:
                    steps.append(_Program(self.num_qubits, run, self._plan))
                self._prog = steps
            self._prog_key = key
        return self._prog

    def program_stats(self) -> dict:
        prog = self.compile()
        if isinstance(prog, _Program):
            return dict(prog.stats)
        total = {f: 0 for f, _ in _lib.QsvProgramStats._fields_ if f != "reserved"}
        for st in prog:
            if isinstance(st, _Program):
                for k, v in st.stats.items():
                    total[k] += v
        total["num_maps"] = sum(1 for st in prog if not isinstance(st, _Program))
        return total

    def plan_stats(self, **kw) -> dict:
        """Host-only planning statistics (no GPU needed)."""
        opts = default_plan_opts(**kw) if kw else self._plan
        basic = [g for g in self.gates if isinstance(g, BasicGate)]  # maps run on the host
        ops = fill_ops(basic)
        st = _lib.QsvProgramStats()
        check(lib.qsv_plan_stats(self.num_qubits, ops, len(basic), C.byref(opts),
                                 C.byref(st)))
        return {f: getattr(st, f) for f, _ in _lib.QsvProgramStats._fields_ if f != "reserved"}

    def update_state(self, state, rng=None) -> None:
        """circuit.py:48-55: one generator (seed / Generator / None) shared by
        every map of the circuit, drawn in gate order."""
        if state.get_qubit_count() != self.num_qubits:
            raise ValueError("state and circuit qubit counts differ")
        if not self.gates:
            return
        if getattr(state, "is_sharded", False):
            # dist.ShardedQuantumState: the sharded engine plans remaps and
            # compiles its own per-rank programs from the gate records
            if not all(isinstance(g, BasicGate) for g in self.gates):
                raise ValueError("quantum maps cannot run on a sharded state")
            state.apply_records([g.record() for g in self.gates])
            return
        prog = self.compile()
        if isinstance(prog, _Program):
            prog.run(state)
            return
        if not isinstance(rng, np.random.Generator):
            rng = np.random.default_rng(rng)
        for step in prog:
            if isinstance(step, _Program):
                step.run(state)
            else:
                step.apply(state, rng)


class ParametricCircuit(Circuit):
    """Circuit with a mutable angle table tracked by gate identity
    (circuit.py:75-125)."""

    def __init__(self, num_qubits: int):
        super().__init__(num_qubits)
        self._params: list[QuantumGate] = []

    def add_parametric_gate(self, gate, position=None) -> None:
        if not gate.is_parametric:
            raise ValueError("gate is not parametric")
        super().add_gate(gate, position)
        self._params.append(gate)

    def remove_gate(self, position: int) -> None:
        if 0 <= position < len(self.gates):
            victim = self.gates[position]
            self._params = [g for g in self._params if g is not victim]
        super().remove_gate(position)

    def get_parameter_count(self) -> int:
        return len(self._params)

    def _param(self, index: int):
        if not 0 <= index < len(self._params):
            raise ValueError(f"parameter index {index} out of range")
        return self._params[index]

    def get_parameter(self, index: int) -> float:
        return self._param(index).angle

    def set_parameter(self, index: int, angle: float) -> None:
        self._param(index).angle = float(angle)

    def get_parametric_gate_position(self, index: int) -> int:
        g = self._param(index)
        for pos, other in enumerate(self.gates):
            if other is g:
                return pos
        raise RuntimeError("parametric gate missing from the gate list")

    def copy(self):
        out = ParametricCircuit(self.num_qubits)
        out.gates = [g.copy() for g in self.gates]
        twin = {id(a): b for a, b in zip(self.gates, out.gates)}
        out._params = [twin[id(g)] for g in self._params]
        out._plan = self._plan
        return out


# ------------------------------------------------------------------ handles
class QuantumCircuit:
    """Qulacs-named handle (bindings __init__.py:91-128)."""

    __slots__ = ("_core",)
    _core_cls = Circuit

    def __init__(self, qubit_count: int):
        self._core = self._core_cls(qubit_count)

    def get_qubit_count(self) -> int:
        return self._core.num_qubits

    def add_gate(self, gate, position=None) -> None:
        self._core.add_gate(unwrap(gate), position)

    def remove_gate(self, position: int) -> None:
        self._core.remove_gate(position)

    def get_gate(self, position: int) -> QuantumGateBase:
        return QuantumGateBase(self._core.get_gate(position))

    def get_gate_count(self) -> int:
        return self._core.get_gate_count()

    def calculate_depth(self) -> int:
        return self._core.calculate_depth()

    def update_quantum_state(self, state, seed=None) -> None:
        self._core.update_state(state, rng=seed)

    def add_observable_rotation_gate(self, observable, angle, num_slices) -> None:
        from ._observable import add_observable_rotation
        add_observable_rotation(self._core, unwrap(observable), angle, num_slices)

    def set_plan_options(self, **kw) -> None:
        self._core.set_plan_options(**kw)

    def program_stats(self) -> dict:
        return self._core.program_stats()

    def plan_stats(self, **kw) -> dict:
        return self._core.plan_stats(**kw)

    def copy(self):
        out = type(self).__new__(type(self))
        out._core = self._core.copy()
        return out


class ParametricQuantumCircuit(QuantumCircuit):
    """Bindings __init__.py:131-149."""

    _core_cls = ParametricCircuit

    def add_parametric_gate(self, gate, position=None) -> None:
        self._core.add_parametric_gate(unwrap(gate), position)

    def get_parameter_count(self) -> int:
        return self._core.get_parameter_count()

    def get_parameter(self, index: int) -> float:
        return self._core.get_parameter(index)

    def set_parameter(self, index: int, angle: float) -> None:
        self._core.set_parameter(index, angle)

    def get_parametric_gate_position(self, index: int) -> int:
        return self._core.get_parametric_gate_position(index)


def circuit_records(circuit) -> list:
    """Neutral records of every gate (fed to the test oracle)."""
    return [g.record() for g in unwrap(circuit).gates]

