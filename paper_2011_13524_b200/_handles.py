"""Qulacs-named gate handle (reference bindings ``_handles.py:14-52``).

A ``QuantumGateBase`` owns one core gate (``_gates``) and forwards to it;
``unwrap`` returns the core object behind any handle.
"""

from __future__ import annotations


def unwrap(obj):
    """Core object behind a handle; raw values pass through."""
    return getattr(obj, "_core", obj)


class QuantumGateBase:
    """Handle for a gate; ``update_quantum_state`` launches it on the GPU."""

    __slots__ = ("_core", "__weakref__")

    def __init__(self, core_gate):
        self._core = core_gate

    def update_quantum_state(self, state) -> None:
        self._core.apply(unwrap(state))

    def add_control_qubit(self, index: int, control_value: int) -> None:
        self._core = self._core.with_control(index, control_value)

    def get_matrix(self):
        return self._core.gate_matrix()

    def get_target_index_list(self) -> list[int]:
        return list(self._core.targets)

    def get_control_index_list(self) -> list[int]:
        return [q for q, _ in self._core.controls]

    def get_name(self) -> str:
        return self._core.name or type(self._core).__name__

    def set_parameter(self, angle: float) -> None:
        self._core.angle = float(angle)

    def get_parameter(self) -> float:
        return self._core.angle

    def copy(self) -> "QuantumGateBase":
        return QuantumGateBase(self._core.copy())

    def __repr__(self) -> str:
        return f"<{self.get_name()} targets={self.get_target_index_list()}>"
