"""User-visible gate fusion (QuantumCircuitOptimizer).

Same passes and the same greedy traversal as the reference optimizer
(``optimizer.py:16-107``), so gate counts after ``optimize_light`` /
``optimize(block_size)`` match the reference's (pinned by
tests/golden/circuits.json).  This is host work on gate descriptions; the
native planner in libqsv does its own, execution-oriented fusion (tile
passes) when the circuit is compiled.
"""

from __future__ import annotations

from ._gates import DenseGate, QuantumGate, merge


def merge_all(circuit) -> DenseGate:
    """Whole circuit folded into one dense gate (optimizer.py:16-32)."""
    acc = None
    for pos, g in enumerate(circuit.gates):
        if not g.mergeable:
            raise ValueError(f"gate at position {pos} cannot be merged")
        acc = g if acc is None else merge(acc, g)
    if acc is None:
        return DenseGate([], [[1.0]])
    if acc is circuit.gates[0]:
        acc = merge(DenseGate([], [[1.0]]), acc)  # densify, never alias the input
    return acc


def commutation_check(first: QuantumGate, second: QuantumGate) -> bool:
    """Provable commutation from per-qubit axis labels: on every shared qubit
    the labels must agree, or one of them must be "any" (optimizer.py:35-49)."""
    for q in set(first.touched_qubits()).intersection(second.touched_qubits()):
        a, b = first.commutation_basis(q), second.commutation_basis(q)
        if "any" in (a, b):
            continue
        if a == "none" or b == "none" or a != b:
            return False
    return True


class _Entry:
    """A gate with its support and mergeability computed once (the passes
    below test them O(gates^2) times; the reference recomputes both on every
    test)."""

    __slots__ = ("gate", "support", "ok")

    def __init__(self, gate):
        self.gate = gate
        self.support = frozenset(gate.touched_qubits())
        self.ok = bool(gate.mergeable)


def _fused(a: _Entry, b: _Entry) -> _Entry:
    return _Entry(merge(a.gate, b.gate))


def optimize_light(circuit) -> None:
    """Merge neighbouring pairs whose supports nest, until a sweep changes
    nothing (optimizer.py:56-70).  A merge stays at position i, so the fused
    gate is immediately tried against its new right neighbour."""
    seq = [_Entry(g) for g in circuit.gates]
    changed = True
    while changed:
        changed = False
        i = 0
        while i + 1 < len(seq):
            a, b = seq[i], seq[i + 1]
            if a.ok and b.ok and (a.support <= b.support or b.support <= a.support):
                seq[i:i + 2] = [_fused(a, b)]
                changed = True
            else:
                i += 1
    circuit.gates[:] = [e.gate for e in seq]


def _partner(seq, i: int, block_size: int):
    """First j > i that gate i can absorb: scanning right, a mergeable gate
    whose union with i's support fits the block wins; a gate that does not
    provably commute with gate i ends the scan (optimizer.py:90-103)."""
    a = seq[i]
    for j in range(i + 1, len(seq)):
        b = seq[j]
        if b.ok and len(a.support | b.support) <= block_size:
            return j
        if not commutation_check(a.gate, b.gate):
            return None
    return None


def optimize_heavy(circuit, block_size: int) -> None:
    """Commutation-aware fusion within ``block_size`` qubits
    (optimizer.py:73-107): gate j slides left to gate i past gates that
    commute with gate i; the fused gate takes gate j's slot, so the gates in
    between keep their order ahead of it, and gate i's position is retried."""
    if block_size < 1:
        raise ValueError("block size must be >= 1")
    seq = [_Entry(g) for g in circuit.gates]
    changed = True
    while changed:
        changed = False
        i = 0
        while i < len(seq):
            a = seq[i]
            j = _partner(seq, i, block_size) if a.ok and len(a.support) <= block_size else None
            if j is None:
                i += 1
                continue
            fused = _fused(a, seq[j])
            del seq[j]
            del seq[i]
            seq.insert(j - 1, fused)
            changed = True
    circuit.gates[:] = [e.gate for e in seq]
