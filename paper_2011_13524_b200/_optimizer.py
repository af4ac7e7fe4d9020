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


def _support(g) -> frozenset:
    return frozenset(g.touched_qubits())


def optimize_light(circuit) -> None:
    """Merge neighbouring pairs whose supports nest, until nothing changes
    (optimizer.py:56-70)."""
    gates = circuit.gates
    again = True
    while again:
        again = False
        i = 0
        while i + 1 < len(gates):
            a, b = gates[i], gates[i + 1]
            if a.mergeable and b.mergeable:
                sa, sb = _support(a), _support(b)
                if sa <= sb or sb <= sa:
                    gates[i:i + 2] = [merge(a, b)]
                    again = True
                    continue  # retry at the same position
            i += 1


def optimize_heavy(circuit, block_size: int) -> None:
    """Slide a later gate left past gates that provably commute with gate i
    and merge it into gate i when the union stays within ``block_size``
    qubits (optimizer.py:73-107)."""
    if block_size < 1:
        raise ValueError("block size must be >= 1")
    gates = circuit.gates
    again = True
    while again:
        again = False
        i = 0
        while i < len(gates):
            a = gates[i]
            if not a.mergeable or len(_support(a)) > block_size:
                i += 1
                continue
            fused = False
            for j in range(i + 1, len(gates)):
                b = gates[j]
                if b.mergeable and len(_support(a) | _support(b)) <= block_size:
                    m = merge(a, b)
                    del gates[j]
                    del gates[i]
                    gates.insert(j - 1, m)
                    again = fused = True
                    break
                if not commutation_check(a, b):
                    break
            if not fused:
                i += 1
