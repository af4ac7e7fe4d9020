"""Quantum-volume-like circuit: layers of random 2-qubit unitaries on a random
pairing of the qubits (dense 4x4 gates through the planner)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rng = np.random.default_rng(0)
c = qs.QuantumCircuit(n)
for _ in range(depth):
    perm = rng.permutation(n)
    for k in range(0, n - 1, 2):
        c.add_gate(qg.RandomUnitary([int(perm[k]), int(perm[k + 1])], seed=int(rng.integers(1 << 30))))
st = qs.QuantumState(n)
st.set_random_state_device(1)
print(c.program_stats(), flush=True)
c.update_quantum_state(st)
torch.cuda.synchronize()
best = 1e9
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    c.update_quantum_state(st)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 1e3)
print(f"qv n={n} depth={depth} gates={c.get_gate_count()} time={best:.4f}s "
      f"per-gate={best / c.get_gate_count() * 1e3:.3f}ms", flush=True)
