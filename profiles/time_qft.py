"""Time a QFT-like circuit (H + controlled phases, no swaps) through the planner."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
c = qs.QuantumCircuit(n)
for i in range(n - 1, -1, -1):
    c.add_gate(qg.H(i))
    for j in range(i - 1, -1, -1):
        g = qg.DiagonalMatrix([i], [1, np.exp(1j * math.pi / (1 << (i - j)))])
        g.add_control_qubit(j, 1)
        c.add_gate(g)
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
print(f"qft n={n} gates={c.get_gate_count()} time={best:.4f}s", flush=True)
