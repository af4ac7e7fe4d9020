"""Time several circuit families with the tile-kernel variant forced to 4 / 5
register bits (QSV_TILE_VARIANT) and with the planner's own choice."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg, workloads  # noqa: E402


def qft(n):
    c = qs.QuantumCircuit(n)
    for i in range(n - 1, -1, -1):
        c.add_gate(qg.H(i))
        for j in range(i - 1, -1, -1):
            g = qg.DiagonalMatrix([i], [1, np.exp(1j * math.pi / (1 << (i - j)))])
            g.add_control_qubit(j, 1)
            c.add_gate(g)
    return c


def timeit(circ, n):
    st = qs.QuantumState(n)
    st.set_random_state_device(1)
    circ.update_quantum_state(st)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        circ.update_quantum_state(st)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


cases = [("cz-ladder-26", lambda: workloads.generate_cz_ladder(26, 20, seed=1), 26),
         ("cz-ladder-30", lambda: workloads.generate_cz_ladder(30, 20, seed=1), 30),
         ("cnot-ring-28", lambda: workloads.generate_cnot_ring(28, seed=1), 28),
         ("vqe-24", lambda: workloads.vqe_ansatz(24), 24),
         ("qft-28", lambda: qft(28), 28)]
for name, make, n in cases:
    row = []
    for v in ("4", "5", ""):
        if v:
            os.environ["QSV_TILE_VARIANT"] = v
        else:
            os.environ.pop("QSV_TILE_VARIANT", None)
        c = make()
        row.append(f"{v or 'auto'}={timeit(c, n):.4f}")
    print(name, " ".join(row), flush=True)
