"""Time Observable.get_expectation_value on the cfg3 instance (VQE ansatz
n=24 + TFIM, 47 terms) and random multi-qubit Pauli sums; check against the
energy the reference produced (-0.201996915076406)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
circ = workloads.vqe_ansatz(n)
obs = workloads.tfim_observable(n)
st = qs.QuantumState(n)
circ.update_quantum_state(st)
v = obs.get_expectation_value(st)
best = 1e9
for _ in range(5):
    t0 = time.perf_counter()
    v = obs.get_expectation_value(st)
    best = min(best, time.perf_counter() - t0)
print(f"n={n} TFIM terms={obs.get_term_count()} energy={v:.15f} expectation_s={best:.6f}")
