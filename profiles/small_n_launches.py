"""cnot-ring(16) (cfg1) through the public API, a few runs: for an ncu launch
list (per-pass kernel durations next to the event-timed circuit).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        python profiles/small_n_launches.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

n = int(os.environ.get("N", "16"))
fam = os.environ.get("FAM", "cnot-ring")
circ = (workloads.generate_cnot_ring(n, seed=1) if fam == "cnot-ring"
        else workloads.generate_cz_ladder(n, 20, seed=1))
st = qs.QuantumState(n)
for _ in range(int(os.environ.get("RUNS", "3"))):
    circ.update_quantum_state(st)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    circ.update_quantum_state(st)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"{fam}({n}) best {best:.4f} ms, {circ.program_stats()['num_steps']} passes")
