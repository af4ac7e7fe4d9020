"""Small states: device time of cnot-ring / cz-ladder at n = 14..20 for tile
sizes L = 8..12 (plan option tile_qubits) and the per-gate path.

    python profiles/time_small_n.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

NS = [int(v) for v in os.environ.get("NS", "14,16,18,20").split(",")]
LS = [int(v) for v in os.environ.get("LS", "0,-1,8,9,10,11,12").split(",")]
for n in NS:
    for fam in ("cnot-ring", "cz-ladder"):
        circ = (workloads.generate_cnot_ring(n, seed=1) if fam == "cnot-ring"
                else workloads.generate_cz_ladder(n, 20, seed=1))
        st = qs.QuantumState(n)
        row = []
        for L in LS:
            if L == 0:
                circ.set_plan_options(use_tiles=0)
            elif L == -1:
                circ.set_plan_options(use_tiles=1, tile_qubits=0)  # engine's choice
            else:
                circ.set_plan_options(use_tiles=1, tile_qubits=L)
            stats = circ.program_stats()
            circ.update_quantum_state(st)
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
            row.append(f"L={ {0: 'gates', -1: 'auto'}.get(L, L)}:{best:.3f}ms/{stats['num_steps']}")
        print(f"{fam} n={n} " + " ".join(row), flush=True)
