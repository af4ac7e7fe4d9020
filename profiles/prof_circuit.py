"""Run one benchmark circuit once (for ncu captures of the tile kernel).

    python profiles/prof_circuit.py [n] [depth] [tile_qubits]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 20
L = int(sys.argv[3]) if len(sys.argv) > 3 else 0
circ = workloads.generate_cz_ladder(n, depth, seed=1)
circ.set_plan_options(use_tiles=1, tile_qubits=L, use_graph=0)
st = qs.QuantumState(n)
st.set_random_state_device(1)
circ.update_quantum_state(st)
st.synchronize()
print(circ.program_stats())
