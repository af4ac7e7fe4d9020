"""Run one benchmark circuit through generated pass kernels (for ncu captures
of k_pass).  python profiles/prof_jit.py [family] [n] [jit]
family: cz-ladder (depth 20) | cnot-ring | vqe"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "cz-ladder"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 28
jit = int(sys.argv[3]) if len(sys.argv) > 3 else 2
circ = {"cz-ladder": lambda: workloads.generate_cz_ladder(n, 20, seed=1),
        "cnot-ring": lambda: workloads.generate_cnot_ring(n, seed=1),
        "vqe": lambda: workloads.vqe_ansatz(n)}[fam]()
circ.set_plan_options(use_graph=0, jit=jit)
st = qs.QuantumState(n)
st.set_random_state_device(1)
circ.update_quantum_state(st)
st.synchronize()
print(circ.program_stats())
