import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_13524_b200 as qs
from paper_2011_13524_b200 import workloads
n = int(sys.argv[1]); L = int(sys.argv[2]); depth = int(sys.argv[3]) if len(sys.argv) > 3 else 20
print("start", n, L, flush=True)
circ = workloads.generate_cz_ladder(n, depth, seed=1)
circ.set_plan_options(use_tiles=1, tile_qubits=L, use_graph=int(os.environ.get("GRAPH", "0")))
print(circ.program_stats(), flush=True)
st = qs.QuantumState(n)
st.set_random_state_device(1)
torch.cuda.synchronize()
for r in range(2):
    t0 = time.time()
    circ.update_quantum_state(st)
    st.synchronize()
    print(f"run {r}: {time.time() - t0:.3f}s norm={st.get_squared_norm():.12f}", flush=True)
