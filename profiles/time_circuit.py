"""Time benchmark circuits through the native planner (device events).

    python profiles/time_circuit.py [n] [depth] [reps]
Prints one line per plan variant.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
variants = [dict(tile_qubits=12, real_frames=rf) for rf in (0, 1)]
if os.environ.get('TC_VARIANTS'):
    variants = eval(os.environ['TC_VARIANTS'])
st = qs.QuantumState(n)
st.set_random_state_device(1)
for fam in ("cz-ladder", "cnot-ring"):
    circ = (workloads.generate_cz_ladder(n, depth, seed=1) if fam == "cz-ladder"
            else workloads.generate_cnot_ring(n, seed=1))
    layers = depth + 1 if fam == "cz-ladder" else 11
    for v in variants:
        circ.set_plan_options(use_tiles=1, **v)
        stats = circ.program_stats()
        circ.update_quantum_state(st)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            circ.update_quantum_state(st)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 1e3)
        print(f"{os.environ.get('QSV_LIB', 'default')} {fam} n={n} {v} passes={stats['num_tile_passes']} "
              f"kernels={stats['num_gate_kernels']} total={best:.4f}s sec/layer={best / layers:.5f}",
              flush=True)
