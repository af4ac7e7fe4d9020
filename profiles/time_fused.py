"""cz-ladder run after the reference optimizer passes (light / heavy(k)):
gate counts and device time through the planner."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402
from paper_2011_13524_b200.circuit import QuantumCircuitOptimizer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
for opt in ("none", "light", "heavy2", "heavy3", "heavy4", "heavy5"):
    c = workloads.generate_cz_ladder(n, 20, seed=1)
    if opt == "light":
        QuantumCircuitOptimizer().optimize_light(c)
    elif opt.startswith("heavy"):
        QuantumCircuitOptimizer().optimize(c, int(opt[-1]))
    st = qs.QuantumState(n)
    st.set_random_state_device(1)
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
    s = c.program_stats()
    print(f"{opt}: gates={c.get_gate_count()} passes={s['num_tile_passes']} "
          f"kernels={s['num_gate_kernels']} fp64={s['fp64_flops'] / 1e12:.2f}TF time={best:.4f}s",
          flush=True)
