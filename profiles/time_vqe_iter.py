"""VQE iterations at n=24 (cfg3): new angles for every parameter, ansatz +
TFIM expectation per iteration; wall time per iteration and which pass kernels
ran (generated vs interpreter), over 12 iterations."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402
from paper_2011_13524_b200._lib import jit_stats  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
circ = workloads.vqe_ansatz(n)
obs = workloads.tfim_observable(n)
st = qs.QuantumState(n)
rng = np.random.default_rng(1)
times = []
for it in range(12):
    for k in range(circ.get_parameter_count()):
        circ.set_parameter(k, float(rng.uniform(0, 2 * np.pi)))
    st.set_zero_state()
    st.synchronize()
    t0 = time.perf_counter()
    circ.update_quantum_state(st)
    e = obs.get_expectation_value(st)
    times.append(time.perf_counter() - t0)
    stats = circ._core.compile().stats
    print(f"iter {it}: {times[-1] * 1e3:.3f} ms  jit passes {stats['num_jit_passes']}/{stats['num_tile_passes']}  energy {e:.6f}", flush=True)
print("median of iterations 3..11:", np.median(times[3:]) * 1e3, "ms", jit_stats())
