"""cfg3 VQE ansatz (n=24) device time with the tile-kernel variant forced to
4 / 5 register bits (QSV_TILE_VARIANT, read at plan time) and the planner's
own choice.

    python profiles/time_vqe_variant.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

n = 24
for var in (None, "4", "5"):
    if var is None:
        os.environ.pop("QSV_TILE_VARIANT", None)
    else:
        os.environ["QSV_TILE_VARIANT"] = var
    circ = workloads.vqe_ansatz(n)
    st = qs.QuantumState(n)
    circ.update_quantum_state(st)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        st.set_zero_state()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        circ.update_quantum_state(st)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"variant={var or 'auto'} ansatz device {best:.3f} ms", flush=True)
