"""First run of a fresh program (interpreter; generated kernels come from the
second run) per tile variant: device ms of run 1 and of the steady state.

    QSV_TILE_VARIANT=3|4 python profiles/first_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for n in [int(v) for v in os.environ.get("NS", "14,16,18").split(",")]:
    for fam in ("cnot-ring", "cz-ladder"):
        row = []
        for seed in (1, 2, 3):
            circ = (workloads.generate_cnot_ring(n, seed=seed) if fam == "cnot-ring"
                    else workloads.generate_cz_ladder(n, 20, seed=seed))
            st = qs.QuantumState(n)
            first = timed(lambda: circ.update_quantum_state(st))
            circ.update_quantum_state(st)
            steady = min(timed(lambda: circ.update_quantum_state(st)) for _ in range(5))
            row.append(f"{first:.3f}/{steady:.3f}")
        print(f"{fam} n={n} first/steady ms: " + " ".join(row), flush=True)
