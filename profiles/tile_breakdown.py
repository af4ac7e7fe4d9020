"""Tile-pass time breakdown: run a benchmark circuit with parts of k_tile
disabled through QSV_TILE_DEBUG (read when a program is planned):
  0 full | 1 skip all gate ops | 2 skip phases (HBM streaming only)
  4 skip diagonal ops | 8 skip 1-qubit dense/real ops

    python profiles/tile_breakdown.py [n] [family] [real_frames ...]
Device time per run (CUDA events, best of 2).  Results with parts disabled
are wrong by construction; only the timings matter.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
fam = sys.argv[2] if len(sys.argv) > 2 else "cz-ladder"
rfs = [int(v) for v in sys.argv[3:]] or [1]
circ = (workloads.generate_cz_ladder(n, 20, seed=1) if fam == "cz-ladder"
        else workloads.generate_cnot_ring(n, seed=1))
st = qs.QuantumState(n)
st.set_random_state_device(1)
for rf in rfs:
    for dbg in (0, 1, 2, 4, 8):
        os.environ["QSV_TILE_DEBUG"] = str(dbg)
        circ.set_plan_options(real_frames=rf)
        stats = circ.program_stats()
        circ.update_quantum_state(st)
        best = 1e9
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            circ.update_quantum_state(st)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 1e3)
        print(f"{fam} n={n} rf={rf} debug={dbg} passes={stats['num_tile_passes']} "
              f"fp64={stats['fp64_flops'] / 1e12:.2f}TF time={best:.4f}s", flush=True)
