"""Full-size parity check of the headline circuit workload (one-off evidence,
not a suite test: the C oracle needs minutes at n=30).

cz-ladder(n, depth, seed=1) -- the circuit bench.py times -- from |0...0>,
run through the native planner (fusion + real frames + tile passes) on the
GPU and gate by gate through the OpenMP C oracle (oracle/qsv_oracle.c) on the
host; prints the max |amplitude error| and the norm drift.

    python profiles/parity_n30.py --qubits 30 --depth 20
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402
from paper_2011_13524_b200._circuit import circuit_records  # noqa: E402
from oracle import c_oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=30)
    ap.add_argument("--depth", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    n, depth = a.qubits, a.depth
    circ = workloads.generate_cz_ladder(n, depth, seed=1)
    recs = circuit_records(circ)

    st = qs.QuantumState(n)
    t0 = time.perf_counter()
    circ.update_quantum_state(st)
    got = st.get_vector()
    t_gpu = time.perf_counter() - t0
    del st

    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[0] = 1.0
    t0 = time.perf_counter()
    for i, rec in enumerate(recs):
        c_oracle.apply_record(ref, n, rec)
        if i % 200 == 0:
            print(f"oracle {i}/{len(recs)} {time.perf_counter() - t0:.0f}s", flush=True)
    t_cpu = time.perf_counter() - t0

    err = 0.0
    step = 1 << 26
    for lo in range(0, 1 << n, step):
        err = max(err, float(np.max(np.abs(got[lo:lo + step] - ref[lo:lo + step]))))
    res = {"workload": f"cz-ladder n={n} depth={depth} seed=1 from |0>",
           "gates": circ.get_gate_count(), "records": len(recs),
           "max_abs_amp_err": err, "bar": 1e-12, "pass": err <= 1e-12,
           "norm2_gpu": float(np.vdot(got, got).real), "norm2_oracle": c_oracle.norm2(ref, n),
           "gpu_s_incl_plan_and_d2h": t_gpu, "oracle_s": t_cpu,
           "oracle_threads": os.cpu_count()}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
