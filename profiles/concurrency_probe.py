"""Do an SM-capped slice swap and a tile pass run concurrently on two streams?

Times (CUDA events, one GPU): a cz-ladder program on state A alone, a k=1
slice swap between states B and C capped at R SMs alone, and both enqueued
on two streams -- once with two torch side streams, once with the swap on
the legacy default stream.  Concurrent means T(both) ~ max, serial ~ sum.

    python profiles/concurrency_probe.py --qubits 27 --sms 16
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402
from paper_2011_13524_b200.dist import CudaShard  # noqa: E402


def timed(fn, streams):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    a.record(main)
    for s in streams:
        s.wait_stream(main)
    fn()
    for s in streams:
        main.wait_stream(s)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=27)
    ap.add_argument("--sms", type=int, default=16)
    a = ap.parse_args()
    n = a.qubits
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    legacy = torch.cuda.default_stream()
    circ = workloads.generate_cz_ladder(n, 4, seed=1)
    A = qs.QuantumState(n)
    A.set_stream(s1.cuda_stream)
    A.set_random_state_device(1)
    B = CudaShard(n, 0, s2.cuda_stream)
    C = CudaShard(n, 0, s2.cuda_stream)
    B.set_sm_limit(a.sms)
    count = 1 << (n - 1)

    def comp():
        circ.update_quantum_state(A)

    def swap():
        B.slice_swap(C.ptr(), [n - 1], 1, 0, 0, count)

    for _ in range(2):
        comp()
        swap()
    torch.cuda.synchronize()
    out = {"qubits": n, "swap_sms": a.sms}
    out["compute_s"] = min(timed(comp, [s1]) for _ in range(3))
    out["swap_s"] = min(timed(swap, [s2]) for _ in range(3))
    out["both_side_streams_s"] = min(timed(lambda: (swap(), comp()), [s1, s2]) for _ in range(3))
    out["both_comp_first_s"] = min(timed(lambda: (comp(), swap()), [s1, s2]) for _ in range(3))
    B.state.set_stream(legacy.cuda_stream)
    out["both_swap_on_legacy_s"] = min(timed(lambda: (swap(), comp()), [s1, legacy])
                                       for _ in range(3))
    out["swap_GBps_hbm"] = 4 * 16 * count / out["swap_s"] / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
