"""Exchange-step timing on one GPU: 4 virtual ranks, remaps of k = 1..3
qubits, "p2p" (qsv_slice_swap, in place) vs "nccl" mode's in-process path
(torch strided copies through a temporary).  On one GPU both are HBM-bound;
the figure is slice bytes moved per second (each swapped element is read and
written on both sides: 4 * 16 B of HBM traffic per element pair).

    python profiles/time_exchange.py --local 28
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2011_13524_b200.dist import CudaShard, ShardedQuantumState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--local", type=int, default=28)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    L, world = a.local, 4
    n = L + 2
    stream = torch.cuda.current_stream()
    out = {}
    for mode in ("p2p", "nccl"):
        st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                                 backend=lambda L_, r: CudaShard(L_, 0, stream.cuda_stream),
                                 exchange=mode)
        for r, s in st.shards.items():
            s.set_random(5 + r)
        for gs, ls, name in (([L], [L - 1], "k1_high"), ([L], [3], "k1_low"),
                             ([L, L + 1], [L - 1, L - 2], "k2_high")):
            st._remap(gs, ls)  # warm
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st._remap(gs, ls)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            k = len(gs)
            moved = world * (1 - 2.0 ** -k) * (16 << L)  # bytes that change shard
            best = min(ts)
            out[f"{mode}_{name}"] = {"s": best, "moved_GBps": moved / best / 1e9,
                                     "hbm_GBps": 2 * moved / best / 1e9}
            print(mode, name, json.dumps(out[f"{mode}_{name}"]), flush=True)
        del st
    print(json.dumps(out))


if __name__ == "__main__":
    main()
