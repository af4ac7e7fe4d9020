"""Exchange / compute overlap on one GPU: cz-ladder(L + 2, depth 20) over 4
virtual ranks (ShardedQuantumState with the product backend: p2p remaps by
qsv_slice_swap), each exchange step either run alone or pipelined block by
block with the segment that follows (``overlap=True``: swaps on the shard
stream with ``overlap_sms`` SMs, the segment prefix of the finished blocks on
a compute stream with the rest).  On one GPU the exchange is HBM traffic
instead of NVLink, but the tile passes are FP64-bound, so the overlap is
visible as a shorter circuit.  Device time with CUDA events.

    python profiles/time_overlap.py --local 28
"""

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2011_13524_b200 import workloads  # noqa: E402
from paper_2011_13524_b200._circuit import circuit_records  # noqa: E402
from paper_2011_13524_b200.dist import ShardedQuantumState  # noqa: E402


def run(n, recs, reps, **kw):
    # circuit-order segments (reorder=False): an exchange step per layer, the
    # regime the overlap is for (the run-ahead planner needs one remap here)
    st = ShardedQuantumState(n, world=4, owned=[0, 1, 2, 3], reorder=False, **kw)
    for r, s in st.shards.items():
        s.set_random(97 + r)
        s.scale(0.5)
    stream = torch.cuda.current_stream()
    st.apply_records(recs)  # warm-up
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        st.stats = {"swaps": 0, "bytes_sent": 0, "segments": 0}
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st.apply_records(recs)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    norm = st.get_squared_norm()
    stats = dict(st.stats)
    st.close()
    del st
    return {"circuit_s": min(ts), "all_s": ts, "norm": norm, "stats": stats}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--local", type=int, default=28)
    ap.add_argument("--depth", type=int, default=20)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--side-stream", action="store_true",
                    help="run the engine on a torch side stream instead of the default stream")
    ap.add_argument("--sms", default="4,8,16,32")
    ap.add_argument("--trace", action="store_true",
                    help="print the block timeline of a few overlapped exchange steps")
    a = ap.parse_args()
    if a.side_stream:
        with torch.cuda.stream(torch.cuda.Stream()):
            return body(a)
    return body(a)


def trace(n, recs, sms, bits):
    st = ShardedQuantumState(n, world=4, owned=[0, 1, 2, 3], overlap=True, overlap_bits=bits,
                             overlap_sms=sms, reorder=False)
    for r, s in st.shards.items():
        s.set_random(97 + r)
        s.scale(0.5)
    st.apply_records(recs)
    torch.cuda.synchronize()
    st.trace = []
    st.apply_records(recs)
    torch.cuda.synchronize()
    t0 = None
    lines = []
    for label, ev in st.trace:
        if label == "start":
            t0 = ev
            lines.append([])
        lines[-1].append(f"{label}@{t0.elapsed_time(ev):.2f}")
    for ln in lines[:6]:
        print(f"trace sms={sms} bits={bits}: " + " ".join(ln), flush=True)
    st.close()


def body(a):
    n = a.local + 2
    if a.trace:
        recs = circuit_records(workloads.generate_cz_ladder(n, a.depth, seed=1))
        for sms in [int(v) for v in a.sms.split(",")]:
            trace(n, recs, sms, 2)
        return
    recs = circuit_records(workloads.generate_cz_ladder(n, a.depth, seed=1))
    out = {"workload": f"cz-ladder n={n} depth={a.depth} seed=1, 4 virtual ranks on one GPU "
                       f"(2^{a.local} amplitudes each)"}
    # serial_sX: exchange steps alone, swaps capped at X SMs (an exchange as
    # slow as X SMs make it -- the regime of an NVLink-bound exchange);
    # overlap_bB_sX: the same swaps pipelined over 2^B blocks
    configs = [("serial", dict(overlap=False))]
    for sms in [int(v) for v in a.sms.split(",")]:
        configs.append((f"serial_s{sms}", dict(overlap=False, exchange_sms=sms)))
        for bits in (1, 2, 3):
            configs.append((f"overlap_b{bits}_s{sms}",
                            dict(overlap=True, overlap_bits=bits, overlap_sms=sms)))
    for name, kw in configs:
        res = run(n, recs, a.reps, **kw)
        res["sec_per_layer"] = res["circuit_s"] / (a.depth + 1)
        out[name] = res
        print(name, json.dumps(res), flush=True)
        assert math.isfinite(res["norm"]) and abs(res["norm"] - 1.0) < 1e-9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
