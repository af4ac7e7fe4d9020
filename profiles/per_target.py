"""Per-target device time of single gates at n=28 (algorithmic GB/s).

    python profiles/per_target.py [n] [gate ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
if os.environ.get("L2_FETCH"):
    # experiment: cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity = 0x05, bytes)
    import ctypes
    torch.cuda.init()
    rt = ctypes.CDLL("libcudart.so.12")
    v = ctypes.c_size_t()
    rt.cudaDeviceGetLimit(ctypes.byref(v), 0x05)
    print("L2 fetch granularity was", v.value, flush=True)
    print("set rc", rt.cudaDeviceSetLimit(0x05, ctypes.c_size_t(int(os.environ["L2_FETCH"]))))
    rt.cudaDeviceGetLimit(ctypes.byref(v), 0x05)
    print("now", v.value, flush=True)
kinds = sys.argv[2:] or ["CZ", "CNOT"]
st = qs.QuantumState(n)
st.set_random_state_device(3)
for kind in kinds:
    row = []
    for t in range(n - 1):
        g = qg.CZ(t, t + 1) if kind == "CZ" else qg.CNOT((t + 1) % n, t) if kind == "CNOT" \
            else getattr(qg, kind)(t)
        frac = 0.25 if kind == "CZ" else 0.5 if kind == "CNOT" else 1.0
        g.update_quantum_state(st)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.update_quantum_state(st)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 1e3)
        row.append(f"{t}:{32 * frac * 2 ** n / best / 1e9:.0f}")
    print(kind, " ".join(row), flush=True)
