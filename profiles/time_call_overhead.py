"""Per-call host overhead of single-gate application (reference budget:
bindings/tests/test_bindings.py:581-590, <= 2 us of binding overhead over the
core call).  Median wall time per call over batches of calls, for the
Qulacs-named handle and the core gate at n=2 and n=10, and the device time of
the same gate, so the host share is visible."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg  # noqa: E402


def median_call(fn, calls=5000, batches=7):
    meds = []
    for _ in range(batches):
        t0 = time.perf_counter()
        for _ in range(calls):
            fn()
        meds.append((time.perf_counter() - t0) / calls)
    return sorted(meds)[len(meds) // 2]


out = {}
for n in (2, 10, 20):
    st = qs.QuantumState(n)
    for name, g in (("X(0)", qg.X(0)), ("RX(3)", qg.RX(min(3, n - 1), 0.3)),
                    ("CNOT(0,1)", qg.CNOT(0, 1))):
        bound = median_call(lambda: g.update_quantum_state(st))
        core = median_call(lambda: g._core.apply(st))
        st.synchronize()
        out[f"n={n} {name}"] = {"handle_us": bound * 1e6, "core_us": core * 1e6,
                                "binding_overhead_us": (bound - core) * 1e6}
        print(f"n={n} {name}: handle {bound*1e6:.2f} us, core {core*1e6:.2f} us", flush=True)
print(json.dumps(out))
