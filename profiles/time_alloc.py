"""State create/copy/destroy cost (the pooled stream-ordered allocator)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13524_b200 as qs  # noqa: E402

for n in (10, 16, 20, 24):
    st = qs.QuantumState(n)
    st.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        c = st.copy()
        del c
    st.synchronize()
    t1 = time.perf_counter()
    for _ in range(200):
        s2 = qs.QuantumState(n)
        del s2
    st.synchronize()
    t2 = time.perf_counter()
    print(f"n={n}: copy+free {(t1 - t0) / 200 * 1e6:.1f} us, create+free {(t2 - t1) / 200 * 1e6:.1f} us",
          flush=True)
