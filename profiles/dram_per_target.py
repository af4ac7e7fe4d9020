"""CZ(t, t+1) and CNOT(t+1, t) of the cfg2 sweep at n=28, one launch each, for
an ncu capture of the physical DRAM traffic next to the touched-byte model
(CZ moves 32*2^(n-2) B, CNOT 32*2^(n-1) B).
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        python profiles/dram_per_target.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg  # noqa: E402

n = 28
st = qs.QuantumState(n)
st.set_random_state_device(3)
for t in (0, 1, 2, 3, 4, 14, 26):
    qg.CZ(t, (t + 1) % n).update_quantum_state(st)
for t in (0, 1, 2, 3, 4, 14, 26):
    qg.CNOT((t + 1) % n, t).update_quantum_state(st)
st.synchronize()
print("ok")
