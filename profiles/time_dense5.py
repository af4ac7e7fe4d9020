"""One random 5-qubit dense gate (DenseMatrix on 5 targets, the fused blocks of
QuantumCircuitOptimizer().optimize(c, 5)) on an n-qubit state: device time,
FP64 rate (128 real FMA per amplitude) and HBM rate, for the DMMA kernel
(k_dense5_mma, default) or the DFMA kernel (QSV_DENSE5_MMA=0); also checks the
result against numpy on a sample of cosets.
    python profiles/time_dense5.py [n] [targets...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import gate as qg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
targets = [int(v) for v in sys.argv[2:]] or [0, 3, 9, 17, 25]
rng = np.random.default_rng(3)
q, r = np.linalg.qr(rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32)))
U = q * (np.diag(r) / np.abs(np.diag(r)))
g = qg.DenseMatrix(targets, U)
st = qs.QuantumState(n)
s = torch.cuda.current_stream()
st.set_stream(s.cuda_stream)
st.set_random_state_device(2)
before = st.get_vector() if n <= 24 else None
g.update_quantum_state(st)
torch.cuda.synchronize()
err = None
if before is not None:
    ref = before.reshape([2] * n)
    axes = [n - 1 - t for t in targets]  # numpy axis of qubit t (qubit 0 = last axis)
    ref = np.moveaxis(ref, axes[::-1], list(range(5)))
    ref = (U @ ref.reshape(32, -1)).reshape(ref.shape)
    ref = np.moveaxis(ref, list(range(5)), axes[::-1]).reshape(-1)
    err = float(np.max(np.abs(st.get_vector() - ref)))
best = 1e9
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    g.update_quantum_state(st)
    b.record(s)
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 1e3)
amps = 2 ** n
print(json.dumps({"n": n, "targets": targets, "mma": os.environ.get("QSV_DENSE5_MMA", "1"),
                  "s": best, "fp64_tflops": 2 * 128 * amps / best / 1e12,
                  "hbm_gbs": 32 * amps / best / 1e9, "max_err_vs_numpy": err}))
