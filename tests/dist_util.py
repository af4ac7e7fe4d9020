"""Test-only shard backend for the sharded engine: a numpy shard driven by
the CPU oracle (lets the host logic of paper_2011_13524_b200.dist run on CPU
with gloo).  Test infrastructure, never used by the product."""

import numpy as np
import torch

from oracle import qsim_oracle as orc


class OracleShard:
    def __init__(self, L, rank):
        self.L = L
        self.a = np.zeros(1 << L, dtype=np.complex128)

    def set_zero(self, one):
        self.a[:] = 0
        if one:
            self.a[0] = 1

    def set_basis(self, k):
        self.a[:] = 0
        self.a[k] = 1

    def load(self, arr):
        self.a[:] = arr

    def get(self):
        return self.a.copy()

    def apply_records(self, records):
        orc.run_records(self.a, self.L, records)

    def norm2(self):
        return orc.squared_norm(self.a)

    def scale(self, f):
        self.a *= f

    def expect_terms(self, terms):
        return orc.expectation(self.a, self.a, self.L, terms)

    def tensor(self):
        return torch.from_numpy(self.a.view(np.float64))

    def sync(self):
        pass


def random_records(n, ngates, seed):
    """Random mix of every record kind with controls and diagonals on all
    qubits (global ones included)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(ngates):
        perm = [int(v) for v in rng.permutation(n)]
        k = int(rng.integers(0, 7))
        if k == 0:
            t = perm[:int(rng.integers(1, 3))]
            d = 1 << len(t)
            z = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
            q, r = np.linalg.qr(z)
            out.append(("dense", tuple(t), q, ()))
        elif k == 1:
            out.append(("pauli", (perm[0],), (1,), ((perm[1], int(rng.integers(2))),)))
        elif k == 2:
            out.append(("diag", (perm[0],), np.array([1, -1], dtype=complex), ((perm[1], 1),)))
        elif k == 3:
            m = int(rng.integers(1, 4))
            out.append(("diag", tuple(perm[:m]), np.exp(1j * rng.uniform(0, 6, 1 << m)), ()))
        elif k == 4:
            m = int(rng.integers(1, 4))
            out.append(("pauli_rot", tuple(perm[:m]), tuple(int(v) for v in rng.integers(1, 4, m)),
                        float(rng.uniform(-6, 6)), ()))
        elif k == 5:
            m = int(rng.integers(1, 3))
            out.append(("pauli", tuple(perm[:m]), tuple(int(v) for v in rng.integers(1, 4, m)), ()))
        else:
            t = (perm[0],)
            z = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
            q, r = np.linalg.qr(z)
            out.append(("dense", t, q, ((perm[1], int(rng.integers(2))), (perm[2], 1))))
    return out
