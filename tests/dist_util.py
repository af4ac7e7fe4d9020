"""Test-only shard backend for the sharded engine: a numpy shard driven by
the CPU oracle (lets the host logic of paper_2011_13524_b200.dist run on CPU
with gloo).  Test infrastructure, never used by the product."""

from multiprocessing import resource_tracker, shared_memory

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

    def prepare(self, records, outer_mask=0):
        return list(records)

    def run(self, records):
        if records:
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


_BUFS = {}  # "pointer" -> numpy array (own shards and mapped peers)


def _spread(j, ls):
    for p in sorted(ls):
        j = ((j >> p) << (p + 1)) | (j & ((1 << p) - 1))
    return j


class SharedOracleShard(OracleShard):
    """OracleShard in POSIX shared memory with the peer-exchange interface
    of CudaShard (ptr / ipc_handle / open_peer / slice_swap): lets the p2p
    exchange protocol of dist.py (halves per owner, barriers, rounds) run
    across gloo processes on CPU, with the shm name standing in for the CUDA
    IPC handle."""

    def __init__(self, L, rank):
        self.L = L
        self.shm = shared_memory.SharedMemory(create=True, size=16 << L)
        self.a = np.ndarray(1 << L, dtype=np.complex128, buffer=self.shm.buf)
        self.a[:] = 0
        self.key = id(self.a)
        _BUFS[self.key] = self.a
        self._peers = {}

    def ptr(self):
        return self.key

    def device_id(self):
        return None

    def can_reach(self, device):
        return True

    def ipc_handle(self):
        return self.shm.name.encode()

    def open_peer(self, handle):
        shm = shared_memory.SharedMemory(name=handle.decode())
        resource_tracker.unregister(shm._name, "shared_memory")  # the owner unlinks
        arr = np.ndarray(1 << self.L, dtype=np.complex128, buffer=shm.buf)
        _BUFS[id(arr)] = arr
        self._peers[id(arr)] = shm
        return id(arr)

    def close_peer(self, key):
        _BUFS.pop(key, None)
        self._peers.pop(key).close()

    def slice_swap(self, peer, ls, d_mine, d_peer, j0, j1):
        j = _spread(np.arange(j0, j1, dtype=np.int64), ls)
        va = sum(((d_mine >> i) & 1) << p for i, p in enumerate(ls))
        vb = sum(((d_peer >> i) & 1) << p for i, p in enumerate(ls))
        b = _BUFS[peer]
        tmp = self.a[j | va].copy()
        self.a[j | va] = b[j | vb]
        b[j | vb] = tmp

    @staticmethod
    def blockwise(prepared):
        return True

    def run_block(self, records, mask, value, stream_ptr=None):
        """The records on the block {x : x & mask == value} only (they do not
        mix blocks): applied to a copy, the block copied back."""
        if not records:
            return
        idx = np.nonzero((np.arange(1 << self.L) & mask) == value)[0]
        tmp = self.a.copy()
        orc.run_records(tmp, self.L, records)
        self.a[idx] = tmp[idx]

    def discard(self, prepared):
        pass

    def set_sm_limit(self, sms):
        pass

    def release(self):
        _BUFS.pop(self.key, None)
        del self.a
        self.shm.close()
        self.shm.unlink()


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


def circuit_of(n, records):
    """QuantumCircuit holding the gates of neutral records, so that tests
    drive the sharded engine through the reference call
    ``circuit.update_quantum_state(state)`` (bindings __init__.py:118-119)."""
    from paper_2011_13524_b200 import QuantumCircuit
    from paper_2011_13524_b200 import _gates as G
    qc = QuantumCircuit(n)
    for rec in records:
        kind = rec[0]
        if kind == "dense":
            g = G.DenseGate(rec[1], rec[2], rec[3])
        elif kind == "diag":
            g = G.DiagonalGate(rec[1], rec[2], rec[3])
        elif kind == "pauli":
            g = G.PauliGate(rec[1], rec[2], rec[3])
        elif kind == "pauli_rot":
            g = G.PauliRotationGate(rec[1], rec[2], rec[3], rec[4])
        else:
            raise ValueError(f"no gate for record kind {kind!r}")
        qc.add_gate(g)
    return qc


def observable_of(n, terms):
    """Observable of (coef, [(qubit, axis)...]) terms, evaluated through the
    reference call ``Observable.get_expectation_value(state)``."""
    from paper_2011_13524_b200 import Observable
    obs = Observable(n)
    for coef, ops in terms:
        obs.add_operator(float(np.real(coef)),
                         " ".join(f"{'IXYZ'[a]} {q}" for q, a in ops))
    return obs


def tfim_terms(n, j=-1.0, h=-0.5):
    """Transverse-field Ising terms (SURVEY 8(d) cfg3 shape): X on every
    qubit, so no shard ever holds the union of the X supports."""
    return ([(j, [(i, 3), (i + 1, 3)]) for i in range(n - 1)]
            + [(h, [(i, 1)]) for i in range(n)])
