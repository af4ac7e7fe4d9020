"""Sharded engine (paper_2011_13524_b200.dist) on CPU: virtual ranks in one
process, and real 2- and 4-process runs over gloo, with the oracle as the
shard backend.  Checks the qubit map, per-rank specialisation of global
controls / diagonals / Z signs, the swap exchange and the reductions."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2011_13524_b200.dist import ShardedQuantumState, specialize

from oracle import qsim_oracle as orc
from dist_util import (OracleShard, SharedOracleShard, circuit_of, observable_of,
                       random_records, tfim_terms)


def _reference(n, records, seed):
    a = orc.haar_state(n, seed)
    return orc.run_records(a, n, records)


@pytest.mark.parametrize("n,world", [(6, 2), (7, 4), (8, 8), (9, 2)])
def test_virtual_ranks_match_oracle(n, world):
    recs = random_records(n, 60, seed=n * 10 + world)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: OracleShard(L, r))
    st.load(orc.haar_state(n, 3))
    circuit_of(n, recs).update_quantum_state(st)
    got = st.get_vector()
    ref = _reference(n, recs, 3)
    assert np.max(np.abs(got - ref)) <= 1e-12
    assert st.stats["swaps"] > 0
    assert abs(st.get_squared_norm() - orc.squared_norm(ref)) <= 1e-12
    terms = [(0.7, [(0, 1), (n - 1, 3)]), (-0.2, [(n - 1, 1)]), (0.4, [(1, 2), (n - 2, 2)]),
             (1.1, [])]
    e = observable_of(n, terms).get_expectation_value(st)
    assert abs(e - orc.expectation(ref, ref, n, terms)) <= 1e-11


def test_cz_ladder_sharded_matches_oracle():
    n = 8
    recs = orc.cz_ladder_records(n, 4, seed=1)
    st = ShardedQuantumState(n, world=4, owned=[0, 1, 2, 3],
                             backend=lambda L, r: OracleShard(L, r))
    st.set_zero_state()
    circuit_of(n, recs).update_quantum_state(st)
    ref = orc.run_records(orc.zero_state(n), n, recs)
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_specialize_controls_and_signs():
    L = 3
    phys = [0, 1, 2, 3]  # qubit 3 is global
    # control on the global qubit: active only on rank 1
    rec = ("pauli", (0,), (1,), ((3, 1),))
    assert specialize(rec, phys, L, 0) is None
    assert specialize(rec, phys, L, 1)[0] == "dense"
    # Z on a global qubit flips the rotation angle on rank 1
    rot = ("pauli_rot", (0, 3), (1, 3), 0.5, ())
    assert specialize(rot, phys, L, 0)[3] == 0.5
    assert specialize(rot, phys, L, 1)[3] == -0.5
    with pytest.raises(ValueError):
        specialize(("dense", (3,), np.eye(2), ()), phys, L, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        recs = random_records(n, 40, seed=77)
        st = ShardedQuantumState(n, backend=lambda L, r: OracleShard(L, r), chunk_bytes=256)
        st.load(orc.haar_state(n, 5))
        circuit_of(n, recs).update_quantum_state(st)
        vec = st.get_vector()
        norm = st.get_squared_norm()
        e = observable_of(n, [(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])]).get_expectation_value(st)
        e_tf = observable_of(n, tfim_terms(n)).get_expectation_value(st)
        q.put((rank, vec, norm, (e, e_tf), dict(st.stats)))
    finally:
        dist.destroy_process_group()


def _worker_p2p(rank, world, port, n, q, overlap_min=20):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        recs = random_records(n, 40, seed=77)
        st = ShardedQuantumState(n, backend=lambda L, r: SharedOracleShard(L, r), exchange="p2p",
                                 overlap_min_qubits=overlap_min)
        st.load(orc.haar_state(n, 5))
        circuit_of(n, recs).update_quantum_state(st)
        vec = st.get_vector()
        e = observable_of(n, [(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])]).get_expectation_value(st)
        mode = st.exchange
        st.close()
        dist.barrier()
        for s in st.shards.values():
            s.release()
        q.put((rank, mode, vec, e, dict(st.stats)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap_min", [(2, 20), (4, 20), (2, 2), (4, 2)])
def test_gloo_processes_p2p_protocol(world, overlap_min):
    """The peer-memory exchange protocol (dist.ShardedQuantumState
    exchange="p2p": mapped peer shards, each owner swapping half of every
    pair's slice, barriers around the step) across processes, with shared
    memory standing in for CUDA IPC.  overlap_min=2: exchange steps are
    pipelined block by block with the following segment (barrier per
    block; 17 qubits, so that a shard leaves block qubits besides a tile)."""
    n = 7 if overlap_min >= 20 else 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_p2p, args=(r, world, port, n, q, overlap_min))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _reference(n, random_records(n, 40, seed=77), 5)
    e_ref = orc.expectation(ref, ref, n, [(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])])
    for rank, mode, vec, e, stats in res:
        assert mode == "p2p"
        assert np.max(np.abs(vec - ref)) <= 1e-12, rank
        assert abs(e - e_ref) <= 1e-11
        assert stats["swaps"] > 0
        assert (stats.get("overlapped", 0) > 0) == (overlap_min < 20)


@pytest.mark.parametrize("world", [2, 8])
def test_virtual_ranks_p2p_protocol(world):
    n = 9
    recs = random_records(n, 60, seed=5)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: SharedOracleShard(L, r), exchange="p2p")
    assert st.exchange == "p2p"
    st.load(orc.haar_state(n, 2))
    circuit_of(n, recs).update_quantum_state(st)
    got = st.get_vector()
    for s in st.shards.values():
        s.release()
    assert np.max(np.abs(got - _reference(n, recs, 2))) <= 1e-12


@pytest.mark.parametrize("world,bits", [(2, 1), (2, 2), (4, 2), (8, 1)])
def test_virtual_ranks_overlapped_remaps(world, bits):
    """Exchange steps pipelined with the segment that follows (block by
    block over 2^bits blocks) give the oracle's state, for random mixed
    records and for the cz-ladder (long overlappable prefixes).  Shards keep
    a 12-qubit tile besides the block qubits."""
    n = 14 + bits + world.bit_length() - 1
    for recs, seed in ((random_records(n, 80, seed=world + bits), 4),
                       (orc.cz_ladder_records(n, 6, seed=2), None)):
        st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                                 backend=lambda L, r: SharedOracleShard(L, r), exchange="p2p",
                                 overlap=True, overlap_bits=bits, overlap_min_qubits=2)
        if seed is None:
            st.set_zero_state()
            ref = orc.run_records(orc.zero_state(n), n, recs)
        else:
            st.load(orc.haar_state(n, seed))
            ref = _reference(n, recs, seed)
        circuit_of(n, recs).update_quantum_state(st)
        got = st.get_vector()
        for s in st.shards.values():
            s.release()
        assert st.stats.get("overlapped", 0) > 0
        assert np.max(np.abs(got - ref)) <= 1e-12


def test_overlap_plan_blocks_and_prefix():
    """The block qubits are the local qubits (not 0..3, not exchanged) whose
    first non-diagonal use comes last; the prefix stops at the first gate
    acting non-diagonally on one of them."""
    n, world = 16, 2  # L = 15
    st = ShardedQuantumState(n, world=world, owned=[0, 1],
                             backend=lambda L, r: SharedOracleShard(L, r), exchange="p2p",
                             overlap=True, overlap_bits=2, overlap_min_qubits=2)
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    seg = [("dense", (15,), h, ())] + [("dense", (q,), h, ()) for q in range(14, -1, -1)]
    seg.insert(3, ("diag", (6,), np.array([1, 1j]), ()))
    # logical 15 (global) swaps with physical 3: H on 15, 14, 13, diag, 12, ...
    blk, phys, prefix = st._overlap_plan([15], [3], seg)
    assert phys[15] == 3 and phys[3] == 15
    # positions 4 and 5 are used last (the H on qubit 3 acts on the global slot)
    assert blk == [4, 5] and prefix == seg.index(("dense", (5,), h, ()))
    assert st._overlap_plan([15], [3], seg[:1]) == ([13, 14], phys, 1)
    st.overlap = False
    assert st._overlap_plan([15], [3], seg) is None
    for s in st.shards.values():
        s.release()


@pytest.mark.parametrize("reorder", [True, False])
def test_reordered_segments_match_oracle(reorder):
    """Segments that run ahead past deferred gates (gates on disjoint qubits
    commute) and the circuit-order planner give the same state: random
    mixed records with controls, and a cz-ladder."""
    n, world = 9, 4
    for recs in (random_records(n, 120, seed=11), orc.cz_ladder_records(n, 5, seed=7)):
        st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                                 backend=lambda L, r: OracleShard(L, r), reorder=reorder)
        st.load(orc.haar_state(n, 2))
        circuit_of(n, recs).update_quantum_state(st)
        ref = _reference(n, recs, 2)
        assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_overlap_auto_only_across_processes():
    """overlap="auto" pipelines exchange steps only when peers are remote."""
    st = ShardedQuantumState(8, world=2, owned=[0, 1],
                             backend=lambda L, r: SharedOracleShard(L, r), exchange="p2p")
    assert st.overlap is False
    for s in st.shards.values():
        s.release()
    with pytest.raises(ValueError):
        ShardedQuantumState(8, world=2, owned=[0, 1], backend=lambda L, r: OracleShard(L, r),
                            overlap="yes")


def test_exchange_mode_selection():
    with pytest.raises(ValueError):
        ShardedQuantumState(5, world=2, owned=[0, 1], backend=lambda L, r: OracleShard(L, r),
                            exchange="p2p")
    with pytest.raises(ValueError):
        ShardedQuantumState(5, world=2, owned=[0, 1], backend=lambda L, r: OracleShard(L, r),
                            exchange="bogus")
    st = ShardedQuantumState(5, world=2, owned=[0, 1], backend=lambda L, r: OracleShard(L, r))
    assert st.exchange == "nccl"


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_processes_match_oracle(world):
    n = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _reference(n, random_records(n, 40, seed=77), 5)
    terms = [(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])]
    e_ref = orc.expectation(ref, ref, n, terms)
    tf_ref = orc.expectation(ref, ref, n, tfim_terms(n)).real
    for rank, vec, norm, (e, e_tf), stats in res:
        assert np.max(np.abs(vec - ref)) <= 1e-12, rank
        assert abs(norm - orc.squared_norm(ref)) <= 1e-12
        assert abs(e - e_ref) <= 1e-11
        assert abs(e_tf - tf_ref) <= 1e-11
        assert stats["swaps"] > 0


def test_multi_qubit_remaps_batch_global_qubits():
    """cz-ladder needs every qubit non-diagonally in every layer.  In circuit
    order (reorder=False) the planner brings all global qubits local in one
    remap per layer (k = log2 P), which moves (1 - 2^-k) of a shard instead
    of k/2 with one swap per qubit.  With segments that run ahead past the
    deferred gates (the default) the low qubits finish the whole circuit
    first: cz-ladder(36, 20) on 8 ranks needs ONE remap of the 3 global
    qubits (120 GB per rank instead of 2.65 TB)."""
    from paper_2011_13524_b200.dist import plan_exchange_bytes
    n, world = 36, 8
    recs = orc.cz_ladder_records(n, 20, seed=1)
    inorder = plan_exchange_bytes(n, world, recs, reorder=False)
    single = plan_exchange_bytes(n, world, recs, lookahead=0, reorder=False)
    assert inorder["qubits_remapped"] >= 3 * 20
    assert inorder["remaps"] <= 22
    assert inorder["bytes_sent_per_rank"] < 0.7 * single["bytes_sent_per_rank"]
    ahead = plan_exchange_bytes(n, world, recs)
    assert ahead["remaps"] == 1 and ahead["qubits_remapped"] == 3
    assert ahead["bytes_sent_per_rank"] == (16 << 33) * 7 / 8
    # small instance, every virtual rank, chunked N-d slice exchanges
    n = 9
    recs = orc.cz_ladder_records(n, 3, seed=2)
    st = ShardedQuantumState(n, world=8, owned=list(range(8)),
                             backend=lambda L, r: OracleShard(L, r), chunk_bytes=64)
    st.load(orc.haar_state(n, 4))
    circuit_of(n, recs).update_quantum_state(st)
    ref = orc.run_records(orc.haar_state(n, 4), n, recs)
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
    assert st.stats["remapped_qubits"] > st.stats["swaps"]


def _worker_k(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        recs = orc.cz_ladder_records(n, 3, seed=3)
        st = ShardedQuantumState(n, backend=lambda L, r: OracleShard(L, r), chunk_bytes=96)
        st.load(orc.haar_state(n, 6))
        circuit_of(n, recs).update_quantum_state(st)
        q.put((rank, st.get_vector(), dict(st.stats)))
    finally:
        dist.destroy_process_group()


def test_gloo_multi_qubit_remap_processes():
    n, world = 8, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_k, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = orc.run_records(orc.haar_state(n, 6), n, orc.cz_ladder_records(n, 3, seed=3))
    for rank, vec, stats in res:
        assert np.max(np.abs(vec - ref)) <= 1e-12, rank
        assert stats["remapped_qubits"] > stats["swaps"]


@pytest.mark.parametrize("n,world", [(6, 2), (8, 4), (9, 8)])
def test_sharded_tfim_expectation(n, world):
    """Observables with X on every qubit (TFIM, sum_i X_i): the union of the
    X/Y supports exceeds a shard, so terms are grouped and each group is
    brought local by its own remap; the state itself is unchanged (only the
    qubit map moves)."""
    recs = random_records(n, 50, seed=n + 3 * world)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: OracleShard(L, r))
    st.set_Haar_random_state(9)
    circuit_of(n, recs).update_quantum_state(st)
    ref = _reference(n, recs, 9)
    for terms in (tfim_terms(n), [(1.0, [(i, 1)]) for i in range(n)],
                  [(0.5, [(i, 2), ((i + 1) % n, 2)]) for i in range(n)]):
        e = observable_of(n, terms).get_expectation_value(st)
        assert isinstance(e, float)
        assert abs(e - orc.expectation(ref, ref, n, terms).real) <= 1e-11
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
    with pytest.raises(ValueError):  # one term wider than a shard
        observable_of(n, [(1.0, [(i, 1) for i in range(n)])]).get_expectation_value(st)


def test_sharded_state_reference_api():
    """The reference calls reach the sharded engine: gate / circuit
    update_quantum_state, Observable.get_expectation_value, get_qubit_count;
    maps and transition amplitudes between sharded states are refused."""
    from paper_2011_13524_b200 import GeneralQuantumOperator, QuantumCircuit, gate
    n, world = 6, 4
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: OracleShard(L, r))
    assert st.get_qubit_count() == n
    st.set_computational_basis(5)
    gate.H(n - 1).update_quantum_state(st)  # global qubit: a remap
    gate.CNOT(n - 1, 0).update_quantum_state(st)
    ref = np.zeros(1 << n, dtype=np.complex128)
    ref[5] = 1
    ref = orc.run_records(ref, n, [gate.H(n - 1)._core.record(),
                                   gate.CNOT(n - 1, 0)._core.record()])
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
    qc = QuantumCircuit(n)
    qc.add_gate(gate.DepolarizingNoise(0, 0.1))
    with pytest.raises(ValueError):
        qc.update_quantum_state(st)
    op = GeneralQuantumOperator(n)
    op.add_operator(1.0, "X 0")
    st2 = ShardedQuantumState(n, world=world, owned=list(range(world)),
                              backend=lambda L, r: OracleShard(L, r))
    with pytest.raises(ValueError):
        op.get_transition_amplitude(st, st2)
    with pytest.raises(ValueError):
        QuantumCircuit(n + 1).update_quantum_state(st)
