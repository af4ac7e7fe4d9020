"""Sharded engine with the CUDA shard backend on one GPU: several virtual
ranks in one process (exchanges through qsv_slice_swap on the other shard's
pointer, or device copies through torch views in "nccl" mode), and several
processes sharing the GPU whose shards are mapped into each other with CUDA
IPC (the cross-process p2p path of a multi-GPU node, gloo for the host
barriers).  Checks per-rank compiled segments, swaps and reductions against
the oracle."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2011_13524_b200.dist import CudaShard, ShardedQuantumState

from oracle import c_oracle, qsim_oracle as orc
from dist_util import circuit_of, observable_of, random_records, tfim_terms

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
@pytest.mark.parametrize("n,world", [(8, 2), (10, 4), (12, 8), (16, 4)])
def test_cuda_virtual_ranks(n, world, exchange):
    import torch
    stream = torch.cuda.current_stream().cuda_stream
    recs = random_records(n, 80, seed=n + world)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream), exchange=exchange)
    assert st.exchange == exchange
    st.load(orc.haar_state(n, 1))
    circuit_of(n, recs).update_quantum_state(st)
    got = st.get_vector()
    ref = c_oracle.run_records(orc.haar_state(n, 1), n, recs)
    assert np.max(np.abs(got - ref)) <= 1e-12
    assert st.stats["swaps"] > 0
    assert abs(st.get_squared_norm() - 1.0) <= 1e-12
    terms = [(0.5, [(n - 1, 1), (0, 3)]), (-1.0, [(n - 2, 2), (1, 1)]), (0.25, [])]
    e = observable_of(n, terms).get_expectation_value(st)
    assert abs(e - orc.expectation(ref, ref, n, terms)) <= 1e-11
    tf = tfim_terms(n)  # X on every qubit: groups of terms remapped in turn
    e = observable_of(n, tf).get_expectation_value(st)
    assert abs(e - orc.expectation(ref, ref, n, tf).real) <= 1e-11


def test_cuda_sharded_cz_ladder():
    import torch
    stream = torch.cuda.current_stream().cuda_stream
    n, world = 18, 8
    recs = orc.cz_ladder_records(n, 6, seed=1)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream))
    st.set_zero_state()
    circuit_of(n, recs).update_quantum_state(st)
    ref = c_oracle.run_records(orc.zero_state(n), n, recs)
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_cuda_sharded_per_gate_mode():
    """Per-gate mode (the sharded benchmark path): direct ABI calls, no programs."""
    import torch
    stream = torch.cuda.current_stream().cuda_stream
    n, world = 12, 4
    recs = random_records(n, 60, seed=9)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream, use_tiles=0, fuse=0))
    st.load(orc.haar_state(n, 2))
    from paper_2011_13524_b200 import QuantumGateBase
    for g in circuit_of(n, recs)._core.gates:  # gate.update_quantum_state(state)
        QuantumGateBase(g).update_quantum_state(st)
    ref = c_oracle.run_records(orc.haar_state(n, 2), n, recs)
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_slice_swap_ranges_and_errors():
    """qsv_slice_swap directly: half ranges, unsorted slice bits, bad input."""
    import torch
    stream = torch.cuda.current_stream().cuda_stream
    L = 10
    a, b = CudaShard(L, 0, stream), CudaShard(L, 0, stream)
    va, vb = orc.haar_state(L, 3), orc.haar_state(L, 4)
    a.load(va)
    b.load(vb)
    ls, dm, dp = [7, 2], 0b10, 0b01  # a's slice x7=0,x2=1 <-> b's slice x7=1,x2=0
    cnt = 1 << (L - 2)
    a.slice_swap(b.ptr(), ls, dm, dp, 0, cnt // 2)
    a.slice_swap(b.ptr(), ls, dm, dp, cnt // 2, cnt)
    x = np.arange(1 << L)
    sa = x[(((x >> 7) & 1) == 0) & (((x >> 2) & 1) == 1)]
    sb = x[(((x >> 7) & 1) == 1) & (((x >> 2) & 1) == 0)]
    ea, eb = va.copy(), vb.copy()
    ea[sa], eb[sb] = vb[sb], va[sa]
    assert np.array_equal(a.get(), ea) and np.array_equal(b.get(), eb)
    with pytest.raises(ValueError):
        a.slice_swap(b.ptr(), [3, 3], 0, 1, 0, 1)
    with pytest.raises(ValueError):
        a.slice_swap(b.ptr(), [3], 0, 1, 0, 1 << L)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, n, q, overlap_min=20):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        st = ShardedQuantumState(n, exchange="p2p", overlap_min_qubits=overlap_min)
        recs = random_records(n, 60, seed=31)
        st.load(orc.haar_state(n, 6))
        circuit_of(n, recs).update_quantum_state(st)
        vec = st.get_vector()
        norm = st.get_squared_norm()
        e = observable_of(n, [(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])]).get_expectation_value(st)
        stats = dict(st.stats)
        mode = st.exchange
        st.close()
        q.put((rank, mode, vec, norm, e, stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap_min", [(2, 20), (4, 20), (2, 4), (4, 4)])
def test_ipc_processes_p2p_exchange(world, overlap_min):
    """One process per shard, shards mapped with CUDA IPC, exchanges by
    qsv_slice_swap on the peer's mapped buffer (each owner swaps half).
    overlap_min=4: exchange steps pipelined with the following segment
    (compute stream + SM-limited swaps, barrier per block; 17 qubits so a
    shard keeps a 12-qubit tile besides the block qubits)."""
    n = 12 if overlap_min >= 20 else 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, n, q, overlap_min))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    recs = random_records(n, 60, seed=31)
    ref = c_oracle.run_records(orc.haar_state(n, 6), n, recs)
    terms = [(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])]
    e_ref = orc.expectation(ref, ref, n, terms)
    for rank, mode, vec, norm, e, stats in res:
        assert mode == "p2p"
        assert np.max(np.abs(vec - ref)) <= 1e-12, rank
        assert abs(norm - 1.0) <= 1e-12
        assert abs(e - e_ref) <= 1e-11
        assert stats["swaps"] > 0
        assert (stats.get("overlapped", 0) > 0) == (overlap_min < 20)


_CFG5_REF = {}


def _cfg5_reference(n):
    """cz-ladder(n, depth 20, seed 1) from |0> by the plain-C oracle
    (computed once per session, shared by the P = 2/4/8 cases)."""
    if n not in _CFG5_REF:
        from paper_2011_13524_b200 import workloads
        from paper_2011_13524_b200._circuit import circuit_records
        recs = circuit_records(workloads.generate_cz_ladder(n, 20, seed=1))
        _CFG5_REF[n] = c_oracle.run_records(orc.zero_state(n), n, recs)
    return _CFG5_REF[n]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_cfg5_shape_sharded_matches_oracle(world):
    """cfg5's workload shape at n=24 (the sharded engine at
    n<=24 on P=2/4/8 vs the oracle): cz-ladder(24, depth 20, seed 1) over P
    virtual ranks (p2p remaps, rank-specialised tiled segments), driven
    through circuit.update_quantum_state / Observable.get_expectation_value,
    against the plain-C oracle at 1e-12 (amplitudes) and 1e-10 relative
    (TFIM energy)."""
    import torch
    from paper_2011_13524_b200 import workloads
    n = 24
    ref = _cfg5_reference(n)
    circ = workloads.generate_cz_ladder(n, 20, seed=1)
    stream = torch.cuda.current_stream().cuda_stream
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream))
    st.set_zero_state()
    circ.update_quantum_state(st)
    assert st.exchange == "p2p" and st.stats["swaps"] > 0
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
    assert abs(st.get_squared_norm() - 1.0) <= 1e-12
    tf = tfim_terms(n)
    e = observable_of(n, tf).get_expectation_value(st)
    e_ref = orc.expectation(ref, ref, n, tf).real
    assert abs(e - e_ref) <= 1e-10 * max(abs(e_ref), 1e-6 * sum(abs(c) for c, _ in tf))


@pytest.mark.parametrize("n,world,bits", [(16, 2, 1), (18, 4, 2), (20, 8, 3)])
def test_cuda_overlapped_remaps(n, world, bits):
    """Exchange steps pipelined with the following segment on the product
    backend: the segment prefix runs block by block (qsv_program_run_fixed)
    on a second stream while SM-capped slice swaps exchange the next block;
    random records and the cz-ladder against the C oracle."""
    for recs, seed in ((random_records(n, 80, seed=n + bits), 3),
                       (orc.cz_ladder_records(n, 8, seed=1), None)):
        st = ShardedQuantumState(n, world=world, owned=list(range(world)), overlap=True,
                                 overlap_bits=bits, overlap_min_qubits=4, overlap_sms=7)
        assert st.exchange == "p2p"
        if seed is None:
            st.set_zero_state()
            ref = c_oracle.run_records(orc.zero_state(n), n, recs)
        else:
            st.load(orc.haar_state(n, seed))
            ref = c_oracle.run_records(orc.haar_state(n, seed), n, recs)
        circuit_of(n, recs).update_quantum_state(st)
        assert st.stats.get("overlapped", 0) > 0
        assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
        assert abs(st.get_squared_norm() - 1.0) <= 1e-12


def test_cfg5_shape_overlapped_matches_oracle():
    """cz-ladder(24, 20) over 4 virtual ranks with every eligible exchange
    step overlapped (L = 22, blocks of 2^20) against the plain-C oracle."""
    from paper_2011_13524_b200 import workloads
    n = 24
    ref = _cfg5_reference(n)
    circ = workloads.generate_cz_ladder(n, 20, seed=1)
    st = ShardedQuantumState(n, world=4, owned=[0, 1, 2, 3], overlap=True,
                             overlap_min_qubits=16)
    st.set_zero_state()
    circ.update_quantum_state(st)
    assert st.stats.get("overlapped", 0) > 0
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12


def test_state_view_and_sm_limit():
    """qsv_state_view aliases a block of its parent (gates on the view act on
    that block only); qsv_set_sm_limit changes no result; bad views raise."""
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import workloads
    from paper_2011_13524_b200._circuit import circuit_records
    n, m = 16, 14
    st = qs.QuantumState(n)
    st.set_Haar_random_state(4)
    full = st.get_vector()
    circ = workloads.generate_cz_ladder(m, 4, seed=3)
    recs = circuit_records(circ)
    v = st._view(2 << m, m)
    v._set_sm_limit(5)
    circ.update_quantum_state(v)
    got = st.get_vector()
    blk = c_oracle.run_records(full[2 << m:3 << m].copy(), m, recs)
    assert np.max(np.abs(got[2 << m:3 << m] - blk)) <= 1e-12
    mask = np.ones(1 << n, dtype=bool)
    mask[2 << m:3 << m] = False
    assert np.array_equal(got[mask], full[mask])
    with pytest.raises(ValueError):
        st._view(3, m)  # not a multiple of 2^m
    with pytest.raises(ValueError):
        st._view(0, n + 1)
    with pytest.raises(ValueError):
        st._view(4 << m, m)  # outside the state
    with pytest.raises(ValueError):
        st._set_sm_limit(-1)


def test_program_run_fixed_blocks():
    """A program planned with an outer mask, run block by block with
    qsv_program_run_fixed, equals the program run once; a mask on a tile
    qubit and a program with per-gate kernels are refused."""
    import ctypes as C
    from paper_2011_13524_b200 import _lib
    from paper_2011_13524_b200._lib import check, lib
    from paper_2011_13524_b200.dist import active_qubits, records_to_ops
    n = 18
    blk = [6, 13]
    mask = sum(1 << p for p in blk)
    rng = np.random.default_rng(5)
    recs = orc.cz_ladder_records(n, 3, seed=4)
    # gates touching the block qubits only diagonally / as controls
    recs = [r for r in recs if not active_qubits(r) & {6, 13}]
    recs.append(("diag", (6, 2), np.exp(1j * rng.uniform(0, 6, 4)), ()))
    recs.append(("dense", (3,), np.array([[0, 1], [1, 0]]), ((13, 1),)))
    ops, keep = records_to_ops(recs)

    def prog(outer):
        o = default = _lib.QsvPlanOpts()
        o.use_tiles, o.fuse, o.use_graph, o.real_frames = 1, 1, 0, 1
        o.outer_mask = outer
        h = C.c_void_p()
        check(lib.qsv_program_create(n, ops, len(recs), C.byref(default), C.byref(h)))
        return h

    import paper_2011_13524_b200 as qs
    st = qs.QuantumState(n)
    st.set_Haar_random_state(8)
    h = prog(mask)
    for j in range(4):
        value = sum(((j >> b) & 1) << p for b, p in enumerate(blk))
        check(lib.qsv_program_run_fixed(h, st._handle(), mask, value))
    ref = c_oracle.run_records(orc.haar_state(n, 8), n, recs)
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
    lib.qsv_program_destroy(h)
    h = prog(0)  # tiles may use qubit 6 / 13 now
    with pytest.raises(ValueError):
        check(lib.qsv_program_run_fixed(h, st._handle(), 1, 0))  # qubit 0 is in every tile
    with pytest.raises(ValueError):
        check(lib.qsv_program_run_fixed(h, st._handle(), mask, 1))  # value outside the mask
    lib.qsv_program_destroy(h)
    one = [("dense", (2,), np.array([[1, 1], [1, -1]]) / np.sqrt(2), ())]  # lone gate: a kernel
    ops1, keep1 = records_to_ops(one)
    o = _lib.QsvPlanOpts()
    o.use_tiles, o.fuse, o.use_graph, o.real_frames, o.outer_mask = 1, 0, 0, 0, 0
    h1 = C.c_void_p()
    check(lib.qsv_program_create(n, ops1, 1, C.byref(o), C.byref(h1)))
    with pytest.raises(RuntimeError):
        check(lib.qsv_program_run_fixed(h1, st._handle(), mask, 0))
    lib.qsv_program_destroy(h1)
