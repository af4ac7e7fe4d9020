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
from dist_util import random_records

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
    st.apply_records(recs)
    got = st.get_vector()
    ref = c_oracle.run_records(orc.haar_state(n, 1), n, recs)
    assert np.max(np.abs(got - ref)) <= 1e-12
    assert st.stats["swaps"] > 0
    assert abs(st.get_squared_norm() - 1.0) <= 1e-12
    terms = [(0.5, [(n - 1, 1), (0, 3)]), (-1.0, [(n - 2, 2), (1, 1)]), (0.25, [])]
    assert abs(st.expectation(terms) - orc.expectation(ref, ref, n, terms)) <= 1e-11


def test_cuda_sharded_cz_ladder():
    import torch
    stream = torch.cuda.current_stream().cuda_stream
    n, world = 18, 8
    recs = orc.cz_ladder_records(n, 6, seed=1)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream))
    st.set_zero_state()
    st.apply_records(recs)
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
    for r in recs:
        st.apply_records([r])
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


def _ipc_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        st = ShardedQuantumState(n, exchange="p2p")
        recs = random_records(n, 60, seed=31)
        st.load(orc.haar_state(n, 6))
        st.apply_records(recs)
        vec = st.get_vector()
        norm = st.get_squared_norm()
        e = st.expectation([(0.3, [(n - 1, 1), (0, 3)]), (0.9, [(1, 2)])])
        stats = dict(st.stats)
        mode = st.exchange
        st.close()
        q.put((rank, mode, vec, norm, e, stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ipc_processes_p2p_exchange(world):
    """One process per shard, shards mapped with CUDA IPC, exchanges by
    qsv_slice_swap on the peer's mapped buffer (each owner swaps half)."""
    n = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, n, q)) for r in range(world)]
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


@pytest.mark.parametrize("world", [2, 4, 8])
def test_cfg5_shape_sharded_matches_single_state(world):
    """cfg5's workload shape at n=24 (the sharded engine at
    n<=24 on P=2/4/8): cz-ladder(24, depth 20, seed 1) over P virtual ranks
    (p2p remaps, rank-specialised tiled segments) against the single-state
    engine, itself pinned to the C oracle at n=30 (profiles/r1_parity_n30.json)."""
    import torch
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import workloads
    from paper_2011_13524_b200._circuit import circuit_records
    n = 24
    circ = workloads.generate_cz_ladder(n, 20, seed=1)
    one = qs.QuantumState(n)
    circ.update_quantum_state(one)
    ref = one.get_vector()
    stream = torch.cuda.current_stream().cuda_stream
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream))
    st.set_zero_state()
    st.apply_records(circuit_records(circ))
    assert st.exchange == "p2p" and st.stats["swaps"] > 0
    assert np.max(np.abs(st.get_vector() - ref)) <= 1e-12
    assert abs(st.get_squared_norm() - 1.0) <= 1e-12
