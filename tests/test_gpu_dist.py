"""Sharded engine with the CUDA shard backend, several virtual ranks on one
GPU (exchanges become device copies through torch views of the libqsv
buffers).  Checks per-rank compiled segments, swaps and reductions against
the oracle."""

import numpy as np
import pytest

from paper_2011_13524_b200.dist import CudaShard, ShardedQuantumState

from oracle import c_oracle, qsim_oracle as orc
from dist_util import random_records

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,world", [(8, 2), (10, 4), (12, 8), (16, 4)])
def test_cuda_virtual_ranks(n, world):
    import torch
    stream = torch.cuda.current_stream().cuda_stream
    recs = random_records(n, 80, seed=n + world)
    st = ShardedQuantumState(n, world=world, owned=list(range(world)),
                             backend=lambda L, r: CudaShard(L, 0, stream))
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
