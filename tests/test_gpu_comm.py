"""NCCL communicator inside libqsv (csrc/qsv_comm.cu) on one GPU: a
one-rank communicator (NCCL refuses two ranks on one device, so the
multi-rank protocol is covered by the gloo tests of dist.py): device
barrier, all-reduce, and the chunked gather / send / recv / scatter slice
exchange against numpy slicing."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _comm():
    from paper_2011_13524_b200 import _lib
    lib = _lib.lib
    assert lib.qsv_comm_available() == 1
    uid = C.create_string_buffer(128)
    _lib.check(lib.qsv_comm_unique_id(uid))
    h = C.c_void_p()
    _lib.check(lib.qsv_comm_create(uid, 1, 0, 0, C.byref(h)))
    return lib, h


def _slice_idx(n, ls, d):
    idx = np.arange(1 << n)
    keep = np.ones(1 << n, dtype=bool)
    for j, b in enumerate(ls):
        keep &= ((idx >> b) & 1) == ((d >> j) & 1)
    return idx[keep]


@pytest.mark.parametrize("n,ls,ds,dr,chunk", [(12, [3], 0, 1, 0), (14, [0, 9], 2, 1, 4096),
                                              (16, [15, 4, 7], 5, 3, 16 * 1000)])
def test_slice_exchange_with_self(n, ls, ds, dr, chunk):
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import _lib
    lib, h = _comm()
    try:
        st = qs.QuantumState(n)
        st.set_Haar_random_state(5)
        before = st.get_vector()
        arr = (C.c_int * len(ls))(*ls)
        _lib.check(lib.qsv_comm_slice_exchange(h, st._handle(), 0, arr, len(ls), ds, dr, chunk))
        got = st.get_vector()
        want = before.copy()
        want[_slice_idx(n, ls, dr)] = before[_slice_idx(n, ls, ds)]
        assert np.array_equal(got, want)
    finally:
        lib.qsv_comm_destroy(h)


def test_barrier_and_allreduce():
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import _lib
    lib, h = _comm()
    try:
        st = qs.QuantumState(4)
        _lib.check(lib.qsv_comm_barrier(h, st._handle()))
        vals = np.array([1.5, -2.25, 3.0])
        _lib.check(lib.qsv_comm_allreduce_sum(h, st._handle(), vals.ctypes.data, 3))
        assert list(vals) == [1.5, -2.25, 3.0]  # one rank: the sum is the value
        r, w = C.c_int(), C.c_int()
        _lib.check(lib.qsv_comm_rank(h, C.byref(r), C.byref(w)))
        assert (r.value, w.value) == (0, 1)
        bad = (C.c_int * 1)(40)
        assert lib.qsv_comm_slice_exchange(h, st._handle(), 0, bad, 1, 0, 1, 0) != 0
        assert lib.qsv_comm_slice_exchange(h, st._handle(), 3, bad, 0, 0, 0, 0) != 0
    finally:
        lib.qsv_comm_destroy(h)
