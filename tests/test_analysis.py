"""State analysis and reshaping: marginal
probabilities, Z-basis sampling, element-wise multiply, tensor_product,
permutate_qubit, drop_qubit.

CPU tests pin the oracle restatement (oracle/qsim_oracle.py) to the
reference's own outputs (tests/golden/analysis.*, made by
tests/golden/make_golden.py).  GPU tests run the CUDA kernels through the
C ABI and compare with the same fixtures and with the oracle at larger n:
bit-exact for sample indices and gathers, <= 1e-12 for probabilities and
products.
"""

import json
import os

import numpy as np
import pytest

from oracle import qsim_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_analysis():
    with open(os.path.join(GOLDEN, "analysis.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLDEN, "analysis.npz"))


# ----------------------------------------------------------------- CPU pins
def test_oracle_marginal_matches_reference():
    meta, _ = load_analysis()
    for c in meta["marginal"]:
        got = orc.marginal_probability(orc.haar_state(c["n"], c["seed"]), c["n"], c["pattern"])
        assert got == c["value"], c


def test_oracle_sampling_matches_reference():
    meta, _ = load_analysis()
    for c in meta["sampling"]:
        got = orc.sampling(orc.haar_state(c["n"], c["seed"]), c["count"], c["sample_seed"])
        assert got == c["samples"], (c["n"], c["count"])


def test_oracle_reshaping_matches_reference():
    meta, outs = load_analysis()
    for c in meta["tensor"]:
        got = orc.tensor_product(orc.haar_state(c["n1"], c["s1"]), orc.haar_state(c["n2"], c["s2"]))
        assert np.array_equal(got, outs[c["key"]])
    for c in meta["permutate"]:
        got = orc.permutate_qubit(orc.haar_state(c["n"], c["seed"]), c["n"], c["order"])
        assert np.array_equal(got, outs[c["key"]])
    for c in meta["drop"]:
        got = orc.drop_qubit(orc.haar_state(c["n"], c["seed"]), c["n"], c["targets"], c["values"])
        assert np.array_equal(got, outs[c["key"]])


# ------------------------------------------------------------------ GPU path
def _qs():
    import paper_2011_13524_b200 as qs
    return qs


def _haar(n, seed):
    s = _qs().QuantumState(n)
    s.set_Haar_random_state(seed)
    return s


@pytest.mark.gpu
def test_gpu_marginal_golden_and_oracle():
    meta, _ = load_analysis()
    for c in meta["marginal"]:
        got = _haar(c["n"], c["seed"]).get_marginal_probability(c["pattern"])
        assert abs(got - c["value"]) <= 1e-12, c
    rng = np.random.default_rng(5)
    for n in (1, 6, 17, 20):
        st = _haar(n, n)
        ref_amps = orc.haar_state(n, n)
        for _ in range(6):
            pat = [int(v) for v in rng.integers(0, 3, size=n)]
            got = st.get_marginal_probability(pat)
            ref = orc.marginal_probability(ref_amps, n, pat)
            assert abs(got - ref) <= 1e-12 * max(1.0, ref), (n, pat)
    # every qubit fixed (deposit path, more fixed bits than widen() handles)
    n = 30
    st = _qs().QuantumState(n)
    st.set_computational_basis((1 << 29) | 5)
    pat = [1, 0, 1] + [0] * 26 + [1]
    assert st.get_marginal_probability(pat) == 1.0
    pat[1] = 1
    assert st.get_marginal_probability(pat) == 0.0
    with pytest.raises(ValueError):
        st.get_marginal_probability([0, 1])
    with pytest.raises(ValueError):
        st.get_marginal_probability([3] + [2] * 29)


@pytest.mark.gpu
def test_gpu_sampling_golden_and_oracle():
    meta, _ = load_analysis()
    for c in meta["sampling"]:
        got = _haar(c["n"], c["seed"]).sampling(c["count"], seed=c["sample_seed"])
        assert got == c["samples"], (c["n"], c["count"])
    for n in (1, 3, 8, 9, 14, 20):
        st = _haar(n, 100 + n)
        got = st.sampling(5000, seed=n)
        ref = orc.sampling(orc.haar_state(n, 100 + n), 5000, n)
        mism = sum(1 for a, b in zip(got, ref) if a != b)
        assert mism == 0, (n, mism)
    # a basis state always samples its index; zero-probability blocks skipped
    st = _qs().QuantumState(22)
    st.set_computational_basis(3_000_001)
    assert set(st.sampling(777, seed=1)) == {3_000_001}
    assert st.sampling(0) == []
    with pytest.raises(ValueError):
        st.sampling(-1)


@pytest.mark.gpu
def test_gpu_reshaping_golden():
    qs = _qs()
    from paper_2011_13524_b200 import state as qstate
    meta, outs = load_analysis()
    for c in meta["tensor"]:
        got = qstate.tensor_product(_haar(c["n1"], c["s1"]), _haar(c["n2"], c["s2"]))
        assert got.get_qubit_count() == c["n1"] + c["n2"]
        assert np.max(np.abs(got.get_vector() - outs[c["key"]])) <= 1e-15
    for c in meta["permutate"]:
        got = qstate.permutate_qubit(_haar(c["n"], c["seed"]), c["order"]).get_vector()
        assert np.array_equal(got, outs[c["key"]])
    for c in meta["drop"]:
        got = qstate.drop_qubit(_haar(c["n"], c["seed"]), c["targets"], c["values"]).get_vector()
        assert np.array_equal(got, outs[c["key"]])
    # more dropped qubits than widen() handles (deposit path)
    n = 31
    st = qs.QuantumState(n)
    st.set_computational_basis((1 << 30) | 2)
    tg = list(range(1, 31))
    vals = [1] + [0] * 28 + [1]
    out = qstate.drop_qubit(st, tg, vals).get_vector()
    assert np.array_equal(out, np.array([1, 0], dtype=np.complex128))
    with pytest.raises(ValueError):
        qstate.permutate_qubit(st, [0, 0] + list(range(2, n)))
    with pytest.raises(ValueError):
        qstate.drop_qubit(st, list(range(n)), [0] * n)


@pytest.mark.gpu
def test_gpu_reshaping_vs_oracle_larger():
    from paper_2011_13524_b200 import state as qstate
    rng = np.random.default_rng(11)
    for n in (14, 20):
        a = orc.haar_state(n, 1)
        st = _haar(n, 1)
        order = [int(q) for q in rng.permutation(n)]
        assert np.array_equal(qstate.permutate_qubit(st, order).get_vector(),
                              orc.permutate_qubit(a, n, order))
        tg = [int(q) for q in rng.choice(n, size=5, replace=False)]
        vals = [int(v) for v in rng.integers(0, 2, size=5)]
        assert np.array_equal(qstate.drop_qubit(st, tg, vals).get_vector(),
                              orc.drop_qubit(a, n, tg, vals))
    b1, b2 = orc.haar_state(12, 2), orc.haar_state(9, 3)
    got = qstate.tensor_product(_haar(12, 2), _haar(9, 3)).get_vector()
    assert np.max(np.abs(got - orc.tensor_product(b1, b2))) <= 1e-15


@pytest.mark.gpu
def test_gpu_multiply_elementwise_function():
    for n in (1, 5, 12):
        st = _haar(n, 4)
        a = orc.haar_state(n, 4)

        def f(i):
            return complex(np.cos(0.1 * i), np.sin(0.3 * i)) * (1 + (i & 3))

        st.multiply_elementwise_function(f)
        ref = orc.multiply_elementwise(a, f)
        assert np.max(np.abs(st.get_vector() - ref)) <= 1e-15
