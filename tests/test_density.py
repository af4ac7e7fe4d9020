"""Density matrices on the GPU: DensityMatrix,
density_from_pure, get_trace and apply_density of basic gates and channels,
against the reference's own outputs (tests/golden/density.*, made by
tests/golden/make_golden.py) at 1e-12."""

import numpy as np
import pytest

from golden_util import core_factory, density_specs, load_density

pytestmark = pytest.mark.gpu


def _run(name):
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import _gates, _maps
    for nm, n, hseed, ops in density_specs():
        if nm != name:
            continue
        if hseed is None:
            rho = qs.DensityMatrix(n)
        else:
            st = qs.QuantumState(n)
            st.set_Haar_random_state(hseed)
            rho = qs.density_from_pure(st)
        for fac, args in ops:
            core_factory(fac, _gates, _maps)(*args).apply_density(rho)
        return rho
    raise KeyError(name)


def test_density_matches_reference():
    meta, outs = load_density()
    for case in meta:
        rho = _run(case["name"])
        got = rho.elements
        assert np.max(np.abs(got - outs[case["name"]])) <= 1e-12, case["name"]
        tr = rho.get_trace()
        assert abs(tr - complex(*case["trace"])) <= 1e-12
        assert np.max(np.abs(got - got.conj().T)) <= 1e-14  # Hermitian


def test_density_from_pure_and_errors():
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import _gates, _maps
    st = qs.QuantumState(4)
    st.set_Haar_random_state(2)
    psi = st.get_vector()
    rho = qs.density_from_pure(st)
    assert np.max(np.abs(rho.elements - np.outer(psi, psi.conj()))) <= 1e-15
    assert rho.dim == 16
    r2 = rho.copy()
    _gates.H(3).apply_density(r2)
    assert np.max(np.abs(rho.elements - np.outer(psi, psi.conj()))) <= 1e-15  # copy is deep
    with pytest.raises(TypeError):
        _maps.AdaptiveGate(_gates.X(0), lambda r: True).apply_density(rho)
    with pytest.raises(ValueError):
        _gates.X(5).apply_density(rho)
    with pytest.raises(ValueError):
        rho.elements = np.eye(3)
