"""Typed ctypes wrapper of the plain-C oracle (liboracle_c.so).

TEST INFRASTRUCTURE ONLY (see qsv_oracle.c).  Applies the neutral gate
records of qsim_oracle.py to a complex128 numpy array in place.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import qsim_oracle as orc

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_VP = C.c_void_p
_I = C.c_int


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle_c.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = C.CDLL(path)
        L.oracle_apply_dense.argtypes = [_VP, _I, _VP, _I, _VP, _VP, _VP, _I]
        L.oracle_apply_diag.argtypes = [_VP, _I, _VP, _I, _VP, _VP, _VP, _I]
        L.oracle_apply_pauli_rot.argtypes = [_VP, _I, _VP, _VP, _I, C.c_double]
        L.oracle_apply_pauli.argtypes = [_VP, _I, _VP, _VP, _I]
        L.oracle_pauli_term.argtypes = [_VP, _VP, _I, _VP, _VP, _I, _VP]
        L.oracle_norm2.argtypes = [_VP, _I, _VP]
        for f in ("oracle_apply_dense", "oracle_apply_diag", "oracle_apply_pauli_rot",
                  "oracle_apply_pauli", "oracle_pauli_term", "oracle_norm2"):
            getattr(L, f).restype = _I
        _LIB = L
    return _LIB


def _ints(v):
    return np.ascontiguousarray(np.array(list(v) or [0], dtype=np.int32))


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def apply_record(psi: np.ndarray, n: int, rec) -> None:
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    L = lib()
    kind = rec[0]
    if kind == "dense" or kind == "diag":
        _, t, payload, ctl = rec
        payload = np.ascontiguousarray(payload, dtype=np.complex128)
        tq, cq, cv = _ints(t), _ints(q for q, _ in ctl), _ints(v for _, v in ctl)
        fn = L.oracle_apply_dense if kind == "dense" else L.oracle_apply_diag
        rc = fn(_ptr(psi), n, _ptr(tq), len(t), _ptr(payload), _ptr(cq), _ptr(cv), len(ctl))
    elif kind == "pauli" and not rec[3]:
        tq, ids = _ints(rec[1]), _ints(rec[2])
        rc = L.oracle_apply_pauli(_ptr(psi), n, _ptr(tq), _ptr(ids), len(rec[1]))
    elif kind == "pauli_rot" and not rec[4]:
        tq, ids = _ints(rec[1]), _ints(rec[2])
        rc = L.oracle_apply_pauli_rot(_ptr(psi), n, _ptr(tq), _ptr(ids), len(rec[1]),
                                      float(rec[3]))
    elif kind == "pauli":
        _, t, ids, ctl = rec
        return apply_record(psi, n, ("dense", t, orc.pauli_matrix(ids), ctl))
    elif kind == "pauli_rot":
        _, t, ids, ang, ctl = rec
        mat = np.cos(ang / 2) * np.eye(1 << len(t)) + 1j * np.sin(ang / 2) * orc.pauli_matrix(ids)
        return apply_record(psi, n, ("dense", t, mat, ctl))
    else:
        raise ValueError(kind)
    if rc != 0:
        raise RuntimeError(f"oracle call failed ({rc})")


def run_records(psi, n, records):
    for rec in records:
        apply_record(psi, n, rec)
    return psi


def pauli_term(bra, ket, n, ops) -> complex:
    tq, ids = _ints(q for q, _ in ops), _ints(a for _, a in ops)
    out = np.zeros(2)
    lib().oracle_pauli_term(_ptr(bra), _ptr(ket), n, _ptr(tq), _ptr(ids), len(ops), _ptr(out))
    return complex(out[0], out[1])


def norm2(psi, n) -> float:
    out = np.zeros(1)
    lib().oracle_norm2(_ptr(psi), n, _ptr(out))
    return float(out[0])
