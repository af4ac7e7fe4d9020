"""Generated expectation passes (csrc/qsv_expect_jit.cu).

CPU: the pass layout and the generated CUDA for several observables, compiled
with NVRTC for sm_100a exactly as libqsv does (no GPU needed): every source
compiles, keeps its accumulators in registers (no local memory), and the
passes cover every term once.

GPU: the first evaluation of an observable runs the generic k_expect_tile,
the second the generated kernels (QSV_EXPECT_JIT=1, the default); both are
checked against the oracle (GeneralOperator._accumulate, observable.py:99-104)
at the north-star bar (1e-10 relative), and the path counters prove which
kernel ran.
"""

import ctypes as C
import re
import subprocess

import numpy as np
import pytest

from paper_2011_13524_b200 import _lib


def tfim_masks(n):
    xms, zms = [], []
    for i in range(n - 1):
        xms.append(0)
        zms.append((1 << i) | (1 << (i + 1)))
    for i in range(n):
        xms.append(1 << i)
        zms.append(0)
    return xms, zms


def random_terms(n, count, seed, max_len=4):
    """(coef, ((qubit, axis), ...)) with axes 1..3 = X, Y, Z."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        k = int(rng.integers(1, max_len + 1))
        qsel = [int(q) for q in rng.choice(n, size=k, replace=False)]
        axes = [int(a) for a in rng.integers(1, 4, size=k)]
        out.append((float(rng.normal()), tuple(zip(qsel, axes))))
    return out


def masks_of(terms):
    xms, zms = [], []
    for _, ops in terms:
        xm = zm = 0
        for q, a in ops:
            if a in (1, 2):
                xm |= 1 << q
            if a in (2, 3):
                zm |= 1 << q
        xms.append(xm)
        zms.append(zm)
    return xms, zms


_NVRTC = None


def nvrtc_compile(src):
    """NVRTC with libqsv's options (csrc/qsv_jit.cu kOpts) -> cubin bytes."""
    global _NVRTC
    if _NVRTC is None:
        _NVRTC = C.CDLL("/usr/local/cuda/lib64/libnvrtc.so")
    nv = _NVRTC
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo",
            b"--device-as-default-execution-space"]
    prog = C.c_void_p()
    assert nv.nvrtcCreateProgram(C.byref(prog), src.encode(), b"qsv_pass.cu", 0, None, None) == 0
    rc = nv.nvrtcCompileProgram(prog, len(opts), (C.c_char_p * len(opts))(*opts))
    n = C.c_size_t()
    nv.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    nv.nvrtcGetProgramLog(prog, log)
    assert rc == 0, log.value.decode()[:3000]
    nv.nvrtcGetCUBINSize(prog, C.byref(n))
    buf = C.create_string_buffer(n.value)
    nv.nvrtcGetCUBIN(prog, buf)
    return buf.raw


def resources(cubin, tmp_path):
    path = tmp_path / "k.cubin"
    path.write_bytes(cubin)
    out = subprocess.run(["cuobjdump", "-res-usage", str(path)], capture_output=True,
                         text=True).stdout
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", out)
    return {k: int(v) for k, v in zip(("reg", "stack", "shared", "local"), m.groups())}


def _accs_per_pass(src):
    return len(re.findall(r"double acc\d+ = 0\.0;", src))


@pytest.mark.parametrize("case", ["tfim24", "tfim28", "random16", "ys14"])
def test_generated_expectation_sources_compile(case, tmp_path):
    if case.startswith("tfim"):
        n = int(case[4:])
        xms, zms = tfim_masks(n)
    elif case == "random16":
        n = 16
        xms, zms = masks_of(random_terms(n, 60, 3))
    else:  # Y-heavy: imaginary pair sums, flips on lane / warp / slot bits
        n = 14
        xms, zms = masks_of([(1.0, ((q, 2), ((q + 5) % n, 2))) for q in range(n)]
                            + [(1.0, ((q, 2),)) for q in range(n)])
    srcs = _lib.expect_jit_sources(n, xms, zms)
    assert sum(_accs_per_pass(s) for s in srcs) == len(xms)  # every term in one pass
    if case == "tfim24":
        assert len(srcs) == 3  # 24 X flips: 12 + 8 + 8 tile qubits (0..3 in every tile)
    for s in srcs[:3]:
        res = resources(nvrtc_compile(s), tmp_path)
        assert res["local"] == 0, res
        assert res["reg"] <= 255, res


def test_unfit_flip_mask_is_unsupported():
    n = 20
    xm = (1 << 20) - 1  # 20 flip qubits > 12 tile qubits
    with pytest.raises(Exception):
        _lib.expect_jit_sources(n, [xm], [0])


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("case", ["tfim14", "tfim20", "tfim24", "random16", "random18y",
                                  "chunked13", "many18"])
def test_generated_expectation_matches_oracle(case):
    import paper_2011_13524_b200 as qs
    from paper_2011_13524_b200 import workloads
    from oracle import qsim_oracle as orc

    if case.startswith("tfim"):
        n = int(case[4:])
        obs = workloads.tfim_observable(n)
        terms = ([(-1.0, ((i, 3), (i + 1, 3))) for i in range(n - 1)]
                 + [(-0.5, ((i, 1),)) for i in range(n)])
    else:
        if case == "random16":
            n, terms = 16, random_terms(16, 60, 5)
        elif case == "many18":  # 43 passes: two copy-back batches, three stream lanes
            n, terms = 18, random_terms(18, 400, 7, max_len=10)
        elif case == "random18y":
            n = 18
            terms = random_terms(18, 40, 6, max_len=6)
            terms += [(0.3, ((q, 2), ((q + 9) % n, 1), ((q + 3) % n, 3))) for q in range(n)]
        else:  # one flip mask with 100 terms: chunks of <= 40 per pass
            n = 13
            rng = np.random.default_rng(9)
            terms = []
            for _ in range(100):
                zq = [int(q) for q in rng.choice(np.arange(2, n), size=3, replace=False)]
                terms.append((float(rng.normal()), ((0, 1), (1, 2)) + tuple((q, 3) for q in zq)))
            terms += [(0.2, ((q, 1),)) for q in (5, 8, 11)]  # >2 flip masks: tile path
        obs = qs.Observable(n)
        for coef, ops in terms:
            obs.add_operator(coef, " ".join(f"{'XYZ'[a - 1]} {q}" for q, a in ops))
    st = qs.QuantumState(n)
    st.set_Haar_random_state(11)
    a = orc.haar_state(n, 11)
    ref = orc.expectation(a, a, n, terms).real
    scale = sum(abs(c) for c, _ in terms)
    bar = 1e-10 * max(abs(ref), 1e-6 * scale)
    before = _lib.expect_path_stats()
    first = obs.get_expectation_value(st)
    second = obs.get_expectation_value(st)
    third = obs.get_expectation_value(st)
    after = _lib.expect_path_stats()
    assert after["jit_passes"] > before["jit_passes"], (before, after)
    assert abs(first - ref) <= bar, (first, ref)
    assert abs(second - ref) <= bar, (second, ref)
    assert second == third  # fixed-order reductions: bit-reproducible
