"""CPU oracle: a numpy restatement of the reference state-vector hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2011_13524_b200/`` imports
this module; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
there only as the checker or as the timed CPU baseline -- never as the
product path.

Every function restates the algorithm of the reference package
``qsimcore`` (arXiv 2011.13524 re-implementation under
``/root/reference/pkg/src/qsimcore``) with the same index decomposition,
the same numpy arithmetic and the same operation order, so that its output
and its CPU cost profile match the reference.  Citations are
``file:line`` into ``/root/reference/pkg/src/qsimcore``.

Parity pin: ``tests/golden/*.npz`` were produced by running the reference
itself (``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py``
checks this module against them bit-for-bit or at 1e-15.

Gate records (the neutral format the product exports for checking)::

    ("dense",     targets, matrix[2^m, 2^m], controls)
    ("diag",      targets, diag[2^m],        controls)
    ("pauli",     targets, pauli_ids,         controls)
    ("pauli_rot", targets, pauli_ids, angle,  controls)

``controls`` is a tuple of ``(qubit, value)`` pairs; bit j of a matrix index
refers to ``targets[j]`` (kernels.py:42-52).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

# Thread chunking of the outer (B0) loop, as the reference's _run_chunked
# (kernels.py:59-70, config.py:13-43): a pool per call, used only when
# threads > 1 and n >= 13, and only by the kernels the reference chunks
# (1-qubit dense, small dense, generic dense, uncontrolled diagonal).
_THREADS = 1
_THRESHOLD = 13


def set_threads(count: int) -> None:
    global _THREADS
    _THREADS = max(1, int(count))


def _chunked(work, length, n):
    if _THREADS <= 1 or n < _THRESHOLD or length < 2:
        work(0, length)
        return
    k = min(_THREADS, length)
    step = -(-length // k)
    spans = [(lo, min(lo + step, length)) for lo in range(0, length, step)]
    with ThreadPoolExecutor(max_workers=k) as pool:
        list(pool.map(lambda sp: work(*sp), spans))


_P1Q = {
    0: np.array([[1, 0], [0, 1]], dtype=np.complex128),
    1: np.array([[0, 1], [1, 0]], dtype=np.complex128),
    2: np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    3: np.array([[1, 0], [0, -1]], dtype=np.complex128),
}


# ---------------------------------------------------------------- indexing
def outer_indices(n: int, fixed) -> np.ndarray:
    """B0: indices with zero bits at ``fixed`` (kernels.py:28-39).

    A dense counter is widened by one zero bit per fixed position, lowest
    position first, so the result is ascending.
    """
    out = np.arange(1 << (n - len(fixed)), dtype=np.intp)
    for pos in sorted(fixed):
        keep = out & ((1 << pos) - 1)
        out = ((out ^ keep) << 1) | keep
    return out


def inner_offsets(targets) -> np.ndarray:
    """B1: offset i has bit ``targets[j]`` set iff bit j of i is set
    (kernels.py:42-52)."""
    cnt = np.arange(1 << len(targets), dtype=np.intp)
    res = np.zeros_like(cnt)
    for j, t in enumerate(targets):
        res |= ((cnt >> j) & 1) << t
    return res


def _cosets(n, targets, controls):
    """kernels.py:73-76 -- B0 over targets+controls, shifted by the
    control-value offset (kernels.py:55-56)."""
    fixed = list(targets) + [q for q, _ in controls]
    shift = 0
    for q, v in controls:
        if v:
            shift |= 1 << q
    return outer_indices(n, fixed) + shift, inner_offsets(targets)


# ---------------------------------------------------------------- kernels
def apply_dense(amps, n, targets, mat, controls=()):
    """kernels.py:79-106: m=0 scalar, m=1 reshape path, m<=2 unrolled
    gather, else gather @ K^T scatter."""
    m = len(targets)
    mat = np.asarray(mat, dtype=np.complex128)
    if mat.shape != (1 << m, 1 << m):
        raise ValueError("matrix shape does not match the target count")
    if m == 0:
        if controls:
            base, _ = _cosets(n, targets, controls)
            amps[base] *= mat[0, 0]
        else:
            amps *= mat[0, 0]
        return
    if m == 1 and not controls:
        # kernels.py:109-123
        v = amps.reshape(-1, 2, 1 << targets[0])

        def one(a, b):
            lo = v[a:b, 0, :]
            hi = v[a:b, 1, :]
            new_lo = mat[0, 0] * lo + mat[0, 1] * hi
            v[a:b, 1, :] = mat[1, 0] * lo + mat[1, 1] * hi
            v[a:b, 0, :] = new_lo

        _chunked(one, v.shape[0], n)
        return
    base, offs = _cosets(n, targets, controls)
    if m <= 2:
        # kernels.py:126-138
        def small(a, b):
            cols = [amps[base[a:b] + o] for o in offs]
            for z in range(len(offs)):
                acc = mat[z, 0] * cols[0]
                for w in range(1, len(offs)):
                    acc += mat[z, w] * cols[w]
                amps[base[a:b] + offs[z]] = acc

        _chunked(small, len(base), n)
        return
    kt = np.ascontiguousarray(mat.T)

    def generic(a, b):
        rows = base[a:b, None] + offs[None, :]
        amps[rows] = amps[rows] @ kt

    _chunked(generic, len(base), n)


def apply_diagonal(amps, n, targets, diag, controls=()):
    """kernels.py:155-173."""
    diag = np.asarray(diag, dtype=np.complex128)
    if diag.shape != (1 << len(targets),):
        raise ValueError("diagonal length does not match the target count")
    if not controls:
        idx = np.arange(amps.size, dtype=np.intp)
        sub = np.zeros(amps.size, dtype=np.intp)
        for j, t in enumerate(targets):
            sub |= ((idx >> t) & 1) << j

        def part(a, b):
            amps[a:b] *= diag[sub[a:b]]

        _chunked(part, amps.size, n)
        return
    base, offs = _cosets(n, targets, controls)
    for z in range(len(offs)):
        amps[base + offs[z]] *= diag[z]


def pauli_masks(targets, ids):
    """kernels.py:188-199: X/Y set the flip mask, Y/Z the sign mask."""
    xm = zm = ny = 0
    for t, p in zip(targets, ids):
        if p == 1 or p == 2:
            xm |= 1 << t
        if p == 2 or p == 3:
            zm |= 1 << t
        if p == 2:
            ny += 1
    return xm, zm, ny


def pauli_action(amps, n, targets, ids):
    """Return P|psi> (kernels.py:202-213)."""
    xm, zm, ny = pauli_masks(targets, ids)
    src = np.arange(amps.size, dtype=np.intp) ^ xm
    out = amps[src].copy() if xm else amps.copy()
    if zm:
        odd = (np.bitwise_count(src & zm) & 1) == 1
        out[odd] *= -1
    if ny % 4:
        out *= 1j ** (ny % 4)
    return out


def pauli_matrix(ids):
    """kernels.py:238-243 -- factor j acts on index bit j."""
    acc = np.ones((1, 1), dtype=np.complex128)
    for p in ids:
        acc = np.kron(_P1Q[p], acc)
    return acc


def apply_pauli(amps, n, targets, ids, controls=()):
    """kernels.py:216-220."""
    if controls:
        apply_dense(amps, n, targets, pauli_matrix(ids), controls)
        return
    amps[:] = pauli_action(amps, n, targets, ids)


def apply_pauli_rotation(amps, n, targets, ids, angle, controls=()):
    """exp(+i angle P / 2) (kernels.py:223-235, gates.py:263-268)."""
    c = np.cos(angle / 2)
    s = np.sin(angle / 2)
    if controls:
        mat = c * np.eye(1 << len(targets), dtype=np.complex128) \
            + 1j * s * pauli_matrix(ids)
        apply_dense(amps, n, targets, mat, controls)
        return
    rot = pauli_action(amps, n, targets, ids)
    amps *= c
    amps += 1j * s * rot


def apply_record(amps, n, rec):
    """Dispatch one neutral gate record onto the matching kernel, as
    ``BasicGate._apply_kernel`` does per payload class (gates.py:98-100,
    140-141, 196-197, 254-255, 287-289)."""
    kind = rec[0]
    if kind == "dense":
        _, t, mat, ctl = rec
        apply_dense(amps, n, tuple(t), mat, tuple(ctl))
    elif kind == "diag":
        _, t, d, ctl = rec
        apply_diagonal(amps, n, tuple(t), d, tuple(ctl))
    elif kind == "pauli":
        _, t, ids, ctl = rec
        apply_pauli(amps, n, tuple(t), tuple(ids), tuple(ctl))
    elif kind == "pauli_rot":
        _, t, ids, ang, ctl = rec
        apply_pauli_rotation(amps, n, tuple(t), tuple(ids), ang, tuple(ctl))
    else:
        raise ValueError(f"unknown gate record kind {kind!r}")


def run_records(amps, n, records):
    """Circuit.update_state's per-gate loop (circuit.py:48-55)."""
    for rec in records:
        apply_record(amps, n, rec)
    return amps


# ---------------------------------------------------------------- maps
def apply_map_record(amps, n, rec, rng, cregs):
    """Quantum maps (maps.py:35-187) on a state vector.  Records:
    ("cptp", kraus_records, register_or_None), ("prob", probs, records),
    ("adaptive", condition, inner_record).  Returns the new amplitude array
    (a CPTP map rebinds it, maps.py:84)."""
    kind = rec[0]
    if kind == "cptp":
        _, kraus, reg = rec
        draw = rng.random()
        cumulative = 0.0
        chosen = branch = None
        for i, k in enumerate(kraus):
            cand = amps.copy()
            apply_record(cand, n, k)
            prob = squared_norm(cand)
            cumulative += prob
            if cumulative >= draw or i == len(kraus) - 1:
                if prob <= 0:
                    continue
                chosen, branch = i, cand
                break
        if chosen is None:
            raise ValueError("all Kraus branches have zero probability")
        branch /= np.sqrt(squared_norm(branch))
        if reg is not None:
            if reg >= len(cregs):
                cregs.extend([0] * (reg + 1 - len(cregs)))
            cregs[reg] = chosen
        return branch
    if kind == "prob":
        _, probs, gates = rec
        draw = rng.random()
        cumulative = 0.0
        for p, g in zip(probs, gates):
            cumulative += p
            if draw < cumulative:
                apply_record(amps, n, g)
                break
        return amps
    if kind == "adaptive":
        _, cond, inner = rec
        if cond(list(cregs)):
            if inner[0] in ("cptp", "prob", "adaptive"):
                return apply_map_record(amps, n, inner, rng, cregs)
            apply_record(amps, n, inner)
        return amps
    apply_record(amps, n, rec)
    return amps


def run_records_rng(amps, n, records, seed):
    """update_state with maps: one default_rng(seed) shared by every map in
    gate order (circuit.py:48-55); returns (amplitudes, classical registers)."""
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    cregs = []
    for rec in records:
        amps = apply_map_record(amps, n, rec, rng, cregs)
    return amps, cregs


# ---------------------------------------------------------------- states
def zero_state(n):
    """state.py:25-30."""
    a = np.zeros(1 << n, dtype=np.complex128)
    a[0] = 1.0
    return a


def haar_state(n, seed):
    """state.py:46-54: PCG64 normals (real block then imaginary block),
    divided by the 2-norm."""
    g = np.random.default_rng(seed)
    raw = g.standard_normal(1 << n) + 1j * g.standard_normal(1 << n)
    return raw / np.linalg.norm(raw)


def squared_norm(a):
    """state.py:75-76."""
    return float(np.real(np.vdot(a, a)))


def inner_product(bra, ket):
    """state.py:136-139."""
    return complex(np.vdot(bra, ket))


def expectation(amps_bra, amps_ket, n, terms):
    """GeneralOperator._accumulate (observable.py:99-104): terms are
    ``(coef, ((qubit, axis), ...))``."""
    total = 0.0 + 0.0j
    for coef, ops in terms:
        qs = tuple(q for q, _ in ops)
        ids = tuple(a for _, a in ops)
        total += complex(coef) * np.vdot(amps_bra, pauli_action(amps_ket, n, qs, ids))
    return total


# ------------------------------------------------- analysis / reshaping
WILDCARD = 2


def marginal_probability(amps, n, pattern):
    """state.py:83-95: sum of |psi|^2 over indices matching 0/1 per qubit,
    WILDCARD (2) leaves a qubit free."""
    probs = np.abs(amps) ** 2
    idx = np.arange(1 << n)
    mask = np.ones(1 << n, dtype=bool)
    for qubit, want in enumerate(pattern):
        if want == WILDCARD:
            continue
        mask &= ((idx >> qubit) & 1) == want
    return float(probs[mask].sum())


def sampling(amps, count, seed):
    """state.py:97-106: cumulative distribution + searchsorted(side=right)
    on draws rng.random(count) * cumulative[-1]."""
    if count == 0:
        return []
    cumulative = np.cumsum(np.abs(amps) ** 2)
    rng = np.random.default_rng(seed)
    draws = rng.random(count) * cumulative[-1]
    return np.searchsorted(cumulative, draws, side="right").tolist()


def multiply_elementwise(amps, func):
    """state.py:116-119: amps *= [func(i) for i in range(dim)]."""
    coefs = np.fromiter((func(i) for i in range(amps.size)), dtype=np.complex128,
                        count=amps.size)
    amps *= coefs
    return amps


def tensor_product(first, second):
    """state.py:142-146: kron(second, first) (first on the low qubits)."""
    return np.kron(second, first)


def permutate_qubit(amps, n, order):
    """state.py:149-161: new qubit i carries old qubit order[i]."""
    src = np.arange(1 << n)
    dst = np.zeros(1 << n, dtype=np.intp)
    for new_q, old_q in enumerate(order):
        dst |= ((src >> old_q) & 1) << new_q
    out = np.zeros(1 << n, dtype=np.complex128)
    out[dst] = amps[src]
    return out


def drop_qubit(amps, n, targets, values):
    """state.py:164-192: project targets onto values, remove them, no
    renormalisation."""
    keep = [q for q in range(n) if q not in set(targets)]
    src = np.arange(1 << len(keep), dtype=np.intp)
    full = np.zeros(1 << len(keep), dtype=np.intp)
    for j, q in enumerate(keep):
        full |= ((src >> j) & 1) << q
    for t, v in zip(targets, values):
        full |= v << t
    return amps[full].copy()


# ---------------------------------------------------------------- workloads
def _rot(q, pid, ang):
    return ("pauli_rot", (q,), (pid,), float(ang), ())


def cz_ladder_records(n, depth, seed, commuting=False):
    """bench.py:28-55: depth+1 RZ-RX-RZ layers (RZ only when commuting)
    with CZ(q, q+1) for q = layer parity, step 2, between them."""
    g = np.random.default_rng(seed)
    out = []
    for layer in range(depth + 1):
        for q in range(n):
            if commuting:
                out.append(_rot(q, 3, g.random() * 2 * np.pi))
            else:
                out.append(_rot(q, 3, g.random() * 2 * np.pi))
                out.append(_rot(q, 1, g.random() * 2 * np.pi))
                out.append(_rot(q, 3, g.random() * 2 * np.pi))
        if layer == depth:
            break
        for q in range(layer % 2, n - 1, 2):
            out.append(("diag", (q + 1,), np.array([1, -1], dtype=np.complex128),
                        ((q, 1),)))
    return out


def cnot_ring_records(n, seed):
    """bench.py:58-81: 11 rotation layers, the first without its leading RZ
    and the last without its trailing RZ, with CNOT((q+1)%n, q) rings in
    between."""
    g = np.random.default_rng(seed)
    out = []
    for layer in range(11):
        for q in range(n):
            if layer != 0:
                out.append(_rot(q, 3, g.random() * 2 * np.pi))
            out.append(_rot(q, 1, g.random() * 2 * np.pi))
            if layer != 10:
                out.append(_rot(q, 3, g.random() * 2 * np.pi))
        if layer != 10:
            for q in range(n):
                out.append(("pauli", (q,), (1,), (((q + 1) % n, 1),)))
    return out
