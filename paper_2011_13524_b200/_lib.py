"""ctypes binding of libqsv.so (the C ABI declared in include/qsv.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: if the shared object is missing the import
fails, and every call that needs a GPU raises when none is present.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# QSV_LIB overrides the in-tree build (used for A/B experiments of kernel variants)
LIB_PATH = os.environ.get("QSV_LIB") or os.path.join(_HERE, "libqsv.so")

QSV_OK = 0
QSV_EINVAL = -1
QSV_ENOMEM = -2
QSV_ECUDA = -3
QSV_EUNSUPPORTED = -4

MAX_TARGETS = 12
MAX_CONTROLS = 16

OP_DENSE = 1
OP_DIAG = 2
OP_PAULI = 3
OP_PAULI_ROT = 4
OP_SPARSE = 5


class QsvOp(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("m", C.c_int32),
        ("targets", C.c_int32 * MAX_TARGETS),
        ("ids", C.c_int32 * MAX_TARGETS),
        ("nc", C.c_int32),
        ("control_qubits", C.c_int32 * MAX_CONTROLS),
        ("control_values", C.c_int32 * MAX_CONTROLS),
        ("angle", C.c_double),
        ("data", C.c_void_p),
        ("nnz", C.c_int32),
        ("sp_rows", C.c_void_p),
        ("sp_cols", C.c_void_p),
    ]


class QsvPlanOpts(C.Structure):
    _fields_ = [
        ("use_tiles", C.c_int32),
        ("tile_qubits", C.c_int32),
        ("fuse", C.c_int32),
        ("use_graph", C.c_int32),
        ("real_frames", C.c_int32),
        ("jit", C.c_int32),
        ("outer_mask", C.c_uint64),
    ]


class QsvProgramStats(C.Structure):
    _fields_ = [
        ("num_ops_in", C.c_int32),
        ("num_steps", C.c_int32),
        ("num_tile_passes", C.c_int32),
        ("num_gate_kernels", C.c_int32),
        ("hbm_bytes", C.c_double),
        ("fp64_flops", C.c_double),
        ("num_jit_passes", C.c_int32),
        ("reserved", C.c_int32),
    ]


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA engine first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
_I = C.c_int
_IP = C.POINTER(C.c_int)
_DP = C.c_void_p
_U64 = C.c_uint64

_SIGS = {
    "qsv_last_error": ([], C.c_char_p),
    "qsv_version": ([], _I),
    "qsv_device_count": ([_IP], _I),
    "qsv_device_info": ([_I, C.c_char_p, _I, _IP, C.POINTER(_U64)], _I),
    "qsv_state_create": ([_I, _I, C.POINTER(_P)], _I),
    "qsv_state_create_shared": ([_I, _I, C.POINTER(_P)], _I),
    "qsv_ipc_export": ([_P, _P], _I),
    "qsv_ipc_open": ([_P, _I, C.POINTER(_P)], _I),
    "qsv_ipc_close": ([_I, _P], _I),
    "qsv_slice_swap": ([_P, _P, _IP, _I, _U64, _U64, _U64, _U64], _I),
    "qsv_state_view": ([_P, _U64, _I, C.POINTER(_P)], _I),
    "qsv_set_sm_limit": ([_P, _I], _I),
    "qsv_state_destroy": ([_P], _I),
    "qsv_state_num_qubits": ([_P, _IP], _I),
    "qsv_state_device_ptr": ([_P, C.POINTER(_P)], _I),
    "qsv_set_stream": ([_P, _P], _I),
    "qsv_get_stream": ([_P, C.POINTER(_P)], _I),
    "qsv_sync": ([_P], _I),
    "qsv_set_zero": ([_P], _I),
    "qsv_set_basis": ([_P, _U64], _I),
    "qsv_load": ([_P, _DP, _U64], _I),
    "qsv_get": ([_P, _DP, _U64], _I),
    "qsv_get_async": ([_P, _DP, _U64], _I),
    "qsv_load_range": ([_P, _DP, _U64, _U64], _I),
    "qsv_get_range": ([_P, _DP, _U64, _U64], _I),
    "qsv_copy": ([_P, _P], _I),
    "qsv_set_random_device": ([_P, _U64], _I),
    "qsv_apply_dense": ([_P, _IP, _I, _DP, _IP, _IP, _I], _I),
    "qsv_apply_diag": ([_P, _IP, _I, _DP, _IP, _IP, _I], _I),
    "qsv_apply_pauli": ([_P, _IP, _IP, _I, _IP, _IP, _I], _I),
    "qsv_apply_pauli_rot": ([_P, _IP, _IP, _I, C.c_double, _IP, _IP, _I], _I),
    "qsv_apply_sparse": ([_P, _IP, _I, _I, _IP, _IP, _DP, _IP, _IP, _I], _I),
    "qsv_norm2": ([_P, C.POINTER(C.c_double)], _I),
    "qsv_scale": ([_P, C.c_double, C.c_double], _I),
    "qsv_add": ([_P, _P], _I),
    "qsv_inner": ([_P, _P, C.POINTER(C.c_double)], _I),
    "qsv_expect": ([_P, _P, _I, _IP, _IP, _IP, _DP, C.POINTER(C.c_double)], _I),
    "qsv_marginal_prob": ([_P, _U64, _U64, C.POINTER(C.c_double)], _I),
    "qsv_sampling": ([_P, _DP, _I, _DP], _I),
    "qsv_mul_elementwise": ([_P, _DP, _U64], _I),
    "qsv_tensor_product": ([_P, _P, _P], _I),
    "qsv_permutate_qubit": ([_P, _IP, _I, _P], _I),
    "qsv_drop_qubit": ([_P, _IP, _IP, _I, _P], _I),
    "qsv_branch_norm2": ([_P, _IP, _I, _DP, C.POINTER(C.c_double)], _I),
    "qsv_conj": ([_P], _I),
    "qsv_trace_pairs": ([_P, C.POINTER(C.c_double)], _I),
    "qsv_program_create": ([_I, C.POINTER(QsvOp), _I, C.POINTER(QsvPlanOpts), C.POINTER(_P)], _I),
    "qsv_program_run": ([_P, _P], _I),
    "qsv_program_run_fixed": ([_P, _P, _U64, _U64], _I),
    "qsv_program_stats_get": ([_P, C.POINTER(QsvProgramStats)], _I),
    "qsv_program_destroy": ([_P], _I),
    "qsv_plan_stats": ([_I, C.POINTER(QsvOp), _I, C.POINTER(QsvPlanOpts),
                        C.POINTER(QsvProgramStats)], _I),
    "qsv_jit_stats": ([C.POINTER(C.c_long)] * 3, _I),
    "qsv_comm_available": ([], _I),
    "qsv_comm_unique_id": ([_P], _I),
    "qsv_comm_create": ([_P, _I, _I, _I, C.POINTER(_P)], _I),
    "qsv_comm_destroy": ([_P], _I),
    "qsv_comm_rank": ([_P, _IP, _IP], _I),
    "qsv_comm_barrier": ([_P, _P], _I),
    "qsv_comm_allreduce_sum": ([_P, _P, _DP, _I], _I),
    "qsv_comm_slice_exchange": ([_P, _P, _I, _IP, _I, _U64, _U64, _U64], _I),
    "qsv_expect_path_stats": ([C.POINTER(C.c_long)] * 2, _I),
    "qsv_expect_jit_source": ([_I, _I, C.POINTER(_U64), C.POINTER(_U64), _I, C.c_char_p,
                               C.c_size_t, _IP], _I),
}

EXPORTED = tuple(_SIGS)

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def check(rc: int) -> None:
    """Map a libqsv return code onto the reference's exception types
    (ValueError for bad arguments, MemoryError for allocation failure)."""
    if rc == QSV_OK:
        return
    msg = lib.qsv_last_error().decode(errors="replace")
    if rc == QSV_EINVAL:
        raise ValueError(msg)
    if rc == QSV_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libqsv error {rc}: {msg}")


def int_array(values):
    values = list(values)
    arr = (C.c_int * max(1, len(values)))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr


def device_info(device: int = 0) -> dict:
    """Name, SM count and memory of a CUDA device (empty if none)."""
    buf = C.create_string_buffer(256)
    sms = C.c_int(0)
    mem = C.c_uint64(0)
    if lib.qsv_device_info(int(device), buf, 256, C.byref(sms), C.byref(mem)) != QSV_OK:
        return {}
    return {"name": buf.value.decode(errors="replace"), "sm_count": sms.value,
            "memory_bytes": mem.value}


def device_count() -> int:
    out = C.c_int(0)
    rc = lib.qsv_device_count(C.byref(out))
    if rc != QSV_OK:
        return 0
    return out.value


def jit_stats() -> dict:
    """Generated tile-pass kernels: NVRTC compiles, disk-cache and in-process
    cache hits so far in this process."""
    a, b, c = C.c_long(), C.c_long(), C.c_long()
    check(lib.qsv_jit_stats(C.byref(a), C.byref(b), C.byref(c)))
    return {"compiles": a.value, "disk_hits": b.value, "mem_hits": c.value}


def expect_jit_sources(num_qubits: int, xms, zms) -> list:
    """CUDA sources of the generated expectation passes qsv_expect would use
    for terms with flip masks ``xms`` and sign masks ``zms`` (no GPU needed)."""
    nt = len(xms)
    xa, za = (_U64 * max(1, nt))(*xms), (_U64 * max(1, nt))(*zms)
    npass = C.c_int()
    check(lib.qsv_expect_jit_source(num_qubits, nt, xa, za, -1, None, 0, C.byref(npass)))
    out = []
    for p in range(npass.value):
        buf = C.create_string_buffer(1 << 22)
        check(lib.qsv_expect_jit_source(num_qubits, nt, xa, za, p, buf, len(buf), C.byref(npass)))
        out.append(buf.value.decode())
    return out


def expect_path_stats() -> dict:
    """Expectation tile passes run so far: generated kernels vs generic kernel."""
    a, b = C.c_long(), C.c_long()
    check(lib.qsv_expect_path_stats(C.byref(a), C.byref(b)))
    return {"jit_passes": a.value, "generic_passes": b.value}
