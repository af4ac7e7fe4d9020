/*
 * qsv.h -- C ABI of the B200 state-vector engine (libqsv.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (qsimcore, /root/reference/pkg/src/qsimcore) has no C ABI; its seam is the
 * Python kernel layer `kernels.apply_*(amps, num_qubits, targets, payload,
 * controls)` reached only through `BasicGate._apply_kernel`
 * (gates.py:98-100).  Each entry point below replaces one function of that
 * layer (or of the state container) and says which.  The Python package
 * `paper_2011_13524_b200` binds these through ctypes;
 * argument validation that raises ValueError in the reference stays in that
 * Python layer, the library re-checks and returns QSV_EINVAL.
 *
 * Conventions
 *   - amplitudes are complex128 = two little-endian float64 (re, im);
 *     qubit i is bit i of the amplitude index (state.py:1-6);
 *   - matrices are row-major 2^m x 2^m interleaved complex; bit j of a
 *     row/column index refers to targets[j] (kernels.py:42-52);
 *   - controls are (qubit, value) pairs, value 0 or 1 (gates.py:108-123);
 *   - every call returns QSV_OK (0) or a negative code; qsv_last_error()
 *     returns a thread-local message for the last failing call;
 *   - work is enqueued on the state's stream (default: the legacy default
 *     stream, so torch.cuda events see it); calls that return host data
 *     (qsv_get, qsv_norm2, qsv_inner, qsv_expect) synchronise that stream;
 *   - a handle is not thread-safe (same contract as the reference,
 *     SPEC.md:177 / _handles.py:1-7).
 */
#ifndef QSV_H
#define QSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSV_OK 0
#define QSV_EINVAL (-1)      /* bad argument  -> Python ValueError   */
#define QSV_ENOMEM (-2)      /* cudaMalloc    -> Python MemoryError  */
#define QSV_ECUDA (-3)       /* CUDA failure  -> Python RuntimeError */
#define QSV_EUNSUPPORTED (-4)

#define QSV_MAX_TARGETS 12   /* largest dense / diagonal target count */
#define QSV_MAX_CONTROLS 16

typedef struct qsv_state qsv_state;
typedef struct qsv_program qsv_program;
typedef struct qsv_comm qsv_comm;

/* ------------------------------------------------------------ library */
const char* qsv_last_error(void);
int qsv_version(void);
int qsv_device_count(int* out);
/* name (NUL-terminated, truncated to name_len), SM count, global memory */
int qsv_device_info(int device, char* name, int name_len, int* sm_count, uint64_t* total_mem);

/* --------------------------------------------------------------- state
 * qsv_state_create        <- StateVector.__init__ (state.py:25-30):
 *                            2^n amplitudes set to |0...0>.
 * qsv_set_zero            <- set_zero_state (state.py:32-34)
 * qsv_set_basis           <- set_computational_basis (state.py:36-44)
 * qsv_load / qsv_get      <- load / get_vector (state.py:63-73); the host
 *                            buffer may be pageable or pinned.
 * qsv_load_range/get_range   partial transfers (shards, chunked I/O).
 * qsv_copy                <- copy (state.py:56-61), device to device.
 * qsv_set_random_device   non-parity device-generated random state for
 *                         benchmark inputs only (set_haar_random stays
 *                         host-side numpy for bit-exact parity).
 */
int qsv_state_create(int num_qubits, int device, qsv_state** out);
int qsv_state_destroy(qsv_state* st);
int qsv_state_num_qubits(const qsv_state* st, int* out);
int qsv_state_device_ptr(const qsv_state* st, void** out);
int qsv_set_stream(qsv_state* st, void* cuda_stream);
int qsv_get_stream(const qsv_state* st, void** cuda_stream);
int qsv_sync(qsv_state* st);

int qsv_set_zero(qsv_state* st);
int qsv_set_basis(qsv_state* st, uint64_t index);
int qsv_load(qsv_state* st, const double* interleaved, uint64_t n_amps);
int qsv_get(const qsv_state* st, double* interleaved_out, uint64_t n_amps);
/* qsv_get_async: enqueue the device->host copy on the state's stream and
 * return; the caller synchronises (qsv_sync) before reading `out`, which
 * should be pinned for the copy to overlap other work. */
int qsv_get_async(const qsv_state* st, double* interleaved_out, uint64_t n_amps);
int qsv_load_range(qsv_state* st, const double* interleaved, uint64_t offset, uint64_t count);
int qsv_get_range(const qsv_state* st, double* interleaved_out, uint64_t offset, uint64_t count);
int qsv_copy(const qsv_state* src, qsv_state* dst);
int qsv_set_random_device(qsv_state* st, uint64_t seed);

/* --------------------------------------------------------------- gates
 * qsv_apply_dense      <- kernels.apply_dense (kernels.py:79-138), any m
 *                         up to QSV_MAX_TARGETS, optional controls.
 * qsv_apply_diag       <- kernels.apply_diagonal (kernels.py:155-173).
 * qsv_apply_pauli      <- kernels.apply_pauli (kernels.py:216-220).
 * qsv_apply_pauli_rot  <- kernels.apply_pauli_rotation
 *                         (kernels.py:223-235): exp(+i angle P / 2).
 * ids are Pauli ids 0=I 1=X 2=Y 3=Z (gates.py:23).
 */
int qsv_apply_dense(qsv_state* st, const int* targets, int m, const double* matrix,
                    const int* control_qubits, const int* control_values, int nc);
int qsv_apply_diag(qsv_state* st, const int* targets, int m, const double* diag,
                   const int* control_qubits, const int* control_values, int nc);
int qsv_apply_pauli(qsv_state* st, const int* targets, const int* ids, int m,
                    const int* control_qubits, const int* control_values, int nc);
int qsv_apply_pauli_rot(qsv_state* st, const int* targets, const int* ids, int m,
                        double angle, const int* control_qubits,
                        const int* control_values, int nc);
/* qsv_apply_sparse  <- kernels.apply_sparse / apply_permutation
 *                      (kernels.py:141-152, 176-185): per coset of the
 *                      targets, out[r] = sum over entries (r, c, v) of
 *                      v * in[c]; rows without entries become 0 (sparse
 *                      matrix product semantics).  A permutation table t is
 *                      the entries (t[s], s, 1).  Cost is O(nnz) per coset
 *                      instead of the dense 4^m. */
int qsv_apply_sparse(qsv_state* st, const int* targets, int m, int nnz, const int* rows,
                     const int* cols, const double* values, const int* control_qubits,
                     const int* control_values, int nc);

/* ------------------------------------------------------- state algebra
 * qsv_norm2   <- get_squared_norm (state.py:75-76)
 * qsv_scale   <- normalize / multiply_coef (state.py:78-81, 108-109)
 * qsv_add     <- add_state (state.py:111-114): dst += src
 * qsv_inner   <- inner_product (state.py:136-139): <bra|ket>
 * qsv_expect  <- GeneralOperator._accumulate (observable.py:99-104):
 *                sum_t coef_t <bra| P_t |ket>.  Term t has term_len[t]
 *                factors, listed consecutively in qubits[] / ids[];
 *                coefs are interleaved complex.  bra may equal ket.
 * All reductions are deterministic (fixed-order two-stage tree).
 */
int qsv_norm2(const qsv_state* st, double* out);
int qsv_scale(qsv_state* st, double re, double im);
int qsv_add(qsv_state* dst, const qsv_state* src);
int qsv_inner(const qsv_state* bra, const qsv_state* ket, double out_re_im[2]);
int qsv_expect(const qsv_state* bra, const qsv_state* ket, int nterms,
               const int* term_len, const int* qubits, const int* ids,
               const double* coefs, double out_re_im[2]);

/* --------------------------------------------- analysis and reshaping
 * qsv_marginal_prob    <- get_marginal_probability (state.py:83-95): sum of
 *                         |psi_x|^2 over x with (x & mask) == value.
 * qsv_sampling         <- sampling (state.py:97-106): uniforms[i] are the
 *                         host draws rng.random(count) (numpy PCG64, for
 *                         seed parity); out[i] = searchsorted(cumsum(|psi|^2),
 *                         uniforms[i] * total, side="right").
 * qsv_mul_elementwise  <- multiply_elementwise_function (state.py:116-119):
 *                         amps *= coefs (coefs evaluated by the caller).
 * qsv_tensor_product   <- tensor_product (state.py:142-146): out =
 *                         kron(second, first), first on the low qubits.
 * qsv_permutate_qubit  <- permutate_qubit (state.py:149-161): new qubit i
 *                         carries old qubit order[i]; out must differ from src.
 * qsv_drop_qubit       <- drop_qubit (state.py:164-192): project targets onto
 *                         values and remove them (not renormalised).
 */
int qsv_marginal_prob(const qsv_state* st, uint64_t mask, uint64_t value, double* out);
int qsv_sampling(const qsv_state* st, const double* uniforms, int count, uint64_t* out);
int qsv_mul_elementwise(qsv_state* st, const double* coefs_interleaved, uint64_t n_amps);
int qsv_tensor_product(const qsv_state* first, const qsv_state* second, qsv_state* out);
int qsv_permutate_qubit(const qsv_state* src, const int* order, int n, qsv_state* out);
int qsv_drop_qubit(const qsv_state* src, const int* targets, const int* values, int k,
                   qsv_state* out);

/* qsv_branch_norm2 <- the branch probability |K_i psi|^2 of CptpMap.apply
 *                     (maps.py:55-73): squared norm of matrix|psi> for a
 *                     2^k x 2^k matrix on k = 1..5 targets, computed coset by
 *                     coset without copying the state (the reference copies
 *                     the state per Kraus operator).  Controls are expanded
 *                     into the matrix by the caller. */
int qsv_branch_norm2(const qsv_state* st, const int* targets, int k, const double* matrix,
                     double* out);

/* Density matrices (state.py:195-222) are held as 2h-qubit vectors,
 * element (r, c) at index (r << h) | c; U rho U^dag is U on qubits h + t and
 * conj(U) on qubits t (two ordinary gate calls).
 * qsv_conj         amps <- conj(amps) (density_from_pure, state.py:219-222)
 * qsv_trace_pairs  <- DensityMatrix.get_trace (state.py:216-217):
 *                     sum_i amps[(i << h) | i] for a 2h-qubit state. */
int qsv_conj(qsv_state* st);
int qsv_trace_pairs(const qsv_state* st, double out_re_im[2]);

/* ------------------------------------------------------------ programs
 * A program is a compiled gate list: the replacement for the per-gate loop
 * of Circuit.update_state (circuit.py:48-55).  qsv_program_create copies the
 * payloads to the device once, fuses runs of gates with the same support and
 * packs the rest into tile passes (several gates per HBM sweep); run replays
 * it on a state of the same width.
 */
#define QSV_OP_DENSE 1
#define QSV_OP_DIAG 2
#define QSV_OP_PAULI 3
#define QSV_OP_PAULI_ROT 4
#define QSV_OP_SPARSE 5       /* data: nnz complex values; sp_rows / sp_cols */

typedef struct qsv_op {
  int32_t kind;                            /* QSV_OP_*                     */
  int32_t m;                               /* target count                 */
  int32_t targets[QSV_MAX_TARGETS];
  int32_t ids[QSV_MAX_TARGETS];            /* Pauli ids (PAULI, PAULI_ROT) */
  int32_t nc;                              /* control count                */
  int32_t control_qubits[QSV_MAX_CONTROLS];
  int32_t control_values[QSV_MAX_CONTROLS];
  double angle;                            /* PAULI_ROT                    */
  const double* data;                      /* DENSE: 4^m, DIAG: 2^m complex, SPARSE: nnz */
  int32_t nnz;                             /* SPARSE: entry count          */
  const int32_t* sp_rows;                  /* SPARSE: row of each entry    */
  const int32_t* sp_cols;                  /* SPARSE: column of each entry */
} qsv_op;

typedef struct qsv_plan_opts {
  int32_t use_tiles;      /* 1: pack gates into tile passes (default)     */
  int32_t tile_qubits;    /* qubits per tile, 0 = engine default           */
  int32_t fuse;           /* 1: fuse same-support runs on the host (def.)  */
  int32_t use_graph;      /* 1: replay through a CUDA graph                */
  int32_t real_frames;    /* 1: run 1-qubit gates as real rotations with   */
                          /*    their phases merged into diagonal flushes */
  int32_t jit;            /* tile passes as runtime-compiled straight-line */
                          /* kernels (NVRTC, cached by structure):        */
                          /* 0 off (interpreter), 1 auto: from the second */
                          /* run (or the first when every pass is cached),*/
                          /* 2 eager: compiled at qsv_program_create      */
  uint64_t outer_mask;    /* qubits never chosen as tile qubits, so the    */
                          /* program can run on the block of amplitudes   */
                          /* with those bits fixed (qsv_program_run_fixed) */
} qsv_plan_opts;

typedef struct qsv_program_stats {
  int32_t num_ops_in;     /* gates given to qsv_program_create             */
  int32_t num_steps;      /* kernels launched per run                      */
  int32_t num_tile_passes;/* of which tile passes                          */
  int32_t num_gate_kernels;
  double hbm_bytes;       /* algorithmic HBM bytes per run                 */
  double fp64_flops;      /* FP64 flops per run (2 per FMA), planner count */
  int32_t num_jit_passes; /* tile passes running as generated kernels      */
  int32_t reserved;
} qsv_program_stats;

int qsv_program_create(int num_qubits, const qsv_op* ops, int nops,
                       const qsv_plan_opts* opts, qsv_program** out);
int qsv_program_run(qsv_program* prog, qsv_state* st);
/* Run on the amplitudes whose bits in `mask` equal `value` only (the other
 * blocks are untouched): the program's tile passes enumerate just those
 * tiles.  `mask` must avoid every tile qubit (plan with outer_mask ⊇ mask)
 * and the program must consist of tile passes only (QSV_EUNSUPPORTED
 * otherwise; qsv_program_stats.num_gate_kernels == 0).  The sharded engine
 * runs a segment block by block this way while the next block is still
 * being exchanged (dist.py _remap_overlapped). */
int qsv_program_run_fixed(qsv_program* prog, qsv_state* st, uint64_t mask, uint64_t value);
int qsv_program_stats_get(const qsv_program* prog, qsv_program_stats* out);
int qsv_program_destroy(qsv_program* prog);
/* Host-only: plan without touching a device (stats only). */
int qsv_plan_stats(int num_qubits, const qsv_op* ops, int nops, const qsv_plan_opts* opts,
                   qsv_program_stats* out);

/* Generated tile-pass kernels compiled by NVRTC in this process (misses of
 * both caches), loaded from the on-disk cubin cache, and reused from the
 * in-process cache (qsv_plan_opts.jit).  No GPU needed. */
int qsv_jit_stats(long* compiles, long* disk_hits, long* mem_hits);

/* Expectation-pass code generation without a device (inspection / tests):
 * the pass layout qsv_expect would use for these terms (flip masks xms[t],
 * sign masks zms[t] over qubits), and the CUDA source of pass `pass` copied
 * into buf (NUL-terminated, truncated to cap).  *num_passes receives the pass
 * count; returns QSV_EUNSUPPORTED when a flip mask does not fit a tile. */
/* Expectation tile passes run so far in this process: through generated
 * kernels (qsv_expect_jit.cu) and through the generic k_expect_tile. */
int qsv_expect_path_stats(long* jit_passes, long* generic_passes);

int qsv_expect_jit_source(int num_qubits, int nterms, const uint64_t* xms, const uint64_t* zms,
                          int pass, char* buf, size_t cap, int* num_passes);

/* --------------------------------------------------------------- sharding
 * Exchange primitives of the sharded engine (dist.py; no reference
 * counterpart -- the reference is single-process).  A shard that
 * takes part in peer exchanges is allocated with qsv_state_create_shared
 * (plain cudaMalloc, so its buffer can be exported with CUDA IPC); a peer
 * process maps it with qsv_ipc_open and passes the mapped pointer to
 * qsv_slice_swap, which exchanges the slice {x : bits ls of x == d_mine} of
 * the local shard with the slice {x : bits ls == d_peer} of the peer buffer
 * in place, one kernel over NVLink (loads and stores to peer memory; no
 * staging buffers, no pack/unpack).  Only slice elements j0 <= j < j1 (in
 * slice order) are touched, so the two owners of a pair can each swap half.
 * The caller orders it against the peer's own work (a barrier before and
 * after an exchange step).  QSV_IPC_HANDLE_BYTES bytes per handle. */
#define QSV_IPC_HANDLE_BYTES 64
#define QSV_MAX_SLICE_BITS 16
int qsv_state_create_shared(int num_qubits, int device, qsv_state** out);
int qsv_ipc_export(const qsv_state* st, void* handle_out);
int qsv_ipc_open(const void* handle, int device, void** peer_amps);
int qsv_ipc_close(int device, void* peer_amps);
int qsv_slice_swap(qsv_state* st, void* peer_amps, const int* ls, int k, uint64_t d_mine,
                   uint64_t d_peer, uint64_t j0, uint64_t j1);

/* Exchange / compute overlap (dist.py _remap_overlapped).  qsv_state_view
 * makes a non-owning state over amplitudes [offset, offset + 2^num_qubits)
 * of `parent` (offset a multiple of 2^num_qubits): the block of a shard
 * whose top qubits are fixed, so a segment of local gates that leaves those
 * qubits alone runs on it (own stream, own reduction scratch) while the
 * rest of the shard is still being exchanged.  The view must be destroyed
 * before its parent and cannot be IPC-exported.  qsv_set_sm_limit caps the
 * SMs used by the tile passes and slice swaps launched for a state (0 = all),
 * so an exchange kernel and a tile pass on two streams share the GPU instead
 * of one waiting for the other's persistent CTAs. */
int qsv_state_view(qsv_state* parent, uint64_t offset, int num_qubits, qsv_state** out);
int qsv_set_sm_limit(qsv_state* st, int sms);

/* ----------------------------------------------------------- communicator
 * NCCL inside libqsv for the sharded engine (dist.py; the north star's
 * "NCCL send/recv" exchange -- no reference counterpart, the reference is
 * single-process).  NCCL is loaded on first use (dlopen libnccl.so.2).
 * Rendezvous: rank 0 calls qsv_comm_unique_id and hands the
 * QSV_COMM_ID_BYTES-byte id to every rank (dist.py broadcasts it), each rank
 * calls qsv_comm_create with its rank and device.  All operations are
 * enqueued on the given state's stream:
 *  - qsv_comm_barrier: one-element all-reduce, a device-side barrier that
 *    orders every rank's earlier shard work before later work (no host wait);
 *  - qsv_comm_allreduce_sum: values[0..count) summed over ranks (count <= 64),
 *    synchronous, results back in `values`;
 *  - qsv_comm_slice_exchange: send the slice {x : bits ls of x == d_send} of
 *    the shard to `peer` and overwrite the slice {x : bits ls == d_recv} with
 *    the slice the peer sends (grouped ncclSend / ncclRecv through staging
 *    buffers of at most chunk_bytes per direction; gather / scatter kernels
 *    pack the strided slices).  Every rank of a pair must call it with the
 *    other as peer; peer == own rank copies within the shard.
 * qsv_comm_available: 1 when libnccl.so.2 can be loaded. */
#define QSV_COMM_ID_BYTES 128
int qsv_comm_available(void);
int qsv_comm_unique_id(void* id_out);
int qsv_comm_create(const void* id, int nranks, int rank, int device, qsv_comm** out);
int qsv_comm_destroy(qsv_comm* comm);
int qsv_comm_rank(const qsv_comm* comm, int* rank, int* nranks);
int qsv_comm_barrier(qsv_comm* comm, qsv_state* st);
int qsv_comm_allreduce_sum(qsv_comm* comm, qsv_state* st, double* values, int count);
int qsv_comm_slice_exchange(qsv_comm* comm, qsv_state* st, int peer, const int* ls, int k,
                            uint64_t d_send, uint64_t d_recv, uint64_t chunk_bytes);

#ifdef __cplusplus
}
#endif

#endif /* QSV_H */
