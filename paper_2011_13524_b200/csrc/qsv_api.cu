// extern "C" entry points of libqsv (declared in include/qsv.h).
#include <cstdarg>
#include <cstring>
#include <cmath>
#include <string>
#include <vector>
#include <map>
#include <algorithm>

#include "qsv_internal.cuh"
#include "qsv_program.cuh"

namespace qsv {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  cudaGetLastError();  // clear sticky-free errors
  return e == cudaErrorMemoryAllocation ? QSV_ENOMEM : QSV_ECUDA;
}

size_t expect_tile_scratch_bytes();
int expect_tile(const double2* a, int n, const std::vector<uint64_t>& xms,
                const std::vector<uint64_t>& zms, void* scratch, std::vector<double>& res,
                cudaStream_t s);
int launch_expect_sweep(const double2* bra, const double2* ket, int n, uint64_t xm,
                        const uint64_t* zm, int nt, double* partials, double* dev_out,
                        cudaStream_t s);

int launch_marginal(const double2* a, int n, uint64_t mask, uint64_t value, double* partials,
                    double* dev_out, cudaStream_t s);
int launch_sampling(const double2* a, int n, const double* dev_u, int count, double* scratch,
                    uint64_t* dev_out, cudaStream_t s);
size_t sampling_scratch_doubles(int n);
int launch_conj(double2* a, uint64_t dim, cudaStream_t s);
int launch_trace_pairs(const double2* a, int h, double* partials, double* dev_out,
                       cudaStream_t s);
int launch_branch_norm(const double2* a, int n, const int* targets, int k, const double2* dE,
                       const uint64_t* dOffs, double* partials, double* dev_out, cudaStream_t s);
int launch_mul_elementwise(double2* a, const double2* f, uint64_t dim, cudaStream_t s);
int launch_kron(const double2* first, int n1, const double2* second, int n2, double2* out,
                cudaStream_t s);
int launch_permute(const double2* in, double2* out, int n, const int* order, cudaStream_t s);
int launch_drop(const double2* in, int n, const int* targets, const int* values, int k,
                double2* out, cudaStream_t s);

__global__ void k_set1(double2* a, uint64_t idx) { a[idx] = make_double2(1.0, 0.0); }

// Device scratch owned by a state: payloads of direct gate calls and
// reduction results.  Grown on demand, reused in stream order.
struct Scratch {
  void* ptr = nullptr;
  size_t cap = 0;
};
static std::map<const qsv_state*, Scratch> g_payload;
static std::map<const qsv_state*, Scratch> g_results;
static std::map<const qsv_state*, Scratch> g_analysis;
static constexpr size_t kPartialBytes = sizeof(double) * 2 * kRedBlocks * kMaxTerms;
// the tile kernel's work counters follow the reduction scratch (zeroed once,
// reset by the last CTA of every tile pass)
static constexpr size_t kScratchBytes = kPartialBytes + 2 * sizeof(unsigned long long);

static cudaError_t alloc_scratch(qsv_state* st) {
  cudaError_t e = dev_alloc(reinterpret_cast<void**>(&st->partials), kScratchBytes, st->device,
                            st->stream);
  if (e != cudaSuccess) return e;
  st->tile_ctr = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<char*>(st->partials) + kPartialBytes);
  return cudaMemsetAsync(st->tile_ctr, 0, 2 * sizeof(unsigned long long), st->stream);
}

// ------------------------------------------------------------ allocator
// State vectors up to kPoolMaxBytes come from the device's stream-ordered
// memory pool (cudaMallocAsync / cudaFreeAsync): freed blocks stay cached up
// to kPoolKeepBytes, so the many short-lived states of copies, channel
// branches, density-matrix terms and benchmark repeats cost neither a
// cudaMalloc nor the implicit device synchronisation of cudaFree.  Larger
// states (the 16-128 GiB shards) use plain cudaMalloc: allocated once, never
// kept in a cache, and peer-accessible for NVLink copies.  An allocation that
// fails trims the pool and retries once.
constexpr size_t kPoolMaxBytes = 1ULL << 30;
constexpr uint64_t kPoolKeepBytes = 4ULL << 30;

cudaError_t dev_alloc(void** p, size_t bytes, int device, cudaStream_t s) {
  if (bytes > kPoolMaxBytes) return cudaMalloc(p, bytes);
  static std::vector<char> configured(64, 0);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) {
    cudaGetLastError();
    return cudaMalloc(p, bytes);
  }
  if (device >= 0 && device < 64 && !configured[device]) {
    uint64_t keep = kPoolKeepBytes;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    configured[device] = 1;
  }
  cudaError_t e = cudaMallocAsync(p, bytes, s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(p, bytes, s);
  }
  return e;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  if (bytes > kPoolMaxBytes) cudaFree(p);
  else cudaFreeAsync(p, s);
}


// Cross-state ordering.  An op queued on `s` (device `dev`) that reads another
// state `src` must (1) start after the work already queued on src's stream and
// (2) finish before anything queued on src's stream later (a gate overwriting
// the amplitudes being read, or the stream-ordered free of src).  Both sides
// are expressed as event waits on the device, no host synchronisation.
static int stream_wait(cudaStream_t waiter, cudaStream_t signaler, int signaler_dev) {
  if (waiter == signaler) return QSV_OK;
  DeviceGuard dg(signaler_dev);
  cudaEvent_t ev;
  QSV_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t e = cudaEventRecord(ev, signaler);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(waiter, ev, 0);
  cudaEventDestroy(ev);  // released once the recorded work completes
  if (e != cudaSuccess) return cuda_fail(e, "cross-state stream ordering");
  return QSV_OK;
}
static int read_begin(const qsv_state* src, cudaStream_t s, int dev) {
  (void)dev;
  return stream_wait(s, src->stream, src->device);
}
static int read_end(const qsv_state* src, cudaStream_t s, int dev) {
  return stream_wait(src->stream, s, dev);
}

static int ensure(Scratch& s, size_t bytes, cudaStream_t stream) {
  if (s.cap >= bytes) return QSV_OK;
  if (s.ptr) {
    QSV_TRY(cudaStreamSynchronize(stream));
    QSV_TRY(cudaFree(s.ptr));
    s.ptr = nullptr;
    s.cap = 0;
  }
  size_t cap = std::max<size_t>(bytes, 4096);
  QSV_TRY(cudaMalloc(&s.ptr, cap));
  s.cap = cap;
  return QSV_OK;
}

std::vector<char> make_payload(const GateDesc& g) {
  std::vector<char> out;
  if (g.kind == QSV_OP_DENSE && g.m >= 5) {
    const size_t D = (size_t)1 << g.m;
    out.resize(D * D * sizeof(double2) + D * sizeof(uint64_t));
    memcpy(out.data(), g.data.data(), D * D * sizeof(double2));
    uint64_t* offs = reinterpret_cast<uint64_t*>(out.data() + D * D * sizeof(double2));
    for (size_t z = 0; z < D; ++z) {
      uint64_t o = 0;
      for (int j = 0; j < g.m; ++j)
        if ((z >> j) & 1) o |= 1ULL << g.targets[j];
      offs[z] = o;
    }
  } else if (g.kind == QSV_OP_DIAG && g.m > 5) {
    out.resize(((size_t)1 << g.m) * sizeof(double2));
    memcpy(out.data(), g.data.data(), out.size());
  } else if (g.kind == QSV_OP_SPARSE) {
    // [values (CSR order)][coset offsets][row pointers][columns]
    const size_t D = (size_t)1 << g.m, nnz = g.data.size();
    std::vector<size_t> order(nnz);
    for (size_t e = 0; e < nnz; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t x, size_t y) { return g.sp_rows[x] < g.sp_rows[y]; });
    out.resize(nnz * sizeof(double2) + D * sizeof(uint64_t) + (D + 1 + nnz) * sizeof(int32_t));
    double2* vals = reinterpret_cast<double2*>(out.data());
    uint64_t* offs = reinterpret_cast<uint64_t*>(out.data() + nnz * sizeof(double2));
    int32_t* rptr = reinterpret_cast<int32_t*>(offs + D);
    int32_t* cols = rptr + D + 1;
    for (size_t e = 0; e < nnz; ++e) {
      vals[e] = make_double2(g.data[order[e]].re, g.data[order[e]].im);
      cols[e] = g.sp_cols[order[e]];
    }
    for (size_t z = 0; z <= D; ++z) rptr[z] = 0;
    for (size_t e = 0; e < nnz; ++e) ++rptr[g.sp_rows[e] + 1];
    for (size_t z = 0; z < D; ++z) rptr[z + 1] += rptr[z];
    for (size_t z = 0; z < D; ++z) {
      uint64_t o = 0;
      for (int j = 0; j < g.m; ++j)
        if ((z >> j) & 1) o |= 1ULL << g.targets[j];
      offs[z] = o;
    }
  }
  return out;
}

static int apply_desc(qsv_state* st, const GateDesc& g0) {
  int rc = validate_gate(st->n, g0);
  if (rc) return rc;
  DeviceGuard dg(st->device);
  GateDesc g = canonicalize(g0);
  std::vector<char> payload = make_payload(g);
  const Cplx* dev = nullptr;
  if (!payload.empty()) {
    Scratch& s = g_payload[st];
    rc = ensure(s, payload.size(), st->stream);
    if (rc) return rc;
    QSV_TRY(cudaMemcpyAsync(s.ptr, payload.data(), payload.size(), cudaMemcpyHostToDevice,
                            st->stream));
    dev = reinterpret_cast<const Cplx*>(s.ptr);
    // pageable source: the copy is staged before return, so the host vector
    // may be freed; the kernel below is ordered after the copy.
  }
  return launch_gate(st->amps, st->n, g, dev, st->stream);
}

static GateDesc make_desc(int kind, const int* targets, const int* ids, int m, const int* cq,
                          const int* cv, int nc) {
  GateDesc g;
  memset(g.targets, 0, sizeof(g.targets));
  memset(g.ids, 0, sizeof(g.ids));
  memset(g.cq, 0, sizeof(g.cq));
  memset(g.cv, 0, sizeof(g.cv));
  g.kind = kind;
  g.m = m;
  g.nc = nc;
  g.angle = 0;
  if (m > 0 && m <= QSV_MAX_TARGETS)
    for (int j = 0; j < m; ++j) {
      g.targets[j] = targets[j];
      g.ids[j] = ids ? ids[j] : 0;
    }
  if (nc > 0 && nc <= QSV_MAX_CONTROLS)
    for (int j = 0; j < nc; ++j) {
      g.cq[j] = cq[j];
      g.cv[j] = cv[j];
    }
  return g;
}

static bool bad_state(const qsv_state* st) {
  if (!st) {
    set_error("null state handle");
    return true;
  }
  return false;
}

}  // namespace qsv

using namespace qsv;

extern "C" {

const char* qsv_last_error(void) { return g_err.c_str(); }

int qsv_version(void) { return 1; }

int qsv_device_count(int* out) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *out = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *out = c;
  return QSV_OK;
}

int qsv_device_info(int device, char* name, int name_len, int* sm_count, uint64_t* total_mem) {
  cudaDeviceProp p;
  QSV_TRY(cudaGetDeviceProperties(&p, device));
  if (name && name_len > 0) {
    strncpy(name, p.name, (size_t)name_len - 1);
    name[name_len - 1] = 0;
  }
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (total_mem) *total_mem = (uint64_t)p.totalGlobalMem;
  return QSV_OK;
}

static int state_create(int num_qubits, int device, bool plain, qsv_state** out) {
  if (!out) {
    set_error("null output pointer");
    return QSV_EINVAL;
  }
  *out = nullptr;
  if (num_qubits < 1 || num_qubits > 40) {
    set_error("qubit count must be in [1, 40], got %d", num_qubits);
    return QSV_EINVAL;
  }
  int ndev = 0;
  QSV_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("device %d out of range (%d devices)", device, ndev);
    return QSV_EINVAL;
  }
  DeviceGuard dg(device);
  qsv_state* st = new qsv_state();
  st->n = num_qubits;
  st->device = device;
  st->dim = 1ULL << num_qubits;
  st->stream = 0;
  st->amps = nullptr;
  st->partials = nullptr;
  st->host_res = nullptr;
  st->plain = plain ? 1 : 0;
  st->view = 0;
  st->sm_limit = 0;
  st->tile_ctr = nullptr;
  const size_t bytes = std::max<size_t>(st->dim * sizeof(double2), 32);
  cudaError_t e = plain ? cudaMalloc(reinterpret_cast<void**>(&st->amps), bytes)
                        : dev_alloc(reinterpret_cast<void**>(&st->amps), bytes, device, st->stream);
  if (e != cudaSuccess) {
    delete st;
    set_error("cannot allocate %zu bytes for a %d-qubit state: %s", bytes, num_qubits,
              cudaGetErrorString(e));
    cudaGetLastError();
    return QSV_ENOMEM;
  }
  e = alloc_scratch(st);
  if (e != cudaSuccess) {
    if (plain) cudaFree(st->amps);
    else dev_free(st->amps, bytes, st->stream);
    delete st;
    return cuda_fail(e, "cudaMalloc(partials)");
  }
  *out = st;
  return qsv_set_zero(st);
}

int qsv_state_create(int num_qubits, int device, qsv_state** out) {
  return state_create(num_qubits, device, false, out);
}

int qsv_state_create_shared(int num_qubits, int device, qsv_state** out) {
  return state_create(num_qubits, device, true, out);
}

int qsv_state_view(qsv_state* parent, uint64_t offset, int num_qubits, qsv_state** out) {
  if (bad_state(parent) || !out) {
    if (!out) set_error("null output pointer");
    return QSV_EINVAL;
  }
  *out = nullptr;
  if (num_qubits < 1 || num_qubits > parent->n) {
    set_error("view qubit count %d outside [1, %d]", num_qubits, parent->n);
    return QSV_EINVAL;
  }
  const uint64_t dim = 1ULL << num_qubits;
  if (offset % dim != 0 || offset >= parent->dim) {
    set_error("view offset %llu is not a multiple of 2^%d inside the state",
              (unsigned long long)offset, num_qubits);
    return QSV_EINVAL;
  }
  DeviceGuard dg(parent->device);
  qsv_state* st = new qsv_state();
  st->n = num_qubits;
  st->device = parent->device;
  st->dim = dim;
  st->stream = parent->stream;
  st->amps = parent->amps + offset;
  st->partials = nullptr;
  st->host_res = nullptr;
  st->plain = 0;
  st->view = 1;
  st->sm_limit = 0;
  st->tile_ctr = nullptr;
  cudaError_t e = alloc_scratch(st);
  if (e != cudaSuccess) {
    delete st;
    return cuda_fail(e, "cudaMalloc(partials)");
  }
  *out = st;
  return QSV_OK;
}

int qsv_set_sm_limit(qsv_state* st, int sms) {
  if (bad_state(st)) return QSV_EINVAL;
  if (sms < 0) {
    set_error("SM limit must be >= 0, got %d", sms);
    return QSV_EINVAL;
  }
  st->sm_limit = sms;
  return QSV_OK;
}

int qsv_state_destroy(qsv_state* st) {
  if (!st) return QSV_OK;
  DeviceGuard dg(st->device);
  // stream-ordered release: the pool reuses the blocks after the work queued
  // on this stream (no host synchronisation for pooled blocks)
  if (st->view) {
    // the parent owns the amplitudes
  } else if (st->plain) {
    cudaStreamSynchronize(st->stream);
    cudaFree(st->amps);
  } else {
    dev_free(st->amps, std::max<size_t>(st->dim * sizeof(double2), 32), st->stream);
  }
  dev_free(st->partials, kScratchBytes, st->stream);
  for (auto* mp : {&g_payload, &g_results, &g_analysis}) {
    auto it = mp->find(st);
    if (it != mp->end()) {
      cudaFree(it->second.ptr);
      mp->erase(it);
    }
  }
  delete st;
  return QSV_OK;
}

int qsv_state_num_qubits(const qsv_state* st, int* out) {
  if (bad_state(st)) return QSV_EINVAL;
  *out = st->n;
  return QSV_OK;
}

int qsv_state_device_ptr(const qsv_state* st, void** out) {
  if (bad_state(st)) return QSV_EINVAL;
  *out = st->amps;
  return QSV_OK;
}

int qsv_set_stream(qsv_state* st, void* stream) {
  if (bad_state(st)) return QSV_EINVAL;
  // work (and the stream-ordered allocation) queued on the old stream must be
  // complete before the new stream touches the state
  DeviceGuard dg(st->device);
  QSV_TRY(cudaStreamSynchronize(st->stream));
  st->stream = reinterpret_cast<cudaStream_t>(stream);
  return QSV_OK;
}

int qsv_get_stream(const qsv_state* st, void** stream) {
  if (bad_state(st)) return QSV_EINVAL;
  *stream = reinterpret_cast<void*>(st->stream);
  return QSV_OK;
}

int qsv_sync(qsv_state* st) {
  if (bad_state(st)) return QSV_EINVAL;
  DeviceGuard dg(st->device);
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_set_zero(qsv_state* st) { return qsv_set_basis(st, 0); }

int qsv_set_basis(qsv_state* st, uint64_t index) {
  if (bad_state(st)) return QSV_EINVAL;
  if (index >= st->dim) {
    set_error("basis index %llu out of range for %d qubits", (unsigned long long)index, st->n);
    return QSV_EINVAL;
  }
  DeviceGuard dg(st->device);
  QSV_TRY(cudaMemsetAsync(st->amps, 0, st->dim * sizeof(double2), st->stream));
  k_set1<<<1, 1, 0, st->stream>>>(st->amps, index);
  QSV_CHECK_LAUNCH("k_set1");
  return QSV_OK;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int qsv_load_range(qsv_state* st, const double* src, uint64_t offset, uint64_t count) {
  if (bad_state(st)) return QSV_EINVAL;
  if (offset > st->dim || count > st->dim - offset) {
    set_error("range [%llu, +%llu) outside a state of %llu amplitudes",
              (unsigned long long)offset, (unsigned long long)count, (unsigned long long)st->dim);
    return QSV_EINVAL;
  }
  if (count == 0) return QSV_OK;
  DeviceGuard dg(st->device);
  QSV_TRY(cudaMemcpyAsync(st->amps + offset, src, count * sizeof(double2), cudaMemcpyHostToDevice,
                          st->stream));
  if (!is_pinned(src)) QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_load(qsv_state* st, const double* src, uint64_t n_amps) {
  if (bad_state(st)) return QSV_EINVAL;
  if (n_amps != st->dim) {
    set_error("expected %llu amplitudes, got %llu", (unsigned long long)st->dim,
              (unsigned long long)n_amps);
    return QSV_EINVAL;
  }
  return qsv_load_range(st, src, 0, n_amps);
}

int qsv_get_range(const qsv_state* st, double* dst, uint64_t offset, uint64_t count) {
  if (bad_state(st)) return QSV_EINVAL;
  if (offset > st->dim || count > st->dim - offset) {
    set_error("range [%llu, +%llu) outside a state of %llu amplitudes",
              (unsigned long long)offset, (unsigned long long)count, (unsigned long long)st->dim);
    return QSV_EINVAL;
  }
  if (count == 0) return QSV_OK;
  DeviceGuard dg(st->device);
  QSV_TRY(cudaMemcpyAsync(dst, st->amps + offset, count * sizeof(double2), cudaMemcpyDeviceToHost,
                          st->stream));
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_get(const qsv_state* st, double* dst, uint64_t n_amps) {
  if (bad_state(st)) return QSV_EINVAL;
  if (n_amps != st->dim) {
    set_error("expected a buffer of %llu amplitudes, got %llu", (unsigned long long)st->dim,
              (unsigned long long)n_amps);
    return QSV_EINVAL;
  }
  return qsv_get_range(st, dst, 0, n_amps);
}

int qsv_get_async(const qsv_state* st, double* dst, uint64_t n_amps) {
  if (bad_state(st)) return QSV_EINVAL;
  if (n_amps != st->dim) {
    set_error("expected a buffer of %llu amplitudes, got %llu", (unsigned long long)st->dim,
              (unsigned long long)n_amps);
    return QSV_EINVAL;
  }
  DeviceGuard dg(st->device);
  QSV_TRY(cudaMemcpyAsync(dst, st->amps, st->dim * sizeof(double2), cudaMemcpyDeviceToHost,
                          st->stream));
  return QSV_OK;
}

int qsv_copy(const qsv_state* src, qsv_state* dst) {
  if (bad_state(src) || bad_state(dst)) return QSV_EINVAL;
  if (src->n != dst->n) {
    set_error("qubit counts differ (%d vs %d)", src->n, dst->n);
    return QSV_EINVAL;
  }
  DeviceGuard dg(dst->device);
  int rc = read_begin(src, dst->stream, dst->device);
  if (rc) return rc;
  if (src->device == dst->device) {
    QSV_TRY(cudaMemcpyAsync(dst->amps, src->amps, src->dim * sizeof(double2),
                            cudaMemcpyDeviceToDevice, dst->stream));
  } else {
    QSV_TRY(cudaMemcpyPeerAsync(dst->amps, dst->device, src->amps, src->device,
                                src->dim * sizeof(double2), dst->stream));
  }
  return read_end(src, dst->stream, dst->device);
}

int qsv_set_random_device(qsv_state* st, uint64_t seed) {
  if (bad_state(st)) return QSV_EINVAL;
  DeviceGuard dg(st->device);
  int rc = launch_random(st->amps, st->dim, seed, st->stream);
  if (rc) return rc;
  double s = 0;
  rc = qsv_norm2(st, &s);
  if (rc) return rc;
  return qsv_scale(st, 1.0 / std::sqrt(s), 0.0);
}

// ------------------------------------------------------------------ gates
int qsv_apply_dense(qsv_state* st, const int* targets, int m, const double* matrix, const int* cq,
                    const int* cv, int nc) {
  if (bad_state(st)) return QSV_EINVAL;
  if (m < 0 || m > QSV_MAX_TARGETS || nc < 0 || nc > QSV_MAX_CONTROLS) {
    set_error("unsupported target/control count (%d, %d)", m, nc);
    return QSV_EINVAL;
  }
  GateDesc g = make_desc(QSV_OP_DENSE, targets, nullptr, m, cq, cv, nc);
  const size_t D = (size_t)1 << m;
  g.data.resize(D * D);
  memcpy(g.data.data(), matrix, D * D * sizeof(Cplx));
  return apply_desc(st, g);
}

int qsv_apply_diag(qsv_state* st, const int* targets, int m, const double* diag, const int* cq,
                   const int* cv, int nc) {
  if (bad_state(st)) return QSV_EINVAL;
  if (m < 0 || m > QSV_MAX_TARGETS || nc < 0 || nc > QSV_MAX_CONTROLS) {
    set_error("unsupported target/control count (%d, %d)", m, nc);
    return QSV_EINVAL;
  }
  GateDesc g = make_desc(QSV_OP_DIAG, targets, nullptr, m, cq, cv, nc);
  g.data.resize((size_t)1 << m);
  memcpy(g.data.data(), diag, g.data.size() * sizeof(Cplx));
  return apply_desc(st, g);
}

int qsv_apply_pauli(qsv_state* st, const int* targets, const int* ids, int m, const int* cq,
                    const int* cv, int nc) {
  if (bad_state(st)) return QSV_EINVAL;
  if (m < 0 || m > QSV_MAX_TARGETS || nc < 0 || nc > QSV_MAX_CONTROLS) {
    set_error("unsupported target/control count (%d, %d)", m, nc);
    return QSV_EINVAL;
  }
  GateDesc g = make_desc(QSV_OP_PAULI, targets, ids, m, cq, cv, nc);
  return apply_desc(st, g);
}

int qsv_apply_sparse(qsv_state* st, const int* targets, int m, int nnz, const int* rows,
                     const int* cols, const double* values, const int* cq, const int* cv, int nc) {
  if (bad_state(st)) return QSV_EINVAL;
  if (m < 0 || m > QSV_MAX_TARGETS || nc < 0 || nc > QSV_MAX_CONTROLS || nnz < 0) {
    set_error("unsupported target/control/entry count (%d, %d, %d)", m, nc, nnz);
    return QSV_EINVAL;
  }
  GateDesc g = make_desc(QSV_OP_SPARSE, targets, nullptr, m, cq, cv, nc);
  g.data.resize(nnz);
  if (nnz) memcpy(g.data.data(), values, nnz * sizeof(Cplx));
  g.sp_rows.assign(rows, rows + nnz);
  g.sp_cols.assign(cols, cols + nnz);
  return apply_desc(st, g);
}

int qsv_apply_pauli_rot(qsv_state* st, const int* targets, const int* ids, int m, double angle,
                        const int* cq, const int* cv, int nc) {
  if (bad_state(st)) return QSV_EINVAL;
  if (m < 0 || m > QSV_MAX_TARGETS || nc < 0 || nc > QSV_MAX_CONTROLS) {
    set_error("unsupported target/control count (%d, %d)", m, nc);
    return QSV_EINVAL;
  }
  GateDesc g = make_desc(QSV_OP_PAULI_ROT, targets, ids, m, cq, cv, nc);
  g.angle = angle;
  return apply_desc(st, g);
}

// ---------------------------------------------------------- reductions
struct Sweep {
  uint64_t xm;
  std::vector<uint64_t> zm;
  std::vector<int> term;  // term index per slot
};

static int run_sweeps(const qsv_state* bra, const qsv_state* ket,
                      const std::vector<Sweep>& sweeps, std::vector<double>& res) {
  DeviceGuard dg(ket->device);
  cudaStream_t s = ket->stream;
  // the host waits for s below, so the bra's later work is ordered already
  int rc0 = read_begin(bra, s, ket->device);
  if (rc0) return rc0;
  const size_t need = sizeof(double) * 2 * kMaxTerms * std::max<size_t>(1, sweeps.size());
  Scratch& sc = g_results[ket];
  int rc = ensure(sc, need, s);
  if (rc) return rc;
  double* dout = reinterpret_cast<double*>(sc.ptr);
  for (size_t i = 0; i < sweeps.size(); ++i) {
    rc = launch_expect_sweep(bra->amps, ket->amps, ket->n, sweeps[i].xm, sweeps[i].zm.data(),
                             (int)sweeps[i].zm.size(), ket->partials,
                             dout + 2 * kMaxTerms * i, s);
    if (rc) return rc;
  }
  res.assign(2 * kMaxTerms * sweeps.size(), 0.0);
  if (!sweeps.empty()) {
    QSV_TRY(cudaMemcpyAsync(res.data(), dout, res.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            s));
  }
  QSV_TRY(cudaStreamSynchronize(s));
  return QSV_OK;
}

int qsv_norm2(const qsv_state* st, double* out) {
  if (bad_state(st)) return QSV_EINVAL;
  std::vector<Sweep> sw(1);
  sw[0].xm = 0;
  sw[0].zm = {0};
  sw[0].term = {0};
  std::vector<double> res;
  int rc = run_sweeps(st, st, sw, res);
  if (rc) return rc;
  *out = res[0];
  return QSV_OK;
}

int qsv_inner(const qsv_state* bra, const qsv_state* ket, double out[2]) {
  if (bad_state(bra) || bad_state(ket)) return QSV_EINVAL;
  if (bra->n != ket->n) {
    set_error("qubit counts differ (%d vs %d)", bra->n, ket->n);
    return QSV_EINVAL;
  }
  if (bra->device != ket->device) {
    set_error("states live on different devices");
    return QSV_EINVAL;
  }
  std::vector<Sweep> sw(1);
  sw[0].xm = 0;
  sw[0].zm = {0};
  sw[0].term = {0};
  std::vector<double> res;
  int rc = run_sweeps(bra, ket, sw, res);
  if (rc) return rc;
  out[0] = res[0];
  out[1] = res[1];
  return QSV_OK;
}

int qsv_expect(const qsv_state* bra, const qsv_state* ket, int nterms, const int* term_len,
               const int* qubits, const int* ids, const double* coefs, double out[2]) {
  if (bad_state(bra) || bad_state(ket)) return QSV_EINVAL;
  if (bra->n != ket->n || bra->device != ket->device) {
    set_error("bra and ket differ in width or device");
    return QSV_EINVAL;
  }
  // group terms by flip mask (one sweep per <= kMaxTerms terms of a group)
  std::map<uint64_t, std::vector<int>> groups;
  std::vector<uint64_t> zms(nterms), xms(nterms);
  std::vector<int> nys(nterms);
  size_t pos = 0;
  for (int t = 0; t < nterms; ++t) {
    uint64_t xm = 0, zm = 0, used = 0;
    int ny = 0;
    for (int f = 0; f < term_len[t]; ++f, ++pos) {
      const int q = qubits[pos], id = ids[pos];
      if (q < 0 || q >= ket->n) {
        set_error("term touches qubit %d but the operator has %d qubits", q, ket->n);
        return QSV_EINVAL;
      }
      if (used & (1ULL << q)) {
        set_error("qubit indices in a Pauli product must be distinct");
        return QSV_EINVAL;
      }
      used |= 1ULL << q;
      if (id < 0 || id > 3) {
        set_error("Pauli ids must be in {0, 1, 2, 3}");
        return QSV_EINVAL;
      }
      if (id == 1 || id == 2) xm |= 1ULL << q;
      if (id == 2 || id == 3) zm |= 1ULL << q;
      if (id == 2) ++ny;
    }
    zms[t] = zm;
    xms[t] = xm;
    nys[t] = ny;
    groups[xm].push_back(t);
  }
  // expectation values with many flip masks: tile passes (qsv_expect_tile.cu)
  std::vector<Cplx> per_term(nterms, Cplx{0, 0});
  bool done = false;
  if (bra == ket && ket->n >= 12 && groups.size() > 2) {
    DeviceGuard dg(ket->device);
    Scratch& sc = g_analysis[ket];
    int rc = ensure(sc, expect_tile_scratch_bytes(), ket->stream);
    if (rc) return rc;
    std::vector<double> tres;
    rc = expect_tile(ket->amps, ket->n, xms, zms, sc.ptr, tres, ket->stream);
    if (rc == QSV_OK) {
      for (int t = 0; t < nterms; ++t) per_term[t] = {tres[2 * t], tres[2 * t + 1]};
      done = true;
    } else if (rc != QSV_EUNSUPPORTED) {
      return rc;
    }
  }
  std::vector<Sweep> sweeps;
  if (!done)
  for (auto& kv : groups) {
    for (size_t i = 0; i < kv.second.size(); i += kMaxTerms) {
      Sweep s;
      s.xm = kv.first;
      for (size_t j = i; j < std::min(kv.second.size(), i + kMaxTerms); ++j) {
        s.term.push_back(kv.second[j]);
        s.zm.push_back(zms[kv.second[j]]);
      }
      sweeps.push_back(s);
    }
  }
  std::vector<double> res;
  if (!done) {
    int rc = run_sweeps(bra, ket, sweeps, res);
    if (rc) return rc;
  }
  // sum_t coef_t * i^ny_t * S_t, accumulated in term order
  for (size_t i = 0; i < sweeps.size(); ++i)
    for (size_t j = 0; j < sweeps[i].term.size(); ++j)
      per_term[sweeps[i].term[j]] = {res[2 * kMaxTerms * i + 2 * j],
                                     res[2 * kMaxTerms * i + 2 * j + 1]};
  static const Cplx ip[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
  double re = 0, im = 0;
  for (int t = 0; t < nterms; ++t) {
    const Cplx p = ip[nys[t] & 3];
    const Cplx S = per_term[t];
    const Cplx v{p.re * S.re - p.im * S.im, p.re * S.im + p.im * S.re};
    const double cr = coefs[2 * t], ci = coefs[2 * t + 1];
    re += cr * v.re - ci * v.im;
    im += cr * v.im + ci * v.re;
  }
  out[0] = re;
  out[1] = im;
  return QSV_OK;
}

int qsv_scale(qsv_state* st, double re, double im) {
  if (bad_state(st)) return QSV_EINVAL;
  DeviceGuard dg(st->device);
  return launch_scale(st->amps, st->dim, make_double2(re, im), st->stream);
}

int qsv_add(qsv_state* dst, const qsv_state* src) {
  if (bad_state(dst) || bad_state(src)) return QSV_EINVAL;
  if (dst->n != src->n || dst->device != src->device) {
    set_error("qubit counts differ");
    return QSV_EINVAL;
  }
  DeviceGuard dg(dst->device);
  int rc = read_begin(src, dst->stream, dst->device);
  if (!rc) rc = launch_add(dst->amps, src->amps, dst->dim, dst->stream);
  if (!rc) rc = read_end(src, dst->stream, dst->device);
  return rc;
}

// ------------------------------------------------- analysis / reshaping
int qsv_marginal_prob(const qsv_state* st, uint64_t mask, uint64_t value, double* out) {
  if (bad_state(st)) return QSV_EINVAL;
  if (st->n < 64 && (mask >> st->n) != 0) {
    set_error("pattern mask touches qubits beyond %d", st->n);
    return QSV_EINVAL;
  }
  DeviceGuard dg(st->device);
  Scratch& sc = g_results[st];
  int rc = ensure(sc, sizeof(double) * 2 * kMaxTerms, st->stream);
  if (rc) return rc;
  double* dout = reinterpret_cast<double*>(sc.ptr);
  rc = launch_marginal(st->amps, st->n, mask, value, st->partials, dout, st->stream);
  if (rc) return rc;
  QSV_TRY(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_sampling(const qsv_state* st, const double* uniforms, int count, uint64_t* out) {
  if (bad_state(st)) return QSV_EINVAL;
  if (count < 0) {
    set_error("sample count must be non-negative");
    return QSV_EINVAL;
  }
  if (count == 0) return QSV_OK;
  DeviceGuard dg(st->device);
  const size_t nd = sampling_scratch_doubles(st->n);
  const size_t bytes = (nd + 2 * (size_t)count) * sizeof(double);
  Scratch& sc = g_analysis[st];
  int rc = ensure(sc, bytes, st->stream);
  if (rc) return rc;
  double* scratch = reinterpret_cast<double*>(sc.ptr);
  double* du = scratch + nd;
  uint64_t* dout = reinterpret_cast<uint64_t*>(du + count);
  QSV_TRY(cudaMemcpyAsync(du, uniforms, sizeof(double) * count, cudaMemcpyHostToDevice,
                          st->stream));
  rc = launch_sampling(st->amps, st->n, du, count, scratch, dout, st->stream);
  if (rc) return rc;
  QSV_TRY(cudaMemcpyAsync(out, dout, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost,
                          st->stream));
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_mul_elementwise(qsv_state* st, const double* coefs, uint64_t n_amps) {
  if (bad_state(st)) return QSV_EINVAL;
  if (n_amps != st->dim) {
    set_error("expected %llu coefficients, got %llu", (unsigned long long)st->dim,
              (unsigned long long)n_amps);
    return QSV_EINVAL;
  }
  DeviceGuard dg(st->device);
  Scratch& sc = g_analysis[st];
  int rc = ensure(sc, st->dim * sizeof(double2), st->stream);
  if (rc) return rc;
  QSV_TRY(cudaMemcpyAsync(sc.ptr, coefs, st->dim * sizeof(double2), cudaMemcpyHostToDevice,
                          st->stream));
  rc = launch_mul_elementwise(st->amps, reinterpret_cast<const double2*>(sc.ptr), st->dim,
                              st->stream);
  if (rc) return rc;
  QSV_TRY(cudaStreamSynchronize(st->stream));  // the scratch is reused by the next call
  return QSV_OK;
}

static int same_device3(const qsv_state* a, const qsv_state* b, const qsv_state* c) {
  if (a->device != b->device || a->device != c->device) {
    set_error("states live on different devices");
    return QSV_EINVAL;
  }
  return QSV_OK;
}

int qsv_tensor_product(const qsv_state* first, const qsv_state* second, qsv_state* out) {
  if (bad_state(first) || bad_state(second) || bad_state(out)) return QSV_EINVAL;
  if (out->n != first->n + second->n) {
    set_error("output has %d qubits, expected %d", out->n, first->n + second->n);
    return QSV_EINVAL;
  }
  if (same_device3(first, second, out)) return QSV_EINVAL;
  DeviceGuard dg(out->device);
  int rc = read_begin(first, out->stream, out->device);
  if (!rc) rc = read_begin(second, out->stream, out->device);
  if (!rc) rc = launch_kron(first->amps, first->n, second->amps, second->n, out->amps, out->stream);
  if (!rc) rc = read_end(first, out->stream, out->device);
  if (!rc) rc = read_end(second, out->stream, out->device);
  return rc;
}

int qsv_permutate_qubit(const qsv_state* src, const int* order, int n, qsv_state* out) {
  if (bad_state(src) || bad_state(out)) return QSV_EINVAL;
  if (n != src->n || out->n != src->n) {
    set_error("order / output width must equal the state's %d qubits", src->n);
    return QSV_EINVAL;
  }
  if (src == out) {
    set_error("permutate_qubit needs a distinct output state");
    return QSV_EINVAL;
  }
  uint64_t seen = 0;
  for (int i = 0; i < n; ++i) {
    if (order[i] < 0 || order[i] >= n || ((seen >> order[i]) & 1ULL)) {
      set_error("order must be a permutation of 0..%d", n - 1);
      return QSV_EINVAL;
    }
    seen |= 1ULL << order[i];
  }
  if (same_device3(src, out, out)) return QSV_EINVAL;
  DeviceGuard dg(out->device);
  int rc = read_begin(src, out->stream, out->device);
  if (!rc) rc = launch_permute(src->amps, out->amps, n, order, out->stream);
  if (!rc) rc = read_end(src, out->stream, out->device);
  return rc;
}

int qsv_drop_qubit(const qsv_state* src, const int* targets, const int* values, int k,
                   qsv_state* out) {
  if (bad_state(src) || bad_state(out)) return QSV_EINVAL;
  if (k < 0 || k >= src->n || out->n != src->n - k) {
    set_error("cannot drop %d of %d qubits into a %d-qubit state", k, src->n, out->n);
    return QSV_EINVAL;
  }
  uint64_t seen = 0;
  for (int i = 0; i < k; ++i) {
    if (targets[i] < 0 || targets[i] >= src->n || ((seen >> targets[i]) & 1ULL)) {
      set_error("targets must be distinct qubits of the state");
      return QSV_EINVAL;
    }
    if (values[i] != 0 && values[i] != 1) {
      set_error("projection values must be 0 or 1");
      return QSV_EINVAL;
    }
    seen |= 1ULL << targets[i];
  }
  if (same_device3(src, out, out)) return QSV_EINVAL;
  DeviceGuard dg(out->device);
  int rc = read_begin(src, out->stream, out->device);
  if (!rc) rc = launch_drop(src->amps, src->n, targets, values, k, out->amps, out->stream);
  if (!rc) rc = read_end(src, out->stream, out->device);
  return rc;
}

int qsv_branch_norm2(const qsv_state* st, const int* targets, int k, const double* matrix,
                     double* out) {
  if (bad_state(st)) return QSV_EINVAL;
  if (k < 1 || k > 5 || k > st->n) {
    set_error("branch norm supports 1..5 target qubits, got %d", k);
    return QSV_EINVAL;
  }
  uint64_t seen = 0;
  for (int j = 0; j < k; ++j) {
    if (targets[j] < 0 || targets[j] >= st->n || ((seen >> targets[j]) & 1ULL)) {
      set_error("targets must be distinct qubits of the state");
      return QSV_EINVAL;
    }
    seen |= 1ULL << targets[j];
  }
  DeviceGuard dg(st->device);
  const size_t D = (size_t)1 << k;
  std::vector<char> host(D * D * sizeof(double2) + D * sizeof(uint64_t) + 2 * sizeof(double));
  memcpy(host.data(), matrix, D * D * sizeof(double2));
  uint64_t* offs = reinterpret_cast<uint64_t*>(host.data() + D * D * sizeof(double2));
  for (size_t w = 0; w < D; ++w) {
    uint64_t o = 0;
    for (int j = 0; j < k; ++j)
      if ((w >> j) & 1) o |= 1ULL << targets[j];
    offs[w] = o;
  }
  Scratch& sc = g_payload[st];
  int rc = ensure(sc, host.size(), st->stream);
  if (rc) return rc;
  char* dev = reinterpret_cast<char*>(sc.ptr);
  QSV_TRY(cudaMemcpyAsync(dev, host.data(), host.size() - 2 * sizeof(double),
                          cudaMemcpyHostToDevice, st->stream));
  double* dout = reinterpret_cast<double*>(dev + host.size() - 2 * sizeof(double));
  rc = launch_branch_norm(st->amps, st->n, targets, k, reinterpret_cast<const double2*>(dev),
                          reinterpret_cast<const uint64_t*>(dev + D * D * sizeof(double2)),
                          st->partials, dout, st->stream);
  if (rc) return rc;
  QSV_TRY(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_conj(qsv_state* st) {
  if (bad_state(st)) return QSV_EINVAL;
  DeviceGuard dg(st->device);
  return launch_conj(st->amps, st->dim, st->stream);
}

int qsv_trace_pairs(const qsv_state* st, double out[2]) {
  if (bad_state(st)) return QSV_EINVAL;
  if (st->n % 2) {
    set_error("a vectorised density matrix has an even qubit count, got %d", st->n);
    return QSV_EINVAL;
  }
  DeviceGuard dg(st->device);
  Scratch& sc = g_results[st];
  int rc = ensure(sc, sizeof(double) * 2 * kMaxTerms, st->stream);
  if (rc) return rc;
  double* dout = reinterpret_cast<double*>(sc.ptr);
  rc = launch_trace_pairs(st->amps, st->n / 2, st->partials, dout, st->stream);
  if (rc) return rc;
  QSV_TRY(cudaMemcpyAsync(out, dout, 2 * sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

}  // extern "C"
