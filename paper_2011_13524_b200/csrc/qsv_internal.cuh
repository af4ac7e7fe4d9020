// Internal definitions shared by the libqsv translation units.
//
// Data layout in HBM: one cudaMalloc'd array of 2^n double2 (re, im), 256 B
// aligned, qubit i = bit i of the index (reference state.py:1-6).  All gate
// kernels update it in place; the only extra device memory is a small
// reduction scratch (kRedBlocks x kMaxTerms x 2 doubles) per state.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../include/qsv.h"

namespace qsv {

constexpr int kThreads = 256;
constexpr int kRedBlocks = 148 * 4;   // fixed grid => deterministic reductions
constexpr int kMaxTerms = 8;          // Pauli terms evaluated per sweep
constexpr int kMaxFixed = QSV_MAX_TARGETS + QSV_MAX_CONTROLS;

void set_error(const char* fmt, ...);
// pooled stream-ordered device memory for blocks up to 1 GiB (qsv_api.cu)
cudaError_t dev_alloc(void** p, size_t bytes, int device, cudaStream_t s);
void dev_free(void* p, size_t bytes, cudaStream_t s);
int cuda_fail(cudaError_t e, const char* what);

#define QSV_TRY(call)                                   \
  do {                                                  \
    cudaError_t e__ = (call);                           \
    if (e__ != cudaSuccess) return ::qsv::cuda_fail(e__, #call); \
  } while (0)

#define QSV_CHECK_LAUNCH(name)                          \
  do {                                                  \
    cudaError_t e__ = cudaGetLastError();               \
    if (e__ != cudaSuccess) return ::qsv::cuda_fail(e__, name); \
  } while (0)

// Sorted positions at which zero bits are inserted into a dense counter, plus
// an OR-ed value (control values).  widen() is the B0 enumeration of the
// reference (kernels.py:28-39, 55-56) done per thread in registers.
struct FixedBits {
  int n;
  uint64_t lowmask[kMaxFixed];
  uint64_t value;
};

__host__ __device__ __forceinline__ uint64_t widen(uint64_t k, const FixedBits& f) {
#pragma unroll 4
  for (int i = 0; i < f.n; ++i) {
    const uint64_t lo = k & f.lowmask[i];
    k = ((k ^ lo) << 1) | lo;
  }
  return k | f.value;
}

FixedBits make_fixed(const int* pos, int npos, uint64_t value);

struct Cplx {
  double re, im;
};

__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a*b, fused
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}

// 256-bit global accesses (sm_100 LDG.E.256 / STG.E.256): two consecutive
// amplitudes per instruction.  Pointers must be 32-byte aligned.
struct Amp2 {
  double2 a, b;
};

__device__ __forceinline__ Amp2 ld2(const double2* p) {
  Amp2 r;
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.a.x), "=d"(r.a.y), "=d"(r.b.x), "=d"(r.b.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ Amp2 ld2_ro(const double2* p) {
  Amp2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.a.x), "=d"(r.a.y), "=d"(r.b.x), "=d"(r.b.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st2(double2* p, Amp2 v) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "d"(v.a.x), "d"(v.a.y), "d"(v.b.x), "d"(v.b.y)
               : "memory");
}
__device__ __forceinline__ double2 ld1(const double2* p) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st1(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
}

// cudaFuncSetAttribute acts on the current device: remember per device
// (bit d of done_mask) whether the dynamic shared-memory limit is raised.
template <typename F>
inline cudaError_t ensure_smem_attr(F* func, int bytes, uint64_t& done_mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && ((done_mask >> dev) & 1ULL)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && dev < 64) done_mask |= 1ULL << dev;
  return e;
}

inline unsigned grid_for(uint64_t units, int per_thread) {
  uint64_t per_block = (uint64_t)kThreads * per_thread;
  uint64_t b = (units + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > 0x7fffffffULL) b = 0x7fffffffULL;
  return (unsigned)b;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace qsv

struct qsv_state {
  int n;
  int device;
  uint64_t dim;
  double2* amps;
  cudaStream_t stream;
  double* partials;   // device reduction scratch
  double* host_res;   // pinned result slots
  int plain;          // amps from cudaMalloc (IPC-exportable shard), not the pool
  int view;           // amps alias another state's buffer (qsv_state_view): not freed
  int sm_limit;       // > 0: tile passes / slice swaps launched for this state use at
                      // most this many SMs (qsv_set_sm_limit; exchange overlap)
  unsigned long long* tile_ctr;  // tile-pass work counters (2, self-resetting; after partials)
};

// ----------------------------------------------------------------------
// gate launchers (qsv_gates.cu)
namespace qsv {

struct GateDesc {
  int kind;  // QSV_OP_*
  int m;
  int targets[QSV_MAX_TARGETS];
  int ids[QSV_MAX_TARGETS];
  int nc;
  int cq[QSV_MAX_CONTROLS];
  int cv[QSV_MAX_CONTROLS];
  double angle;
  std::vector<Cplx> data;  // DENSE: 4^m, DIAG: 2^m, SPARSE: nnz values
  std::vector<int32_t> sp_rows, sp_cols;  // SPARSE entries (row, column)
  // real-frame form of an uncontrolled 1-qubit dense gate (tile planner):
  // data = R diag(rf_b) with R = rf_r real; the tile encoder applies
  // diag(rf_b) inside a merged diagonal flush and R as real arithmetic
  int rf = 0;
  Cplx rf_b[2] = {{1, 0}, {1, 0}};
  double rf_r[4] = {0, 0, 0, 0};
};

int validate_gate(int n, const GateDesc& g);
// Launch one gate on amps (dim = 2^n) on stream.  dev_data, when non-null,
// points at a device copy of g.data (needed for m >= 6 dense / m >= 5 diag).
int launch_gate(double2* amps, int n, const GateDesc& g, const Cplx* dev_data,
                cudaStream_t stream);
// Algorithmic HBM bytes the reference model attributes to this gate.
double gate_hbm_bytes(int n, const GateDesc& g);
// Simplifications applied before launch (subset phase, rotation -> 2x2 ...)
GateDesc canonicalize(const GateDesc& g);

int launch_scale(double2* amps, uint64_t dim, double2 f, cudaStream_t s);
int launch_add(double2* dst, const double2* src, uint64_t dim, cudaStream_t s);
int launch_random(double2* amps, uint64_t dim, uint64_t seed, cudaStream_t s);

}  // namespace qsv
