// Gate-application kernels (sm_100a) -- the replacement for the reference's
// kernels.apply_* layer (/root/reference/pkg/src/qsimcore/kernels.py).
//
// Every kernel is an in-place streaming update of the state in HBM.  The
// reference's materialised B0 index arrays (kernels.py:28-56) become
// per-thread bit insertion (widen()); the gathers become 256-bit loads of two
// neighbouring amplitudes wherever the lowest fixed bit is >= 1, so every
// warp moves whole 32-byte sectors and consecutive lanes touch consecutive
// sectors.  Byte counts per launch (the roofline numerator) are in
// gate_hbm_bytes() and DESIGN.md.
#include <cmath>
#include <cstring>
#include <algorithm>

#include "qsv_internal.cuh"

namespace qsv {

FixedBits make_fixed(const int* pos, int npos, uint64_t value) {
  FixedBits f;
  int tmp[kMaxFixed];
  for (int i = 0; i < npos; ++i) tmp[i] = pos[i];
  std::sort(tmp, tmp + npos);
  f.n = npos;
  for (int i = 0; i < kMaxFixed; ++i) f.lowmask[i] = 0;
  for (int i = 0; i < npos; ++i) f.lowmask[i] = (1ULL << tmp[i]) - 1ULL;
  f.value = value;
  return f;
}

constexpr int kUnroll = 2;  // units per thread, loads issued before compute

// --------------------------------------------------------------------------
// 2x2 on pairs (i0, i0 | tbit), optionally controlled: replaces
// _apply_dense_1q (kernels.py:109-123) and the m=1 controlled branch of
// _apply_dense_small (kernels.py:126-138).
//   MODE 0 (VEC2):  lowest fixed bit >= 1 -> unit = two neighbouring pairs,
//                   one 256-bit load on each side.
//   MODE 1 (TGT0):  target is bit 0, controls >= 1 -> unit = one pair held in
//                   one 256-bit word.
//   MODE 2 (SCALAR): a control sits on bit 0 -> 16-byte accesses.
//   MODE 3 (PAIR):   a control sits on bit 0 -> the aligned 32-byte pairs are
//                    read and written whole (default; see k_diag MODE 2).
struct Mat2 {
  double2 m00, m01, m10, m11;
};

// QSV_DIAG_PAIR=0 selects the 16-byte paths for controls on bit 0 (A/B measurements)
static bool diag_pair_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QSV_DIAG_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_pair2x2(double2* __restrict__ a, FixedBits fb, uint64_t tbit, Mat2 M, uint64_t units) {
  const uint64_t first = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x;
  if (MODE == 0) {
    Amp2 lo[kUnroll], hi[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u << 1, fb);
        lo[j] = ld2(a + idx[j]);
        hi[j] = ld2(a + idx[j] + tbit);
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        Amp2 nl, nh;
        nl.a = cfma(M.m01, hi[j].a, cmul(M.m00, lo[j].a));
        nh.a = cfma(M.m11, hi[j].a, cmul(M.m10, lo[j].a));
        nl.b = cfma(M.m01, hi[j].b, cmul(M.m00, lo[j].b));
        nh.b = cfma(M.m11, hi[j].b, cmul(M.m10, lo[j].b));
        st2(a + idx[j], nl);
        st2(a + idx[j] + tbit, nh);
      }
    }
  } else if (MODE == 1) {
    Amp2 v[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u, fb);
        v[j] = ld2(a + idx[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        Amp2 o;
        o.a = cfma(M.m01, v[j].b, cmul(M.m00, v[j].a));
        o.b = cfma(M.m11, v[j].b, cmul(M.m10, v[j].a));
        st2(a + idx[j], o);
      }
    }
  } else if (MODE == 3) {
    // control on bit 0: each side's aligned 32-byte pair is read and written
    // whole (full-sector stores; the neighbour fails the control, so no other
    // thread touches it)
    Amp2 lo[kUnroll], hi[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u, fb);
        lo[j] = ld2(a + (idx[j] & ~1ULL));
        hi[j] = ld2(a + (idx[j] & ~1ULL) + tbit);
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        if (idx[j] & 1) {
          const double2 x = lo[j].b, y = hi[j].b;
          lo[j].b = cfma(M.m01, y, cmul(M.m00, x));
          hi[j].b = cfma(M.m11, y, cmul(M.m10, x));
        } else {
          const double2 x = lo[j].a, y = hi[j].a;
          lo[j].a = cfma(M.m01, y, cmul(M.m00, x));
          hi[j].a = cfma(M.m11, y, cmul(M.m10, x));
        }
        st2(a + (idx[j] & ~1ULL), lo[j]);
        st2(a + (idx[j] & ~1ULL) + tbit, hi[j]);
      }
    }
  } else {
    double2 x[kUnroll], y[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u, fb);
        x[j] = ld1(a + idx[j]);
        y[j] = ld1(a + idx[j] + tbit);
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        st1(a + idx[j], cfma(M.m01, y[j], cmul(M.m00, x[j])));
        st1(a + idx[j] + tbit, cfma(M.m11, y[j], cmul(M.m10, x[j])));
      }
    }
  }
}

// --------------------------------------------------------------------------
// Diagonal: psi_x *= d[sub(x)] over the amplitudes whose control bits match
// (kernels.py:155-173).  The table lives in shared memory (m <= 8) or is read
// through the read-only path (m > 8).  MODE 0: lowest fixed bit >= 1 (or no
// controls) -> 256-bit accesses; MODE 1: control on bit 0, 16-byte accesses;
// MODE 2: control on bit 0, the touched amplitude's aligned 32-byte pair is
// read and written whole (the neighbour unchanged, and untouched by any other
// thread since it fails the bit-0 control): a full-sector store instead of a
// 16-byte partial write, which HBM serves as read-modify-write (CZ on qubits
// 0 and 1).
struct DiagSmall {
  double2 d[32];
};

struct TPos {
  int p[QSV_MAX_TARGETS];
};

template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_diag(double2* __restrict__ a, FixedBits fb, int m, DiagSmall small,
           const double2* __restrict__ big, TPos tpos, uint64_t units) {
  __shared__ double2 tab[256];
  const int D = 1 << m;
  if (m <= 8) {
    for (int i = threadIdx.x; i < D; i += blockDim.x) tab[i] = (m <= 5) ? small.d[i] : big[i];
    __syncthreads();
  }
  const int* tp = tpos.p;
  auto sub_of = [&](uint64_t x) {
    int s = 0;
#pragma unroll
    for (int j = 0; j < 12; ++j)
      if (j < m) s |= (int)((x >> tp[j]) & 1ULL) << j;
    return s;
  };
  auto lookup = [&](int s) { return m <= 8 ? tab[s] : __ldg(big + s); };
  const uint64_t first = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x;
  if (MODE == 0) {
    Amp2 v[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u << 1, fb);
        v[j] = ld2(a + idx[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        Amp2 o;
        o.a = cmul(v[j].a, lookup(sub_of(idx[j])));
        o.b = cmul(v[j].b, lookup(sub_of(idx[j] + 1)));
        st2(a + idx[j], o);
      }
    }
  } else if (MODE == 2) {
    Amp2 v[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u, fb);
        v[j] = ld2(a + (idx[j] & ~1ULL));
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        const double2 f = lookup(sub_of(idx[j]));
        if (idx[j] & 1) v[j].b = cmul(v[j].b, f);
        else v[j].a = cmul(v[j].a, f);
        st2(a + (idx[j] & ~1ULL), v[j]);
      }
    }
  } else {
    double2 v[kUnroll];
    uint64_t idx[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) {
        idx[j] = widen(u, fb);
        v[j] = ld1(a + idx[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const uint64_t u = first + (uint64_t)j * kThreads;
      if (u < units) st1(a + idx[j], cmul(v[j], lookup(sub_of(idx[j]))));
    }
  }
}

// Single-target diagonal (RZ, S, T, U1, ... without controls): the two
// entries stay in registers; pure streaming, every amplitude read and written
// once with 256-bit accesses.
__global__ void __launch_bounds__(kThreads)
    k_diag1(double2* __restrict__ a, int t, double2 d0, double2 d1, uint64_t units) {
  const uint64_t first = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x;
  Amp2 v[kUnroll];
#pragma unroll
  for (int j = 0; j < kUnroll; ++j) {
    const uint64_t u = first + (uint64_t)j * kThreads;
    if (u < units) v[j] = ld2(a + (u << 1));
  }
#pragma unroll
  for (int j = 0; j < kUnroll; ++j) {
    const uint64_t u = first + (uint64_t)j * kThreads;
    if (u < units) {
      const uint64_t x = u << 1;
      const bool ba = (x >> t) & 1ULL;
      const bool bb = ((x + 1) >> t) & 1ULL;
      Amp2 o;
      o.a = cmul(v[j].a, ba ? d1 : d0);
      o.b = cmul(v[j].b, bb ? d1 : d0);
      st2(a + x, o);
    }
  }
}

// --------------------------------------------------------------------------
// Dense 2^K x 2^K on one coset per thread (K = 2..4): replaces the unrolled
// gather of _apply_dense_small (kernels.py:126-138) and the zgemm path
// (kernels.py:100-106).  The matrix travels as a __grid_constant__ kernel
// parameter: every lane reads the same element at the same time, so the
// constant cache broadcasts it.
template <int K>
struct MatK {
  double2 m[1 << (2 * K)];
};

template <int K>
__global__ void __launch_bounds__(128)
    k_dense_reg(double2* __restrict__ a, FixedBits fb, const __grid_constant__ MatK<K> M,
                uint64_t tb0, uint64_t tb1, uint64_t tb2, uint64_t tb3, uint64_t tb4,
                uint64_t ncos) {
  constexpr int D = 1 << K;
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ncos) return;
  const uint64_t tb[5] = {tb0, tb1, tb2, tb3, tb4};
  const uint64_t base = widen(k, fb);
  double2 in[D];
#pragma unroll
  for (int w = 0; w < D; ++w) {
    uint64_t off = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if ((w >> j) & 1) off |= tb[j];
    in[w] = a[base + off];
  }
#pragma unroll
  for (int z = 0; z < D; ++z) {
    double2 acc = cmul(M.m[z * D], in[0]);
#pragma unroll
    for (int w = 1; w < D; ++w) acc = cfma(M.m[z * D + w], in[w], acc);
    uint64_t off = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if ((z >> j) & 1) off |= tb[j];
    a[base + off] = acc;
  }
}

// Dense for K >= 5: cosets staged in shared memory, rows computed by the
// block's threads, matrix read through L2 (generic path; merged gates from
// optimize_heavy(5) and merge_all land here).
__global__ void __launch_bounds__(kThreads)
    k_dense_smem(double2* __restrict__ a, FixedBits fb, int K, const double2* __restrict__ mat,
                 const uint64_t* __restrict__ offs, uint64_t ncos) {
  extern __shared__ double2 sm[];
  const int D = 1 << K;
  const int per_block = max(1, kThreads / D);  // cosets per block
  for (uint64_t c0 = (uint64_t)blockIdx.x * per_block; c0 < ncos;
       c0 += (uint64_t)gridDim.x * per_block) {
    const uint64_t rem = ncos - c0;
    const int nco = rem < (uint64_t)per_block ? (int)rem : per_block;
    for (int i = threadIdx.x; i < nco * D; i += blockDim.x) {
      const int c = i / D, w = i % D;
      sm[i] = a[widen(c0 + c, fb) + offs[w]];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nco * D; i += blockDim.x) {
      const int c = i / D, z = i % D;
      const double2* row = mat + (uint64_t)z * D;
      const double2* in = sm + c * D;
      double2 acc = make_double2(0.0, 0.0);
      for (int w = 0; w < D; ++w) acc = cfma(__ldg(row + w), in[w], acc);
      a[widen(c0 + c, fb) + offs[z]] = acc;
    }
    __syncthreads();
  }
}

// Dense K = 5 (fused blocks of optimize_heavy(5), kernels.py:100-106): the
// 32x32 matrix is staged in shared memory once per block and read as
// broadcasts; each thread holds one coset's 32 amplitudes in registers and
// computes its 32 outputs (1024 complex FMA per coset, FP64-bound).
__global__ void __launch_bounds__(kThreads)
    k_dense5(double2* __restrict__ a, FixedBits fb, const double2* __restrict__ mat,
             const uint64_t* __restrict__ offs, uint64_t ncos) {
  constexpr int D = 32;
  __shared__ double2 sM[D * D];
  __shared__ uint64_t sO[D];
  for (int i = threadIdx.x; i < D * D; i += kThreads) sM[i] = mat[i];
  if (threadIdx.x < D) sO[threadIdx.x] = offs[threadIdx.x];
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t c = (uint64_t)blockIdx.x * kThreads + threadIdx.x; c < ncos; c += stride) {
    const uint64_t x0 = widen(c, fb);
    double2 in[D];
#pragma unroll
    for (int w = 0; w < D; ++w) in[w] = ld1(a + (x0 | sO[w]));
#pragma unroll 4
    for (int z = 0; z < D; ++z) {
      double2 acc = cmul(sM[z * D], in[0]);
#pragma unroll
      for (int w = 1; w < D; ++w) acc = cfma(sM[z * D + w], in[w], acc);
      st1(a + (x0 | sO[z]), acc);
    }
  }
}

// Dense K = 5 on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).  A fused
// 5-qubit block is a 32x32 complex matrix times 32-amplitude cosets, i.e. the
// real GEMM [Or; Oi] = [[Mr, -Mi], [Mi, Mr]] [Ir; Ii] with a 64x64 A and one
// column per coset.  A warp takes 8 cosets (one n = 8 column tile): each lane
// (g = lane / 4, t = lane % 4) loads the 8 amplitudes w = t (mod 4) of coset
// g -- exactly its B fragments for the 16 k-steps -- then runs 8 row tiles x 16
// k-steps = 128 DMMA with the 8 row-tile accumulators interleaved (8
// independent chains), and stores its D fragments: rows g, g+8, g+16, g+24
// (real parts from row tiles 0..3, imaginary from 4..7) of cosets 2t, 2t+1.
// A fragments come from shared memory pre-permuted into fragment order (one
// conflict-free 256-byte LDS per DMMA).  Same FLOPs as k_dense5 (128 real
// FMA per amplitude), on the DMMA pipe (measured 36.4 vs 31.7 TFLOP/s DFMA,
// profiles/fp64_peak.json).  Reference: the zgemm path kernels.py:100-106.
constexpr int kMmaThreads = 256;
__global__ void __launch_bounds__(kMmaThreads)
    k_dense5_mma(double2* __restrict__ a, FixedBits fb, const double2* __restrict__ mat,
                 const uint64_t* __restrict__ offs, uint64_t ncos) {
  __shared__ double sA[8 * 16 * 32];  // [row tile][k step][lane]
  __shared__ uint64_t sO[32];
  for (int i = threadIdx.x; i < 8 * 16 * 32; i += kMmaThreads) {
    const int r = i >> 9, st = (i >> 5) & 15, ln = i & 31;
    const int row = 8 * r + (ln >> 2), col = 4 * st + (ln & 3);  // into the 64x64 real A
    const double2 m = mat[(row & 31) * 32 + (col & 31)];
    // [[Mr, -Mi], [Mi, Mr]]
    sA[i] = (row < 32) == (col < 32) ? m.x : (row < 32 ? -m.y : m.y);
  }
  if (threadIdx.x < 32) sO[threadIdx.x] = offs[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const uint64_t warps = (uint64_t)gridDim.x * (kMmaThreads / 32);
  const uint64_t ntile = (ncos + 7) / 8;
  for (uint64_t ct = (uint64_t)blockIdx.x * (kMmaThreads / 32) + (threadIdx.x >> 5); ct < ntile;
       ct += warps) {
    const uint64_t cin = ct * 8 + g;
    double b[16];
    if (cin < ncos) {
      const uint64_t x0 = widen(cin, fb);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 v = ld1(a + (x0 | sO[4 * q + t]));
        b[q] = v.x;
        b[8 + q] = v.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) b[q] = 0.0;
    }
    double d[8][2];
#pragma unroll
    for (int r = 0; r < 8; ++r) d[r][0] = d[r][1] = 0.0;
#pragma unroll
    for (int st = 0; st < 16; ++st) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const double av = sA[((r << 4) | st) * 32 + lane];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[r][0]), "+d"(d[r][1])
                     : "d"(av), "d"(b[st]));
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t cout = ct * 8 + 2 * t + h;
      if (cout >= ncos) continue;
      const uint64_t x0 = widen(cout, fb);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        st1(a + (x0 | sO[8 * r + g]), make_double2(d[r][h], d[r + 4][h]));
    }
  }
}

// QSV_DENSE5_MMA=0 keeps the DFMA kernel (A/B)
bool dense5_mma_enabled() {
  static const int on = [] {
    const char* e = getenv("QSV_DENSE5_MMA");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// Sparse / permutation (kernels.py:141-152, 176-185): cosets staged in shared
// memory like k_dense_smem, each output row summed over its CSR entries
// (O(nnz) per coset instead of 4^K).  Payload: values, coset offsets,
// row pointers, columns.
__global__ void __launch_bounds__(kThreads)
    k_sparse_smem(double2* __restrict__ a, FixedBits fb, int K, const double2* __restrict__ vals,
                  const uint64_t* __restrict__ offs, const int32_t* __restrict__ rptr,
                  const int32_t* __restrict__ cols, uint64_t ncos) {
  extern __shared__ double2 sm[];
  const int D = 1 << K;
  const int per_block = max(1, kThreads / D);  // cosets per block
  for (uint64_t c0 = (uint64_t)blockIdx.x * per_block; c0 < ncos;
       c0 += (uint64_t)gridDim.x * per_block) {
    const uint64_t rem = ncos - c0;
    const int nco = rem < (uint64_t)per_block ? (int)rem : per_block;
    for (int i = threadIdx.x; i < nco * D; i += blockDim.x) {
      const int c = i / D, w = i % D;
      sm[i] = a[widen(c0 + c, fb) + offs[w]];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nco * D; i += blockDim.x) {
      const int c = i / D, z = i % D;
      const double2* in = sm + c * D;
      double2 acc = make_double2(0.0, 0.0);
      for (int e = __ldg(rptr + z); e < __ldg(rptr + z + 1); ++e)
        acc = cfma(__ldg(vals + e), in[__ldg(cols + e)], acc);
      a[widen(c0 + c, fb) + offs[z]] = acc;
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// Pauli product on pairs (i, j = i ^ xmask) (kernels.py:202-235):
//   new_i = alpha psi_i + beta phi(j) psi_j,  new_j = alpha psi_j + beta phi(i) psi_i
//   phi(x) = i^ny (-1)^popc(x & zmask)
// (alpha, beta) = (0, 1) for the Pauli gate, (cos a/2, i sin a/2) for the
// rotation exp(i a P / 2).  The pair is enumerated with the top bit of xmask
// inserted as zero.  MODE 0: pivot >= 1 -> two neighbouring pairs per unit,
// 256-bit loads on both sides; MODE 1: xmask == 1 -> the pair is one 256-bit
// word.
template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_pauli_pairs(double2* __restrict__ a, FixedBits piv, uint64_t xm, uint64_t zm, double2 alpha,
                  double2 bph, uint64_t units) {
  const uint64_t first = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x;
  auto sgn = [&](uint64_t x, double2 v) {
    return (__popcll(x & zm) & 1) ? make_double2(-v.x, -v.y) : v;
  };
  if (MODE == 0) {
    Amp2 P[kUnroll], Q[kUnroll];
    uint64_t ii[kUnroll], jj[kUnroll];
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {
      const uint64_t u = first + (uint64_t)r * kThreads;
      if (u < units) {
        ii[r] = widen(u << 1, piv);
        jj[r] = (ii[r] ^ xm) & ~1ULL;
        P[r] = ld2(a + ii[r]);
        Q[r] = ld2(a + jj[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {
      const uint64_t u = first + (uint64_t)r * kThreads;
      if (u < units) {
        const bool sw = xm & 1ULL;
        const uint64_t i0 = ii[r], i1 = ii[r] + 1;
        const uint64_t j0 = i0 ^ xm, j1 = i1 ^ xm;
        const double2 pi0 = P[r].a, pi1 = P[r].b;
        const double2 pj0 = sw ? Q[r].b : Q[r].a;
        const double2 pj1 = sw ? Q[r].a : Q[r].b;
        const double2 ni0 = cfma(bph, sgn(j0, pj0), cmul(alpha, pi0));
        const double2 ni1 = cfma(bph, sgn(j1, pj1), cmul(alpha, pi1));
        const double2 nj0 = cfma(bph, sgn(i0, pi0), cmul(alpha, pj0));
        const double2 nj1 = cfma(bph, sgn(i1, pi1), cmul(alpha, pj1));
        Amp2 oP, oQ;
        oP.a = ni0;
        oP.b = ni1;
        oQ.a = sw ? nj1 : nj0;
        oQ.b = sw ? nj0 : nj1;
        st2(a + ii[r], oP);
        st2(a + jj[r], oQ);
      }
    }
  } else {
    Amp2 v[kUnroll];
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {
      const uint64_t u = first + (uint64_t)r * kThreads;
      if (u < units) v[r] = ld2(a + (u << 1));
    }
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {
      const uint64_t u = first + (uint64_t)r * kThreads;
      if (u < units) {
        const uint64_t i = u << 1, j = i + 1;
        Amp2 o;
        o.a = cfma(bph, sgn(j, v[r].b), cmul(alpha, v[r].a));
        o.b = cfma(bph, sgn(i, v[r].a), cmul(alpha, v[r].b));
        st2(a + i, o);
      }
    }
  }
}

// Z-type Pauli / rotation (xmask == 0): psi_x *= f[popc(x & zmask) & 1].
__global__ void __launch_bounds__(kThreads)
    k_parity_diag(double2* __restrict__ a, uint64_t zm, double2 f0, double2 f1, uint64_t units) {
  const uint64_t first = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x;
  Amp2 v[kUnroll];
#pragma unroll
  for (int r = 0; r < kUnroll; ++r) {
    const uint64_t u = first + (uint64_t)r * kThreads;
    if (u < units) v[r] = ld2(a + (u << 1));
  }
#pragma unroll
  for (int r = 0; r < kUnroll; ++r) {
    const uint64_t u = first + (uint64_t)r * kThreads;
    if (u < units) {
      const uint64_t x = u << 1;
      const int pa = __popcll(x & zm) & 1;
      const int pb = __popcll((x + 1) & zm) & 1;
      Amp2 o;
      o.a = cmul(v[r].a, pa ? f1 : f0);
      o.b = cmul(v[r].b, pb ? f1 : f0);
      st2(a + x, o);
    }
  }
}

// --------------------------------------------------------------------------
// State algebra helpers
__global__ void __launch_bounds__(kThreads)
    k_scale(double2* __restrict__ a, double2 f, uint64_t units) {
  const uint64_t u = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (u >= units) return;
  Amp2 v = ld2(a + (u << 1));
  v.a = cmul(v.a, f);
  v.b = cmul(v.b, f);
  st2(a + (u << 1), v);
}

__global__ void __launch_bounds__(kThreads)
    k_add(double2* __restrict__ dst, const double2* __restrict__ src, uint64_t units) {
  const uint64_t u = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (u >= units) return;
  Amp2 v = ld2(dst + (u << 1));
  Amp2 w = ld2_ro(src + (u << 1));
  v.a.x += w.a.x;
  v.a.y += w.a.y;
  v.b.x += w.b.x;
  v.b.y += w.b.y;
  st2(dst + (u << 1), v);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Non-parity benchmark initialiser: complex Gaussian from a counter hash
// (Box-Muller); the caller normalises.
__global__ void __launch_bounds__(kThreads)
    k_random(double2* __restrict__ a, uint64_t seed, uint64_t dim) {
  const uint64_t x = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (x >= dim) return;
  const uint64_t h1 = mix64(seed * 0x9e3779b97f4a7c15ULL + 2 * x + 1);
  const uint64_t h2 = mix64(h1 ^ 0xd1b54a32d192ed03ULL);
  const double u1 = ((h1 >> 11) + 1) * (1.0 / 9007199254740993.0);
  const double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  a[x] = make_double2(r * c, r * s);
}

// ==========================================================================
// host side

static inline double2 D2(Cplx c) { return make_double2(c.re, c.im); }

static bool is_one(Cplx c) { return c.re == 1.0 && c.im == 0.0; }

GateDesc canonicalize(const GateDesc& g0) {
  GateDesc g = g0;
  if (g.kind == QSV_OP_PAULI_ROT) {
    const double c = std::cos(g.angle / 2), s = std::sin(g.angle / 2);
    if (g.m == 1 && g.nc == 0 && g.ids[0] == 3) {  // RZ: diag(e^{+ia/2}, e^{-ia/2})
      g.kind = QSV_OP_DIAG;
      g.data = {{c, s}, {c, -s}};
      return canonicalize(g);
    }
    if (g.nc > 0 || g.m == 1) {
      // c I + i s P as a dense matrix (kernels.py:227-230 for the controlled
      // case; the 1-qubit uncontrolled case is the same 2x2 on one pair)
      const int D = 1 << g.m;
      std::vector<Cplx> P((size_t)D * D, Cplx{0, 0});
      for (int col = 0; col < D; ++col) {
        // P e_col: flip X/Y bits, phase from Y/Z bits of the source (col)
        int row = col;
        Cplx ph{1, 0};
        for (int j = 0; j < g.m; ++j) {
          const int id = g.ids[j];
          const int bit = (col >> j) & 1;
          if (id == 1 || id == 2) row ^= 1 << j;
          if (id == 3 && bit) ph = {-ph.re, -ph.im};
          if (id == 2) ph = bit ? Cplx{ph.im, -ph.re} : Cplx{-ph.im, ph.re};  // *(-i) or *(+i)
        }
        P[(size_t)row * D + col] = ph;
      }
      g.kind = QSV_OP_DENSE;
      g.data.assign((size_t)D * D, Cplx{0, 0});
      for (int r = 0; r < D; ++r)
        for (int col = 0; col < D; ++col) {
          Cplx p = P[(size_t)r * D + col];
          // c*delta + i*s*p
          g.data[(size_t)r * D + col] = {(r == col ? c : 0.0) - s * p.im, s * p.re};
        }
      return g;
    }
    return g;
  }
  if (g.kind == QSV_OP_PAULI && g.nc > 0) {
    const int D = 1 << g.m;
    g.kind = QSV_OP_DENSE;
    g.data.assign((size_t)D * D, Cplx{0, 0});
    for (int col = 0; col < D; ++col) {
      int row = col;
      Cplx ph{1, 0};
      for (int j = 0; j < g.m; ++j) {
        const int id = g.ids[j];
        const int bit = (col >> j) & 1;
        if (id == 1 || id == 2) row ^= 1 << j;
        if (id == 3 && bit) ph = {-ph.re, -ph.im};
        if (id == 2) ph = bit ? Cplx{ph.im, -ph.re} : Cplx{-ph.im, ph.re};
      }
      g.data[(size_t)row * D + col] = ph;
    }
    return g;
  }
  if (g.kind == QSV_OP_DENSE && g.m == 0) {
    g.kind = QSV_OP_DIAG;
    return canonicalize(g);
  }
  if (g.kind == QSV_OP_DIAG) {
    // entries equal to 1 leave their amplitudes untouched: if only one entry
    // differs, move the targets into the control set (touch 2^(n-m-c) amps)
    const int D = 1 << g.m;
    int diff = -1, ndiff = 0;
    for (int z = 0; z < D; ++z)
      if (!is_one(g.data[z])) {
        diff = z;
        ++ndiff;
      }
    if (ndiff == 0) {
      g.m = 0;
      g.data = {{1, 0}};
      g.nc = -1;  // marks a no-op
      return g;
    }
    if (ndiff == 1 && g.m > 0 && g.nc + g.m <= QSV_MAX_CONTROLS) {
      for (int j = 0; j < g.m; ++j) {
        g.cq[g.nc] = g.targets[j];
        g.cv[g.nc] = (diff >> j) & 1;
        ++g.nc;
      }
      g.data = {g.data[diff]};
      g.m = 0;
    }
    return g;
  }
  return g;
}

int validate_gate(int n, const GateDesc& g) {
  if (g.m < 0 || g.m > QSV_MAX_TARGETS) {
    set_error("target count %d outside [0, %d]", g.m, QSV_MAX_TARGETS);
    return QSV_EINVAL;
  }
  if (g.nc < 0 || g.nc > QSV_MAX_CONTROLS) {
    set_error("control count %d outside [0, %d]", g.nc, QSV_MAX_CONTROLS);
    return QSV_EINVAL;
  }
  uint64_t used = 0;
  for (int j = 0; j < g.m; ++j) {
    const int t = g.targets[j];
    if (t < 0 || t >= n) {
      set_error("gate touches qubit %d but the state has %d qubits", t, n);
      return QSV_EINVAL;
    }
    if (used & (1ULL << t)) {
      set_error("target qubits must be distinct");
      return QSV_EINVAL;
    }
    used |= 1ULL << t;
  }
  for (int j = 0; j < g.nc; ++j) {
    const int q = g.cq[j];
    if (q < 0 || q >= n) {
      set_error("gate touches qubit %d but the state has %d qubits", q, n);
      return QSV_EINVAL;
    }
    if (used & (1ULL << q)) {
      set_error("control qubit %d overlaps a target or another control", q);
      return QSV_EINVAL;
    }
    if (g.cv[j] != 0 && g.cv[j] != 1) {
      set_error("control values must be 0 or 1");
      return QSV_EINVAL;
    }
    used |= 1ULL << q;
  }
  if (g.kind == QSV_OP_SPARSE) {
    const int D = 1 << g.m;
    if (g.sp_rows.size() != g.data.size() || g.sp_cols.size() != g.data.size()) {
      set_error("sparse entries: rows, columns and values differ in length");
      return QSV_EINVAL;
    }
    for (size_t e = 0; e < g.data.size(); ++e)
      if (g.sp_rows[e] < 0 || g.sp_rows[e] >= D || g.sp_cols[e] < 0 || g.sp_cols[e] >= D) {
        set_error("sparse entry (%d, %d) outside a %dx%d matrix", g.sp_rows[e], g.sp_cols[e], D,
                  D);
        return QSV_EINVAL;
      }
  }
  if (g.kind == QSV_OP_PAULI || g.kind == QSV_OP_PAULI_ROT) {
    for (int j = 0; j < g.m; ++j)
      if (g.ids[j] < 0 || g.ids[j] > 3) {
        set_error("Pauli ids must be in {0, 1, 2, 3}");
        return QSV_EINVAL;
      }
    if (g.kind == QSV_OP_PAULI_ROT && !std::isfinite(g.angle)) {
      set_error("rotation angle must be finite");
      return QSV_EINVAL;
    }
  } else if (g.kind == QSV_OP_DENSE) {
    if (g.data.size() != (size_t)1 << (2 * g.m)) {
      set_error("matrix size does not match %d targets", g.m);
      return QSV_EINVAL;
    }
  } else if (g.kind == QSV_OP_DIAG) {
    if (g.data.size() != (size_t)1 << g.m) {
      set_error("diagonal length does not match %d targets", g.m);
      return QSV_EINVAL;
    }
  } else if (g.kind != QSV_OP_SPARSE) {  // sparse entries checked above
    set_error("unknown op kind %d", g.kind);
    return QSV_EINVAL;
  }
  return QSV_OK;
}

static void pauli_masks(const GateDesc& g, uint64_t* xm, uint64_t* zm, int* ny) {
  *xm = *zm = 0;
  *ny = 0;
  for (int j = 0; j < g.m; ++j) {
    const int id = g.ids[j];
    if (id == 1 || id == 2) *xm |= 1ULL << g.targets[j];
    if (id == 2 || id == 3) *zm |= 1ULL << g.targets[j];
    if (id == 2) ++*ny;
  }
}

static const Cplx kIpow[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};

static Cplx mulc(Cplx a, Cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

double gate_hbm_bytes(int n, const GateDesc& g0) {
  // touched amplitudes x 32 B (read + write); SURVEY.md 8(d)
  GateDesc g = canonicalize(g0);
  if (g.nc < 0) return 0.0;
  double amps = std::ldexp(1.0, n);
  if (g.kind == QSV_OP_DIAG || g.kind == QSV_OP_DENSE) amps = std::ldexp(1.0, n - g.nc);
  return 32.0 * amps;
}

int launch_gate(double2* a, int n, const GateDesc& g0, const Cplx* dev_data, cudaStream_t s) {
  GateDesc g = canonicalize(g0);
  if (g.nc < 0) return QSV_OK;  // identity
  const uint64_t dim = 1ULL << n;
  int fixed[kMaxFixed];
  uint64_t cval = 0;
  for (int j = 0; j < g.nc; ++j) {
    fixed[j] = g.cq[j];
    if (g.cv[j]) cval |= 1ULL << g.cq[j];
  }
  int lowest_ctl = 64;
  for (int j = 0; j < g.nc; ++j) lowest_ctl = std::min(lowest_ctl, g.cq[j]);

  if (g.kind == QSV_OP_SPARSE) {
    if (!dev_data) {
      set_error("internal: sparse gate needs a device payload");
      return QSV_EINVAL;
    }
    int fixed2[kMaxFixed];
    for (int j = 0; j < g.nc; ++j) fixed2[j] = g.cq[j];
    for (int j = 0; j < g.m; ++j) fixed2[g.nc + j] = g.targets[j];
    FixedBits fb2 = make_fixed(fixed2, g.nc + g.m, cval);
    const int D = 1 << g.m;
    const size_t nnz = g.data.size();
    const char* base = reinterpret_cast<const char*>(dev_data);
    const double2* vals = reinterpret_cast<const double2*>(base);
    const uint64_t* offs = reinterpret_cast<const uint64_t*>(base + nnz * sizeof(double2));
    const int32_t* rptr = reinterpret_cast<const int32_t*>(offs + D);
    const int32_t* cols = rptr + D + 1;
    const uint64_t ncos = dim >> (g.nc + g.m);
    const int per_block = std::max(1, kThreads / D);
    const size_t smem = sizeof(double2) * (size_t)per_block * D;
    static uint64_t attr_done = 0;
    QSV_TRY(ensure_smem_attr(k_sparse_smem, 200 * 1024, attr_done));
    uint64_t nblk = (ncos + per_block - 1) / per_block;
    nblk = std::max<uint64_t>(1, std::min<uint64_t>(nblk, 148ULL * 64));
    k_sparse_smem<<<(unsigned)nblk, kThreads, smem, s>>>(a, fb2, g.m, vals, offs, rptr, cols, ncos);
    QSV_CHECK_LAUNCH("k_sparse_smem");
    return QSV_OK;
  }

  if (g.kind == QSV_OP_DIAG) {
    if (g.m == 1 && g.nc == 0) {
      const uint64_t units = dim / 2;
      k_diag1<<<grid_for(units, kUnroll), kThreads, 0, s>>>(a, g.targets[0], D2(g.data[0]),
                                                           D2(g.data[1]), units);
      QSV_CHECK_LAUNCH("k_diag1");
      return QSV_OK;
    }
    if (g.m > 5 && !dev_data) {
      set_error("internal: diagonal with %d targets needs a device table", g.m);
      return QSV_EINVAL;
    }
    FixedBits fb = make_fixed(fixed, g.nc, cval);
    DiagSmall small;
    memset(&small, 0, sizeof(small));
    if (g.m <= 5)
      for (int z = 0; z < (1 << g.m); ++z) small.d[z] = D2(g.data[z]);
    TPos tp;
    for (int j = 0; j < QSV_MAX_TARGETS; ++j) tp.p[j] = j < g.m ? g.targets[j] : 0;
    const double2* big = reinterpret_cast<const double2*>(dev_data);
    const uint64_t cnt = dim >> g.nc;
    if (lowest_ctl >= 1 && cnt >= 2) {
      const uint64_t units = cnt / 2;
      k_diag<0><<<grid_for(units, kUnroll), kThreads, 0, s>>>(a, fb, g.m, small, big, tp, units);
    } else if (lowest_ctl == 0 && dim >= 2 && diag_pair_mode()) {
      k_diag<2><<<grid_for(cnt, kUnroll), kThreads, 0, s>>>(a, fb, g.m, small, big, tp, cnt);
    } else {
      k_diag<1><<<grid_for(cnt, kUnroll), kThreads, 0, s>>>(a, fb, g.m, small, big, tp, cnt);
    }
    QSV_CHECK_LAUNCH("k_diag");
    return QSV_OK;
  }

  if (g.kind == QSV_OP_PAULI || g.kind == QSV_OP_PAULI_ROT) {
    // uncontrolled here (canonicalize turned controlled ones into dense)
    uint64_t xm, zm;
    int ny;
    pauli_masks(g, &xm, &zm, &ny);
    Cplx alpha{0, 0}, beta{1, 0};
    if (g.kind == QSV_OP_PAULI_ROT) {
      alpha = {std::cos(g.angle / 2), 0};
      beta = {0, std::sin(g.angle / 2)};
    }
    const Cplx bph = mulc(beta, kIpow[ny & 3]);
    if (xm == 0) {
      // psi_x *= alpha + bph * (-1)^parity
      const Cplx f0{alpha.re + bph.re, alpha.im + bph.im};
      const Cplx f1{alpha.re - bph.re, alpha.im - bph.im};
      if (zm == 0 && f0.re == 1.0 && f0.im == 0.0) return QSV_OK;
      const uint64_t units = dim / 2;
      k_parity_diag<<<grid_for(units, kUnroll), kThreads, 0, s>>>(a, zm, D2(f0), D2(f1), units);
      QSV_CHECK_LAUNCH("k_parity_diag");
      return QSV_OK;
    }
    const int pivot = 63 - __builtin_clzll(xm);
    FixedBits piv = make_fixed(&pivot, 1, 0);
    if (pivot >= 1) {
      const uint64_t units = dim / 4;
      k_pauli_pairs<0><<<grid_for(units, kUnroll), kThreads, 0, s>>>(a, piv, xm, zm, D2(alpha),
                                                                     D2(bph), units);
    } else {
      const uint64_t units = dim / 2;
      k_pauli_pairs<1><<<grid_for(units, kUnroll), kThreads, 0, s>>>(a, piv, xm, zm, D2(alpha),
                                                                     D2(bph), units);
    }
    QSV_CHECK_LAUNCH("k_pauli_pairs");
    return QSV_OK;
  }

  // dense
  const int m = g.m;
  for (int j = 0; j < m; ++j) fixed[g.nc + j] = g.targets[j];
  FixedBits fb = make_fixed(fixed, g.nc + m, cval);
  const uint64_t ncos = dim >> (g.nc + m);
  if (m == 1) {
    Mat2 M{D2(g.data[0]), D2(g.data[1]), D2(g.data[2]), D2(g.data[3])};
    const int t = g.targets[0];
    const uint64_t tbit = 1ULL << t;
    if (t >= 1 && lowest_ctl >= 1 && ncos >= 2) {
      const uint64_t units = ncos / 2;
      k_pair2x2<0><<<grid_for(units, kUnroll), kThreads, 0, s>>>(a, fb, tbit, M, units);
    } else if (t == 0) {
      k_pair2x2<1><<<grid_for(ncos, kUnroll), kThreads, 0, s>>>(a, fb, tbit, M, ncos);
    } else if (diag_pair_mode()) {
      k_pair2x2<3><<<grid_for(ncos, kUnroll), kThreads, 0, s>>>(a, fb, tbit, M, ncos);
    } else {
      k_pair2x2<2><<<grid_for(ncos, kUnroll), kThreads, 0, s>>>(a, fb, tbit, M, ncos);
    }
    QSV_CHECK_LAUNCH("k_pair2x2");
    return QSV_OK;
  }
  uint64_t tb[5] = {0, 0, 0, 0, 0};
  for (int j = 0; j < m && j < 5; ++j) tb[j] = 1ULL << g.targets[j];
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, (ncos + 127) / 128);
  if (m >= 2 && m <= 4) {
    switch (m) {
      case 2: {
        MatK<2> M;
        for (int i = 0; i < 16; ++i) M.m[i] = D2(g.data[i]);
        k_dense_reg<2><<<blocks, 128, 0, s>>>(a, fb, M, tb[0], tb[1], tb[2], tb[3], tb[4], ncos);
        break;
      }
      case 3: {
        MatK<3> M;
        for (int i = 0; i < 64; ++i) M.m[i] = D2(g.data[i]);
        k_dense_reg<3><<<blocks, 128, 0, s>>>(a, fb, M, tb[0], tb[1], tb[2], tb[3], tb[4], ncos);
        break;
      }
      case 4: {
        MatK<4> M;
        for (int i = 0; i < 256; ++i) M.m[i] = D2(g.data[i]);
        k_dense_reg<4><<<blocks, 128, 0, s>>>(a, fb, M, tb[0], tb[1], tb[2], tb[3], tb[4], ncos);
        break;
      }
    }
    QSV_CHECK_LAUNCH("k_dense_reg");
    return QSV_OK;
  }
  // m >= 5: shared-memory cosets, matrix + offsets from device memory
  if (!dev_data) {
    set_error("internal: dense gate with %d targets needs a device matrix", m);
    return QSV_EINVAL;
  }
  const int D = 1 << m;
  const uint64_t* offs = reinterpret_cast<const uint64_t*>(dev_data + (size_t)D * D);
  if (m == 5 && dense5_mma_enabled() && ncos >= 8) {
    const uint64_t tiles = (ncos + 7) / 8;
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((tiles + kMmaThreads / 32 - 1) / (kMmaThreads / 32), 148ULL * 8));
    k_dense5_mma<<<grid, kMmaThreads, 0, s>>>(a, fb, reinterpret_cast<const double2*>(dev_data),
                                              offs, ncos);
    QSV_CHECK_LAUNCH("k_dense5_mma");
    return QSV_OK;
  }
  if (m == 5) {
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((ncos + kThreads - 1) / kThreads, 148ULL * 8));
    k_dense5<<<grid, kThreads, 0, s>>>(a, fb, reinterpret_cast<const double2*>(dev_data), offs,
                                       ncos);
    QSV_CHECK_LAUNCH("k_dense5");
    return QSV_OK;
  }
  const int per_block = std::max(1, kThreads / D);
  const size_t smem = sizeof(double2) * (size_t)per_block * D;
  if (smem > 48 * 1024) {
    static uint64_t attr_done = 0;
    QSV_TRY(ensure_smem_attr(k_dense_smem, 200 * 1024, attr_done));
  }
  uint64_t nblk = (ncos + per_block - 1) / per_block;
  nblk = std::min<uint64_t>(nblk, 148ULL * 64);
  k_dense_smem<<<(unsigned)nblk, kThreads, smem, s>>>(a, fb, m, reinterpret_cast<const double2*>(dev_data),
                                                       offs, ncos);
  QSV_CHECK_LAUNCH("k_dense_smem");
  return QSV_OK;
}

int launch_scale(double2* a, uint64_t dim, double2 f, cudaStream_t s) {
  if (dim < 2) {
    // 1-amplitude states cannot exist (n >= 1), but keep the guard
    return QSV_OK;
  }
  const uint64_t units = dim / 2;
  k_scale<<<grid_for(units, 1), kThreads, 0, s>>>(a, f, units);
  QSV_CHECK_LAUNCH("k_scale");
  return QSV_OK;
}

int launch_add(double2* dst, const double2* src, uint64_t dim, cudaStream_t s) {
  const uint64_t units = dim / 2;
  k_add<<<grid_for(units, 1), kThreads, 0, s>>>(dst, src, units);
  QSV_CHECK_LAUNCH("k_add");
  return QSV_OK;
}

int launch_random(double2* a, uint64_t dim, uint64_t seed, cudaStream_t s) {
  k_random<<<grid_for(dim, 1), kThreads, 0, s>>>(a, seed, dim);
  QSV_CHECK_LAUNCH("k_random");
  return QSV_OK;
}

}  // namespace qsv
