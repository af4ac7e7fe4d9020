// State analysis and reshaping: marginal probabilities, Z-basis sampling,
// element-wise multiply, tensor product, qubit permutation, qubit dropping.
//
// Replaces the numpy implementations of the reference container
// (state.py:83-114 and the module functions state.py:142-192):
//   get_marginal_probability  probs[mask].sum()           -> masked reduction
//   sampling                  cumsum + searchsorted       -> block sums, scan,
//                                                            per-draw search
//   multiply_elementwise_function  amps *= coefs          -> one HBM pass
//   tensor_product            np.kron(second, first)      -> one write pass
//   permutate_qubit / drop_qubit  fancy-index gathers     -> gather kernels
// All are HBM-bound byte movers: coalesced on the written side, 16-byte
// accesses, and deterministic (fixed-order) reductions.
#include <algorithm>
#include <cmath>
#include <vector>

#include "qsv_internal.cuh"

namespace qsv {

static unsigned stream_grid(uint64_t units) {
  return (unsigned)std::min<uint64_t>(std::max<uint64_t>(1, (units + kThreads - 1) / kThreads),
                                      148ULL * 16);
}

// Index with the free bits of u deposited at pos[0..nf) over a fixed value:
// used instead of widen() when more than kMaxFixed qubits are fixed.
struct Deposit {
  int nf;
  int8_t pos[64];
  uint64_t value;
};

__device__ __forceinline__ uint64_t deposit(uint64_t u, const Deposit& d) {
  uint64_t x = d.value;
  for (int i = 0; i < d.nf; ++i) x |= ((u >> i) & 1ULL) << d.pos[i];
  return x;
}

static Deposit make_deposit(int n, uint64_t fixed_mask, uint64_t value) {
  Deposit d;
  d.nf = 0;
  d.value = value & fixed_mask;
  for (int q = 0; q < n; ++q)
    if (!((fixed_mask >> q) & 1ULL)) d.pos[d.nf++] = (int8_t)q;
  return d;
}

// ---------------------------------------------------------------- marginal
// sum over x with (x & mask) == value of |psi_x|^2; free bits enumerated by
// widen() so only the 2^(n-k) matching amplitudes are read.
__global__ void __launch_bounds__(kThreads)
    k_marginal(const double2* __restrict__ a, FixedBits fb, uint64_t units,
               double* __restrict__ partials) {
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t u = (uint64_t)blockIdx.x * kThreads + threadIdx.x; u < units; u += stride) {
    const double2 v = ld1(a + widen(u, fb));
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads)
    k_marginal_dep(const double2* __restrict__ a, Deposit dp, uint64_t units,
                   double* __restrict__ partials) {
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t u = (uint64_t)blockIdx.x * kThreads + threadIdx.x; u < units; u += stride) {
    const double2 v = ld1(a + deposit(u, dp));
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void k_sum_partials(const double* __restrict__ partials, int nblocks,
                               double* __restrict__ out) {
  __shared__ double s[kThreads];
  double v = 0;
  for (int b = threadIdx.x; b < nblocks; b += kThreads) v += partials[b];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// ------------------------------------------------------------ branch norm
// ||E psi||^2 for a 2^K x 2^K matrix E on K qubits without materialising
// E psi: per coset, u = E v and accumulate |u|^2 (CptpMap branch
// probabilities, maps.py:55-73, where the reference copies the whole state
// per Kraus operator).  E and the coset offsets live in shared memory.
template <int K>
__global__ void __launch_bounds__(kThreads)
    k_branch_norm(const double2* __restrict__ a, FixedBits fb, const double2* __restrict__ E,
                  const uint64_t* __restrict__ offs, uint64_t units,
                  double* __restrict__ partials) {
  constexpr int D = 1 << K;
  __shared__ double2 sE[D * D];
  __shared__ uint64_t sO[D];
  for (int i = threadIdx.x; i < D * D; i += kThreads) sE[i] = E[i];
  if (threadIdx.x < D) sO[threadIdx.x] = offs[threadIdx.x];
  __syncthreads();
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t u = (uint64_t)blockIdx.x * kThreads + threadIdx.x; u < units; u += stride) {
    const uint64_t x0 = widen(u, fb);
    double2 v[D];
#pragma unroll
    for (int w = 0; w < D; ++w) v[w] = __ldg(a + (x0 | sO[w]));
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double2 t = cmul(sE[r * D], v[0]);
#pragma unroll
      for (int w = 1; w < D; ++w) t = cfma(sE[r * D + w], v[w], t);
      acc = fma(t.x, t.x, fma(t.y, t.y, acc));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

// scratch: E (4^k double2) followed by 2^k offsets, already on the device
int launch_branch_norm(const double2* a, int n, const int* targets, int k, const double2* dE,
                       const uint64_t* dOffs, double* partials, double* dev_out, cudaStream_t s) {
  int pos[8];
  for (int j = 0; j < k; ++j) pos[j] = targets[j];
  std::sort(pos, pos + k);
  FixedBits fb = make_fixed(pos, k, 0);
  const uint64_t units = 1ULL << (n - k);
  const unsigned grid = (unsigned)std::min<uint64_t>(kRedBlocks, std::max<uint64_t>(
                                                          1, (units + kThreads - 1) / kThreads));
  switch (k) {
    case 1: k_branch_norm<1><<<grid, kThreads, 0, s>>>(a, fb, dE, dOffs, units, partials); break;
    case 2: k_branch_norm<2><<<grid, kThreads, 0, s>>>(a, fb, dE, dOffs, units, partials); break;
    case 3: k_branch_norm<3><<<grid, kThreads, 0, s>>>(a, fb, dE, dOffs, units, partials); break;
    case 4: k_branch_norm<4><<<grid, kThreads, 0, s>>>(a, fb, dE, dOffs, units, partials); break;
    case 5: k_branch_norm<5><<<grid, kThreads, 0, s>>>(a, fb, dE, dOffs, units, partials); break;
    default:
      set_error("branch norm supports 1..5 qubits, got %d", k);
      return QSV_EINVAL;
  }
  QSV_CHECK_LAUNCH("k_branch_norm");
  k_sum_partials<<<1, kThreads, 0, s>>>(partials, (int)grid, dev_out);
  QSV_CHECK_LAUNCH("k_sum_partials");
  return QSV_OK;
}

// ------------------------------------------------ density-matrix helpers
// A density matrix rho (2^h x 2^h, row-major) is held as a 2h-qubit vector:
// element (r, c) at index (r << h) | c, so U rho U^dag is U on the row
// qubits (h + t) and conj(U) on the column qubits (t).
__global__ void __launch_bounds__(kThreads)
    k_conj(double2* __restrict__ a, uint64_t dim) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t x = (uint64_t)blockIdx.x * kThreads + threadIdx.x; x < dim; x += stride) {
    double2 v = a[x];
    v.y = -v.y;
    a[x] = v;
  }
}

// sum_i rho[i][i] = sum_i a[(i << h) | i]; per-block partials (re, im)
__global__ void __launch_bounds__(kThreads)
    k_trace_pairs(const double2* __restrict__ a, int h, double* __restrict__ partials) {
  double re = 0.0, im = 0.0;
  const uint64_t count = 1ULL << h;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < count; i += stride) {
    const double2 v = __ldg(a + ((i << h) | i));
    re += v.x;
    im += v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  __shared__ double red[2][kThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = re;
    red[1][threadIdx.x >> 5] = im;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sr = 0, si = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      sr += red[0][w];
      si += red[1][w];
    }
    partials[blockIdx.x] = sr;
    partials[gridDim.x + blockIdx.x] = si;
  }
}

int launch_conj(double2* a, uint64_t dim, cudaStream_t s) {
  k_conj<<<stream_grid(dim), kThreads, 0, s>>>(a, dim);
  QSV_CHECK_LAUNCH("k_conj");
  return QSV_OK;
}

int launch_trace_pairs(const double2* a, int h, double* partials, double* dev_out,
                       cudaStream_t s) {
  const uint64_t count = 1ULL << h;
  const unsigned grid = (unsigned)std::min<uint64_t>(
      kRedBlocks / 2, std::max<uint64_t>(1, (count + kThreads - 1) / kThreads));
  k_trace_pairs<<<grid, kThreads, 0, s>>>(a, h, partials);
  QSV_CHECK_LAUNCH("k_trace_pairs");
  k_sum_partials<<<1, kThreads, 0, s>>>(partials, (int)grid, dev_out);
  QSV_CHECK_LAUNCH("k_sum_partials");
  k_sum_partials<<<1, kThreads, 0, s>>>(partials + grid, (int)grid, dev_out + 1);
  QSV_CHECK_LAUNCH("k_sum_partials");
  return QSV_OK;
}

// ---------------------------------------------------------------- sampling
// The cumulative distribution is defined blockwise: block b holds amplitudes
// [b*BS, (b+1)*BS); cum(j) = P[b] + r_j where r_j is the sequential running
// sum of |psi|^2 inside the block and P the exclusive scan of the block sums
// B[b] = r_last.  The search recomputes r_j with the same code, so the
// values it compares against are exactly the ones the block sums used.
constexpr int kSampleBlockLog = 8;  // 256 amplitudes per block

__device__ __forceinline__ double prob(double2 v) { return fma(v.x, v.x, v.y * v.y); }

__global__ void __launch_bounds__(kThreads)
    k_block_sums(const double2* __restrict__ a, int bs_log, uint64_t nblocks,
                 double* __restrict__ bsum) {
  const uint64_t b = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (b >= nblocks) return;
  const uint64_t bs = 1ULL << bs_log;
  const double2* p = a + (b << bs_log);
  double r = 0.0;
  if (bs >= 2) {
    for (uint64_t j = 0; j < bs; j += 2) {
      const Amp2 v = ld2_ro(p + j);
      r += prob(v.a);
      r += prob(v.b);
    }
  } else {
    r += prob(p[0]);
  }
  bsum[b] = r;
}

// Exclusive scan, three kernels: per-segment totals, a one-block scan of the
// totals, per-segment scan with the offset.  Segment = kThreads * kScanPer.
constexpr int kScanPer = 16;
constexpr uint64_t kScanSeg = (uint64_t)kThreads * kScanPer;

__device__ __forceinline__ double block_excl_scan(double v, double* sh, double* total) {
  // inclusive warp scan, then warp totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  double ex = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) ex = 0.0;
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const double t = sh[w];
      sh[w] = run;
      run += t;
    }
    sh[kThreads / 32] = run;
  }
  __syncthreads();
  const double excl = sh[warp] + ex;
  *total = sh[kThreads / 32];
  __syncthreads();
  return excl;
}

__global__ void __launch_bounds__(kThreads)
    k_seg_totals(const double* __restrict__ in, uint64_t count, double* __restrict__ seg) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanSeg + (uint64_t)threadIdx.x * kScanPer;
  double s = 0;
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < count) s += in[base + k];
  __shared__ double sh[kThreads / 32 + 1];
  double tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) seg[blockIdx.x] = tot;
}

// one block: exclusive scan of nseg totals in place (sequential per thread)
__global__ void __launch_bounds__(kThreads)
    k_scan_totals(double* __restrict__ seg, uint64_t nseg) {
  const uint64_t per = (nseg + kThreads - 1) / kThreads;
  const uint64_t lo = (uint64_t)threadIdx.x * per;
  double s = 0;
  for (uint64_t k = 0; k < per; ++k)
    if (lo + k < nseg) s += seg[lo + k];
  __shared__ double sh[kThreads / 32 + 1];
  double tot;
  double run = block_excl_scan(s, sh, &tot);
  for (uint64_t k = 0; k < per; ++k)
    if (lo + k < nseg) {
      const double t = seg[lo + k];
      seg[lo + k] = run;
      run += t;
    }
}

__global__ void __launch_bounds__(kThreads)
    k_seg_scan(const double* __restrict__ in, uint64_t count, const double* __restrict__ seg,
               double* __restrict__ out) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanSeg + (uint64_t)threadIdx.x * kScanPer;
  double s = 0;
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < count) s += in[base + k];
  __shared__ double sh[kThreads / 32 + 1];
  double tot;
  double run = seg[blockIdx.x] + block_excl_scan(s, sh, &tot);
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < count) {
      const double t = in[base + k];
      out[base + k] = run;
      run += t;
    }
}

// one thread per draw: v = u * total; first index j with cum(j) > v
// (np.searchsorted(cumulative, v, side="right"), state.py:104-106)
__global__ void __launch_bounds__(kThreads)
    k_search(const double2* __restrict__ a, int bs_log, uint64_t nblocks,
             const double* __restrict__ P, const double* __restrict__ bsum,
             const double* __restrict__ u, int count, uint64_t* __restrict__ out) {
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= count) return;
  const double total = P[nblocks - 1] + bsum[nblocks - 1];
  const double v = u[i] * total;
  // largest b with P[b] <= v  (P[0] = 0 <= v)
  uint64_t lo = 0, hi = nblocks;  // invariant: P[lo] <= v, answer in [lo, hi)
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (P[mid] <= v) lo = mid;
    else hi = mid;
  }
  const uint64_t bs = 1ULL << bs_log;
  const uint64_t dim = nblocks << bs_log;
  uint64_t found = dim - 1;
  for (uint64_t b = lo; b < nblocks; ++b) {
    const double2* p = a + (b << bs_log);
    double r = 0.0;
    bool hit = false;
    for (uint64_t j = 0; j < bs; ++j) {
      r += prob(p[j]);
      if (P[b] + r > v) {
        found = (b << bs_log) + j;
        hit = true;
        break;
      }
    }
    if (hit) break;
  }
  out[i] = found;
}

// ------------------------------------------------------- elementwise / kron
__global__ void __launch_bounds__(kThreads)
    k_mul_elementwise(double2* __restrict__ a, const double2* __restrict__ f, uint64_t units) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t u = (uint64_t)blockIdx.x * kThreads + threadIdx.x; u < units; u += stride) {
    const uint64_t x = u << 1;
    Amp2 v = ld2(a + x);
    const Amp2 c = ld2_ro(f + x);
    v.a = cmul(v.a, c.a);
    v.b = cmul(v.b, c.b);
    st2(a + x, v);
  }
}

// out[(s << n1) | f] = second[s] * first[f]   (np.kron(second, first))
__global__ void __launch_bounds__(kThreads)
    k_kron(const double2* __restrict__ first, int n1, const double2* __restrict__ second,
           double2* __restrict__ out, uint64_t dim) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t fmask = (1ULL << n1) - 1;
  for (uint64_t x = (uint64_t)blockIdx.x * kThreads + threadIdx.x; x < dim; x += stride)
    st1(out + x, cmul(__ldg(second + (x >> n1)), __ldg(first + (x & fmask))));
}

struct QubitOrder {
  int n;
  int8_t src[64];  // output bit i <- input bit src[i]
};

// out[d] = in[s], bit order[i] of s = bit i of d (state.py:150-163)
__global__ void __launch_bounds__(kThreads)
    k_permute(const double2* __restrict__ in, double2* __restrict__ out, QubitOrder ord,
              uint64_t dim) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t d = (uint64_t)blockIdx.x * kThreads + threadIdx.x; d < dim; d += stride) {
    uint64_t s = 0;
    for (int i = 0; i < ord.n; ++i) s |= ((d >> i) & 1ULL) << ord.src[i];
    st1(out + d, __ldg(in + s));
  }
}

// out[k] = in[widen(k)]: projected qubits fixed to their values (state.py:166-192)
__global__ void __launch_bounds__(kThreads)
    k_gather_dep(const double2* __restrict__ in, double2* __restrict__ out, Deposit dp,
                 uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k < count; k += stride)
    st1(out + k, __ldg(in + deposit(k, dp)));
}

__global__ void __launch_bounds__(kThreads)
    k_gather_fixed(const double2* __restrict__ in, double2* __restrict__ out, FixedBits fb,
                   uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k < count; k += stride)
    st1(out + k, __ldg(in + widen(k, fb)));
}


int launch_marginal(const double2* a, int n, uint64_t mask, uint64_t value, double* partials,
                    double* dev_out, cudaStream_t s) {
  int pos[64];
  int k = 0;
  for (int q = 0; q < n; ++q)
    if ((mask >> q) & 1ULL) pos[k++] = q;
  const uint64_t units = 1ULL << (n - k);
  const unsigned grid = (unsigned)std::min<uint64_t>(kRedBlocks, std::max<uint64_t>(
                                                          1, (units + kThreads - 1) / kThreads));
  if (k > kMaxFixed) {  // few matching amplitudes: deposit the free bits
    k_marginal_dep<<<grid, kThreads, 0, s>>>(a, make_deposit(n, mask, value), units, partials);
  } else {
    FixedBits fb = make_fixed(pos, k, value & mask);
    k_marginal<<<grid, kThreads, 0, s>>>(a, fb, units, partials);
  }
  QSV_CHECK_LAUNCH("k_marginal");
  k_sum_partials<<<1, kThreads, 0, s>>>(partials, (int)grid, dev_out);
  QSV_CHECK_LAUNCH("k_sum_partials");
  return QSV_OK;
}

// scratch: 2 * nblocks + nseg doubles; u/out on the device
int launch_sampling(const double2* a, int n, const double* dev_u, int count, double* scratch,
                    uint64_t* dev_out, cudaStream_t s) {
  const int bs_log = std::min(kSampleBlockLog, n);
  const uint64_t nblocks = 1ULL << (n - bs_log);
  double* bsum = scratch;
  double* P = scratch + nblocks;
  double* seg = P + nblocks;
  const uint64_t nseg = (nblocks + kScanSeg - 1) / kScanSeg;
  k_block_sums<<<grid_for(nblocks, 1), kThreads, 0, s>>>(a, bs_log, nblocks, bsum);
  QSV_CHECK_LAUNCH("k_block_sums");
  k_seg_totals<<<(unsigned)nseg, kThreads, 0, s>>>(bsum, nblocks, seg);
  QSV_CHECK_LAUNCH("k_seg_totals");
  k_scan_totals<<<1, kThreads, 0, s>>>(seg, nseg);
  QSV_CHECK_LAUNCH("k_scan_totals");
  k_seg_scan<<<(unsigned)nseg, kThreads, 0, s>>>(bsum, nblocks, seg, P);
  QSV_CHECK_LAUNCH("k_seg_scan");
  if (count > 0) {
    k_search<<<grid_for((uint64_t)count, 1), kThreads, 0, s>>>(a, bs_log, nblocks, P, bsum,
                                                               dev_u, count, dev_out);
    QSV_CHECK_LAUNCH("k_search");
  }
  return QSV_OK;
}

size_t sampling_scratch_doubles(int n) {
  const int bs_log = std::min(kSampleBlockLog, n);
  const uint64_t nblocks = 1ULL << (n - bs_log);
  return 2 * nblocks + (nblocks + kScanSeg - 1) / kScanSeg + 1;
}

int launch_mul_elementwise(double2* a, const double2* f, uint64_t dim, cudaStream_t s) {
  const uint64_t units = dim / 2;
  k_mul_elementwise<<<stream_grid(units), kThreads, 0, s>>>(a, f, units);
  QSV_CHECK_LAUNCH("k_mul_elementwise");
  return QSV_OK;
}

int launch_kron(const double2* first, int n1, const double2* second, int n2, double2* out,
                cudaStream_t s) {
  const uint64_t dim = 1ULL << (n1 + n2);
  k_kron<<<stream_grid(dim), kThreads, 0, s>>>(first, n1, second, out, dim);
  QSV_CHECK_LAUNCH("k_kron");
  return QSV_OK;
}

int launch_permute(const double2* in, double2* out, int n, const int* order, cudaStream_t s) {
  QubitOrder o;
  o.n = n;
  for (int i = 0; i < n; ++i) o.src[i] = (int8_t)order[i];
  const uint64_t dim = 1ULL << n;
  k_permute<<<stream_grid(dim), kThreads, 0, s>>>(in, out, o, dim);
  QSV_CHECK_LAUNCH("k_permute");
  return QSV_OK;
}

int launch_drop(const double2* in, int n, const int* targets, const int* values, int k,
                double2* out, cudaStream_t s) {
  std::vector<std::pair<int, int>> tv;
  for (int i = 0; i < k; ++i) tv.push_back({targets[i], values[i]});
  std::sort(tv.begin(), tv.end());
  uint64_t mask = 0, val = 0;
  for (int i = 0; i < k; ++i) {
    mask |= 1ULL << tv[i].first;
    if (tv[i].second) val |= 1ULL << tv[i].first;
  }
  const uint64_t count = 1ULL << (n - k);
  if (k > kMaxFixed) {
    k_gather_dep<<<stream_grid(count), kThreads, 0, s>>>(in, out, make_deposit(n, mask, val),
                                                         count);
  } else {
    int pos[kMaxFixed];
    for (int i = 0; i < k; ++i) pos[i] = tv[i].first;
    FixedBits fb = make_fixed(pos, k, val);
    k_gather_fixed<<<stream_grid(count), kThreads, 0, s>>>(in, out, fb, count);
  }
  QSV_CHECK_LAUNCH("k_gather");
  return QSV_OK;
}

}  // namespace qsv
