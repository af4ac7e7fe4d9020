// Pauli-sum expectation values in tile passes: many X/Y flip masks per HBM
// read of the state.
//
// The reference evaluates sum_t c_t <psi|P_t|psi> term by term, each term a
// full copy (pauli_action) plus a zdotc (observable.py:99-104).  The sweep
// kernels of qsv_reduce.cu already read the state once per distinct flip
// mask; a Hamiltonian such as the transverse-field Ising model (one X_i per
// qubit) still needs n + 1 sweeps.  Here a pass fixes a set S of 12 tile
// qubits (qubits 0..3 plus the flip qubits of as many masks as fit); a CTA
// loads a 2^12-amplitude tile into shared memory and evaluates every term
// whose flip mask lies in S, so TFIM at n = 24 takes 3 reads instead of 25.
//
//   S_t = sum_x conj(psi_x) psi_{x ^ xm_t} (-1)^popc((x ^ xm_t) & zm_t)
// (the host multiplies by coef_t * i^ny_t, as for the sweeps).  Terms that
// share a flip mask share the products conj(psi_x) psi_{x ^ xm}, which each
// thread keeps in registers while it adds them with the terms' signs.
// Reductions are warp shuffles, then per-warp shared slots, then a fixed-order
// block and grid sum: results are bit-reproducible run to run.
#include <algorithm>
#include <cstring>
#include <vector>

#include "qsv_internal.cuh"

namespace qsv {

constexpr int kXTileQubits = 12;
constexpr int kXThreads = 256;
constexpr int kXPer = (1 << kXTileQubits) / kXThreads;  // amplitudes per thread (16)
constexpr int kXMaxTerms = 64;                          // terms per pass
constexpr int kXWarps = kXThreads / 32;

struct XGroup {
  uint32_t xl;     // flip mask over the tile's local bits
  int32_t first;   // first term of the group
  int32_t count;
  int32_t pad;
};

struct XTerm {
  uint32_t zl;     // sign mask over local bits
  uint32_t kmask;  // bit k: parity of ((k * 256) ^ xl) & zl over the k-indexed local bits
                   // (bits 8..11) and of the flip mask's low bits: the per-amplitude
                   // sign is bit k of kmask ^ parity(tid & zl_lo & ~...) (see kernel)
  uint64_t zg;     // sign mask over the other (tile-constant) bits
};

struct XPass {
  int32_t ngroups, nterms;
  int32_t spos[kXTileQubits];  // local bit j -> qubit
  XGroup groups[kXMaxTerms];
  XTerm terms[kXMaxTerms];
};

__global__ void __launch_bounds__(kXThreads, 2)
    k_expect_tile(const double2* __restrict__ a, const XPass* __restrict__ gp, FixedBits tb,
                  uint64_t ntiles, double* __restrict__ partials) {
  extern __shared__ double2 sm[];  // 2^12 amplitudes (64 KiB, dynamic)
  __shared__ XPass P;
  __shared__ uint64_t s_hi[kXPer];
  __shared__ double2 s_acc[kXWarps][kXMaxTerms];
  {
    const int* src = reinterpret_cast<const int*>(gp);
    int* dst = reinterpret_cast<int*>(&P);
    for (int i = threadIdx.x; i < (int)(sizeof(XPass) / 4); i += kXThreads) dst[i] = src[i];
  }
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kXPer) {
    uint64_t h = 0;
    for (int b = 0; b < 4; ++b)
      if ((tid >> b) & 1) h |= 1ULL << P.spos[8 + b];
    s_hi[tid] = h;
  }
  for (int i = tid; i < kXWarps * kXMaxTerms; i += kXThreads)
    s_acc[i / kXMaxTerms][i % kXMaxTerms] = make_double2(0.0, 0.0);
  uint64_t lo = 0;
  for (int b = 0; b < 8; ++b)
    if ((tid >> b) & 1) lo |= 1ULL << P.spos[b];
  __syncthreads();

  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = widen(tile, tb);
#pragma unroll
    for (int k = 0; k < kXPer; ++k) sm[k * kXThreads + tid] = ld1(a + (base | lo | s_hi[k]));
    __syncthreads();
    double2 v[kXPer];  // this thread's amplitudes, shared by every group
#pragma unroll
    for (int k = 0; k < kXPer; ++k) v[k] = sm[k * kXThreads + tid];
    for (int g = 0; g < P.ngroups; ++g) {
      const uint32_t xl = P.groups[g].xl;
      double2 p[kXPer];
#pragma unroll
      for (int k = 0; k < kXPer; ++k) {
        const double2 w = xl ? sm[(uint32_t)(k * kXThreads + tid) ^ xl] : v[k];
        p[k] = make_double2(fma(v[k].x, w.x, v[k].y * w.y), fma(v[k].x, w.y, -v[k].y * w.x));
      }
      const int t1 = P.groups[g].first + P.groups[g].count;
      for (int t = P.groups[g].first; t < t1; ++t) {
        const XTerm T = P.terms[t];
        // sign of x ^ xl for x = k * 256 + tid: tile part, thread part, k part
        const uint32_t tpar =
            (uint32_t)((__popcll(base & T.zg) ^ __popc((uint32_t)tid & T.zl & 0xffu)) & 1);
        const uint32_t M = T.kmask ^ (0u - tpar);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < kXPer; ++k) {
          const bool neg = (M >> k) & 1u;
          acc.x += neg ? -p[k].x : p[k].x;
          acc.y += neg ? -p[k].y : p[k].y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        if (lane == 0) {
          s_acc[warp][t].x += acc.x;
          s_acc[warp][t].y += acc.y;
        }
      }
    }
    __syncthreads();  // the tile buffer is refilled next iteration
  }
  if (tid < P.nterms) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < kXWarps; ++w) {
      s.x += s_acc[w][tid].x;
      s.y += s_acc[w][tid].y;
    }
    partials[((size_t)blockIdx.x * kXMaxTerms + tid) * 2 + 0] = s.x;
    partials[((size_t)blockIdx.x * kXMaxTerms + tid) * 2 + 1] = s.y;
  }
}

// out[t] = sum over blocks of partials[block][t] (fixed order, one block per term)
__global__ void __launch_bounds__(kXThreads)
    k_expect_tile_final(const double* __restrict__ partials, int nblocks, double* __restrict__ out) {
  __shared__ double sre[kXThreads], sim[kXThreads];
  const int t = blockIdx.x;
  double re = 0, im = 0;
  for (int b = threadIdx.x; b < nblocks; b += kXThreads) {
    re += partials[((size_t)b * kXMaxTerms + t) * 2 + 0];
    im += partials[((size_t)b * kXMaxTerms + t) * 2 + 1];
  }
  sre[threadIdx.x] = re;
  sim[threadIdx.x] = im;
  __syncthreads();
  for (int o = kXThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sre[threadIdx.x] += sre[threadIdx.x + o];
      sim[threadIdx.x] += sim[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * t] = sre[0];
    out[2 * t + 1] = sim[0];
  }
}

// --------------------------------------------------------------- host side
struct XTermIn {
  uint64_t xm, zm;
  int index;  // caller's term index
};

// Pack terms into passes: each pass is a tile set of 12 qubits (0..3 plus
// flip qubits) and at most kXMaxTerms terms.  Returns false if some flip mask
// does not fit a tile (the caller then uses the sweep kernels).
static bool pack_passes(int n, const std::vector<XTermIn>& terms,
                        std::vector<std::pair<uint64_t, std::vector<int>>>& passes) {
  if (n < kXTileQubits) return false;
  const uint64_t low = 0xFULL;
  // distinct flip masks in first-appearance order
  std::vector<uint64_t> masks;
  for (const XTermIn& t : terms)
    if (std::find(masks.begin(), masks.end(), t.xm) == masks.end()) masks.push_back(t.xm);
  for (uint64_t m : masks)
    if (__builtin_popcountll(m | low) > kXTileQubits) return false;
  std::vector<char> done(masks.size(), 0);
  size_t left = masks.size();
  while (left) {
    uint64_t S = low;
    std::vector<int> members;
    int nterms = 0;
    for (size_t i = 0; i < masks.size(); ++i) {
      if (done[i]) continue;
      if (__builtin_popcountll(S | masks[i]) > kXTileQubits) continue;
      int cnt = 0;
      for (const XTermIn& t : terms) cnt += t.xm == masks[i];
      if (nterms + cnt > kXMaxTerms && nterms > 0) continue;
      if (cnt > kXMaxTerms) return false;
      S |= masks[i];
      nterms += cnt;
      done[i] = 1;
      --left;
      for (size_t k = 0; k < terms.size(); ++k)
        if (terms[k].xm == masks[i]) members.push_back((int)k);
    }
    // pad S with the lowest unused qubits
    for (int q = 0; q < n && __builtin_popcountll(S) < kXTileQubits; ++q) S |= 1ULL << q;
    passes.push_back({S, members});
  }
  return true;
}

// Evaluate S_t for every term (bra == ket); results (re, im) per caller index
// land in res[2 * index].  Returns QSV_EUNSUPPORTED when the masks do not
// fit tiles.  scratch must hold sizeof(XPass) + 2 * grid * kXMaxTerms doubles
// + 2 * kXMaxTerms doubles.
constexpr int kXBatch = 32;  // passes launched back to back before one synchronisation

size_t expect_tile_scratch_bytes() {
  return ((sizeof(XPass) * kXBatch + 255) / 256) * 256 +
         sizeof(double) * (2 * (size_t)296 * kXMaxTerms + 2 * kXMaxTerms * kXBatch);
}

int expect_tile(const double2* a, int n, const std::vector<uint64_t>& xms,
                const std::vector<uint64_t>& zms, void* scratch, std::vector<double>& res,
                cudaStream_t s) {
  std::vector<XTermIn> terms;
  for (size_t i = 0; i < xms.size(); ++i) terms.push_back({xms[i], zms[i], (int)i});
  std::vector<std::pair<uint64_t, std::vector<int>>> passes;
  if (!pack_passes(n, terms, passes)) return QSV_EUNSUPPORTED;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  const uint64_t ntiles = 1ULL << (n - kXTileQubits);
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)std::min(num_sms * 2, 296));
  char* base = reinterpret_cast<char*>(scratch);
  XPass* dpass0 = reinterpret_cast<XPass*>(base);
  double* partials = reinterpret_cast<double*>(base + ((sizeof(XPass) * kXBatch + 255) / 256) * 256);
  double* dout0 = partials + 2 * (size_t)296 * kXMaxTerms;
  res.assign(2 * xms.size(), 0.0);
  // passes run back to back (stream order protects the shared partials);
  // results come back with one copy and one synchronisation per batch
  std::vector<std::vector<int>> orders;
  std::vector<double> hout;
  auto drain = [&]() -> int {
    if (orders.empty()) return QSV_OK;
    hout.resize(2 * kXMaxTerms * orders.size());
    QSV_TRY(cudaMemcpyAsync(hout.data(), dout0, hout.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    QSV_TRY(cudaStreamSynchronize(s));
    for (size_t b = 0; b < orders.size(); ++b)
      for (size_t k = 0; k < orders[b].size(); ++k) {
        res[2 * terms[orders[b][k]].index] = hout[2 * kXMaxTerms * b + 2 * k];
        res[2 * terms[orders[b][k]].index + 1] = hout[2 * kXMaxTerms * b + 2 * k + 1];
      }
    orders.clear();
    return QSV_OK;
  };
  for (auto& ps : passes) {
    if ((int)orders.size() == kXBatch) {
      const int rc = drain();
      if (rc) return rc;
    }
    XPass* dpass = dpass0 + orders.size();
    double* dout = dout0 + 2 * kXMaxTerms * orders.size();
    XPass P;
    memset(&P, 0, sizeof(P));
    const uint64_t S = ps.first;
    int local_of[64];
    for (int q = 0; q < 64; ++q) local_of[q] = -1;
    int j = 0;
    for (int q = 0; q < n; ++q)
      if ((S >> q) & 1ULL) {
        P.spos[j] = q;
        local_of[q] = j++;
      }
    // groups of terms with the same flip mask, in member order
    std::vector<int> order;
    std::vector<uint64_t> gm;
    for (int k : ps.second)
      if (std::find(gm.begin(), gm.end(), terms[k].xm) == gm.end()) gm.push_back(terms[k].xm);
    for (uint64_t m : gm) {
      XGroup G;
      G.first = (int32_t)order.size();
      G.count = 0;
      G.pad = 0;
      G.xl = 0;
      for (int q = 0; q < n; ++q)
        if ((m >> q) & 1ULL) G.xl |= 1u << local_of[q];
      for (int k : ps.second)
        if (terms[k].xm == m) {
          XTerm T;
          T.zl = 0;
          T.kmask = 0;
          T.zg = 0;
          for (int q = 0; q < n; ++q)
            if ((terms[k].zm >> q) & 1ULL) {
              if (local_of[q] >= 0) T.zl |= 1u << local_of[q];
              else T.zg |= 1ULL << q;
            }
          // parity((x ^ xl) & zl) = parity(tid & zl & 0xff) ^ parity((k << 8) & zl)
          //                          ^ parity(xl & zl)
          for (int kk = 0; kk < kXPer; ++kk)
            if ((__builtin_popcount(((uint32_t)kk << 8) & T.zl) ^
                 __builtin_popcount(G.xl & T.zl)) & 1)
              T.kmask |= 1u << kk;
          P.terms[order.size()] = T;
          order.push_back(k);
          ++G.count;
        }
      P.groups[P.ngroups++] = G;
    }
    P.nterms = (int32_t)order.size();
    QSV_TRY(cudaMemcpyAsync(dpass, &P, sizeof(P), cudaMemcpyHostToDevice, s));
    int pos[kXTileQubits];
    for (int b = 0; b < kXTileQubits; ++b) pos[b] = P.spos[b];
    FixedBits tb = make_fixed(pos, kXTileQubits, 0);
    const size_t smem = sizeof(double2) << kXTileQubits;
    static uint64_t attr_done = 0;
    QSV_TRY(ensure_smem_attr(k_expect_tile, (int)smem, attr_done));
    k_expect_tile<<<grid, kXThreads, smem, s>>>(a, dpass, tb, ntiles, partials);
    QSV_CHECK_LAUNCH("k_expect_tile");
    k_expect_tile_final<<<P.nterms, kXThreads, 0, s>>>(partials, (int)grid, dout);
    QSV_CHECK_LAUNCH("k_expect_tile_final");
    orders.push_back(order);
  }
  return drain();
}

}  // namespace qsv
