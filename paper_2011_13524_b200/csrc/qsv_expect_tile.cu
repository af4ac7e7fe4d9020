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
constexpr int kXMaxTerms = 44;                          // terms per pass
constexpr int kXWarps = kXThreads / 32;
constexpr int kXTileAmps = 1 << kXTileQubits;

struct XGroup {
  uint32_t xl;     // flip mask over the tile's local bits
  int32_t first;   // first term of the group
  int32_t count;
  int32_t hb;      // pairing bit (highest bit of xl; -1 for xl == 0)
};

struct XTerm {
  uint32_t zl;     // sign mask over local bits
  uint32_t zk;     // its k part: bits 8..11 of zl (sign (-1)^popc(k & zk) over slot k)
  uint64_t zg;     // sign mask over the other (tile-constant) bits
  uint32_t imag;   // parity(xl & zl): the pair sums are imaginary (and carry a - sign)
  uint32_t pad;
};

struct XPass {
  int32_t ngroups, nterms;
  int32_t spos[kXTileQubits];  // local bit j -> qubit
  XGroup groups[kXMaxTerms];
  XTerm terms[kXMaxTerms];
};

// dynamic shared memory: two tile buffers (the next tile streams in with
// cp.async while this one is evaluated) + one accumulator per (term, thread);
// a term's sum is purely real or purely imaginary (XTerm::imag), one double
constexpr size_t kXSmemBytes =
    2 * sizeof(double2) * kXTileAmps + sizeof(double) * kXMaxTerms * kXThreads;
static_assert(kXSmemBytes + sizeof(XPass) + 1024 <= 232448, "expectation tile smem");

// sum_k (-1)^popc(k & z) x[k] over 16 slots: four uniform-branch folds,
// 15 additions of depth 4
__device__ __forceinline__ double fold16(const double (&x)[16], uint32_t z) {
  double a[8], b[4], c[2];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (z & 8) ? x[k] - x[k + 8] : x[k] + x[k + 8];
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = (z & 4) ? a[k] - a[k + 4] : a[k] + a[k + 4];
#pragma unroll
  for (int k = 0; k < 2; ++k) c[k] = (z & 2) ? b[k] - b[k + 2] : b[k] + b[k + 2];
  return (z & 1) ? c[0] - c[1] : c[0] + c[1];
}

// in-place 16-point Walsh-Hadamard transform: x[z] = sum_k (-1)^popc(k & z) x[k]
__device__ __forceinline__ void wht16(double (&x)[16]) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1)
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (!(k & h)) {
        const double u = x[k], w = x[k + h];
        x[k] = u + w;
        x[k + h] = u - w;
      }
}

__device__ __forceinline__ double pick16(const double (&x)[16], uint32_t z) {
  switch (z & 15u) {
    case 0: return x[0];
    case 1: return x[1];
    case 2: return x[2];
    case 3: return x[3];
    case 4: return x[4];
    case 5: return x[5];
    case 6: return x[6];
    case 7: return x[7];
    case 8: return x[8];
    case 9: return x[9];
    case 10: return x[10];
    case 11: return x[11];
    case 12: return x[12];
    case 13: return x[13];
    case 14: return x[14];
    default: return x[15];
  }
}

__device__ __forceinline__ void x_cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void x_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void x_cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// products p = conj(psi_x) psi_{x ^ xl} of the 8 slots k whose bit J equals b
// (b is per thread; selects instead of branches), zero in the other 8
template <int J>
__device__ __forceinline__ void pair_products(const double2 (&v)[kXPer], const double2* sm,
                                              int tid, uint32_t xl, uint32_t b,
                                              double (&re)[kXPer], double (&im)[kXPer]) {
#pragma unroll
  for (int i = 0; i < kXPer / 2; ++i) {
    const int k0 = ((i >> J) << (J + 1)) | (i & ((1 << J) - 1));
    const int k1 = k0 | (1 << J);
    const double2 x = b ? v[k1] : v[k0];
    const uint32_t k = b ? (uint32_t)k1 : (uint32_t)k0;
    const double2 w = sm[(k * kXThreads + (uint32_t)tid) ^ xl];
    const double r = fma(x.x, w.x, x.y * w.y);
    const double m = fma(x.x, w.y, -x.y * w.x);
    re[k0] = b ? 0.0 : r;
    re[k1] = b ? r : 0.0;
    im[k0] = b ? 0.0 : m;
    im[k1] = b ? m : 0.0;
  }
}

// S_t = sum_x conj(psi_x) psi_{x ^ xl} (-1)^popc((x ^ xl) & zl) over the tile,
// accumulated per thread across all of the CTA's tiles (one shared-memory
// read-modify-write per term and tile instead of a warp reduction), reduced
// once at the end.  For xl != 0 the pairs x, x ^ xl contribute
// sigma(x ^ xl) (p + c conj p) with p = conj(psi_x) psi_{x ^ xl} and
// c = (-1)^popc(xl & zl): 2 Re p or 2i Im p, so only the half of the tile with
// bit hb = 0 is visited and only the needed part of p is formed.
__global__ void __launch_bounds__(kXThreads, 1)
    k_expect_tile(const double2* __restrict__ a, const XPass* __restrict__ gp, FixedBits tb,
                  uint64_t ntiles, double* __restrict__ partials) {
  extern __shared__ double2 xdyn[];
  double* acc = reinterpret_cast<double*>(xdyn + 2 * kXTileAmps);  // [term][thread]
  __shared__ XPass P;
  __shared__ uint64_t s_hi[kXPer];
  __shared__ double s_red[kXWarps];
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
  for (int t = 0; t < P.nterms; ++t) acc[t * kXThreads + tid] = 0.0;
  uint64_t lo = 0;
  for (int b = 0; b < 8; ++b)
    if ((tid >> b) & 1) lo |= 1ULL << P.spos[b];
  // thread part of every term's sign, tile-invariant
  uint64_t tsg = 0;
  for (int t = 0; t < P.nterms; ++t)
    tsg |= (uint64_t)(__popc((uint32_t)tid & P.terms[t].zl & 0xffu) & 1) << t;
  __syncthreads();

  auto issue = [&](uint64_t tile, int buf) {
    const uint64_t base = widen(tile, tb);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(xdyn + buf * kXTileAmps);
#pragma unroll
    for (int k = 0; k < kXPer; ++k)
      x_cp_async16(sb + (uint32_t)(k * kXThreads + tid) * 16u, a + (base | lo | s_hi[k]));
    x_cp_commit();
  };
  uint64_t tile = blockIdx.x;
  int buf = 0;
  if (tile < ntiles) issue(tile, 0);
  for (; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const uint64_t next = tile + gridDim.x;
    if (next < ntiles) {
      issue(next, buf ^ 1);
      x_cp_wait<1>();
    } else {
      x_cp_wait<0>();
    }
    __syncthreads();
    const double2* sm = xdyn + buf * kXTileAmps;
    const uint64_t base = widen(tile, tb);
    double2 v[kXPer];
#pragma unroll
    for (int k = 0; k < kXPer; ++k) v[k] = sm[k * kXThreads + tid];
    for (int g = 0; g < P.ngroups; ++g) {
      const XGroup G = P.groups[g];
      const int t1 = G.first + G.count;
      double re[kXPer], im[kXPer];
      double f = 1.0;
      if (G.xl == 0) {
#pragma unroll
        for (int k = 0; k < kXPer; ++k) {
          re[k] = fma(v[k].x, v[k].x, v[k].y * v[k].y);
          im[k] = 0.0;
        }
      } else {
        // every thread visits 8 of its 16 slots, so no lane or warp idles:
        // a pairing bit on the slots (hb >= 8) is visited from its 0 side; a
        // pairing bit on the thread bits (then the slot part of xl is 0) is
        // visited by the bit-0 thread on slots 0..7 and by the bit-1 thread
        // on slots 8..15 (each pair once; the summand is symmetric in which
        // end visits it)
        f = 2.0;
        const uint32_t b = G.hb >= 8 ? 0u : ((uint32_t)tid >> G.hb) & 1u;
        switch (G.hb >= 8 ? G.hb - 8 : 3) {
          case 0: pair_products<0>(v, sm, tid, G.xl, b, re, im); break;
          case 1: pair_products<1>(v, sm, tid, G.xl, b, re, im); break;
          case 2: pair_products<2>(v, sm, tid, G.xl, b, re, im); break;
          default: pair_products<3>(v, sm, tid, G.xl, b, re, im); break;
        }
      }
      // a slot sign pattern (-1)^popc(k & zk) is one Walsh-Hadamard
      // coefficient: groups with many terms transform once and pick, small
      // groups fold per term
      const bool many = G.count >= 4;
      if (many) {
        wht16(re);
        if (G.xl) wht16(im);
      }
      for (int t = G.first; t < t1; ++t) {
        const XTerm T = P.terms[t];
        const uint32_t neg = (uint32_t)((__popcll(base & T.zg) ^ (tsg >> t) ^ T.imag) & 1);
        double val;
        if (many) val = T.imag ? pick16(im, T.zk) : pick16(re, T.zk);
        else val = T.imag ? fold16(im, T.zk) : fold16(re, T.zk);
        acc[t * kXThreads + tid] = fma(neg ? -f : f, val, acc[t * kXThreads + tid]);
      }
    }
    __syncthreads();  // this buffer is refilled by the prefetch two tiles on
  }
  // per term: fixed-order block sum of the per-thread accumulators
  for (int t = 0; t < P.nterms; ++t) {
    double s = acc[t * kXThreads + tid];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_red[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double r = 0.0;
      for (int w = 0; w < kXWarps; ++w) r += s_red[w];
      const bool imag = P.terms[t].imag;
      partials[((size_t)blockIdx.x * kXMaxTerms + t) * 2 + 0] = imag ? 0.0 : r;
      partials[((size_t)blockIdx.x * kXMaxTerms + t) * 2 + 1] = imag ? r : 0.0;
    }
    __syncthreads();
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
int launch_expect_tile_final(const double* partials, int nblocks, int nterms, double* out,
                             cudaStream_t s) {
  k_expect_tile_final<<<nterms, kXThreads, 0, s>>>(partials, nblocks, out);
  QSV_CHECK_LAUNCH("k_expect_tile_final");
  return QSV_OK;
}

void expect_generic_pass_done();
int expect_tile_jit(const double2* a, int n, const std::vector<uint64_t>& xms,
                    const std::vector<uint64_t>& zms, void* scratch, std::vector<double>& res,
                    cudaStream_t s);

struct XTermIn {
  uint64_t xm, zm;
  int index;  // caller's term index
};

// Pack terms into passes: each pass is a tile set of 12 qubits (0..3 plus
// flip qubits) and at most kXMaxTerms terms; a flip mask with more terms is
// split into chunks.  Returns false if some flip mask does not fit a tile
// (the caller then uses the sweep kernels).
static bool pack_passes(int n, const std::vector<XTermIn>& terms,
                        std::vector<std::pair<uint64_t, std::vector<int>>>& passes) {
  if (n < kXTileQubits) return false;
  const uint64_t low = 0xFULL;
  // units: (flip mask, up to kXMaxTerms of its terms), masks in first-appearance order
  std::vector<uint64_t> masks;
  for (const XTermIn& t : terms)
    if (std::find(masks.begin(), masks.end(), t.xm) == masks.end()) masks.push_back(t.xm);
  std::vector<std::pair<uint64_t, std::vector<int>>> units;
  for (uint64_t m : masks) {
    if (__builtin_popcountll(m | low) > kXTileQubits) return false;
    std::vector<int> chunk;
    for (size_t k = 0; k < terms.size(); ++k) {
      if (terms[k].xm != m) continue;
      chunk.push_back((int)k);
      if ((int)chunk.size() == kXMaxTerms) {
        units.push_back({m, chunk});
        chunk.clear();
      }
    }
    if (!chunk.empty()) units.push_back({m, chunk});
  }
  std::vector<char> done(units.size(), 0);
  size_t left = units.size();
  while (left) {
    uint64_t S = low;
    std::vector<int> members;
    int nterms = 0;
    for (size_t i = 0; i < units.size(); ++i) {
      if (done[i]) continue;
      if (__builtin_popcountll(S | units[i].first) > kXTileQubits) continue;
      const int cnt = (int)units[i].second.size();
      if (nterms + cnt > kXMaxTerms) continue;
      S |= units[i].first;
      nterms += cnt;
      done[i] = 1;
      --left;
      members.insert(members.end(), units[i].second.begin(), units[i].second.end());
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

size_t expect_jit_scratch_bytes();  // qsv_expect_jit.cu (generated passes' layout)

size_t expect_tile_scratch_bytes() {
  const size_t generic = ((sizeof(XPass) * kXBatch + 255) / 256) * 256 +
                         sizeof(double) * (2 * (size_t)296 * kXMaxTerms + 2 * kXMaxTerms * kXBatch);
  return std::max(generic, expect_jit_scratch_bytes());
}

int expect_tile(const double2* a, int n, const std::vector<uint64_t>& xms,
                const std::vector<uint64_t>& zms, void* scratch, std::vector<double>& res,
                cudaStream_t s) {
  {  // generated pass kernels when compiled for this observable (qsv_expect_jit.cu)
    const int rc = expect_tile_jit(a, n, xms, zms, scratch, res, s);
    if (rc != QSV_EUNSUPPORTED) return rc;
  }
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
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)std::min(num_sms, 296));
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
      G.xl = 0;
      for (int q = 0; q < n; ++q)
        if ((m >> q) & 1ULL) G.xl |= 1u << local_of[q];
      G.hb = G.xl ? 31 - __builtin_clz(G.xl) : -1;
      for (int k : ps.second)
        if (terms[k].xm == m) {
          XTerm T;
          memset(&T, 0, sizeof(T));
          for (int q = 0; q < n; ++q)
            if ((terms[k].zm >> q) & 1ULL) {
              if (local_of[q] >= 0) T.zl |= 1u << local_of[q];
              else T.zg |= 1ULL << q;
            }
          // parity((x ^ xl) & zl) = parity(tid & zl & 0xff) ^ parity(k & zk)
          //                          ^ parity(xl & zl)
          T.zk = (T.zl >> 8) & 0xFu;
          T.imag = (uint32_t)(__builtin_popcount(G.xl & T.zl) & 1);
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
    const size_t smem = kXSmemBytes;
    static uint64_t attr_done = 0;
    QSV_TRY(ensure_smem_attr(k_expect_tile, (int)smem, attr_done));
    k_expect_tile<<<grid, kXThreads, smem, s>>>(a, dpass, tb, ntiles, partials);
    QSV_CHECK_LAUNCH("k_expect_tile");
    k_expect_tile_final<<<P.nterms, kXThreads, 0, s>>>(partials, (int)grid, dout);
    QSV_CHECK_LAUNCH("k_expect_tile_final");
    expect_generic_pass_done();
    orders.push_back(order);
  }
  return drain();
}

}  // namespace qsv
