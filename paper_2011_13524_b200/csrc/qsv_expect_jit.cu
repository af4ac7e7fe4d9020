// Pauli-sum expectation passes as generated straight-line kernels.
//
// Same decomposition as k_expect_tile (qsv_expect_tile.cu): a pass fixes a
// set S of 12 tile qubits (qubits 0..3 plus flip qubits), a CTA streams
// 2^12-amplitude tiles through shared memory and evaluates every term whose
// flip mask lies in S.  The generic kernel reads the pass description from
// shared memory at run time, keeps one accumulator per (term, thread) in
// shared memory and picks slot signs through a 16-way switch; ncu shows it
// issue-bound on address / predicate work at 8 warps per SM
// (profiles/r1_expect_tile_n24.md).  Here the pass's structure -- which
// local bit every qubit sits on, each group's flip mask, each term's sign
// masks -- is compiled into the kernel:
//
//  * layout per pass: local bits 0..3 = qubits 0..3 (lanes read 256-byte
//    runs), then the pass's flip qubits on the register slot bits 8..11
//    first (a flip there pairs two registers of one thread: no data
//    movement), then on lane bit 4 and warp bits 5..7 (partner read from the
//    tile in shared memory);
//  * per group, only the product part its terms need (Re or Im of
//    conj(psi_x) psi_{x ^ xm}) on the half of the pairs that has the pairing
//    bit clear;
//  * a term's slot signs (-1)^popc(k & zk) are literal: a group with three
//    or more terms runs one in-place Walsh-Hadamard transform over its 8 / 16
//    products and reads each term's coefficient at a literal index, smaller
//    groups add with literal signs;
//  * thread-bit signs are one per-thread bit mask computed at kernel start,
//    tile-bit signs one POPC per term and tile (none when the term's Z mask
//    lies inside the tile);
//  * one register accumulator per term; a fixed-order block reduction at the
//    end, then the shared k_expect_tile_final (bit-reproducible).
//
// The source depends only on the observable's structure, so VQE iterations
// (same Hamiltonian, new state) reuse the compiled kernels; NVRTC and the
// caches are qsv_jit.cu's.  Reference: GeneralOperator._accumulate
// observable.py:99-104 (one P|psi> copy + zdotc per term).
#include <algorithm>
#include <cstring>
#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "qsv_internal.cuh"
#include "qsv_jit.cuh"

namespace qsv {

// shared with qsv_expect_tile.cu
constexpr int kEjTileQubits = 12;
constexpr int kEjThreads = 256;
constexpr int kEjMaxTermsStride = 44;  // partials stride (k_expect_tile_final)
constexpr int kEjLanes = 3;            // passes in flight at once (forked streams)
int launch_expect_tile_final(const double* partials, int nblocks, int nterms, double* out,
                             cudaStream_t s);

namespace ej {

constexpr int kEjMaxTerms = 40;  // terms per pass (one register accumulator each)

struct EjTerm {
  int index;      // caller's term index
  uint32_t zl;    // Z mask over local bits
  uint64_t zg;    // Z mask over the other qubits
  bool imag;      // parity(xl & zl): the term reads Im p
};
struct EjGroup {
  uint32_t xl = 0;
  std::vector<EjTerm> terms;
};
struct EjPass {
  int spos[kEjTileQubits];
  std::vector<EjGroup> groups;
  int nterms = 0;
  std::string src;
  JitKernel k;
};
struct EjPlan {
  int n = 0;
  std::vector<EjPass> passes;
  long evals = 0;
  bool tried = false;
  bool ready = false;  // every pass has a kernel
};

std::mutex g_ej_mu;
std::atomic<long> g_ej_jit_passes{0}, g_ej_generic_passes{0};
// plans are shared_ptr so an evaluation keeps its plan alive while another
// thread trims the cache; compile decisions are taken under g_ej_mu
std::unordered_map<std::string, std::shared_ptr<EjPlan>> g_ej_plans;

std::string hex64(uint64_t v) {
  char b[32];
  snprintf(b, sizeof(b), "0x%llxull", (unsigned long long)v);
  return b;
}
std::string hex32(uint32_t v) {
  char b[24];
  snprintf(b, sizeof(b), "0x%xu", v);
  return b;
}
std::string I(long v) { return std::to_string(v); }

// Units (flip mask, <= kEjMaxTerms of its terms) packed first-fit into tile
// sets of 12 qubits; false if a flip mask does not fit a tile.
bool ej_pack(int n, const std::vector<uint64_t>& xms, const std::vector<uint64_t>& zms,
             std::vector<EjPass>& passes) {
  if (n < kEjTileQubits) return false;
  const uint64_t low = 0xFULL;
  // units: (flip mask, <= kEjMaxTerms of its terms); flip-free terms (Z
  // products) fit any tile and are dealt out afterwards to balance the passes
  std::vector<uint64_t> masks;
  for (uint64_t m : xms)
    if (m && std::find(masks.begin(), masks.end(), m) == masks.end()) masks.push_back(m);
  struct Unit {
    uint64_t xm;
    std::vector<int> terms;
  };
  std::vector<Unit> units;
  for (uint64_t m : masks) {
    if (__builtin_popcountll(m | low) > kEjTileQubits) return false;
    Unit u{m, {}};
    for (size_t t = 0; t < xms.size(); ++t) {
      if (xms[t] != m) continue;
      u.terms.push_back((int)t);
      if ((int)u.terms.size() == kEjMaxTerms) {
        units.push_back(u);
        u.terms.clear();
      }
    }
    if (!u.terms.empty()) units.push_back(u);
  }
  std::vector<int> diag;
  for (size_t t = 0; t < xms.size(); ++t)
    if (!xms[t]) diag.push_back((int)t);
  // 1. flip units first-fit into tile sets of 12 qubits
  struct Sel {
    uint64_t S;
    std::vector<int> members;  // unit indices
    std::vector<int> dterms;   // flip-free terms dealt to this pass
    int nterms;
  };
  std::vector<Sel> sel;
  std::vector<char> done(units.size(), 0);
  size_t left = units.size();
  while (left) {
    Sel P{low, {}, {}, 0};
    for (size_t i = 0; i < units.size(); ++i) {
      if (done[i]) continue;
      if (__builtin_popcountll(P.S | units[i].xm) > kEjTileQubits) continue;
      if (P.nterms + (int)units[i].terms.size() > kEjMaxTerms) continue;
      P.S |= units[i].xm;
      P.nterms += (int)units[i].terms.size();
      done[i] = 1;
      --left;
      P.members.push_back((int)i);
    }
    sel.push_back(std::move(P));
  }
  // 2. flip-free terms to the passes with the fewest terms (registers: one
  // accumulator per term), new passes only when every pass is full
  for (int t : diag) {
    Sel* best = nullptr;
    for (Sel& P : sel)
      if (P.nterms < kEjMaxTerms && (!best || P.nterms < best->nterms)) best = &P;
    if (!best) {
      sel.push_back(Sel{low, {}, {}, 0});
      best = &sel.back();
    }
    best->dterms.push_back(t);
    ++best->nterms;
  }
  for (Sel& Q : sel) {
    uint64_t S = Q.S;
    // local layout: qubits 0..3 on bits 0..3; flip qubits on the slot bits
    // 8..11 first (most-used first), then bit 4, then the warp bits 5..7;
    // the lowest unused qubits fill what is left
    std::vector<std::pair<int, int>> use;  // (-groups using it, qubit)
    for (int q = 4; q < n; ++q) {
      if (!((S >> q) & 1ULL)) continue;
      int cnt = 0;
      for (int i : Q.members) cnt += (int)((units[i].xm >> q) & 1ULL);
      use.push_back({-cnt, q});
    }
    std::sort(use.begin(), use.end());
    static const int kPref[8] = {8, 9, 10, 11, 4, 5, 6, 7};
    EjPass P;
    for (int b = 0; b < 4; ++b) P.spos[b] = b;
    int slot = 0;
    for (auto& u : use) P.spos[kPref[slot++]] = u.second;
    for (int q = 4; q < n && slot < 8; ++q)
      if (!((S >> q) & 1ULL)) {
        S |= 1ULL << q;
        P.spos[kPref[slot++]] = q;
      }
    int local_of[64];
    for (int q = 0; q < 64; ++q) local_of[q] = -1;
    for (int j = 0; j < kEjTileQubits; ++j) local_of[P.spos[j]] = j;
    auto add_terms = [&](uint64_t xm, const std::vector<int>& ts) {
      EjGroup* G = nullptr;
      uint32_t xl = 0;
      for (int q = 0; q < n; ++q)
        if ((xm >> q) & 1ULL) xl |= 1u << local_of[q];
      for (EjGroup& g : P.groups)
        if (g.xl == xl) G = &g;
      if (!G) {
        P.groups.push_back(EjGroup{});
        G = &P.groups.back();
        G->xl = xl;
      }
      for (int t : ts) {
        EjTerm T{t, 0, 0, false};
        for (int q = 0; q < n; ++q)
          if ((zms[t] >> q) & 1ULL) {
            if (local_of[q] >= 0) T.zl |= 1u << local_of[q];
            else T.zg |= 1ULL << q;
          }
        T.imag = (__builtin_popcount(xl & T.zl) & 1) != 0;
        G->terms.push_back(T);
        ++P.nterms;
      }
    };
    if (!Q.dterms.empty()) add_terms(0, Q.dterms);
    for (int i : Q.members) add_terms(units[i].xm, units[i].terms);
    passes.push_back(std::move(P));
  }
  return true;
}

// ---------------------------------------------------------------- generator
struct EjGen {
  std::string o;
  void line(const std::string& s) {
    o += s;
    o += '\n';
  }
};

// in-place Walsh-Hadamard transform over m values named base0..base{m-1}
void emit_wht(EjGen& g, const std::string& base, int m) {
  for (int h = 1; h < m; h <<= 1)
    for (int k = 0; k < m; ++k)
      if (!(k & h)) {
        const std::string a = base + I(k), b = base + I(k + h);
        g.line("  { const double u_ = " + a + ", w_ = " + b + "; " + a + " = u_ + w_; " + b +
               " = u_ - w_; }");
      }
}

// QSV_EXPECT_BULK=1: tiles move with cp.async.bulk + mbarrier (A/B; the
// source differs, so the two variants are cached separately)
// QSV_EXPECT_REGLOAD=1: register-staged tile loads (A/B; measured slower:
// TFIM n=28 2.75 -> 3.10 ms, profiles/r2_expect_bulk_ab.md), default cp.async
bool ej_regload() {
  static const int on = [] {
    const char* e = getenv("QSV_EXPECT_REGLOAD");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

bool ej_bulk() {
  static const int on = [] {
    const char* e = getenv("QSV_EXPECT_BULK");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

std::string ej_source(const EjPass& P) {
  EjGen g;
  g.line(R"JIT(typedef unsigned long long u64;
typedef unsigned int uint32_t;
struct FixedBits { int n; u64 lowmask[28]; u64 value; };
__device__ __forceinline__ u64 widen(u64 k, const FixedBits& f) {
#pragma unroll 4
  for (int i = 0; i < f.n; ++i) { const u64 lo = k & f.lowmask[i]; k = ((k ^ lo) << 1) | lo; }
  return k | f.value;
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gp) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gp) : "memory");
}
// x with its sign bit flipped when s != 0
__device__ __forceinline__ double fneg(double x, u64 s) {
  return __longlong_as_double(__double_as_longlong(x) ^ (s << 63));
}
struct XParams { const double2* a; u64 ntiles; double* partials; FixedBits tb; };
)JIT");
  const int nt = P.nterms;
  g.line("extern \"C\" __global__ void __launch_bounds__(256, 1) k_pass(const __grid_constant__ XParams P) {");
  g.line("  extern __shared__ double2 sbuf[];");
  g.line("  __shared__ double red[8][" + I(std::max(1, nt)) + "];");
  g.line("  const uint32_t tid = threadIdx.x;");
  // thread's HBM offset part (local bits 0..7 = tid bits) and slot parts
  {
    std::string lo = "  const u64 lo = 0ull";
    for (int b = 0; b < 8; ++b)
      lo += " | ((u64)((tid >> " + I(b) + ") & 1u) << " + I(P.spos[b]) + ")";
    g.line(lo + ";");
  }
  uint64_t hi[16];
  for (int k = 0; k < 16; ++k) {
    hi[k] = 0;
    for (int b = 0; b < 4; ++b)
      if ((k >> b) & 1) hi[k] |= 1ULL << P.spos[8 + b];
  }
  // per-thread sign bits: bit t = parity(thread part of x & z_t), plus the
  // slot-bit-3 sign of split-visit groups (threads with the pairing bit set
  // visit slots 8..15)
  g.line("  u64 hm = 0ull;");
  {
    int t = 0;
    for (const EjGroup& G : P.groups) {
      const uint32_t xs = G.xl >> 8, xt = G.xl & 0xffu;
      const bool split = G.xl != 0 && xs == 0;
      const int hb = xt ? 31 - __builtin_clz(xt) : -1;
      for (const EjTerm& T : G.terms) {
        std::string e = "(uint32_t)__popc(tid & " + hex32(T.zl & 0xffu) + ")";
        if (split && ((T.zl >> 11) & 1u)) e += " + ((tid >> " + I(hb) + ") & 1u)";
        if ((T.zl & 0xffu) || (split && ((T.zl >> 11) & 1u)))
          g.line("  hm |= (u64)((" + e + ") & 1u) << " + I(t) + ";");
        ++t;
      }
    }
  }
  for (int t = 0; t < nt; ++t) g.line("  double acc" + I(t) + " = 0.0;");
  // register staging: each thread loads its 16 amplitudes of the next tile
  // into registers while the current one is evaluated (64 more registers,
  // so only for passes with at most 24 accumulators), and stores the tile to
  // shared memory itself only when a group needs partner amplitudes from
  // other threads -- a 128-bit register store costs a quarter of the
  // shared-memory wavefronts of the cp.async copy-in (one per 32-byte sector)
  bool need_smem = false;
  for (const EjGroup& G : P.groups) need_smem = need_smem || (G.xl & 0xffu) != 0;
  const bool regload = ej_regload() && !ej_bulk() && P.nterms <= 24;
  if (regload) {
    g.line("  u64 tile = blockIdx.x;");
    g.line("  int buf = 0;");
    g.line("  double2 nx[16];");
    g.line("  if (tile < P.ntiles) {");
    g.line("    const u64 gb = widen(tile, P.tb) | lo;");
    for (int k = 0; k < 16; ++k)
      g.line("    nx[" + I(k) + "] = __ldg(P.a + (gb | " + hex64(hi[k]) + "));");
    g.line("  }");
    g.line("  for (; tile < P.ntiles; tile += gridDim.x, buf ^= 1) {");
    g.line("    double2 v[16];");
    g.line("#pragma unroll");
    g.line("    for (int k = 0; k < 16; ++k) v[k] = nx[k];");
    g.line("    const u64 nxt = tile + gridDim.x;");
    g.line("    if (nxt < P.ntiles) {");
    g.line("      const u64 gb = widen(nxt, P.tb) | lo;");
    for (int k = 0; k < 16; ++k)
      g.line("      nx[" + I(k) + "] = __ldg(P.a + (gb | " + hex64(hi[k]) + "));");
    g.line("    }");
    g.line("    double2* smw = sbuf + (buf << 12);");
    if (need_smem) {
      g.line("#pragma unroll");
      g.line("    for (int k = 0; k < 16; ++k) smw[(k << 8) + tid] = v[k];");
      g.line("    __syncthreads();");
    }
    g.line("    const double2* sm = smw;");
    g.line("    (void)sm;");
    g.line("    const u64 base = widen(tile, P.tb);");
    g.line("    (void)base;");
  } else if (ej_bulk()) {
    // Blackwell bulk copies: each thread moves one 256-byte run (16
    // amplitudes of qubits 0..3) with cp.async.bulk, completion counted by
    // an mbarrier per buffer (tx bytes), instead of 16 cp.async of 16 bytes
    {
      std::string lr = "  const u64 lorun = 0ull";
      for (int b = 0; b < 4; ++b)
        lr += " | ((u64)((tid >> " + I(b) + ") & 1u) << " + I(P.spos[4 + b]) + ")";
      for (int b = 0; b < 4; ++b)
        lr += " | ((u64)((tid >> " + I(4 + b) + ") & 1u) << " + I(P.spos[8 + b]) + ")";
      g.line(lr + ";");
    }
    g.line(R"JIT(  __shared__ __align__(8) u64 mbar[2];
  const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(sbuf);
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  // run tid: slot k = tid >> 4, first thread (tid & 15) << 4 -> smem element k*256 + (tid&15)*16
  const uint32_t sofs = ((((tid >> 4) << 8) | ((tid & 15u) << 4)) << 4);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 256;" ::"r"(mb0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 256;" ::"r"(mb0 + 8) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](u64 t, int b) {
    const double2* src = P.a + (widen(t, P.tb) | lorun);
    const uint32_t mb = mb0 + 8u * (uint32_t)b;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 256;" ::"r"(mb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                 ::"r"(sb0 + ((uint32_t)b << 16) + sofs), "l"(src), "r"(mb) : "memory");
  };
  auto wait = [&](int b, uint32_t parity) {
    const uint32_t mb = mb0 + 8u * (uint32_t)b;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb), "r"(parity) : "memory");
  };
  u64 tile = blockIdx.x;
  int buf = 0;
  uint32_t it = 0;
  if (tile < P.ntiles) issue(tile, 0);
  for (; tile < P.ntiles; tile += gridDim.x, ++it) {
    buf = (int)(it & 1u);
    wait(buf, (it >> 1) & 1u);
    __syncthreads();
    const u64 nxt = tile + gridDim.x;
    if (nxt < P.ntiles) issue(nxt, buf ^ 1);)JIT");
  } else {
  g.line(R"JIT(  const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(sbuf);
  u64 tile = blockIdx.x;
  int buf = 0;
  if (tile < P.ntiles) {
    const u64 gb = widen(tile, P.tb) | lo;)JIT");
  for (int k = 0; k < 16; ++k)
    g.line("    cp_async16(sb0 + ((" + I(k * 256) + "u + tid) << 4), P.a + (gb | " + hex64(hi[k]) +
           "));");
  g.line(R"JIT(    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (; tile < P.ntiles; tile += gridDim.x, buf ^= 1) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const u64 nxt = tile + gridDim.x;
    if (nxt < P.ntiles) {
      const uint32_t sbn = sb0 + ((uint32_t)(buf ^ 1) << 16);
      const u64 gb = widen(nxt, P.tb) | lo;)JIT");
  for (int k = 0; k < 16; ++k)
    g.line("      cp_async16(sbn + ((" + I(k * 256) + "u + tid) << 4), P.a + (gb | " +
           hex64(hi[k]) + "));");
  g.line(R"JIT(      asm volatile("cp.async.commit_group;" ::: "memory");
    })JIT");
  }
  if (!regload)
  g.line(R"JIT(    const double2* sm = sbuf + (buf << 12);
    const u64 base = widen(tile, P.tb);
    (void)base;
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = sm[(k << 8) + tid];)JIT");
  int t0 = 0;
  for (const EjGroup& G : P.groups) {
    const uint32_t xs = G.xl >> 8, xt = G.xl & 0xffu;
    bool need_re = false, need_im = false;
    for (const EjTerm& T : G.terms) (T.imag ? need_im : need_re) = true;
    g.line("    { // group xl=" + hex32(G.xl) + ", " + I((long)G.terms.size()) + " terms");
    int m;                       // products formed per thread
    std::vector<int> kofs;       // visited slot of product i (empty: slot i, split groups)
    if (G.xl == 0) {
      m = 16;
      for (int k = 0; k < 16; ++k) {
        g.line("      double r" + I(k) + " = fma(v[" + I(k) + "].x, v[" + I(k) + "].x, v[" + I(k) +
               "].y * v[" + I(k) + "].y);");
        kofs.push_back(k);
      }
    } else {
      m = 8;
      for (int i = 0; i < m; ++i) {
        if (need_re) g.line("      double r" + I(i) + ";");
        if (need_im) g.line("      double m" + I(i) + ";");
      }
      if (xt) g.line("      const double2* pp = sm + (tid ^ " + hex32(xt) + ");");
      std::vector<std::pair<std::string, std::string>> xy;  // (x, y) of product i
      if (xs) {
        const int hb = 31 - __builtin_clz(xs);
        for (int k = 0; k < 16; ++k)
          if (!((k >> hb) & 1)) kofs.push_back(k);
        for (int i = 0; i < 8; ++i) {
          const int k = kofs[i], kp = k ^ (int)xs;
          xy.push_back({"v[" + I(k) + "]", xt ? "pp[" + I(kp << 8) + "]" : "v[" + I(kp) + "]"});
        }
      } else {
        // pairing bit on the thread bits: the thread with it clear visits
        // slots 0..7, its partner slots 8..15 (each pair once, no idle lanes)
        const int hb = 31 - __builtin_clz(xt);
        g.line("      const uint32_t b_ = (tid >> " + I(hb) + ") & 1u;");
        g.line("      const double2* qq = pp + (b_ << 11);");
        for (int i = 0; i < 8; ++i)
          xy.push_back({"(b_ ? v[" + I(i + 8) + "] : v[" + I(i) + "])", "qq[" + I(i << 8) + "]"});
      }
      for (int i = 0; i < 8; ++i) {
        g.line("      { const double2 x_ = " + xy[i].first + ", y_ = " + xy[i].second + ";");
        if (need_re) g.line("        r" + I(i) + " = fma(x_.x, y_.x, x_.y * y_.y);");
        if (need_im) g.line("        m" + I(i) + " = fma(x_.x, y_.y, -x_.y * y_.x);");
        g.line("      }");
      }
    }
    // index of product i's sign bit pattern: product i sits at slot kofs[i]
    // (slot-bit groups / xl == 0) or at slot i (+8 folded into hm) for split
    // groups; W_t = sum_i (-1)^popc(slot_i & zk_t) q_i
    auto slot_of = [&](int i) { return kofs.empty() ? i : kofs[i]; };
    for (int part = 0; part < 2; ++part) {
      const bool im = part == 1;
      if (im ? !need_im : !need_re) continue;
      const std::string q = im ? "m" : "r";
      int cnt = 0;
      for (const EjTerm& T : G.terms) cnt += T.imag == im;
      const bool wht = cnt >= (m == 16 ? 5 : 4);
      if (wht) emit_wht(g, q, m);
      int t = t0;
      for (const EjTerm& T : G.terms) {
        if (T.imag != im) {
          ++t;
          continue;
        }
        const uint32_t zk = (T.zl >> 8) & 0xFu;
        std::string W;
        if (wht) {
          // coefficient index: the sign pattern over products i
          int idx = 0;
          for (int b = 0; (1 << b) < m; ++b) {
            const int s = slot_of(1 << b);  // slot bit pattern of product bit b
            if (__builtin_popcount((uint32_t)s & zk) & 1) idx |= 1 << b;
          }
          W = q + I(idx);
        } else {
          W = "(";
          for (int i = 0; i < m; ++i) {
            const bool neg = __builtin_popcount((uint32_t)slot_of(i) & zk) & 1;
            if (i == 0) W += neg ? "-" + q + "0" : q + "0";
            else W += (neg ? " - " : " + ") + q + I(i);
          }
          W += ")";
        }
        std::string sgn = "(hm >> " + I(t) + ")";
        if (T.zg) sgn = "(" + sgn + " ^ (u64)__popcll(base & " + hex64(T.zg) + "))";
        g.line("      acc" + I(t) + " += fneg(" + W + ", " + sgn + " & 1ull);");
        ++t;
      }
    }
    g.line("    }");
    t0 += (int)G.terms.size();
  }
  g.line("  }");
  // fixed-order block reduction: warp trees, then warps in order
  g.line("  const int lane = tid & 31, warp = tid >> 5;");
  {
    int t = 0;
    for (const EjGroup& G : P.groups)
      for (const EjTerm& T : G.terms) {
        (void)T;
        g.line("  { double s_ = acc" + I(t) + ";");
        g.line("#pragma unroll");
        g.line("    for (int o_ = 16; o_ > 0; o_ >>= 1) s_ += __shfl_xor_sync(0xffffffffu, s_, o_);");
        g.line("    if (lane == 0) red[warp][" + I(t) + "] = s_; }");
        ++t;
      }
  }
  g.line("  __syncthreads();");
  g.line("  if (tid < " + I(nt) + ") {");
  g.line("    double s = 0.0;");
  g.line("#pragma unroll");
  g.line("    for (int w = 0; w < 8; ++w) s += red[w][tid];");
  // scale: 2 for pair groups, -1 for imaginary terms; slot re / im
  {
    uint64_t imask = 0, pmask = 0;
    int t = 0;
    for (const EjGroup& G : P.groups)
      for (const EjTerm& T : G.terms) {
        if (T.imag) imask |= 1ULL << t;
        if (G.xl) pmask |= 1ULL << t;
        ++t;
      }
    g.line("    const bool isim = (" + hex64(imask) + " >> tid) & 1ull;");
    g.line("    if ((" + hex64(pmask) + " >> tid) & 1ull) s *= 2.0;");
    g.line("    if (isim) s = -s;");
  }
  g.line("    double* o = P.partials + ((size_t)blockIdx.x * " + I(kEjMaxTermsStride) + " + tid) * 2;");
  g.line("    o[0] = isim ? 0.0 : s;");
  g.line("    o[1] = isim ? s : 0.0;");
  g.line("  }");
  g.line("}");
  return g.o;
}

struct EjParams {
  const double2* a;
  unsigned long long ntiles;
  double* partials;
  FixedBits tb;
};

#define QSV_TRY_RC(call)         \
  do {                           \
    const int rc__ = (call);     \
    if (rc__ != QSV_OK) return rc__; \
  } while (0)

int jit_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("QSV_EXPECT_JIT");
    mode = e ? atoi(e) : 1;
  }
  return mode;
}

}  // namespace ej

using namespace ej;

// QSV_EXPECT_STREAMS: passes of one evaluation in flight at once (1: all on
// the caller's stream, the pre-overlap behaviour)
int ej_lanes() {
  static const int v = [] {
    const char* e = getenv("QSV_EXPECT_STREAMS");
    const int k = e ? atoi(e) : kEjLanes;
    return std::max(1, std::min(k, kEjLanes));
  }();
  return v;
}

// per-device auxiliary streams and fork / join events of the pass lanes
struct EjLaneSet {
  cudaStream_t streams[kEjLanes] = {};
  cudaEvent_t fork = nullptr, join[kEjLanes] = {};
};
EjLaneSet* ej_lane_set(int dev) {
  static EjLaneSet sets[64];
  static bool made[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  EjLaneSet& L = sets[dev];
  if (!made[dev]) {
    for (int k = 1; k < kEjLanes; ++k) {
      if (cudaStreamCreateWithFlags(&L.streams[k], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&L.join[k], cudaEventDisableTiming) != cudaSuccess)
        return nullptr;
    }
    if (cudaEventCreateWithFlags(&L.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    made[dev] = true;
  }
  return &L;
}

size_t expect_jit_scratch_bytes() {
  return sizeof(double) * ((size_t)kEjLanes * 2 * 296 * kEjMaxTermsStride +
                           2 * (size_t)kEjMaxTermsStride * 32);
}

// Evaluate every term's S_t through generated pass kernels.  Returns
// QSV_EUNSUPPORTED when the generated path is off or not (yet) compiled for
// this observable -- the caller then runs the generic k_expect_tile.  Mode
// (QSV_EXPECT_JIT): 0 off, 1 (default) compile on the observable's second
// evaluation (or use kernels already in the caches), 2 compile on the first.
int expect_tile_jit(const double2* a, int n, const std::vector<uint64_t>& xms,
                    const std::vector<uint64_t>& zms, void* scratch, std::vector<double>& res,
                    cudaStream_t s) {
  const int mode = jit_mode();
  if (mode == 0 || n < kEjTileQubits) return QSV_EUNSUPPORTED;
  std::string key(reinterpret_cast<const char*>(&n), sizeof(n));
  key.append(reinterpret_cast<const char*>(xms.data()), xms.size() * sizeof(uint64_t));
  key.append(reinterpret_cast<const char*>(zms.data()), zms.size() * sizeof(uint64_t));
  std::shared_ptr<EjPlan> plan;
  std::lock_guard<std::mutex> lk(g_ej_mu);
  if (g_ej_plans.size() > 256) g_ej_plans.clear();
  auto it = g_ej_plans.find(key);
  if (it == g_ej_plans.end()) {
    auto p = std::make_shared<EjPlan>();
    p->n = n;
    if (!ej_pack(n, xms, zms, p->passes)) return QSV_EUNSUPPORTED;
    for (EjPass& P : p->passes) P.src = ej_source(P);
    if (const char* dir = getenv("QSV_JIT_DUMP")) {
      for (size_t i = 0; i < p->passes.size(); ++i)
        if (FILE* f = fopen((std::string(dir) + "/xpass_" + std::to_string(i) + ".cu").c_str(), "w")) {
          fputs(p->passes[i].src.c_str(), f);
          fclose(f);
        }
    }
    it = g_ej_plans.emplace(key, std::move(p)).first;
  }
  plan = it->second;
  ++plan->evals;
  if (!plan->tried) {
    bool cached = true;
    for (const EjPass& P : plan->passes) cached = cached && jit_cached(P.src);
    if (mode == 2 || cached || plan->evals >= 2) {
      plan->tried = true;
      std::vector<const std::string*> srcs;
      for (const EjPass& P : plan->passes) srcs.push_back(&P.src);
      std::vector<JitKernel> ks;
      std::string err;
      QSV_TRY_RC(jit_kernels(srcs, ks, &err));
      bool all = true;
      for (size_t i = 0; i < ks.size(); ++i) {
        plan->passes[i].k = ks[i];
        all = all && ks[i].kernel;
      }
      plan->ready = all;
      if (!err.empty() && getenv("QSV_JIT_VERBOSE")) fprintf(stderr, "qsv expect jit: %s\n", err.c_str());
    }
  }
  if (!plan->ready) return QSV_EUNSUPPORTED;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  const uint64_t ntiles = 1ULL << (n - kEjTileQubits);
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)std::min(num_sms, 296));
  // scratch (expect_jit_scratch_bytes()): partials of kEjLanes passes, then
  // up to kEjBatch passes' results, copied back with one synchronisation per
  // batch.  The passes only read the state and write their own partials, so
  // they run on kEjLanes forked streams (pass p on lane p mod kEjLanes, its
  // reduction after it on the same lane): one pass's ramp and tail overlap
  // the next pass's sweep instead of idling HBM between kernels.
  constexpr size_t kEjBatch = 32;
  double* partials = reinterpret_cast<double*>(scratch);
  double* dout = partials + kEjLanes * 2 * (size_t)296 * kEjMaxTermsStride;
  const size_t smem = 2 * sizeof(double2) * (1u << kEjTileQubits);
  res.assign(2 * xms.size(), 0.0);
  std::vector<double> hout;
  const int lanes = std::min<int>(ej_lanes(), (int)plan->passes.size());
  cudaStream_t ls[kEjLanes];
  for (int k = 0; k < kEjLanes; ++k) ls[k] = s;
  EjLaneSet* L = nullptr;
  if (lanes > 1) {
    int dev = 0;
    cudaGetDevice(&dev);
    L = ej_lane_set(dev);
    if (!L) return QSV_EUNSUPPORTED;
    QSV_TRY(cudaEventRecord(L->fork, s));
    for (int k = 1; k < lanes; ++k) {
      ls[k] = L->streams[k];
      QSV_TRY(cudaStreamWaitEvent(ls[k], L->fork, 0));
    }
  }
  for (size_t p0 = 0; p0 < plan->passes.size(); p0 += kEjBatch) {
    const size_t p1 = std::min(plan->passes.size(), p0 + kEjBatch);
    for (size_t p = p0; p < p1; ++p) {
      const EjPass& P = plan->passes[p];
      const int lane = lanes > 1 ? (int)(p % lanes) : 0;
      double* part = partials + lane * 2 * (size_t)296 * kEjMaxTermsStride;
      EjParams prm;
      memset(&prm, 0, sizeof(prm));
      prm.a = a;
      prm.ntiles = ntiles;
      prm.partials = part;
      prm.tb = make_fixed(P.spos, kEjTileQubits, 0);
      QSV_TRY_RC(jit_set_smem(P.k, smem));
      void* args[] = {&prm};
      QSV_TRY(cudaLaunchKernel(reinterpret_cast<const void*>(P.k.kernel), dim3(grid),
                               dim3(kEjThreads), args, smem, ls[lane]));
      QSV_TRY_RC(launch_expect_tile_final(part, (int)grid, P.nterms,
                                          dout + 2 * kEjMaxTermsStride * (p - p0), ls[lane]));
      ++g_ej_jit_passes;
    }
    if (L) {  // join the lanes into s before the copy back
      for (int k = 1; k < lanes; ++k) {
        QSV_TRY(cudaEventRecord(L->join[k], ls[k]));
        QSV_TRY(cudaStreamWaitEvent(s, L->join[k], 0));
      }
    }
    hout.resize(2 * kEjMaxTermsStride * (p1 - p0));
    QSV_TRY(cudaMemcpyAsync(hout.data(), dout, hout.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    QSV_TRY(cudaStreamSynchronize(s));
    if (L && p1 < plan->passes.size()) {  // next batch: fork again
      QSV_TRY(cudaEventRecord(L->fork, s));
      for (int k = 1; k < lanes; ++k) QSV_TRY(cudaStreamWaitEvent(ls[k], L->fork, 0));
    }
    for (size_t p = p0; p < p1; ++p) {
      int t = 0;
      for (const EjGroup& G : plan->passes[p].groups)
        for (const EjTerm& T : G.terms) {
          res[2 * T.index] = hout[2 * kEjMaxTermsStride * (p - p0) + 2 * t];
          res[2 * T.index + 1] = hout[2 * kEjMaxTermsStride * (p - p0) + 2 * t + 1];
          ++t;
        }
    }
  }
  return QSV_OK;
}

}  // namespace qsv

extern "C" int qsv_expect_jit_source(int num_qubits, int nterms, const uint64_t* xms,
                                     const uint64_t* zms, int pass, char* buf, size_t cap,
                                     int* num_passes) {
  if (num_qubits < 1 || num_qubits > 63 || nterms < 0 || (nterms && (!xms || !zms)) ||
      !num_passes)
    return QSV_EINVAL;
  std::vector<qsv::ej::EjPass> passes;
  if (!qsv::ej::ej_pack(num_qubits, std::vector<uint64_t>(xms, xms + nterms),
                    std::vector<uint64_t>(zms, zms + nterms), passes))
    return QSV_EUNSUPPORTED;
  *num_passes = (int)passes.size();
  if (pass < 0 || pass >= (int)passes.size()) return buf ? QSV_EINVAL : QSV_OK;
  if (buf && cap) {
    const std::string src = qsv::ej::ej_source(passes[pass]);
    const size_t n = std::min(cap - 1, src.size());
    memcpy(buf, src.data(), n);
    buf[n] = 0;
  }
  return QSV_OK;
}

namespace qsv {
void expect_generic_pass_done() { ++ej::g_ej_generic_passes; }
}  // namespace qsv

extern "C" int qsv_expect_path_stats(long* jit_passes, long* generic_passes) {
  if (!jit_passes || !generic_passes) return QSV_EINVAL;
  *jit_passes = qsv::ej::g_ej_jit_passes.load();
  *generic_passes = qsv::ej::g_ej_generic_passes.load();
  return QSV_OK;
}
