// Tile passes: several gates per HBM sweep, plus the program planner.
//
// The reference applies a circuit gate by gate, each gate one full sweep of
// the 2^n array (circuit.py:54-55 -> kernels.apply_*).  Here the planner
// packs consecutive gates into passes.  A pass fixes a set S of L "tile"
// qubits (always including qubits 0..3, so HBM runs are >= 256 B); one CTA
// loads the 2^L amplitudes that share the values of all other qubits into
// shared memory, applies every gate of the pass, and writes the tile back.
// A gate can join a pass when its NON-diagonal targets lie in S: diagonal
// factors and controls on qubits outside S are constants of the tile.
//
// Inside a tile the gates run in "phases": each thread holds 2^kRegBits
// amplitudes whose local indices differ in kRegBits register bits, so every
// gate acting on register bits is pure register arithmetic; a phase boundary
// is one shared-memory round trip (XOR-swizzled, bank-conflict free).
// A CTA holds kGroups independent tile groups with their own named barriers,
// so one group's HBM copies and transposes overlap the other's FP64 math.
//
// HBM bytes per pass: 32 * 2^n (read + write once), independent of the number
// of gates in it; FP64 work: 8 FMA per amplitude per 1-qubit dense gate.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <cstdlib>

#include "qsv_tile.cuh"

namespace qsv {

// ===================================================================== device

__device__ __forceinline__ uint32_t swz(uint32_t l) {
  return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u);
}

struct TileCtx {
  uint64_t base;       // global bits of this tile
  uint32_t lt;         // thread's local base (thread bits placed)
  uint32_t rb[kRegBits];  // local bit mask of each register slot
};

__device__ __forceinline__ uint32_t lidx(const TileCtx& c, int j) {
  uint32_t l = c.lt;
#pragma unroll
  for (int i = 0; i < kRegBits; ++i)
    if ((j >> i) & 1) l |= c.rb[i];
  return l;
}

__device__ __forceinline__ bool lcond(const TileOp& op, uint32_t l) {
  return (l & op.lmask) == op.lval;
}

// A control / pattern test (l & mask) == val split into the thread's part
// (fixed for the phase) and the register-slot part (compile-time in j).
struct SplitCond {
  bool t_ok;
  uint32_t rm, rv;  // over register slots
};

__device__ __forceinline__ SplitCond split_cond(const TileCtx& c, uint32_t mask, uint32_t val) {
  SplitCond sc;
  sc.rm = 0;
  sc.rv = 0;
  uint32_t regmask = 0;
#pragma unroll
  for (int i = 0; i < kRegBits; ++i) {
    regmask |= c.rb[i];
    if (mask & c.rb[i]) {
      sc.rm |= 1u << i;
      if (val & c.rb[i]) sc.rv |= 1u << i;
    }
  }
  const uint32_t tm = mask & ~regmask;
  sc.t_ok = (c.lt & tm) == (val & tm);
  return sc;
}

__device__ __forceinline__ bool jcond(const SplitCond& sc, int j) {
  return ((uint32_t)j & sc.rm) == sc.rv;
}

// sign flip on the integer pipe (keeps the FP64 pipe for the math)
__device__ __forceinline__ double2 neg_if(double2 v, bool f) {
  const int s = f ? (int)0x80000000 : 0;
  return make_double2(__hiloint2double(__double2hiint(v.x) ^ s, __double2loint(v.x)),
                      __hiloint2double(__double2hiint(v.y) ^ s, __double2loint(v.y)));
}

template <int I, bool CTRL>
__device__ __forceinline__ void t_dense1_body(double2 (&v)[kRegs], const SplitCond& sc,
                                              double2 m00, double2 m01, double2 m10,
                                              double2 m11) {
#pragma unroll
  for (int j = 0; j < kRegs; ++j) {
    if ((j >> I) & 1) continue;
    const int q = j | (1 << I);
    const double2 x = v[j], y = v[q];
    const double2 nx = cfma(m01, y, cmul(m00, x));
    const double2 ny = cfma(m11, y, cmul(m10, x));
    if (CTRL) {  // predicated select, no branch
      const bool ok = jcond(sc, j);
      v[j].x = ok ? nx.x : x.x;
      v[j].y = ok ? nx.y : x.y;
      v[q].x = ok ? ny.x : y.x;
      v[q].y = ok ? ny.y : y.y;
    } else {
      v[j] = nx;
      v[q] = ny;
    }
  }
}

template <int I>
__device__ __forceinline__ void t_dense1(double2 (&v)[kRegs], const TileCtx& c, const TileOp& op,
                                         const double2* data) {
  const double2 m00 = (data[op.data + 0]), m01 = (data[op.data + 1]);
  const double2 m10 = (data[op.data + 2]), m11 = (data[op.data + 3]);
  SplitCond sc{true, 0, 0};
  if (op.lmask) {
    sc = split_cond(c, op.lmask, op.lval);
    if (!sc.t_ok) return;
  }
  if (sc.rm)
    t_dense1_body<I, true>(v, sc, m00, m01, m10, m11);
  else
    t_dense1_body<I, false>(v, sc, m00, m01, m10, m11);
}

__device__ __forceinline__ void t_apply(double2 (&v)[kRegs], const TileCtx& c, const TileOp& op,
                                        const double2* data) {
  // tile-constant part of the op
  if (op.gmask && ((c.base & op.gmask) != op.gval)) return;
  switch (op.kind) {
    case T_DENSE1:
      switch (op.slots) {
        case 1: t_dense1<0>(v, c, op, data); break;
        case 2: t_dense1<1 % kRegBits>(v, c, op, data); break;
        case 4: t_dense1<2 % kRegBits>(v, c, op, data); break;
        case 8: t_dense1<3 % kRegBits>(v, c, op, data); break;
        case 16: t_dense1<4 % kRegBits>(v, c, op, data); break;
      }
      break;
    case T_DENSE1XR: {
      const double2* M = data + op.data;
      const SplitCond sc{true, 0, 0};
      t_dense1_body<0, false>(v, sc, M[0], M[1], M[2], M[3]);
      t_dense1_body<1 % kRegBits, false>(v, sc, M[4], M[5], M[6], M[7]);
      if (op.m > 2) t_dense1_body<2 % kRegBits, false>(v, sc, M[8], M[9], M[10], M[11]);
      if (op.m > 3) t_dense1_body<3 % kRegBits, false>(v, sc, M[12], M[13], M[14], M[15]);
      if (op.m > 4) t_dense1_body<4 % kRegBits, false>(v, sc, M[16], M[17], M[18], M[19]);
      break;
    }
    case T_PHASE: {
      const SplitCond sc = split_cond(c, op.lmask, op.lval);
      if (!sc.t_ok) break;
      if (op.flags & 2) {
#pragma unroll
        for (int j = 0; j < kRegs; ++j) v[j] = neg_if(v[j], jcond(sc, j));
      } else {
        const double2 f = (data[op.data]);
#pragma unroll
        for (int j = 0; j < kRegs; ++j) {
          const double2 w = cmul(v[j], f);
          const bool ok = jcond(sc, j);
          v[j].x = ok ? w.x : v[j].x;
          v[j].y = ok ? w.y : v[j].y;
        }
      }
      break;
    }
    case T_DIAG: {
      const SplitCond sc = split_cond(c, op.lmask, op.lval);
      if (!sc.t_ok) break;
      // per target: tile/thread constant bit, or register slot
      int fixed_sub = 0;
      int slot[4] = {-1, -1, -1, -1};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t >= op.m) continue;
        const int p = op.tpos[t];
        if (p < 0) {
          fixed_sub |= (int)((c.base >> (-p - 1)) & 1ULL) << t;
        } else {
          int s = -1;
#pragma unroll
          for (int i = 0; i < kRegBits; ++i)
            if (c.rb[i] == (1u << p)) s = i;
          if (s < 0) fixed_sub |= (int)((c.lt >> p) & 1u) << t;
          slot[t] = s;
        }
      }
      const double2* tab = data + op.data;
      if (op.m == 1 && slot[0] >= 0) {
        const double2 d0 = tab[0], d1 = tab[1];
        const int s0 = slot[0];
#pragma unroll
        for (int j = 0; j < kRegs; ++j) {
          const double2 w = cmul(v[j], ((j >> s0) & 1) ? d1 : d0);
          const bool ok = jcond(sc, j);
          v[j].x = ok ? w.x : v[j].x;
          v[j].y = ok ? w.y : v[j].y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < kRegs; ++j) {
          int sub = fixed_sub;
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (slot[t] >= 0) sub |= ((j >> slot[t]) & 1) << t;
          const double2 w = cmul(v[j], tab[sub]);
          const bool ok = jcond(sc, j);
          v[j].x = ok ? w.x : v[j].x;
          v[j].y = ok ? w.y : v[j].y;
        }
      }
      break;
    }
    case T_PARITY: {
      const double2 f0 = (data[op.data]), f1 = (data[op.data + 1]);
      // parity = tile part ^ thread part ^ register part
      int par0 = (__popcll(c.base & op.zg) ^ __popc(c.lt & op.zl)) & 1;
      uint32_t rz = 0;
#pragma unroll
      for (int i = 0; i < kRegBits; ++i)
        if (op.zl & c.rb[i]) rz |= 1u << i;
#pragma unroll
      for (int j = 0; j < kRegs; ++j) {
        const int p = (par0 ^ __popc((uint32_t)j & rz)) & 1;
        v[j] = cmul(v[j], p ? f1 : f0);
      }
      break;
    }
  }
}

// ---- shared-memory ops: a phase of their own, all threads over cosets
template <int K>
__device__ __forceinline__ void s_dense(double2* sm, int L, const TileOp& op,
                                        const double2* data, int tid) {
  constexpr int D = 1 << K;
  int sorted[K];
#pragma unroll
  for (int j = 0; j < K; ++j) sorted[j] = op.tpos[j];
#pragma unroll
  for (int i = 1; i < K; ++i)
#pragma unroll
    for (int j = K - 1; j >= i; --j)
      if (sorted[j - 1] > sorted[j]) {
        const int t = sorted[j];
        sorted[j] = sorted[j - 1];
        sorted[j - 1] = t;
      }
  const uint32_t ncos = 1u << (L - K);
  for (uint32_t cidx = tid; cidx < ncos; cidx += kGroupThreads) {
    uint32_t l0 = cidx;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t lo = l0 & ((1u << sorted[j]) - 1u);
      l0 = ((l0 ^ lo) << 1) | lo;
    }
    if (op.lmask && !lcond(op, l0)) continue;
    double2 in[D];
#pragma unroll
    for (int w = 0; w < D; ++w) {
      uint32_t l = l0;
#pragma unroll
      for (int j = 0; j < K; ++j)
        if ((w >> j) & 1) l |= 1u << op.tpos[j];
      in[w] = sm[swz(l)];
    }
#pragma unroll
    for (int z = 0; z < D; ++z) {
      double2 acc = cmul((data[op.data + z * D]), in[0]);
#pragma unroll
      for (int w = 1; w < D; ++w) acc = cfma((data[op.data + z * D + w]), in[w], acc);
      uint32_t l = l0;
#pragma unroll
      for (int j = 0; j < K; ++j)
        if ((z >> j) & 1) l |= 1u << op.tpos[j];
      sm[swz(l)] = acc;
    }
  }
}

__device__ __forceinline__ void s_pauli(double2* sm, int L, const TileOp& op,
                                        const double2* data, int tid, int gpar) {
  const uint32_t xml = (uint32_t)op.slots;
  const int pivot = 31 - __clz(xml);
  const double2 alpha = (data[op.data]), bph = (data[op.data + 1]);
  const uint32_t np = 1u << (L - 1);
  for (uint32_t p = tid; p < np; p += kGroupThreads) {
    const uint32_t lo = p & ((1u << pivot) - 1u);
    const uint32_t l = ((p ^ lo) << 1) | lo;
    const uint32_t q = l ^ xml;
    const double2 x = sm[swz(l)], y = sm[swz(q)];
    const int pl = (__popc(l & op.zl) ^ gpar) & 1;
    const int pq = (__popc(q & op.zl) ^ gpar) & 1;
    const double2 sy = pq ? make_double2(-y.x, -y.y) : y;
    const double2 sx = pl ? make_double2(-x.x, -x.y) : x;
    sm[swz(l)] = cfma(bph, sy, cmul(alpha, x));
    sm[swz(q)] = cfma(bph, sx, cmul(alpha, y));
  }
}

__device__ __noinline__ void s_apply(double2* sm, int L, const TileOp& op,
                                     const double2* data, uint64_t base, int tid) {
  if (op.gmask && ((base & op.gmask) != op.gval)) return;
  if (op.kind == S_PAULI) {
    s_pauli(sm, L, op, data, tid, __popcll(base & op.zg) & 1);
    return;
  }
  switch (op.m) {
    case 1: s_dense<1>(sm, L, op, data, tid); break;
    case 2: s_dense<2>(sm, L, op, data, tid); break;
    case 3: s_dense<3>(sm, L, op, data, tid); break;
    case 4: s_dense<4>(sm, L, op, data, tid); break;
  }
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kTidBits = kMaxTileQubits - kRegBits;  // log2(kGroupThreads)

// global offset of the local index bits above kTidBits (loop index k of the copies)
__device__ __forceinline__ uint64_t hi_part(const TilePassDev* pd, int L, int k) {
  uint64_t g = 0;
#pragma unroll
  for (int b = 0; b < kRegBits; ++b)
    if (kTidBits + b < L && ((k >> b) & 1)) g |= 1ULL << pd->spos[kTidBits + b];
  return g;
}

__device__ __forceinline__ void group_sync(int group) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "n"(kGroupThreads) : "memory");
}

// Persistent tile kernel.  Each CTA = kGroups groups of kGroupThreads threads;
// group g of CTA b walks tiles g + kGroups * (b + k * gridDim.x).  A group
// copies its tile HBM -> shared memory (cp.async, XOR-swizzled 16-byte
// slots), runs the phases with its own named barrier, and writes it back;
// the groups drift apart so copies/transposes of one overlap the math of the
// other.  The pass program is staged in shared memory once per CTA.
__global__ void __launch_bounds__(kCtaThreads, 1)
    k_tile(double2* __restrict__ a, const TilePassDev* __restrict__ pd,
           const TilePhase* __restrict__ phases, const TileOp* __restrict__ g_ops,
           const double2* __restrict__ g_data, FixedBits tb, uint64_t ntiles, int nops,
           int ndata) {
  extern __shared__ double2 smem_all[];
  __shared__ uint64_t s_hi[kRegs];       // HBM offset of copy-index bits >= kTidBits
  const int L = pd->L;
  const uint32_t tile_amps = 1u << L;
  const int group = threadIdx.x / kGroupThreads;
  const int tid = threadIdx.x % kGroupThreads;
  const int nphases = (pd->debug & 2) ? 0 : pd->nphases;
  const bool skip_ops = pd->debug & 1;
  const int dbg = pd->debug;
  // [tile g0][tile g1][ops][data][phases]
  TileOp* ops = reinterpret_cast<TileOp*>(smem_all + (size_t)kGroups * tile_amps);
  double2* data = reinterpret_cast<double2*>(ops + nops);
  TilePhase* s_ph = reinterpret_cast<TilePhase*>(data + ndata);
  {
    const int4* src = reinterpret_cast<const int4*>(g_ops);
    int4* dst = reinterpret_cast<int4*>(ops);
    for (int i = threadIdx.x; i < nops * (int)(sizeof(TileOp) / 16); i += kCtaThreads)
      dst[i] = src[i];
    for (int i = threadIdx.x; i < ndata; i += kCtaThreads) data[i] = g_data[i];
    const int words = pd->nphases * (int)(sizeof(TilePhase) / 4);
    const int* psrc = reinterpret_cast<const int*>(phases);
    int* pdst = reinterpret_cast<int*>(s_ph);
    for (int i = threadIdx.x; i < words; i += kCtaThreads) pdst[i] = psrc[i];
    if (threadIdx.x < kRegs) s_hi[threadIdx.x] = hi_part(pd, L, threadIdx.x);
  }
  // local bits below kTidBits of the copy index l = k * kGroupThreads + tid
  uint64_t lo_part = 0;
  for (int b = 0; b < kTidBits && b < L; ++b)
    if ((tid >> b) & 1) lo_part |= 1ULL << pd->spos[b];
  const int nk = (int)((tile_amps + kGroupThreads - 1) / kGroupThreads);
  const bool copy_thread = (uint32_t)tid < tile_amps;
  const int nthr = pd->nthrbits;
  const bool active = tid < (1 << nthr);
  double2* sm = smem_all + (size_t)group * tile_amps;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  __syncthreads();

  for (uint64_t tile = (uint64_t)blockIdx.x * kGroups + group; tile < ntiles;
       tile += (uint64_t)gridDim.x * kGroups) {
    const uint64_t base = widen(tile, tb);
    const uint64_t gb = base | lo_part;
    if (copy_thread) {
      for (int k = 0; k < nk; ++k) {
        const uint32_t l = (uint32_t)k * kGroupThreads + tid;
        cp_async16(sbase + swz(l) * 16u, a + (gb | s_hi[k]));
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    group_sync(group);

    for (int ph = 0; ph < nphases; ++ph) {
      const TilePhase& P = s_ph[ph];
      const int ob = P.op_begin, oe = P.op_end;
      if (P.type != 0) {
        for (int o = ob; o < (skip_ops ? ob : oe); ++o) {
          s_apply(sm, L, ops[o], data, base, tid);
          group_sync(group);
        }
        continue;
      }
      TileCtx c;
      c.base = base;
      c.lt = 0;
      for (int j = 0; j < nthr; ++j)
        if ((tid >> j) & 1) c.lt |= 1u << P.thrpos[j];
#pragma unroll
      for (int i = 0; i < kRegBits; ++i) c.rb[i] = 1u << P.regpos[i];
      if (active) {
        // the swizzle is XOR-linear: swz(lt | r) = swz(lt) ^ swz(r)
        uint32_t srb[kRegBits];
#pragma unroll
        for (int i = 0; i < kRegBits; ++i) srb[i] = swz(c.rb[i]);
        const uint32_t slt = swz(c.lt);
        double2 v[kRegs];
#pragma unroll
        for (int j = 0; j < kRegs; ++j) {
          uint32_t ad = slt;
#pragma unroll
          for (int i = 0; i < kRegBits; ++i)
            if ((j >> i) & 1) ad ^= srb[i];
          v[j] = sm[ad];
        }
        for (int o = ob; o < (skip_ops ? ob : oe); ++o) {
          const TileOp& op = ops[o];
          if (!((dbg & 4) && op.kind != T_DENSE1 && op.kind != T_DENSE1XR) &&
              !((dbg & 8) && (op.kind == T_DENSE1 || op.kind == T_DENSE1XR)))
            t_apply(v, c, op, data);
        }
#pragma unroll
        for (int j = 0; j < kRegs; ++j) {
          uint32_t ad = slt;
#pragma unroll
          for (int i = 0; i < kRegBits; ++i)
            if ((j >> i) & 1) ad ^= srb[i];
          sm[ad] = v[j];
        }
      }
      group_sync(group);
    }

    // shared -> HBM (same mapping as the load)
    if (copy_thread) {
      for (int k = 0; k < nk; ++k) {
        const uint32_t l = (uint32_t)k * kGroupThreads + tid;
        st1(a + (gb | s_hi[k]), sm[swz(l)]);
      }
    }
    group_sync(group);  // the tile buffer is refilled next iteration
  }
}

// ======================================================================= host

namespace {

struct M2 {
  Cplx m[4];
};

M2 mat_of_1q(const GateDesc& g) {
  // canonical 1-qubit uncontrolled gate -> 2x2
  M2 r;
  if (g.kind == QSV_OP_DENSE) {
    for (int i = 0; i < 4; ++i) r.m[i] = g.data[i];
  } else if (g.kind == QSV_OP_DIAG) {
    r.m[0] = g.data[0];
    r.m[1] = {0, 0};
    r.m[2] = {0, 0};
    r.m[3] = g.data[1];
  } else {  // PAULI, one target
    const int id = g.ids[0];
    Cplx z{0, 0}, one{1, 0};
    if (id == 1) r = {{z, one, one, z}};
    else if (id == 2) r = {{z, {0, -1}, {0, 1}, z}};
    else if (id == 3) r = {{one, z, z, {-1, 0}}};
    else r = {{one, z, z, one}};
  }
  return r;
}

Cplx cm(Cplx a, Cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
Cplx ca(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }

M2 mul(const M2& A, const M2& B) {  // A * B
  M2 r;
  r.m[0] = ca(cm(A.m[0], B.m[0]), cm(A.m[1], B.m[2]));
  r.m[1] = ca(cm(A.m[0], B.m[1]), cm(A.m[1], B.m[3]));
  r.m[2] = ca(cm(A.m[2], B.m[0]), cm(A.m[3], B.m[2]));
  r.m[3] = ca(cm(A.m[2], B.m[1]), cm(A.m[3], B.m[3]));
  return r;
}

bool is_zero(Cplx c) { return c.re == 0.0 && c.im == 0.0; }

bool is_1q(const GateDesc& g) {
  if (g.m != 1 || g.nc != 0) return false;
  return g.kind == QSV_OP_DENSE || g.kind == QSV_OP_DIAG || g.kind == QSV_OP_PAULI;
}

bool is_diagonal_gate(const GateDesc& g) {
  if (g.kind == QSV_OP_DIAG) return true;
  if (g.kind == QSV_OP_PAULI || g.kind == QSV_OP_PAULI_ROT) {
    for (int j = 0; j < g.m; ++j)
      if (g.ids[j] == 1 || g.ids[j] == 2) return false;
    return true;
  }
  return false;
}

GateDesc desc_from_m2(int q, const M2& M) {
  GateDesc g;
  memset(g.targets, 0, sizeof(g.targets));
  memset(g.ids, 0, sizeof(g.ids));
  memset(g.cq, 0, sizeof(g.cq));
  memset(g.cv, 0, sizeof(g.cv));
  g.m = 1;
  g.nc = 0;
  g.angle = 0;
  g.targets[0] = q;
  if (is_zero(M.m[1]) && is_zero(M.m[2])) {
    g.kind = QSV_OP_DIAG;
    g.data = {M.m[0], M.m[3]};
  } else {
    g.kind = QSV_OP_DENSE;
    g.data = {M.m[0], M.m[1], M.m[2], M.m[3]};
  }
  return g;
}

// Merge runs of uncontrolled 1-qubit gates on the same qubit into one 2x2
// (a pending product per qubit, flushed before the next gate that does not
// commute with it).  Diagonal pendings commute with diagonal gates.
std::vector<GateDesc> fuse_1q(int n, const std::vector<GateDesc>& in) {
  std::vector<GateDesc> out;
  std::vector<int> has(n, 0);
  std::vector<M2> pend(n);
  std::vector<int> pend_cnt(n, 0);
  auto pend_diag = [&](int q) { return is_zero(pend[q].m[1]) && is_zero(pend[q].m[2]); };
  auto flush = [&](int q) {
    if (!has[q]) return;
    out.push_back(canonicalize(desc_from_m2(q, pend[q])));
    if (out.back().nc < 0) out.pop_back();  // identity
    has[q] = 0;
    pend_cnt[q] = 0;
  };
  for (const GateDesc& g : in) {
    if (is_1q(g)) {
      const int q = g.targets[0];
      const M2 M = mat_of_1q(g);
      pend[q] = has[q] ? mul(M, pend[q]) : M;
      has[q] = 1;
      ++pend_cnt[q];
      continue;
    }
    const bool gdiag = is_diagonal_gate(g);
    auto touch = [&](int q) {
      if (has[q] && !(gdiag && pend_diag(q))) flush(q);
    };
    for (int j = 0; j < g.m; ++j) touch(g.targets[j]);
    for (int j = 0; j < g.nc; ++j) touch(g.cq[j]);
    out.push_back(g);
  }
  for (int q = 0; q < n; ++q) flush(q);
  return out;
}

// qubits that must be tile (local) qubits for the gate to run in a tile;
// returns false if the gate cannot run inside a tile at all
bool active_qubits(const GateDesc& g, uint64_t* act) {
  *act = 0;
  if (g.kind == QSV_OP_DENSE) {
    if (g.m > 4) return false;
    for (int j = 0; j < g.m; ++j) *act |= 1ULL << g.targets[j];
    return true;
  }
  if (g.kind == QSV_OP_DIAG) return g.m <= 4;
  if (g.kind == QSV_OP_PAULI || g.kind == QSV_OP_PAULI_ROT) {
    if (g.nc) return false;  // canonical controlled Paulis are dense
    for (int j = 0; j < g.m; ++j)
      if (g.ids[j] == 1 || g.ids[j] == 2) *act |= 1ULL << g.targets[j];
    return true;
  }
  return false;
}

uint64_t touched_mask(const GateDesc& g) {
  uint64_t m = 0;
  for (int j = 0; j < g.m; ++j) m |= 1ULL << g.targets[j];
  for (int j = 0; j < g.nc; ++j) m |= 1ULL << g.cq[j];
  return m;
}

int popc64(uint64_t x) { return __builtin_popcountll(x); }

struct PassSel {
  uint64_t S;                 // tile qubits
  std::vector<int> taken;     // indices into the gate list, in order
};

// Greedy pass: scan gates in order; take a gate when no deferred gate shares
// a qubit with it and its active qubits fit in S (growing S up to L).
PassSel select_pass(int n, int L, const std::vector<GateDesc>& gates,
                    const std::vector<uint64_t>& act, const std::vector<char>& ok,
                    const std::vector<char>& done, size_t first) {
  PassSel ps;
  const int c = std::min(kLowQubits, n);
  ps.S = (c >= 64) ? ~0ULL : ((1ULL << c) - 1);
  uint64_t blocked = 0;
  const uint64_t all = (n >= 64) ? ~0ULL : ((1ULL << n) - 1);
  size_t budget = kTileProgramBudget;  // staged program must fit in shared memory
  for (size_t i = first; i < gates.size(); ++i) {
    if (done[i]) continue;
    const GateDesc& g = gates[i];
    size_t cost = sizeof(TileOp) + sizeof(TilePhase) + 32;
    if (g.kind == QSV_OP_DENSE) cost += sizeof(double2) << (2 * g.m);
    if (g.kind == QSV_OP_DIAG) cost += sizeof(double2) << g.m;
    if (cost > budget) break;
    const uint64_t T = touched_mask(gates[i]);
    if (!ok[i] || (T & blocked)) {
      blocked |= T;
      if ((blocked & all) == all) break;
      continue;
    }
    const uint64_t A = act[i];
    if ((A & ~ps.S) == 0) {
      ps.taken.push_back((int)i);
      budget -= cost;
    } else if (popc64(ps.S | A) <= L) {
      ps.S |= A;
      ps.taken.push_back((int)i);
      budget -= cost;
    } else {
      blocked |= T;
      if ((blocked & all) == all) break;
    }
  }
  // pad S to exactly L qubits with the lowest unused qubits
  for (int q = 0; q < n && popc64(ps.S) < L; ++q) ps.S |= 1ULL << q;
  return ps;
}

void put(std::vector<char>& buf, size_t off, const void* src, size_t bytes) {
  if (buf.size() < off + bytes) buf.resize(off + bytes);
  memcpy(buf.data() + off, src, bytes);
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// choose thread-bit order: the first three lane bits should have distinct
// residues mod 3 so the XOR swizzle keeps 16-byte smem accesses conflict free
void order_thread_bits(std::vector<int>& tb) {
  for (size_t k = 0; k < 3 && k < tb.size(); ++k) {
    for (size_t j = k; j < tb.size(); ++j) {
      bool clash = false;
      for (size_t p = 0; p < k; ++p)
        if (tb[p] % 3 == tb[j] % 3) clash = true;
      if (!clash) {
        std::swap(tb[k], tb[j]);
        break;
      }
    }
  }
}

struct Encoded {
  TilePassDev pd;
  std::vector<TilePhase> phases;
  std::vector<TileOp> ops;
  std::vector<Cplx> data;
};

// Build phases and ops of one pass.
Encoded encode_pass(int n, int L, uint64_t S, const std::vector<const GateDesc*>& pg) {
  Encoded e;
  memset(&e.pd, 0, sizeof(e.pd));
  e.pd.L = L;
  e.pd.nthrbits = L - kRegBits;
  e.pd.smask = S;
  int local_of[64];
  for (int q = 0; q < 64; ++q) local_of[q] = -1;
  {
    int j = 0;
    for (int q = 0; q < n; ++q)
      if ((S >> q) & 1ULL) {
        e.pd.spos[j] = q;
        local_of[q] = j++;
      }
  }
  // current register phase
  bool open = false;
  uint32_t R = 0;
  size_t op_begin = 0;
  std::vector<std::pair<size_t, int>> d1;  // (op index, local bit) of T_DENSE1 ops
  auto close = [&]() {
    if (!open) return;
    // register slots in order of first use by a 1-qubit dense op, so runs of
    // such ops land on slots 0, 1, ... and can be batched
    std::vector<int> order;
    for (auto& pr : d1)
      if (std::find(order.begin(), order.end(), pr.second) == order.end())
        order.push_back(pr.second);
    for (int b = 0; b < L; ++b)
      if (((R >> b) & 1u) && std::find(order.begin(), order.end(), b) == order.end())
        order.push_back(b);
    for (int b = L - 1; b >= 0 && (int)order.size() < kRegBits; --b)
      if (std::find(order.begin(), order.end(), b) == order.end()) order.push_back(b);
    uint32_t Rall = 0;
    for (int b : order) Rall |= 1u << b;
    TilePhase ph;
    memset(&ph, 0, sizeof(ph));
    ph.type = 0;
    int slot_of[32];
    for (int b = 0; b < 32; ++b) slot_of[b] = -1;
    for (int i = 0; i < kRegBits; ++i) {
      ph.regpos[i] = order[i];
      slot_of[order[i]] = i;
    }
    std::vector<int> tb;
    for (int b = 0; b < L; ++b)
      if (!((Rall >> b) & 1u)) tb.push_back(b);
    order_thread_bits(tb);
    for (size_t k = 0; k < tb.size(); ++k) ph.thrpos[k] = tb[k];
    for (auto& pr : d1) e.ops[pr.first].slots = 1 << slot_of[pr.second];
    // batch runs of >= 2 uncontrolled 1-qubit dense ops on slots 0, 1, ... in order
    {
      std::vector<TileOp> merged;
      const size_t end = e.ops.size();
      size_t k = op_begin;
      while (k < end) {
        int len = 0;
        while (k + len < end && len < kRegBits) {
          const TileOp& o = e.ops[k + len];
          if (!(o.kind == T_DENSE1 && o.slots == (1 << len) && o.lmask == 0 && o.gmask == 0 &&
                o.data == e.ops[k].data + 4 * len))
            break;
          ++len;
        }
        if (len >= 2) {
          TileOp b = e.ops[k];
          b.kind = T_DENSE1XR;
          b.m = len;
          b.slots = (1 << len) - 1;
          merged.push_back(b);
          k += len;
        } else {
          merged.push_back(e.ops[k]);
          ++k;
        }
      }
      e.ops.resize(op_begin);
      e.ops.insert(e.ops.end(), merged.begin(), merged.end());
    }
    ph.op_begin = (int)op_begin;
    ph.op_end = (int)e.ops.size();
    e.phases.push_back(ph);
    open = false;
    R = 0;
    d1.clear();
  };
  auto open_reg = [&]() {
    if (open) return;
    open = true;
    R = 0;
    op_begin = e.ops.size();
  };
  for (const GateDesc* gp : pg) {
    const GateDesc& g = *gp;
    TileOp op;
    memset(&op, 0, sizeof(op));
    for (int c = 0; c < g.nc; ++c) {
      const int q = g.cq[c];
      if (local_of[q] >= 0) {
        op.lmask |= 1u << local_of[q];
        if (g.cv[c]) op.lval |= 1u << local_of[q];
      } else {
        op.gmask |= 1ULL << q;
        if (g.cv[c]) op.gval |= 1ULL << q;
      }
    }
    op.data = (uint32_t)e.data.size();
    if (g.kind == QSV_OP_DENSE && g.m == 1) {
      const int b = local_of[g.targets[0]];
      open_reg();
      if (!((R >> b) & 1u) && __builtin_popcount(R) >= kRegBits) {
        close();
        open_reg();
      }
      R |= 1u << b;
      op.kind = T_DENSE1;
      const Cplx* M = g.data.data();
      if (is_zero(M[0]) && is_zero(M[3]) && M[1].re == 1.0 && M[1].im == 0.0 &&
          M[2].re == 1.0 && M[2].im == 0.0)
        op.flags |= 1;
      e.data.insert(e.data.end(), g.data.begin(), g.data.end());
      d1.push_back({e.ops.size(), b});
      e.ops.push_back(op);
      continue;
    }
    if (g.kind == QSV_OP_DENSE) {  // m = 2..4: shared-memory op
      close();
      op.kind = S_DENSE;
      op.m = g.m;
      for (int t = 0; t < g.m; ++t) op.tpos[t] = local_of[g.targets[t]];
      e.data.insert(e.data.end(), g.data.begin(), g.data.end());
      TilePhase ph;
      memset(&ph, 0, sizeof(ph));
      ph.type = 1;
      ph.op_begin = (int)e.ops.size();
      e.ops.push_back(op);
      ph.op_end = (int)e.ops.size();
      e.phases.push_back(ph);
      continue;
    }
    if (g.kind == QSV_OP_DIAG) {
      open_reg();
      if (g.m == 0) {
        op.kind = T_PHASE;
        const Cplx f = g.data[0];
        if (f.re == -1.0 && f.im == 0.0) op.flags |= 2;
        e.data.push_back(f);
      } else {
        op.kind = T_DIAG;
        op.m = g.m;
        for (int t = 0; t < g.m; ++t) {
          const int q = g.targets[t];
          op.tpos[t] = local_of[q] >= 0 ? local_of[q] : -(q + 1);
        }
        e.data.insert(e.data.end(), g.data.begin(), g.data.end());
      }
      e.ops.push_back(op);
      continue;
    }
    // PAULI / PAULI_ROT, uncontrolled
    uint64_t xm = 0, zm = 0;
    int ny = 0;
    for (int t = 0; t < g.m; ++t) {
      const int id = g.ids[t];
      if (id == 1 || id == 2) xm |= 1ULL << g.targets[t];
      if (id == 2 || id == 3) zm |= 1ULL << g.targets[t];
      if (id == 2) ++ny;
    }
    Cplx alpha{0, 0}, beta{1, 0};
    if (g.kind == QSV_OP_PAULI_ROT) {
      alpha = {std::cos(g.angle / 2), 0};
      beta = {0, std::sin(g.angle / 2)};
    }
    static const Cplx ip[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    const Cplx bph = cm(beta, ip[ny & 3]);
    for (int q = 0; q < n; ++q)
      if ((zm >> q) & 1ULL) {
        if (local_of[q] >= 0) op.zl |= 1u << local_of[q];
        else op.zg |= 1ULL << q;
      }
    if (xm == 0) {
      open_reg();
      op.kind = T_PARITY;
      e.data.push_back(ca(alpha, bph));
      e.data.push_back({alpha.re - bph.re, alpha.im - bph.im});
      e.ops.push_back(op);
      continue;
    }
    close();
    op.kind = S_PAULI;
    uint32_t xl = 0;
    for (int q = 0; q < n; ++q)
      if ((xm >> q) & 1ULL) xl |= 1u << local_of[q];
    op.slots = (int32_t)xl;
    e.data.push_back(alpha);
    e.data.push_back(bph);
    TilePhase ph;
    memset(&ph, 0, sizeof(ph));
    ph.type = 1;
    ph.op_begin = (int)e.ops.size();
    e.ops.push_back(op);
    ph.op_end = (int)e.ops.size();
    e.phases.push_back(ph);
  }
  close();
  e.pd.nphases = (int)e.phases.size();
  if (const char* dbg = getenv("QSV_TILE_DEBUG")) e.pd.debug = atoi(dbg);
  return e;
}

// FP64 flops of one gate applied to a 2^n state (2 per FMA): a complex
// multiply-add is 8 flops, a complex multiply 6, a sign flip 0.
double gate_fp64_flops(int n, const GateDesc& g) {
  const double amps = std::ldexp(1.0, n - g.nc);
  if (g.kind == QSV_OP_DENSE) return amps * 8.0 * (double)(1 << g.m);
  if (g.kind == QSV_OP_DIAG) {
    if (g.m == 0 && g.data.size() == 1 && g.data[0].re == -1.0 && g.data[0].im == 0.0) return 0.0;
    return amps * 6.0;
  }
  return std::ldexp(1.0, n) * 14.0;  // Pauli rotation: alpha*x + beta*phase*y
}

void add_gate_step(int n, const GateDesc& g, std::vector<Step>& steps, std::vector<char>& payload,
                   qsv_program_stats* stats) {
  Step st;
  st.type = 0;
  st.gate = g;
  st.tile = -1;
  std::vector<char> pl = make_payload(g);
  st.has_payload = !pl.empty();
  st.payload_off = 0;
  if (st.has_payload) {
    const size_t off = align_up(payload.size(), 256);
    put(payload, off, pl.data(), pl.size());
    st.payload_off = off;
  }
  steps.push_back(st);
  stats->num_gate_kernels += 1;
  stats->num_steps += 1;
  stats->hbm_bytes += gate_hbm_bytes(n, g);
  stats->fp64_flops += gate_fp64_flops(n, g);
}

}  // namespace

int plan_program(int n, const std::vector<GateDesc>& gates_in, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats) {
  std::vector<GateDesc> gates = opts.fuse ? fuse_1q(n, gates_in) : gates_in;
  int L = opts.tile_qubits > 0 ? opts.tile_qubits : kMaxTileQubits;
  L = std::min(std::min(L, kMaxTileQubits), n);
  const bool tiles_on = opts.use_tiles && n >= kRegBits + 1 && L >= kRegBits + 1;
  if (!tiles_on) {
    for (const GateDesc& g : gates) add_gate_step(n, g, steps, payload, stats);
    return QSV_OK;
  }
  const size_t G = gates.size();
  std::vector<uint64_t> act(G, 0);
  std::vector<char> ok(G, 0), done(G, 0);
  for (size_t i = 0; i < G; ++i) ok[i] = active_qubits(gates[i], &act[i]) && popc64(act[i]) <= L;
  size_t first = 0;
  while (true) {
    while (first < G && done[first]) ++first;
    if (first >= G) break;
    if (!ok[first]) {
      add_gate_step(n, gates[first], steps, payload, stats);
      done[first] = 1;
      continue;
    }
    PassSel ps = select_pass(n, L, gates, act, ok, done, first);
    if (ps.taken.size() == 1) {
      // a lone gate is cheaper as its own streaming kernel
      add_gate_step(n, gates[ps.taken[0]], steps, payload, stats);
      done[ps.taken[0]] = 1;
      continue;
    }
    std::vector<const GateDesc*> pg;
    for (int k : ps.taken) {
      pg.push_back(&gates[k]);
      done[k] = 1;
    }
    Encoded e = encode_pass(n, L, ps.S, pg);
    TilePlan tp;
    tp.L = L;
    for (int q = 0; q < n; ++q)
      if ((ps.S >> q) & 1ULL) tp.qubits.push_back(q);
    tp.nphases = (int)e.phases.size();
    tp.nops = (int)e.ops.size();
    tp.ndata = (int)e.data.size();
    tp.num_gates = (int)pg.size();
    tp.hbm_bytes = 32.0 * std::ldexp(1.0, n);
    for (const GateDesc* gp : pg) stats->fp64_flops += gate_fp64_flops(n, *gp);
    // payload: [TilePassDev][phases][ops][data]
    size_t off = align_up(payload.size(), 256);
    tp.dev_off = off;
    put(payload, off, &e.pd, sizeof(e.pd));
    off = align_up(off + sizeof(e.pd), 16);
    put(payload, off, e.phases.data(), e.phases.size() * sizeof(TilePhase));
    off = align_up(off + e.phases.size() * sizeof(TilePhase), 16);
    put(payload, off, e.ops.data(), e.ops.size() * sizeof(TileOp));
    off = align_up(off + e.ops.size() * sizeof(TileOp), 16);
    put(payload, off, e.data.data(), std::max<size_t>(1, e.data.size()) * sizeof(Cplx));
    Step st;
    st.type = 1;
    st.tile = (int)tiles.size();
    st.has_payload = true;
    st.payload_off = tp.dev_off;
    tiles.push_back(tp);
    steps.push_back(st);
    stats->num_tile_passes += 1;
    stats->num_steps += 1;
    stats->hbm_bytes += tp.hbm_bytes;
  }
  return QSV_OK;
}

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s) {
  const char* basep = (const char*)dev_payload + tp.dev_off;
  size_t off = align_up(sizeof(TilePassDev), 16);
  const TilePassDev* pd = reinterpret_cast<const TilePassDev*>(basep);
  const TilePhase* ph = reinterpret_cast<const TilePhase*>(basep + off);
  off = align_up(off + tp.nphases * sizeof(TilePhase), 16);
  const TileOp* ops = reinterpret_cast<const TileOp*>(basep + off);
  off = align_up(off + tp.nops * sizeof(TileOp), 16);
  const double2* data = reinterpret_cast<const double2*>(basep + off);
  int pos[kMaxTileQubits];
  for (int j = 0; j < tp.L; ++j) pos[j] = tp.qubits[j];
  FixedBits tb = make_fixed(pos, tp.L, 0);
  const size_t smem = kGroups * (sizeof(double2) << tp.L) + tp.nops * sizeof(TileOp) +
                      tp.ndata * sizeof(double2) + tp.nphases * sizeof(TilePhase);
  if (smem > kTileSmemLimit) {
    set_error("tile pass program (%d ops, %d phases) does not fit in shared memory", tp.nops,
              tp.nphases);
    return QSV_EUNSUPPORTED;
  }
  static int attr_dev = -1;
  static int num_sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    QSV_TRY(cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kTileSmemLimit));
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    attr_dev = dev;
  }
  const uint64_t ntiles = 1ULL << (n - tp.L);
  const uint64_t ctas = (ntiles + kGroups - 1) / kGroups;
  const unsigned grid = (unsigned)std::min<uint64_t>(ctas, (uint64_t)num_sms);
  k_tile<<<grid, kCtaThreads, smem, s>>>(amps, pd, ph, ops, data, tb, ntiles, tp.nops,
                                          tp.ndata);
  QSV_CHECK_LAUNCH("k_tile");
  return QSV_OK;
}

}  // namespace qsv
