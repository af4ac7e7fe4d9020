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
#include <stdexcept>
#include <mutex>
#include <string>
#include <unordered_map>

#include "qsv_tile.cuh"

#ifndef QSV_TILE_REGBITS
#error "qsv_tile_impl.cuh is included by qsv_tile_r4.cu / qsv_tile_r5.cu"
#endif

namespace qsv {
namespace QSV_TILE_NS {

constexpr int kRegBits = QSV_TILE_REGBITS;  // amplitudes per thread = 2^kRegBits
constexpr int kRegs = 1 << kRegBits;
constexpr int kGroupThreads = (1 << kMaxTileQubits) / kRegs;  // threads per tile group
#ifndef QSV_TILE_GROUPS
#define QSV_TILE_GROUPS 2
#endif
// widest dense gate run inside a tile pass (shared-memory phase).  5-target
// blocks stay standalone (k_dense5 is FP64-bound either way, and a 32-input
// s_dense in the same kernel raises the interpreter's register spills).
#ifndef QSV_TILE_MAX_DENSE
#define QSV_TILE_MAX_DENSE 4
#endif
constexpr int kGroups = QSV_TILE_GROUPS;  // independent tile groups per CTA
constexpr int kCtaThreads = kGroups * kGroupThreads;
// shared memory left for the staged pass program (ops, data, phases)
constexpr int kTileProgramBudget =
    kTileSmemLimit - kGroups * (16 << kMaxTileQubits) - 1024;

// ===================================================================== device

__device__ __forceinline__ uint32_t swz(uint32_t l) {
  return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u);
}

// Register-phase ops arrive in "slot space" (the encoder rewrites them when
// the phase's register slots are known): a control / pattern over local bits
// is split into its thread part (lmask, lval over the non-register local
// bits) and its register part (zl = rm | rv << 16 over slots), so a thread
// needs only its tile base and its thread bits.
struct TileCtx {
  uint64_t base;       // global bits of this tile
  uint32_t lt;         // thread's local base (thread bits placed)
};

__device__ __forceinline__ bool lcond(const TileOp& op, uint32_t l) {
  return (l & op.lmask) == op.lval;
}

struct SplitCond {
  bool t_ok;
  uint32_t rm, rv;  // over register slots
};

__device__ __forceinline__ SplitCond split_cond(const TileCtx& c, const TileOp& op) {
  SplitCond sc;
  sc.rm = op.zl & 0xffffu;
  sc.rv = op.zl >> 16;
  sc.t_ok = (c.lt & op.lmask) == op.lval;
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
  if (op.lmask | op.zl) {
    sc = split_cond(c, op);
    if (!sc.t_ok) return;
  }
  if (sc.rm)
    t_dense1_body<I, true>(v, sc, m00, m01, m10, m11);
  else
    t_dense1_body<I, false>(v, sc, m00, m01, m10, m11);
}

// real 2x2 [[a, b], [c, d]]: 4 FP64 ops per amplitude instead of 8
template <int I, bool CTRL>
__device__ __forceinline__ void t_real1_body(double2 (&v)[kRegs], const SplitCond& sc, double a,
                                             double b, double c, double d) {
#pragma unroll
  for (int j = 0; j < kRegs; ++j) {
    if ((j >> I) & 1) continue;
    const int q = j | (1 << I);
    const double2 x = v[j], y = v[q];
    const double2 nx = make_double2(fma(b, y.x, a * x.x), fma(b, y.y, a * x.y));
    const double2 ny = make_double2(fma(d, y.x, c * x.x), fma(d, y.y, c * x.y));
    if (CTRL) {
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

// X on a register slot: a predicated swap, no arithmetic
template <int I>
__device__ __forceinline__ void t_swap_body(double2 (&v)[kRegs], const SplitCond& sc) {
#pragma unroll
  for (int j = 0; j < kRegs; ++j) {
    if ((j >> I) & 1) continue;
    const int q = j | (1 << I);
    const double2 x = v[j], y = v[q];
    const bool ok = jcond(sc, j);
    v[j].x = ok ? y.x : x.x;
    v[j].y = ok ? y.y : x.y;
    v[q].x = ok ? x.x : y.x;
    v[q].y = ok ? x.y : y.y;
  }
}

template <int I>
__device__ __forceinline__ void t_real1(double2 (&v)[kRegs], const TileCtx& c, const TileOp& op,
                                        const double2* data) {
  SplitCond sc{true, 0, 0};
  if (op.lmask | op.zl) {
    sc = split_cond(c, op);
    if (!sc.t_ok) return;
  }
  if (op.flags & 1) {  // X
    t_swap_body<I>(v, sc);
    return;
  }
  const double2 ab = data[op.data], cd = data[op.data + 1];
  if (sc.rm)
    t_real1_body<I, true>(v, sc, ab.x, ab.y, cd.x, cd.y);
  else
    t_real1_body<I, false>(v, sc, ab.x, ab.y, cd.x, cd.y);
}

template <int NS>
__device__ __forceinline__ void t_real_prefix(double2 (&v)[kRegs], const double2* M) {
  const SplitCond sc{true, 0, 0};
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const double2 ab = M[2 * i], cd = M[2 * i + 1];
    switch (i) {
      case 0: t_real1_body<0, false>(v, sc, ab.x, ab.y, cd.x, cd.y); break;
      case 1: t_real1_body<1 % kRegBits, false>(v, sc, ab.x, ab.y, cd.x, cd.y); break;
      case 2: t_real1_body<2 % kRegBits, false>(v, sc, ab.x, ab.y, cd.x, cd.y); break;
      case 3: t_real1_body<3 % kRegBits, false>(v, sc, ab.x, ab.y, cd.x, cd.y); break;
      default: t_real1_body<4 % kRegBits, false>(v, sc, ab.x, ab.y, cd.x, cd.y); break;
    }
  }
}

// batched uncontrolled 1-qubit ops on the slots of a mask (slot order)
__device__ __forceinline__ void t_real1x(double2 (&v)[kRegs], const TileOp& op,
                                         const double2* data) {
  const double2* M = data + op.data;
  const SplitCond sc{true, 0, 0};
  const int s = op.slots;
#define QSV_REAL_SLOT(I)                                                   \
  if ((s >> (I)) & 1) {                                                    \
    const double2 ab = M[0], cd = M[1];                                    \
    t_real1_body<(I) % kRegBits, false>(v, sc, ab.x, ab.y, cd.x, cd.y);    \
    M += 2;                                                                \
  }
  // prefix masks (slots 0..m-1, the usual shape: slots are assigned in order
  // of first use) run as straight-line code, no merges of v after branches
  switch (s) {
    case (1 << kRegBits) - 1: t_real_prefix<kRegBits>(v, M); return;
    case (1 << (kRegBits - 1)) - 1: t_real_prefix<kRegBits - 1>(v, M); return;
    case (1 << (kRegBits - 2)) - 1: t_real_prefix<kRegBits - 2>(v, M); return;
    default: break;
  }
  QSV_REAL_SLOT(0) QSV_REAL_SLOT(1) QSV_REAL_SLOT(2) QSV_REAL_SLOT(3) QSV_REAL_SLOT(4)
#undef QSV_REAL_SLOT
}

__device__ __forceinline__ void t_dense1x(double2 (&v)[kRegs], const TileOp& op,
                                          const double2* data) {
  const double2* M = data + op.data;
  const SplitCond sc{true, 0, 0};
  const int s = op.slots;
#define QSV_DENSE_SLOT(I)                                                  \
  if ((s >> (I)) & 1) {                                                    \
    t_dense1_body<(I) % kRegBits, false>(v, sc, M[0], M[1], M[2], M[3]);   \
    M += 4;                                                                \
  }
  QSV_DENSE_SLOT(0) QSV_DENSE_SLOT(1) QSV_DENSE_SLOT(2) QSV_DENSE_SLOT(3) QSV_DENSE_SLOT(4)
#undef QSV_DENSE_SLOT
}

// sign flip of amplitude slot J when bit J of `bits` is set: one shift and
// two LOP3 on the integer pipe, no FP64 work
template <int J>
__device__ __forceinline__ double2 neg_bit(double2 v, uint32_t bits) {
  const int s = (int)((bits << (31 - J)) & 0x80000000u);
  return make_double2(__hiloint2double(__double2hiint(v.x) ^ s, __double2loint(v.x)),
                      __hiloint2double(__double2hiint(v.y) ^ s, __double2loint(v.y)));
}

template <int J>
struct NegAll {
  __device__ __forceinline__ static void run(double2 (&v)[kRegs], uint32_t bits) {
    NegAll<J - 1>::run(v, bits);
    v[J] = neg_bit<J>(v[J], bits);
  }
};
template <>
struct NegAll<0> {
  __device__ __forceinline__ static void run(double2 (&v)[kRegs], uint32_t bits) {
    v[0] = neg_bit<0>(v[0], bits);
  }
};

// merged diagonal: v[j] *= T[j] * C(thread) * (-1)^(sign(j, thread))
__device__ __forceinline__ uint32_t flush_sign_bits(const TileCtx& c, const FlushSign* sg, int nr,
                                                    uint32_t bits) {
  for (int r = 0; r < nr; ++r) {
    const FlushSign R = sg[r];
    if ((c.lt & R.lm) == R.lv && (c.base & R.gm) == R.gv) bits ^= R.col;
  }
  return bits;
}

// merged diagonal with a table: v[j] *= T[j] * C(thread) * (-1)^(sign(j, thread))
// (straight-line: the multiply and the sign pass always run)
__device__ __forceinline__ void t_flush(double2 (&v)[kRegs], const TileCtx& c, const TileOp& op,
                                        const double2* data) {
  const double2* T = data + op.data;
  const FlushSign* sg = reinterpret_cast<const FlushSign*>(T + kRegs);
  const uint32_t bits = flush_sign_bits(c, sg, op.m, 0u);
  if (op.slots) {  // per-thread factors of non-register qubits (rare)
    const FlushFactor* fc = reinterpret_cast<const FlushFactor*>(sg + op.m);
    double2 C = make_double2(1.0, 0.0);
    for (int f = 0; f < op.slots; ++f) {
      const int p = fc[f].pos;
      const int bit = p >= 0 ? (int)((c.lt >> p) & 1u) : (int)((c.base >> (-p - 1)) & 1ULL);
      C = cmul(C, bit ? fc[f].d1 : fc[f].d0);
    }
#pragma unroll
    for (int j = 0; j < kRegs; ++j) v[j] = cmul(v[j], C);
  }
#pragma unroll
  for (int j = 0; j < kRegs; ++j) v[j] = cmul(v[j], T[j]);
  if (bits) NegAll<kRegs - 1>::run(v, bits);
}

// merged phase rules: per-thread scalar C and per-slot factors ph[i] (on the
// amplitudes whose slot i is 1): 4 FP64 ops per amplitude for the scalar and
// 2 per slot, however many controlled phases were merged
__device__ __forceinline__ void t_phases(double2 (&v)[kRegs], const TileCtx& c, const TileOp& op,
                                         const double2* data) {
  const FlushPhase* pr = reinterpret_cast<const FlushPhase*>(data + op.data);
  double2 C = make_double2(1.0, 0.0);
  double2 ph[kRegBits];
#pragma unroll
  for (int i = 0; i < kRegBits; ++i) ph[i] = make_double2(1.0, 0.0);
  for (int r = 0; r < op.m; ++r) {
    const FlushPhase R = pr[r];
    if ((c.lt & R.lm) != R.lv || (c.base & R.gm) != R.gv) continue;
    switch (R.slot) {
      case 0: ph[0] = cmul(ph[0], R.f); break;
      case 1: ph[1 % kRegBits] = cmul(ph[1 % kRegBits], R.f); break;
      case 2: ph[2 % kRegBits] = cmul(ph[2 % kRegBits], R.f); break;
      case 3: ph[3 % kRegBits] = cmul(ph[3 % kRegBits], R.f); break;
      case 4: ph[4 % kRegBits] = cmul(ph[4 % kRegBits], R.f); break;
      default: C = cmul(C, R.f); break;
    }
  }
  if (op.flags & 1) {
#pragma unroll
    for (int j = 0; j < kRegs; ++j) v[j] = cmul(v[j], C);
  }
#pragma unroll
  for (int i = 0; i < kRegBits; ++i) {
    if (!((op.slots >> i) & 1)) continue;
#pragma unroll
    for (int j = 0; j < kRegs; ++j)
      if ((j >> i) & 1) v[j] = cmul(v[j], ph[i]);
  }
}

// sign-only merged diagonal (CZ-type patterns): integer XORs, no FP64 work
__device__ __forceinline__ void t_signs(double2 (&v)[kRegs], const TileCtx& c, const TileOp& op,
                                        const double2* data) {
  const FlushSign* sg = reinterpret_cast<const FlushSign*>(data + op.data);
  const uint32_t bits = flush_sign_bits(c, sg, op.m, op.lmask);
  NegAll<kRegs - 1>::run(v, bits);
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
    case T_REAL1:
      switch (op.slots) {
        case 1: t_real1<0>(v, c, op, data); break;
        case 2: t_real1<1 % kRegBits>(v, c, op, data); break;
        case 4: t_real1<2 % kRegBits>(v, c, op, data); break;
        case 8: t_real1<3 % kRegBits>(v, c, op, data); break;
        case 16: t_real1<4 % kRegBits>(v, c, op, data); break;
      }
      break;
    case T_REAL1X:
      t_real1x(v, op, data);
      break;
    case T_DENSE1X:
      t_dense1x(v, op, data);
      break;
    case T_FLUSH:
      t_flush(v, c, op, data);
      break;
    case T_SIGNS:
      t_signs(v, c, op, data);
      break;
    case T_PHASES:
      t_phases(v, c, op, data);
      break;
    case T_PHASE: {
      const SplitCond sc = split_cond(c, op);
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
      const SplitCond sc = split_cond(c, op);
      if (!sc.t_ok) break;
      // per target: register slot (0..7), thread bit (8 + bit) or tile bit (< 0)
      int fixed_sub = 0;
      int slot[4] = {-1, -1, -1, -1};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t >= op.m) continue;
        const int p = op.tpos[t];
        if (p < 0) fixed_sub |= (int)((c.base >> (-p - 1)) & 1ULL) << t;
        else if (p >= 8) fixed_sub |= (int)((c.lt >> (p - 8)) & 1u) << t;
        else slot[t] = p;
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
      const uint32_t rz = (uint32_t)op.m;  // register part (slot mask)
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
#pragma unroll(K >= 5 ? 1 : D)  // 5 targets: keep the 32 inputs + one row live only
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
#if QSV_TILE_MAX_DENSE >= 5
    case 5: s_dense<5>(sm, L, op, data, tid); break;
#endif
  }
}

// One register phase of one thread: load its 2^kRegBits amplitudes from the
// tile in shared memory, run the phase's ops in registers, store them back.
__device__ __forceinline__ void reg_phase(double2* sm, const TilePhase& P, const TileOp* ops,
                                       const double2* data, uint64_t base, int tid, int nthr,
                                       bool skip_ops, int dbg) {
  TileCtx c;
  c.base = base;
  c.lt = P.thr_lo[tid & 15] | P.thr_hi[(tid >> 4) & 15];
  // the swizzle is XOR-linear: swz(lt | r) = swz(lt) ^ swz(r)
  uint32_t srb[kRegBits];
#pragma unroll
  for (int i = 0; i < kRegBits; ++i) srb[i] = swz(1u << P.regpos[i]);
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
  const int ob = P.op_begin, oe = skip_ops ? P.op_begin : P.op_end;
  for (int o = ob; o < oe; ++o) {
    const TileOp& op = ops[o];
    const bool dense1 = op.kind == T_DENSE1 || op.kind == T_DENSE1X || op.kind == T_REAL1 ||
                        op.kind == T_REAL1X;
    if (!((dbg & 4) && !dense1) && !((dbg & 8) && dense1)) t_apply(v, c, op, data);
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
// a group takes its next tile from a global work counter (ctr[0], fetched one
// tile ahead so the atomic's latency hides behind the current tile), so CTAs
// that become resident late -- e.g. while an exchange kernel holds some SMs
// (dist.py overlap) -- simply process fewer tiles.  The last CTA to finish
// resets both counters (ctr[1] counts finished CTAs) for the next launch on
// the stream.  A group
// copies its tile HBM -> shared memory (cp.async, XOR-swizzled 16-byte
// slots), runs the phases with its own named barrier, and writes it back;
// the groups drift apart so copies/transposes of one overlap the math of the
// other.  The pass program is staged in shared memory once per CTA.
__global__ void __launch_bounds__(kCtaThreads, 1)
    k_tile(double2* __restrict__ a, const TilePassDev* __restrict__ pd,
           const TilePhase* __restrict__ phases, const TileOp* __restrict__ g_ops,
           const double2* __restrict__ g_data, FixedBits tb, uint64_t ntiles, int nops,
           int ndata, unsigned long long* __restrict__ ctr, int nostagger) {
  extern __shared__ double2 smem_all[];
  __shared__ unsigned long long s_next[kGroups];
  __shared__ uint64_t s_hi[kRegs + 1];   // HBM offset of copy-index bits >= kTidBits (+ flag)
  __shared__ uint64_t s_lo[kCtaThreads]; // HBM offset of copy-index bits < kTidBits
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
  // local bits below kTidBits of the copy index l = k * kGroupThreads + tid,
  // kept in shared memory (re-read per copy) rather than in registers
  {
    uint64_t lo_part = 0;
    for (int b = 0; b < kTidBits && b < L; ++b)
      if ((tid >> b) & 1) lo_part |= 1ULL << pd->spos[b];
    s_lo[threadIdx.x] = lo_part;
  }
  const int nk = (int)((tile_amps + kGroupThreads - 1) / kGroupThreads);
  const bool copy_thread = (uint32_t)tid < tile_amps;
  const int nthr = pd->nthrbits;
  const bool active = tid < (1 << nthr);
  double2* sm = smem_all + (size_t)group * tile_amps;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  // Stagger: the two groups run identical work, so started together they
  // stay in lockstep and load / store their tiles at the same time, leaving
  // the FP64 pipe idle meanwhile.  Group 1 starts once group 0 is half way
  // through its first tile, so one group's HBM traffic overlaps the other's
  // math from then on.
  volatile int* s_go = reinterpret_cast<volatile int*>(&s_hi[kRegs]);
  if (threadIdx.x == 0) *s_go = (kGroups < 2 || nostagger || (pd->debug & 16)) ? kGroups : 0;
  __syncthreads();
  if (group > 0)
    while (*s_go < group) __nanosleep(256);
  bool first = true;

  if (tid == 0) s_next[group] = atomicAdd(ctr, 1ULL);
  group_sync(group);
  uint64_t tile = s_next[group];
  while (tile < ntiles) {
    unsigned long long next = 0;
    if (tid == 0) next = atomicAdd(ctr, 1ULL);  // the group's following tile
    const uint64_t base = widen(tile, tb);
    if (copy_thread) {
      const uint64_t gb = base | s_lo[threadIdx.x];
      if (L == kMaxTileQubits) {
        // full tile: unrolled, swz(k * G + tid) = swz(k * G) ^ swz(tid) (XOR-linear)
        const uint32_t st = swz((uint32_t)tid);
#pragma unroll
        for (int k = 0; k < kRegs; ++k)
          cp_async16(sbase + ((swz((uint32_t)k * kGroupThreads) ^ st) << 4), a + (gb | s_hi[k]));
      } else {
        for (int k = 0; k < nk; ++k) {
          const uint32_t l = (uint32_t)k * kGroupThreads + tid;
          cp_async16(sbase + swz(l) * 16u, a + (gb | s_hi[k]));
        }
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    group_sync(group);

    for (int ph = 0; ph < nphases; ++ph) {
      // release group k once group 0 is k / kGroups of the way through its first tile
      if (group == 0 && first && tid == 0 && ph * kGroups >= (*s_go + 1) * nphases &&
          *s_go < kGroups - 1)
        *s_go = *s_go + 1;
      const TilePhase& P = s_ph[ph];
      const int ob = P.op_begin, oe = P.op_end;
      if (P.type != 0) {
        for (int o = ob; o < (skip_ops ? ob : oe); ++o) {
          s_apply(sm, L, ops[o], data, base, tid);
          group_sync(group);
        }
        continue;
      }
      if (active) reg_phase(sm, P, ops, data, base, tid, nthr, skip_ops, dbg);
      group_sync(group);
    }

    // shared -> HBM (same mapping as the load)
    if (copy_thread) {
      const uint64_t gb = base | s_lo[threadIdx.x];
      if (L == kMaxTileQubits) {
        const uint32_t st = swz((uint32_t)tid);
#pragma unroll
        for (int k = 0; k < kRegs; ++k)
          st1(a + (gb | s_hi[k]), sm[swz((uint32_t)k * kGroupThreads) ^ st]);
      } else {
        for (int k = 0; k < nk; ++k) {
          const uint32_t l = (uint32_t)k * kGroupThreads + tid;
          st1(a + (gb | s_hi[k]), sm[swz(l)]);
        }
      }
    }
    if (tid == 0) s_next[group] = next;
    group_sync(group);  // the tile buffer is refilled next iteration
    if (group == 0 && first && tid == 0) *s_go = kGroups;
    first = false;
    tile = s_next[group];
  }
  if (group == 0 && tid == 0) *s_go = kGroups;  // no tile / no phase: release the others
  __syncthreads();
  if (threadIdx.x == 0) {
    // every atomic of this CTA is done; the last CTA resets the counters
    __threadfence();
    if (atomicAdd(ctr + 1, 1ULL) == gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
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
    if (g.m > QSV_TILE_MAX_DENSE) return false;  // wider blocks run as k_dense5 / k_dense_smem
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
                    const std::vector<char>& done, size_t first, uint64_t outer,
                    uint64_t seed = 0) {
  PassSel ps;
  const int c = std::min(kLowQubits, n);
  ps.S = (c >= 64) ? ~0ULL : ((1ULL << c) - 1);
  ps.S |= seed;
  uint64_t blocked = 0;
  const uint64_t all = (n >= 64) ? ~0ULL : ((1ULL << n) - 1);
  size_t budget = kTileProgramBudget;  // staged program must fit in shared memory
  for (size_t i = first; i < gates.size(); ++i) {
    if (done[i]) continue;
    const GateDesc& g = gates[i];
    size_t cost = sizeof(TileOp) + sizeof(TilePhase) + 32;
    if (g.kind == QSV_OP_DENSE) cost += sizeof(double2) << (2 * g.m);
    if (g.kind == QSV_OP_DIAG) cost += sizeof(double2) << g.m;
    // merged diagonal flushes: at most one table per R op, one rule per D op
    if (g.kind == QSV_OP_DENSE && g.m == 1) cost += sizeof(TileOp) + sizeof(double2) * kRegs;
    else cost += sizeof(FlushFactor);
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
  // pad S to exactly L qubits with the lowest unused qubits (never an
  // outer-mask qubit: those stay outside so blocks can run separately)
  for (int q = 0; q < n && popc64(ps.S) < L; ++q)
    if (!((outer >> q) & 1)) ps.S |= 1ULL << q;
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
  double fp64_ops_per_amp = 0;  // FP64 pipe operations per amplitude
};

Cplx cconj(Cplx a) { return {a.re, -a.im}; }
bool is_one_c(Cplx a) { return a.re == 1.0 && a.im == 0.0; }
bool is_real_mat(const Cplx* M, int n) {
  for (int i = 0; i < n; ++i)
    if (M[i].im != 0.0) return false;
  return true;
}

// Register-phase scheduling.  Inside one register phase every op is either
// an R op (a 2x2 acting non-diagonally on one register slot, possibly with
// controls) or a D op (diagonal).  D ops commute with each other and with R
// ops on other qubits, so the phase is re-ordered into alternating layers
// "all ready D ops, then all ready R ops": each D layer becomes ONE merged
// T_FLUSH (a 2^kRegBits table over the register slots, linear sign rules
// for sign patterns that involve thread / tile bits, per-thread factors for
// 1-qubit diagonals on non-register qubits) and each R layer runs as
// batched register arithmetic.
struct PhaseOp {
  TileOp op;
  std::vector<Cplx> data;
  bool isR = false;
  uint32_t nd = 0, sup = 0;  // local bits acted on non-diagonally / touched
};

void emit_op(Encoded& e, TileOp op, const std::vector<Cplx>& data) {
  op.data = (uint32_t)e.data.size();
  e.data.insert(e.data.end(), data.begin(), data.end());
  e.ops.push_back(op);
}

double d_op_cost(const TileOp& op) {
  if (op.kind == T_PHASE) return (op.flags & 2) ? 0.0 : 4.0;
  if (op.kind == T_PHASES)
    return ((op.flags & 1) ? 4.0 : 0.0) + 2.0 * __builtin_popcount((uint32_t)op.slots);
  return 4.0;  // T_DIAG / T_PARITY: one complex multiply per amplitude
}

// Merge a layer of D ops: returns the ops that could not be merged.
std::vector<PhaseOp> emit_flush(Encoded& e, const std::vector<PhaseOp>& dl, const int* regpos) {
  uint32_t Rall = 0;
  int slot_of[32];
  for (int b = 0; b < 32; ++b) slot_of[b] = -1;
  for (int i = 0; i < kRegBits; ++i) {
    Rall |= 1u << regpos[i];
    slot_of[regpos[i]] = i;
  }
  std::vector<Cplx> T(kRegs, Cplx{1, 0});
  std::vector<FlushSign> signs;
  std::vector<FlushFactor> facs;
  std::vector<FlushPhase> phrules;
  auto unit = [](Cplx f) { return std::fabs(std::hypot(f.re, f.im) - 1.0) <= 1e-14; };
  // factor f where (thread pattern lm/lv, tile pattern gm/gv) holds and, if
  // jm has a bit, where that register slot equals the bit of jv
  auto add_phase = [&](uint32_t lm, uint32_t lv, uint64_t gm, uint64_t gv, uint32_t jm,
                       uint32_t jv, Cplx f) {
    FlushPhase r;
    memset(&r, 0, sizeof(r));
    r.lm = lm;
    r.lv = lv;
    r.gm = gm;
    r.gv = gv;
    if (!jm) {
      r.slot = -1;
      r.f = make_double2(f.re, f.im);
      phrules.push_back(r);
      return;
    }
    const int sl = __builtin_ctz(jm);
    if (jv & jm) {
      r.slot = sl;
      r.f = make_double2(f.re, f.im);
      phrules.push_back(r);
    } else {  // factor on slot == 0: f overall, conj(f) where the slot is 1
      r.slot = -1;
      r.f = make_double2(f.re, f.im);
      phrules.push_back(r);
      r.slot = sl;
      r.f = make_double2(f.re, -f.im);
      phrules.push_back(r);
    }
  };
  std::vector<PhaseOp> rest;
  bool changed = false;
  auto jpat = [&](uint32_t mask, uint32_t val, uint32_t* jm, uint32_t* jv) {
    *jm = 0;
    *jv = 0;
    for (int b = 0; b < 32; ++b)
      if (((mask >> b) & 1u) && slot_of[b] >= 0) {
        *jm |= 1u << slot_of[b];
        if ((val >> b) & 1u) *jv |= 1u << slot_of[b];
      }
  };
  for (const PhaseOp& po : dl) {
    const TileOp& op = po.op;
    if (op.kind == T_PHASE) {
      const Cplx f = (op.flags & 2) ? Cplx{-1, 0} : po.data[0];
      uint32_t jm, jv;
      jpat(op.lmask, op.lval, &jm, &jv);
      const uint32_t tm = op.lmask & ~Rall;
      if (op.gmask == 0 && tm == 0) {
        for (int j = 0; j < kRegs; ++j)
          if (((uint32_t)j & jm) == jv) T[j] = cm(T[j], f);
        changed = true;
        continue;
      }
      if (!(f.re == -1.0 && f.im == 0.0) && unit(f) && __builtin_popcount(jm) <= 1) {
        add_phase(tm, op.lval & tm, op.gmask, op.gval, jm, jv, f);
        changed = true;
        continue;
      }
      if (f.re == -1.0 && f.im == 0.0 && __builtin_popcount(jm) <= 1) {
        FlushSign r;
        memset(&r, 0, sizeof(r));
        r.lm = tm;
        r.lv = op.lval & tm;
        r.gm = op.gmask;
        r.gv = op.gval;
        // slots j where the register part of the pattern holds
        for (int j = 0; j < kRegs; ++j)
          if (((uint32_t)j & jm) == jv) r.col |= 1u << j;
        signs.push_back(r);
        changed = true;
        continue;
      }
    } else if (op.kind == T_DIAG) {
      bool all_reg = true;
      for (int t = 0; t < op.m; ++t)
        if (op.tpos[t] < 0 || slot_of[(int)op.tpos[t]] < 0) all_reg = false;
      if (all_reg && op.gmask == 0 && (op.lmask & ~Rall) == 0) {
        uint32_t jm, jv;
        jpat(op.lmask, op.lval, &jm, &jv);
        for (int j = 0; j < kRegs; ++j) {
          if (((uint32_t)j & jm) != jv) continue;
          int sub = 0;
          for (int t = 0; t < op.m; ++t) sub |= ((j >> slot_of[(int)op.tpos[t]]) & 1) << t;
          T[j] = cm(T[j], po.data[sub]);
        }
        changed = true;
        continue;
      }
      if (op.m == 1 && (op.lmask & Rall) == 0 && (op.lmask || op.gmask) &&
          unit(po.data[0]) && unit(po.data[1])) {
        // 1-qubit diagonal with controls on thread / tile bits
        const int p = op.tpos[0];
        const uint32_t tm = op.lmask, tv = op.lval;
        if (p >= 0 && slot_of[p] >= 0) {
          const uint32_t jm = 1u << slot_of[p];
          add_phase(tm, tv, op.gmask, op.gval, 0, 0, po.data[0]);
          const Cplx r = cm(po.data[1], cconj(po.data[0]));  // d1 / d0 for unit d0
          add_phase(tm, tv, op.gmask, op.gval, jm, jm, r);
        } else if (p >= 0) {  // target on a thread bit
          add_phase(tm | (1u << p), tv, op.gmask, op.gval, 0, 0, po.data[0]);
          add_phase(tm | (1u << p), tv | (1u << p), op.gmask, op.gval, 0, 0, po.data[1]);
        } else {  // target on a tile bit
          const uint64_t gb = 1ULL << (-p - 1);
          add_phase(tm, tv, op.gmask | gb, op.gval, 0, 0, po.data[0]);
          add_phase(tm, tv, op.gmask | gb, op.gval | gb, 0, 0, po.data[1]);
        }
        changed = true;
        continue;
      }
      if (op.m == 1 && op.lmask == 0 && op.gmask == 0) {  // non-register qubit
        FlushFactor f;
        memset(&f, 0, sizeof(f));
        f.pos = op.tpos[0];
        f.d0 = make_double2(po.data[0].re, po.data[0].im);
        f.d1 = make_double2(po.data[1].re, po.data[1].im);
        facs.push_back(f);
        changed = true;
        continue;
      }
    }
    rest.push_back(po);
  }
  if (!changed) return rest;
  if (!phrules.empty()) {  // one T_PHASES op after the flush (diagonals commute)
    TileOp pop;
    memset(&pop, 0, sizeof(pop));
    pop.kind = T_PHASES;
    pop.m = (int32_t)phrules.size();
    std::vector<Cplx> pdata;
    int scalar = 0;
    for (const FlushPhase& r : phrules) {
      if (r.slot < 0) scalar = 1;
      else pop.slots |= 1 << r.slot;
      Cplx w[3];
      memcpy(w, &r, sizeof(r));
      for (int k = 0; k < 3; ++k) pdata.push_back(w[k]);
    }
    pop.flags = scalar;
    rest.insert(rest.begin(), PhaseOp{});
    rest.front().op = pop;
    rest.front().data = pdata;  // emitted (and costed) by the caller with the other `rest` ops
  }
  bool table = false;
  uint32_t tsign = 0;
  for (int j = 0; j < kRegs; ++j) {
    if (T[j].im != 0.0 || (T[j].re != 1.0 && T[j].re != -1.0)) table = true;
    if (T[j].re == -1.0 && T[j].im == 0.0) tsign |= 1u << j;
  }
  if (!table && tsign == 0 && signs.empty() && facs.empty()) return rest;
  if (!facs.empty()) table = true;  // factors ride on the table flush
  TileOp op;
  memset(&op, 0, sizeof(op));
  op.kind = table ? T_FLUSH : T_SIGNS;
  op.flags = table ? 1 : 0;
  op.m = (int32_t)signs.size();
  op.slots = (int32_t)facs.size();
  op.lmask = table ? 0 : tsign;
  std::vector<Cplx> data;
  if (table) data = T;
  for (const FlushSign& r : signs) {
    Cplx w[2];
    memcpy(w, &r, sizeof(r));
    data.push_back(w[0]);
    data.push_back(w[1]);
  }
  for (const FlushFactor& f : facs) {
    Cplx w[3];
    memcpy(w, &f, sizeof(f));
    for (int k = 0; k < 3; ++k) data.push_back(w[k]);
  }
  emit_op(e, op, data);
  e.fp64_ops_per_amp += (table ? 4.0 : 0.0) + (facs.empty() ? 0.0 : 4.0);
  return rest;
}

// QSV_JIT_DIRECT_STORE=0: generated passes write tiles back through shared
// memory even when the last phase could store from registers (A/B)
inline bool jit_direct_store() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_DIRECT_STORE");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// recorded pass selections by gate-list structure (plan_program)
inline std::mutex g_sel_mu;
inline std::unordered_map<std::string, std::vector<PassSel>> g_sel_cache;

// QSV_PASS_SEARCH: 0 plain greedy, 1 multi-start, 2 multi-start with one
// pass of lookahead.  Unset: plan_program (qsv_tile_select.cu) plans modes 1
// and 2 and keeps the plan with fewer passes; this default only serves
// callers that plan once.
inline int pass_search() {
  static const int mode = [] {
    const char* e = getenv("QSV_PASS_SEARCH");
    return e ? atoi(e) : 2;
  }();
  return tl_pass_search >= 0 ? tl_pass_search : mode;
}

inline int max_pass_phases() {
  static const int v = [] {
    const char* e = getenv("QSV_MAX_PASS_PHASES");
    return e ? std::max(1, atoi(e)) : 1 << 30;
  }();
  return v;
}

// QSV_JIT_WARP_LOCAL=0: every phase transition uses the group barrier (A/B)
inline bool jit_warp_local() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_WARP_LOCAL");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_NOHOIST=0: let the compiler hoist per-phase thread deposits out of
// the tile loop (A/B)
inline bool jit_nohoist() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_NOHOIST");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_ADDR_SPLIT=0: slot addresses as sm[slt ^ c] (one LOP3 + LEA per
// LDS/STS) instead of per-phase base pointers with immediate offsets (A/B)
inline bool jit_addr_split() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_ADDR_SPLIT");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_SIGN_FOLD=0: flush signs as (bits << k) & 0x80000000 then two
// xors, instead of the mask folded into each xor (A/B)
inline bool jit_sign_fold() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_SIGN_FOLD");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_STATIC=0: passes with no more tiles than resident CTAs still pull
// tiles from the work counter (A/B)
inline bool jit_static_tiles() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_STATIC");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_LATE_SYNC=1: the tile's group barrier and the next-tile index
// publication move from the top of the tile loop to the first shared-memory
// store, after the HBM loads.  Off: mixed (cnot-ring(30) 315.7 -> 307.8 ms,
// cz-ladder(30) 223.5 -> 225.1 ms, (28) 49.8 -> 50.7 ms;
// profiles/r2_late_sync_ab.md)
inline bool jit_late_sync() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_LATE_SYNC");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

// QSV_JIT_LATE_WAIT=1: passes with statically assigned tiles wait for their
// predecessor (PDL) at the first HBM load instead of kernel start.  Off:
// mixed (cnot-ring(18) 0.133 -> 0.120 ms, (16) 0.095 -> 0.092, but (17)
// 0.110 -> 0.125; profiles/r2_late_wait_ab.md)
inline bool jit_late_wait() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_LATE_WAIT");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

// QSV_JIT_DIRECT_LOAD=0: tiles always enter through cp.async copy-in (A/B)
inline bool jit_direct_load() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_DIRECT_LOAD");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_DIRECT_ANY=1: direct stores whenever qubits 0..3 sit on lane or
// register bits; default: only when the last phase's lanes hold them in order
// (fully coalesced; measured 1-2% faster on cz-ladder, equal on cnot-ring)
inline bool jit_direct_any() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_DIRECT_ANY");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

// QSV_JIT_PARTIAL_BARRIERS=0: transitions that keep some warp positions still
// synchronise the whole group (A/B)
inline bool jit_partial_barriers() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_PARTIAL_BARRIERS");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// QSV_JIT_SHUFFLE=1: warp-local phase transitions as lane <-> register bit
// swaps with warp shuffles (and lanes aligned by the encoder for them).  Off
// by default: measured slower (cz-ladder(30) 222.7 -> 233.1 ms, cnot-ring(30)
// 303.6 -> 310.8 ms) -- four 32-bit shuffles plus selects per moved amplitude
// cost more issue slots than the 128-bit shared-memory round trip they save
inline bool jit_shuffle_transitions() {
  static const int on = [] {
    const char* e = getenv("QSV_JIT_SHUFFLE");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

inline int jit_stagger_max_phases() {
  static const int v = [] {
    const char* e = getenv("QSV_STAGGER_MAX_PHASES");
    return e ? atoi(e) : 1 << 30;
  }();
  return v;
}

// QSV_PDL=1: generated pass kernels launch with programmatic dependent launch
// (the next pass queued while this one drains).  Off by default: measured
// slower on every small-state circuit (cnot-ring(14) 0.117 -> 0.138 ms,
// cz-ladder(16) 0.180 -> 0.207 ms; profiles/r2_small_n_pdl.txt)
// QSV_PDL_LATE=1 (with QSV_PDL=1): trigger the dependent launch after each
// CTA's last tile instead of at kernel start (A/B)
inline bool jit_pdl_late() {
  static const int on = [] {
    const char* e = getenv("QSV_PDL_LATE");
    return e ? atoi(e) : 0;
  }();
  return on != 0;
}

// 0 never, 1 always, -1 (unset) per program: the planner marks programs of
// shallow passes (TilePlan.pdl, qsv_tile_select.cu)
inline int jit_pdl_mode() {
  static const int v = [] {
    const char* e = getenv("QSV_PDL");
    return e ? atoi(e) : -1;
  }();
  return v;
}
inline bool jit_pdl() { return jit_pdl_mode() == 1; }

// QSV_ONE_FMA=0 keeps the plain real rotations (A/B experiments)
inline bool one_fma_rotations() {
  static const int on = [] {
    const char* e = getenv("QSV_ONE_FMA");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

// FP64 instructions per amplitude of a real 2x2 on a register slot: a
// multiply and an FMA per output component, or one FMA when the matrix has a
// unit diagonal / anti-diagonal (the one-FMA form of realify)
inline double real_rot_ops(const std::vector<Cplx>& d) {
  if (d.size() >= 2 && ((d[0].re == 1.0 && d[1].im == 1.0) || (d[0].im == 1.0 && d[1].re == 1.0)))
    return 2.0;
  return 4.0;
}



void emit_rlayer(Encoded& e, const std::vector<PhaseOp>& rl) {
  // uncontrolled 1-qubit ops are collected into slot-mask batches; a batch
  // stays open while every op emitted after it commutes with the joiner
  struct Batch {
    bool real;
    int slots = 0;
    std::vector<Cplx> mat[kRegBits];
    size_t pos;  // index into `seq`
    uint32_t after_nd = 0, after_sup = 0;
  };
  std::vector<int> seq;              // >= 0: rl index, < 0: -(batch)-1
  std::vector<Batch> batches;
  int open = -1;
  for (size_t k = 0; k < rl.size(); ++k) {
    const PhaseOp& po = rl[k];
    const int slot = __builtin_ctz((uint32_t)po.op.slots);
    const bool real = po.op.kind == T_REAL1;
    const bool plain = po.op.lmask == 0 && po.op.gmask == 0 && !(po.op.flags & 1);
    if (plain) {
      if (open >= 0) {
        Batch& B = batches[open];
        if (B.real == real && !((B.slots >> slot) & 1) && !(po.nd & B.after_sup) &&
            !(po.sup & B.after_nd)) {
          B.slots |= 1 << slot;
          B.mat[slot] = po.data;
          continue;
        }
      }
      Batch B;
      B.real = real;
      B.slots = 1 << slot;
      B.mat[slot] = po.data;
      B.pos = seq.size();
      batches.push_back(B);
      open = (int)batches.size() - 1;
      seq.push_back(-open - 1);
      continue;
    }
    seq.push_back((int)k);
    if (open >= 0) {
      batches[open].after_nd |= po.nd;
      batches[open].after_sup |= po.sup;
    }
  }
  for (int x : seq) {
    if (x >= 0) {
      const PhaseOp& po = rl[x];
      emit_op(e, po.op, po.data);
      e.fp64_ops_per_amp +=
          (po.op.flags & 1) ? 0.0 : (po.op.kind == T_REAL1 ? real_rot_ops(po.data) : 8.0);
      continue;
    }
    const Batch& B = batches[-x - 1];
    TileOp op;
    memset(&op, 0, sizeof(op));
    std::vector<Cplx> data;
    const int cnt = __builtin_popcount(B.slots);
    if (cnt == 1) {
      const int slot = __builtin_ctz(B.slots);
      op.kind = B.real ? T_REAL1 : T_DENSE1;
      op.slots = B.slots;
      data = B.mat[slot];
    } else {
      op.kind = B.real ? T_REAL1X : T_DENSE1X;
      op.slots = B.slots;
      op.m = cnt;
      for (int i = 0; i < kRegBits; ++i)
        if ((B.slots >> i) & 1) data.insert(data.end(), B.mat[i].begin(), B.mat[i].end());
    }
    emit_op(e, op, data);
    for (int i = 0; i < kRegBits; ++i)
      if ((B.slots >> i) & 1) e.fp64_ops_per_amp += B.real ? real_rot_ops(B.mat[i]) : 8.0;
  }
}

// Rewrite a register-phase op into slot space once the phase's register
// slots are known: controls / patterns split into a thread part (lmask,
// lval) and a register part (zl = rm | rv << 16); diagonal targets become a
// slot (0..7) or 8 + thread bit; parity masks a slot mask in m.
void to_slot_space(TileOp& op, const int* slot_of, uint32_t Rall) {
  auto split = [&](uint32_t mask, uint32_t val) {
    uint32_t rm = 0, rv = 0;
    for (int b = 0; b < 32; ++b)
      if (((mask >> b) & 1u) && slot_of[b] >= 0) {
        rm |= 1u << slot_of[b];
        if ((val >> b) & 1u) rv |= 1u << slot_of[b];
      }
    op.zl = rm | (rv << 16);
    op.lmask = mask & ~Rall;
    op.lval = val & ~Rall;
  };
  switch (op.kind) {
    case T_DENSE1:
    case T_REAL1:
    case T_PHASE:
      split(op.lmask, op.lval);
      break;
    case T_DIAG:
      split(op.lmask, op.lval);
      for (int t = 0; t < op.m; ++t) {
        const int p = op.tpos[t];
        if (p >= 0) op.tpos[t] = (int8_t)(slot_of[p] >= 0 ? slot_of[p] : 8 + p);
      }
      break;
    case T_PARITY: {
      uint32_t rz = 0;
      for (int b = 0; b < 32; ++b)
        if (((op.zl >> b) & 1u) && slot_of[b] >= 0) rz |= 1u << slot_of[b];
      op.m = (int32_t)rz;
      op.zl &= ~Rall;
      break;
    }
    default:
      break;  // T_FLUSH and the batches are built in slot space
  }
}

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
  // 1-qubit dense gates by local target bit, in pass order (warp-bit choice)
  std::vector<std::vector<size_t>> uses(L);
  for (size_t i = 0; i < pg.size(); ++i)
    if (pg[i]->kind == QSV_OP_DENSE && pg[i]->m == 1 && local_of[pg[i]->targets[0]] >= 0)
      uses[local_of[pg[i]->targets[0]]].push_back(i);
  size_t gi = 0;  // index of the gate being encoded
  auto next_use = [&](int b) -> size_t {
    auto it = std::lower_bound(uses[b].begin(), uses[b].end(), gi);
    return it == uses[b].end() ? (size_t)-1 : *it;
  };
  std::vector<int> cur_warp;  // warp-index bit positions of the last register phase
  std::vector<int> prev_warp, prev_lanes;  // the last register phase's warp / lane bits
  // current register phase: ops collected with their own data, scheduled at close
  bool open = false;
  uint32_t R = 0;
  std::vector<PhaseOp> cur;
  std::vector<int> d1bit;  // local target bit of each 1-qubit op in `cur` (-1 otherwise)
  std::vector<PhaseOp> carry;  // trailing D layer handed to the next register phase
  // carry_ok: the next phase is a register phase, so a trailing D layer can
  // be merged into that phase's first flush instead of running on its own
  auto close = [&](bool carry_ok) {
    if (!open) return;
    // register slots in order of first use by a 1-qubit op, then the other
    // R bits, then filled with the highest remaining bits
    std::vector<int> order;
    for (int b : d1bit)
      if (b >= 0 && std::find(order.begin(), order.end(), b) == order.end()) order.push_back(b);
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
    // thread bits: lanes (tid bits 0..4) then warp-index bits.  The warp
    // bits are kept from phase to phase while no register bit needs them, so
    // a transition only permutes data inside each warp and the generated
    // kernel synchronises it with __syncwarp instead of the group barrier;
    // when they must change, the new warp bits are the non-register bits
    // whose next 1-qubit use lies furthest ahead (they stay warp bits longest)
    const int nwarp = std::max(0, (L - kRegBits) - 5);
    if ((int)cur_warp.size() != nwarp) cur_warp.assign(nwarp, -1);
    // Only the warp positions whose bit became a register bit change, the
    // others keep their bit at the same index: a transition then moves data
    // only among the warps that differ in the changed positions, and the
    // generated kernel synchronises just those (named barrier per subset).
    // Replacements: local bits 0..3 (the 256-byte HBM runs) stay lane bits
    // where possible (the direct loads / stores need them), then the bit
    // whose next 1-qubit use lies furthest ahead.
    {
      std::vector<int> cand;
      for (int b = 0; b < L; ++b)
        if (!((Rall >> b) & 1u) && std::find(cur_warp.begin(), cur_warp.end(), b) == cur_warp.end())
          cand.push_back(b);
      std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) {
        if ((x < kLowQubits) != (y < kLowQubits)) return y < kLowQubits;
        const size_t nx = next_use(x), ny = next_use(y);
        return nx != ny ? nx > ny : x > y;
      });
      size_t ci = 0;
      for (int& w : cur_warp)
        if (w < 0 || ((Rall >> w) & 1u)) w = cand[ci++];
    }
    std::vector<int> tb;
    for (int b = 0; b < L; ++b)
      if (!((Rall >> b) & 1u) &&
          std::find(cur_warp.begin(), cur_warp.end(), b) == cur_warp.end())
        tb.push_back(b);
    const int nlane = std::min<int>(5, (int)tb.size());
    if (jit_shuffle_transitions() && cur_warp == prev_warp && (int)prev_lanes.size() == nlane &&
        nlane == (int)tb.size()) {
      // warp bits unchanged after a register phase: keep every lane bit that
      // is still a thread bit at its lane position and put the new ones (the
      // previous phase's register bits) in the freed positions, so the
      // transition is a set of lane <-> register bit swaps the generated
      // kernel does with warp shuffles (no shared memory, no barrier)
      std::vector<int> lanes(nlane, -1), avail = tb;
      for (int p = 0; p < nlane; ++p) {
        auto it = std::find(avail.begin(), avail.end(), prev_lanes[p]);
        if (it != avail.end()) {
          lanes[p] = *it;
          avail.erase(it);
        }
      }
      size_t ai = 0;
      for (int p = 0; p < nlane; ++p)
        if (lanes[p] < 0) lanes[p] = avail[ai++];
      tb = lanes;
    } else {
      order_thread_bits(tb);
    }
    prev_lanes.assign(tb.begin(), tb.begin() + nlane);
    prev_warp = cur_warp;
    tb.insert(tb.end(), cur_warp.begin(), cur_warp.end());
    for (size_t k = 0; k < tb.size(); ++k) ph.thrpos[k] = tb[k];
    for (int v = 0; v < 16; ++v) {
      ph.thr_lo[v] = ph.thr_hi[v] = 0;
      for (int j = 0; j < 4; ++j) {
        if (((v >> j) & 1) && j < (int)tb.size()) ph.thr_lo[v] |= 1u << tb[j];
        if (((v >> j) & 1) && j + 4 < (int)tb.size()) ph.thr_hi[v] |= 1u << tb[j + 4];
      }
    }
    // classify
    const size_t K = cur.size();
    for (size_t k = 0; k < K; ++k) {
      PhaseOp& po = cur[k];
      if (d1bit[k] >= 0) {
        po.op.slots = 1 << slot_of[d1bit[k]];
        po.isR = true;
        po.nd = 1u << d1bit[k];
        po.sup = po.nd | po.op.lmask;
      } else {
        po.isR = false;
        po.nd = 0;
        if (po.op.kind == T_PHASE) po.sup = po.op.lmask;
        else if (po.op.kind == T_PARITY) po.sup = po.op.zl;
        else {
          po.sup = po.op.lmask;
          for (int t = 0; t < po.op.m; ++t)
            if (po.op.tpos[t] >= 0) po.sup |= 1u << po.op.tpos[t];
        }
      }
    }
    // dependencies (i < j): R-R share a non-diagonal bit, R-D share the R bit
    std::vector<std::vector<int>> pred(K);
    for (size_t j = 0; j < K; ++j)
      for (size_t i = 0; i < j; ++i) {
        const PhaseOp &a = cur[i], &b = cur[j];
        bool dep;
        if (a.isR && b.isR) dep = (a.nd & b.sup) || (b.nd & a.sup);
        else if (a.isR) dep = a.nd & b.sup;
        else if (b.isR) dep = b.nd & a.sup;
        else dep = false;
        if (dep) pred[j].push_back((int)i);
      }
    std::vector<char> done(K, 0);
    size_t left = K;
    ph.op_begin = (int)e.ops.size();
    while (left) {
      auto ready = [&](size_t k) {
        for (int p : pred[k])
          if (!done[p]) return false;
        return true;
      };
      std::vector<PhaseOp> dl, rl;
      for (size_t k = 0; k < K; ++k)
        if (!done[k] && !cur[k].isR && ready(k)) dl.push_back(cur[k]);
      for (size_t k = 0; k < K; ++k)
        if (!done[k] && !cur[k].isR && ready(k)) done[k] = 1;
      for (size_t k = 0; k < K; ++k)  // preds have lower indices: one scan closes chains
        if (!done[k] && cur[k].isR && ready(k)) {
          done[k] = 1;
          rl.push_back(cur[k]);
        }
      left -= dl.size() + rl.size();
      if (dl.empty() && rl.empty()) break;  // cannot happen (the DAG is acyclic)
      if (carry_ok && rl.empty() && left == 0) {
        carry = dl;
        break;
      }
      for (const PhaseOp& po : emit_flush(e, dl, ph.regpos)) {
        emit_op(e, po.op, po.data);
        e.fp64_ops_per_amp += d_op_cost(po.op);
      }
      emit_rlayer(e, rl);
    }
    ph.op_end = (int)e.ops.size();
    for (int o = ph.op_begin; o < ph.op_end; ++o) to_slot_space(e.ops[o], slot_of, Rall);
    if (ph.op_end > ph.op_begin) e.phases.push_back(ph);
    open = false;
    R = 0;
    cur.clear();
    d1bit.clear();
  };
  auto open_reg = [&]() {
    if (open) return;
    open = true;
    R = 0;
    for (const PhaseOp& po : carry) {
      cur.push_back(po);
      d1bit.push_back(-1);
    }
    carry.clear();
  };
  auto push_cur = [&](const TileOp& op, std::vector<Cplx> data, int bit) {
    PhaseOp po;
    po.op = op;
    po.data = std::move(data);
    cur.push_back(po);
    d1bit.push_back(bit);
  };
  for (size_t gix = 0; gix < pg.size(); ++gix) {
    gi = gix;
    const GateDesc& g = *pg[gix];
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
    if (g.kind == QSV_OP_DENSE && g.m == 1) {
      const int b = local_of[g.targets[0]];
      open_reg();
      if (!((R >> b) & 1u) && __builtin_popcount(R) >= kRegBits) {
        close(true);
        open_reg();
      }
      R |= 1u << b;
      if (g.rf) {  // diag(b) as a D op in front of the real rotation
        if (!(is_one_c(g.rf_b[0]) && is_one_c(g.rf_b[1]))) {
          TileOp dop;
          memset(&dop, 0, sizeof(dop));
          dop.kind = T_DIAG;
          dop.m = 1;
          dop.tpos[0] = (int8_t)b;
          push_cur(dop, {g.rf_b[0], g.rf_b[1]}, -1);
        }
        op.kind = T_REAL1;
        if (g.rf_r[0] == 0.0 && g.rf_r[3] == 0.0 && g.rf_r[1] == 1.0 && g.rf_r[2] == 1.0)
          op.flags |= 1;
        push_cur(op, {{g.rf_r[0], g.rf_r[1]}, {g.rf_r[2], g.rf_r[3]}}, b);
        continue;
      }
      const Cplx* M = g.data.data();
      if (is_zero(M[0]) && is_zero(M[3]) && is_one_c(M[1]) && is_one_c(M[2])) op.flags |= 1;
      std::vector<Cplx> data;
      if (is_real_mat(M, 4)) {
        op.kind = T_REAL1;
        data = {{M[0].re, M[1].re}, {M[2].re, M[3].re}};  // (a, b), (c, d) as double2
      } else {
        op.kind = T_DENSE1;
        op.flags &= ~1;
        data.assign(g.data.begin(), g.data.end());
      }
      push_cur(op, std::move(data), b);
      continue;
    }
    if (g.kind == QSV_OP_DENSE) {  // m = 2..4: shared-memory op
      close(false);
      op.kind = S_DENSE;
      op.m = g.m;
      for (int t = 0; t < g.m; ++t) op.tpos[t] = local_of[g.targets[t]];
      TilePhase ph;
      memset(&ph, 0, sizeof(ph));
      ph.type = 1;
      ph.op_begin = (int)e.ops.size();
      emit_op(e, op, g.data);
      ph.op_end = (int)e.ops.size();
      e.phases.push_back(ph);
      e.fp64_ops_per_amp += 4.0 * (double)(1 << g.m);
      prev_lanes.clear();
      continue;
    }
    if (g.kind == QSV_OP_DIAG) {
      open_reg();
      if (g.m == 0) {
        op.kind = T_PHASE;
        const Cplx f = g.data[0];
        if (f.re == -1.0 && f.im == 0.0) op.flags |= 2;
        push_cur(op, {f}, -1);
      } else {
        op.kind = T_DIAG;
        op.m = g.m;
        for (int t = 0; t < g.m; ++t) {
          const int q = g.targets[t];
          op.tpos[t] = local_of[q] >= 0 ? local_of[q] : -(q + 1);
        }
        push_cur(op, g.data, -1);
      }
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
      push_cur(op, {ca(alpha, bph), {alpha.re - bph.re, alpha.im - bph.im}}, -1);
      continue;
    }
    close(false);
    op.kind = S_PAULI;
    uint32_t xl = 0;
    for (int q = 0; q < n; ++q)
      if ((xm >> q) & 1ULL) xl |= 1u << local_of[q];
    op.slots = (int32_t)xl;
    TilePhase ph;
    memset(&ph, 0, sizeof(ph));
    ph.type = 1;
    ph.op_begin = (int)e.ops.size();
    emit_op(e, op, {alpha, bph});
    ph.op_end = (int)e.ops.size();
    e.phases.push_back(ph);
    e.fp64_ops_per_amp += 8.0;
    prev_lanes.clear();
  }
  gi = pg.size();
  close(false);
  e.pd.nphases = (int)e.phases.size();
  if (const char* dbg = getenv("QSV_TILE_DEBUG")) e.pd.debug = atoi(dbg);
  return e;
}

// ------------------------------------------------------- real frames
// U = diag(a) R diag(b) with R real (Euler: RZ RY RZ up to phase); false if
// U has no such form (non-unitary shapes), then it stays complex.
bool euler_real(const M2& U, Cplx a[2], Cplx b[2], double R[4]) {
  auto mag = [](Cplx z) { return std::hypot(z.re, z.im); };
  auto ph = [&](Cplx z) {
    const double r = mag(z);
    return Cplx{z.re / r, z.im / r};
  };
  double mx = 0;
  for (int i = 0; i < 4; ++i) mx = std::max(mx, mag(U.m[i]));
  if (!(mx > 0) || !std::isfinite(mx)) return false;
  const double eps = 1e-12 * mx;
  const Cplx U00 = U.m[0], U01 = U.m[1], U10 = U.m[2], U11 = U.m[3];
  Cplx a0{1, 0}, a1{1, 0}, b1{1, 0};
  const bool h0 = mag(U00) > eps, h1 = mag(U10) > eps;
  if (h0) a0 = ph(U00);
  if (h1) a1 = ph(U10);
  if (h0 && mag(U01) > eps) b1 = cm(ph(U01), cconj(a0));
  else if (h1 && mag(U11) > eps) b1 = cm(ph(U11), cconj(a1));
  if (!h0) {
    if (!(mag(U01) > eps)) return false;
    a0 = cm(ph(U01), cconj(b1));
  }
  if (!h1) {
    if (!(mag(U11) > eps)) return false;
    a1 = cm(ph(U11), cconj(b1));
  }
  // phases up to sign, canonical (real part > 0, or = 0 with imaginary part
  // > 0): the sign goes into the real matrix R instead, so a real U (e.g. an
  // RY whose cosine turns negative) keeps unit phases and the pass structure
  // (which factors are exactly 1) does not flip with the angle's sign --
  // generated pass kernels stay cached across parameter updates
  // (also snapped to exact +-1 / +-i within a few ulps: whether a factor is
  // exactly 1 must not depend on rounding either)
  auto canon = [](Cplx z) {
    constexpr double tol = 1e-15;
    if (std::fabs(z.im) <= tol && std::fabs(std::fabs(z.re) - 1.0) <= tol) z = {z.re < 0 ? -1.0 : 1.0, 0.0};
    else if (std::fabs(z.re) <= tol && std::fabs(std::fabs(z.im) - 1.0) <= tol) z = {0.0, z.im < 0 ? -1.0 : 1.0};
    return (z.re < 0 || (z.re == 0 && z.im < 0)) ? Cplx{-z.re, -z.im} : z;
  };
  a0 = canon(a0);
  a1 = canon(a1);
  b1 = canon(b1);
  const Cplx A[2] = {a0, a1}, B[2] = {{1, 0}, b1};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      const Cplx z = cm(cm(cconj(A[i]), U.m[2 * i + j]), cconj(B[j]));
      if (std::fabs(z.im) > 1e-13 * mx) return false;
      R[2 * i + j] = z.re;
    }
  a[0] = a0;
  a[1] = a1;
  b[0] = B[0];
  b[1] = B[1];
  return true;
}

// qubits a gate acts on non-diagonally
uint64_t nondiag_mask(const GateDesc& g) {
  uint64_t m = 0;
  if (g.kind == QSV_OP_DENSE || g.kind == QSV_OP_SPARSE) {
    for (int j = 0; j < g.m; ++j) m |= 1ULL << g.targets[j];
  } else if (g.kind == QSV_OP_PAULI || g.kind == QSV_OP_PAULI_ROT) {
    for (int j = 0; j < g.m; ++j)
      if (g.ids[j] == 1 || g.ids[j] == 2) m |= 1ULL << g.targets[j];
  }
  return m;
}

// an uncontrolled 1-qubit diagonal in either canonical form
bool diag_1q(const GateDesc& g, int* q, Cplx d[2]) {
  if (g.kind != QSV_OP_DIAG) return false;
  if (g.m == 1 && g.nc == 0) {
    *q = g.targets[0];
    d[0] = g.data[0];
    d[1] = g.data[1];
    return true;
  }
  if (g.m == 0 && g.nc == 1) {
    *q = g.cq[0];
    d[g.cv[0] ? 1 : 0] = g.data[0];
    d[g.cv[0] ? 0 : 1] = {1, 0};
    return true;
  }
  return false;
}

GateDesc diag_desc(int q, Cplx d0, Cplx d1) {
  M2 D;
  D.m[0] = d0;
  D.m[1] = {0, 0};
  D.m[2] = {0, 0};
  D.m[3] = d1;
  return canonicalize(desc_from_m2(q, D));
}

// Every uncontrolled 1-qubit dense gate U on q is written U = diag(a) R diag(b)
// with R real: diag(b) (applied first) is emitted as a diagonal gate right
// before R (the tile encoder merges such diagonals of one register phase
// into a single T_FLUSH), diag(a) stays pending on q and is folded into the
// next gate on q.  1-qubit diagonals join the pending factor.
// A gate is only split when the next gate acting non-diagonally on its qubit
// is again an uncontrolled 1-qubit gate (which absorbs diag(a)); otherwise
// (a CNOT target, a multi-qubit gate, the end of the circuit) it stays one
// complex 2x2 that absorbs the pending factor, so no extra flush is needed.
bool is_plain_1q_dense(const GateDesc& g) {
  return g.kind == QSV_OP_DENSE && g.m == 1 && g.nc == 0;
}

std::vector<GateDesc> realify(int n, const std::vector<GateDesc>& in) {
  // split[i]: the next non-diagonal gate on the target of gate i is plain 1q
  std::vector<char> split(in.size(), 0);
  {
    std::vector<int> next_plain(n, 0);  // scanning backwards
    for (size_t k = in.size(); k-- > 0;) {
      const GateDesc& g = in[k];
      if (is_plain_1q_dense(g)) split[k] = next_plain[g.targets[0]];
      const uint64_t nd = nondiag_mask(g);
      for (int q = 0; q < n; ++q)
        if ((nd >> q) & 1ULL) next_plain[q] = is_plain_1q_dense(g);
    }
  }
  std::vector<GateDesc> out;
  std::vector<Cplx> p0(n, Cplx{1, 0}), p1(n, Cplx{1, 0});
  std::vector<char> has(n, 0);
  auto push = [&](const GateDesc& g) {
    if (g.nc >= 0) out.push_back(g);
  };
  auto flush = [&](int q) {
    if (!has[q]) return;
    push(diag_desc(q, p0[q], p1[q]));
    has[q] = 0;
    p0[q] = p1[q] = {1, 0};
  };
  for (size_t i = 0; i < in.size(); ++i) {
    const GateDesc& g = in[i];
    int q;
    Cplx d[2];
    if (diag_1q(g, &q, d)) {
      p0[q] = cm(d[0], p0[q]);
      p1[q] = cm(d[1], p1[q]);
      has[q] = !(is_one_c(p0[q]) && is_one_c(p1[q]));
      continue;
    }
    if (g.kind == QSV_OP_DENSE && g.m == 1 && g.nc == 0) {
      q = g.targets[0];
      M2 U;
      for (int k = 0; k < 4; ++k) U.m[k] = g.data[k];
      if (has[q]) {  // U . diag(p)
        U.m[0] = cm(U.m[0], p0[q]);
        U.m[2] = cm(U.m[2], p0[q]);
        U.m[1] = cm(U.m[1], p1[q]);
        U.m[3] = cm(U.m[3], p1[q]);
        has[q] = 0;
        p0[q] = p1[q] = {1, 0};
      }
      Cplx a[2], b[2];
      double Rm[4];
      if (!split[i] || !euler_real(U, a, b, Rm)) {
        push(canonicalize(desc_from_m2(q, U)));
        continue;
      }
      // One-FMA form: R = D . M with D diagonal and M unit-diagonal
      // ([[1, r1/r0], [r2/r3, 1]], D = diag(r0, r3)) or, when r0 = 0 (R is
      // anti-diagonal), M = [[0, 1], [1, 0]] with D = diag(r1, r2).  D joins
      // the pending diagonal diag(a) of the qubit (applied with the next gate
      // on it or in a merged flush), so the rotation itself costs one FMA
      // per output component instead of a multiply and an FMA.  The
      // intermediate fl(x + t y) is later scaled by r0, so the result keeps
      // a relative error of one rounding (no growth from a large t).  The
      // structure (unit entries) does not depend on the angle, so generated
      // pass kernels stay cached across parameter updates.
      double D[2] = {1.0, 1.0};
      if (one_fma_rotations()) {
        if (Rm[0] != 0.0 && Rm[3] != 0.0) {
          D[0] = Rm[0];
          D[1] = Rm[3];
          const double t1 = Rm[1] / Rm[0], t2 = Rm[2] / Rm[3];
          Rm[0] = 1.0;
          Rm[1] = t1;
          Rm[2] = t2;
          Rm[3] = 1.0;
        } else if (Rm[1] != 0.0 && Rm[2] != 0.0) {
          D[0] = Rm[1];
          D[1] = Rm[2];
          Rm[0] = 0.0;
          Rm[1] = 1.0;
          Rm[2] = 1.0;
          Rm[3] = 0.0;
        }
      }
      // one gate carrying both factors, so the pass packer cannot separate
      // diag(b) from R (R diag(b) is what a standalone kernel applies)
      M2 RB;
      RB.m[0] = {Rm[0] * b[0].re, Rm[0] * b[0].im};
      RB.m[1] = {Rm[1] * b[1].re, Rm[1] * b[1].im};
      RB.m[2] = {Rm[2] * b[0].re, Rm[2] * b[0].im};
      RB.m[3] = {Rm[3] * b[1].re, Rm[3] * b[1].im};
      GateDesc gr = desc_from_m2(q, RB);
      if (gr.kind == QSV_OP_DENSE) {
        gr.rf = 1;
        gr.rf_b[0] = b[0];
        gr.rf_b[1] = b[1];
        for (int k = 0; k < 4; ++k) gr.rf_r[k] = Rm[k];
      }
      push(canonicalize(gr));
      p0[q] = {a[0].re * D[0], a[0].im * D[0]};
      p1[q] = {a[1].re * D[1], a[1].im * D[1]};
      has[q] = !(is_one_c(p0[q]) && is_one_c(p1[q]));
      continue;
    }
    const uint64_t nd = nondiag_mask(g);
    for (int k = 0; k < n; ++k)
      if ((nd >> k) & 1ULL) flush(k);
    out.push_back(g);
  }
  for (int q = 0; q < n; ++q) flush(q);
  return out;
}

// FP64 flops of one gate applied to a 2^n state (2 per FMA): a complex
// multiply-add is 8 flops, a complex multiply 6, a sign flip 0.
double gate_fp64_flops(int n, const GateDesc& g) {
  const double amps = std::ldexp(1.0, n - g.nc);
  if (g.kind == QSV_OP_DENSE) return amps * 8.0 * (double)(1 << g.m);
  if (g.kind == QSV_OP_SPARSE) return amps * 8.0 * (double)g.data.size() / (double)(1 << g.m);
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

#include "qsv_tile_jit.cuh"

}  // namespace

bool tiles_enabled(int n, const qsv_plan_opts& opts) {
  int L = opts.tile_qubits > 0 ? opts.tile_qubits : kMaxTileQubits;
  L = std::min(std::min(L, kMaxTileQubits), n);
  return opts.use_tiles && n >= kRegBits + 1 && L >= kRegBits + 1;
}

// host-side gate-list passes shared by both variants: 1-qubit fusion and
// real frames (the latter only when tile passes run)
std::vector<GateDesc> preprocess(int n, const std::vector<GateDesc>& gates_in,
                                 const qsv_plan_opts& opts) {
  std::vector<GateDesc> gates = opts.fuse ? fuse_1q(n, gates_in) : gates_in;
  if (tiles_enabled(n, opts) && opts.real_frames) gates = realify(n, gates);
  return gates;
}

int plan_program(int n, const std::vector<GateDesc>& gates_in, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats, PlanMix* mix,
                 bool preprocessed) {
  std::vector<GateDesc> gates = preprocessed ? gates_in : preprocess(n, gates_in, opts);
  int L = opts.tile_qubits > 0 ? opts.tile_qubits : kMaxTileQubits;
  L = std::min(std::min(L, kMaxTileQubits), n);
  const bool tiles_on = tiles_enabled(n, opts);
  if (!tiles_on) {
    for (const GateDesc& g : gates) add_gate_step(n, g, steps, payload, stats);
    return QSV_OK;
  }
  const size_t G = gates.size();
  std::vector<uint64_t> act(G, 0);
  std::vector<char> ok(G, 0), done(G, 0);
  // a gate fits a tile only together with the always-present low qubits
  const uint64_t lowq = (n >= 64) ? ~0ULL : ((1ULL << std::min(kLowQubits, n)) - 1);
  for (size_t i = 0; i < G; ++i)
    ok[i] = active_qubits(gates[i], &act[i]) && popc64(act[i] | lowq) <= L &&
            !(act[i] & opts.outer_mask);
  // Pass selections depend only on the gate list's structure (kinds, widths,
  // qubits, active masks), not on angles: a ParametricCircuit recompiled
  // after set_parameter replays the recorded selections instead of running
  // the tile-set search again (the lookahead search costs a few ms).
  std::string fp;
  {
    const uint64_t hdr[6] = {(uint64_t)n, (uint64_t)L, opts.outer_mask, (uint64_t)pass_search(),
                             (uint64_t)max_pass_phases(), (uint64_t)G};
    fp.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    for (size_t i = 0; i < G; ++i) {
      const GateDesc& g = gates[i];
      const uint64_t rec[5] = {(uint64_t)g.kind | ((uint64_t)g.m << 8) | ((uint64_t)g.nc << 16),
                               act[i], (uint64_t)ok[i], touched_mask(g),
                               (uint64_t)(g.kind == QSV_OP_DENSE && g.m == 1)};
      fp.append(reinterpret_cast<const char*>(rec), sizeof(rec));
    }
  }
  std::vector<PassSel> replay, record;
  size_t replay_at = 0;
  {
    std::lock_guard<std::mutex> lk(g_sel_mu);
    auto it = g_sel_cache.find(fp);
    if (it != g_sel_cache.end()) replay = it->second;
  }
  const bool replaying = !replay.empty();
  size_t first = 0;
  while (true) {
    while (first < G && done[first]) ++first;
    if (first >= G) break;
    if (!ok[first]) {
      add_gate_step(n, gates[first], steps, payload, stats);
      done[first] = 1;
      continue;
    }
    PassSel ps;
    if (replaying && replay_at < replay.size()) {
      ps = replay[replay_at++];
    } else {
    ps = select_pass(n, L, gates, act, ok, done, first, opts.outer_mask);
    if (pass_search()) {
      // Multi-start: the greedy lets the first pending gates decide the tile
      // set; also seed it with the active qubits of the first pending gate on
      // each qubit and keep the pass that takes the most gates (for
      // nearest-neighbour circuits the best window is often not the one at
      // the lowest pending gate).  Mode 2 scores a candidate by its gates
      // plus the best next pass after it.
      auto seeds_of = [&](const std::vector<char>& dn, size_t from) {
        std::vector<uint64_t> seeds;
        uint64_t seen = 0;
        for (size_t i = from; i < G && seen != ~0ULL; ++i) {
          if (dn[i] || !ok[i]) continue;
          const uint64_t A = act[i] & ~lowq;
          if (!A || (A & seen) == A) continue;
          seen |= A;
          if (popc64(A | lowq) <= L && std::find(seeds.begin(), seeds.end(), A) == seeds.end())
            seeds.push_back(A);
          if ((int)seeds.size() >= 2 * n) break;
        }
        return seeds;
      };
      auto best_single = [&](const std::vector<char>& dn, size_t from) {
        size_t best = select_pass(n, L, gates, act, ok, dn, from, opts.outer_mask).taken.size();
        for (uint64_t sd : seeds_of(dn, from))
          best = std::max(best,
                          select_pass(n, L, gates, act, ok, dn, from, opts.outer_mask, sd).taken.size());
        return best;
      };
      std::vector<PassSel> cands;
      cands.push_back(ps);
      for (uint64_t sd : seeds_of(done, first))
        cands.push_back(select_pass(n, L, gates, act, ok, done, first, opts.outer_mask, sd));
      size_t best_score = 0, best_i = 0;
      std::vector<char> dn;
      for (size_t c = 0; c < cands.size(); ++c) {
        size_t score = cands[c].taken.size();
        if (pass_search() >= 2 && score > 0) {
          dn = done;
          for (int k : cands[c].taken) dn[k] = 1;
          size_t nf = first;
          while (nf < G && dn[nf]) ++nf;
          if (nf < G) score += best_single(dn, nf);
        }
        if (score > best_score) {
          best_score = score;
          best_i = c;
        }
      }
      ps = std::move(cands[best_i]);
    }
    }  // selection (searched or replayed)
    if (popc64(ps.S) < L || (ps.S & opts.outer_mask)) {
      set_error("outer mask leaves too few tile qubits (%d qubits, tile %d)", n, L);
      return QSV_EINVAL;
    }
    if (ps.taken.empty()) ps.taken.push_back((int)first);  // cannot happen (ok[] checks fit)
    if (ps.taken.size() == 1 && !opts.outer_mask) {
      // a lone gate is cheaper as its own streaming kernel (not when the
      // program must run block by block: there every step is a tile pass)
      add_gate_step(n, gates[ps.taken[0]], steps, payload, stats);
      done[ps.taken[0]] = 1;
      if (!replaying) record.push_back(ps);
      continue;
    }
    std::vector<const GateDesc*> pg;
    for (int k : ps.taken) pg.push_back(&gates[k]);
    Encoded e = encode_pass(n, L, ps.S, pg);
    // deep passes: cap the phase count (the generated code of a phase is
    // ~10 KB of SASS; far beyond the instruction cache every tile refetches
    // it).  A prefix of the taken gates is itself a valid pass: the rest stay
    // pending and start the next pass (QSV_MAX_PASS_PHASES, A/B).
    const int cap = max_pass_phases();
    while ((int)e.phases.size() > cap && pg.size() > 1) {
      const size_t keep = std::max<size_t>(1, pg.size() * (size_t)cap / e.phases.size());
      pg.resize(std::min(pg.size() - 1, keep));
      e = encode_pass(n, L, ps.S, pg);
    }
    ps.taken.resize(pg.size());
    for (int k : ps.taken) done[k] = 1;
    if (!replaying) record.push_back(ps);
    if (getenv("QSV_PLAN_DUMP")) {
      fprintf(stderr, "pass %zu: %zu gates, %zu phases, %zu ops, %zu data, fp64 ops/amp %.1f\n",
              tiles.size(), pg.size(), e.phases.size(), e.ops.size(), e.data.size(),
              e.fp64_ops_per_amp);
      for (const TilePhase& ph : e.phases) {
        fprintf(stderr, "  phase type %d regs", ph.type);
        for (int i = 0; i < kRegBits; ++i) fprintf(stderr, " %d", ph.regpos[i]);
        fprintf(stderr, " :");
        for (int o = ph.op_begin; o < ph.op_end; ++o) {
          const TileOp& op = e.ops[o];
          fprintf(stderr, " %d/%x", op.kind, op.slots);
          if (op.kind == T_FLUSH || op.kind == T_SIGNS) fprintf(stderr, "[t%d s%d f%d]", op.flags & 1, op.m, op.slots);
        }
        fprintf(stderr, "\n");
      }
    }
    TilePlan tp;
    tp.variant = kRegBits;
    tp.L = L;
    // the interpreter's thread-base tables hold 8 thread bits
    tp.jit_only = L - kRegBits > 8;
    if (tp.jit_only && !opts.jit) {
      set_error("tile of %d qubits with %d amplitudes per thread needs generated kernels", L,
                kRegs);
      return QSV_EUNSUPPORTED;
    }
    if (opts.jit && sizeof(JitParamHead) + sizeof(double2) * std::max<size_t>(1, e.data.size()) <=
                        kJitMaxParamBytes) {
      try {
        JitSource js = jit_pass_source(e, L);
        tp.jit_seen = js.seen;
        tp.jit_src = std::move(js.src);
        tp.jit_threads = js.threads;
        tp.jit_groups = js.groups;
        tp.jit_smem = js.smem;
        tp.jit_data = e.data;
        if (tp.jit_data.empty()) tp.jit_data.push_back(Cplx{0, 0});
        if (const char* dir = getenv("QSV_JIT_DUMP")) {  // inspection: one file per pass
          const std::string path =
              std::string(dir) + "/pass_r" + std::to_string(kRegBits) + "_" + std::to_string(tiles.size()) + ".cu";
          if (FILE* f = fopen(path.c_str(), "w")) {
            fputs(tp.jit_src.c_str(), f);
            fclose(f);
          }
        }
      } catch (const std::exception&) {
        tp.jit_src.clear();  // this pass stays on the interpreter
      }
    }
    if (mix) {
      for (const TileOp& op : e.ops) {
        const int cnt = __builtin_popcount((uint32_t)op.slots);
        if (op.kind == T_REAL1 || op.kind == T_REAL1X) mix->real_ops += cnt;
        if (op.kind == T_DENSE1 || op.kind == T_DENSE1X) mix->complex_ops += cnt;
        if (op.kind == S_DENSE && op.m >= 5) mix->wide_dense += 1;
        else if (op.kind == S_DENSE || op.kind == S_PAULI) mix->complex_ops += 1;
      }
    }
    for (int q = 0; q < n; ++q)
      if ((ps.S >> q) & 1ULL) tp.qubits.push_back(q);
    tp.nphases = (int)e.phases.size();
    tp.nops = (int)e.ops.size();
    tp.ndata = (int)e.data.size();
    tp.num_gates = (int)pg.size();
    tp.hbm_bytes = 32.0 * std::ldexp(1.0, n);
    stats->fp64_flops += 2.0 * e.fp64_ops_per_amp * std::ldexp(1.0, n);
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
  if (!replaying && !record.empty()) {
    std::lock_guard<std::mutex> lk(g_sel_mu);
    if (g_sel_cache.size() >= 64) g_sel_cache.clear();
    g_sel_cache.emplace(std::move(fp), std::move(record));
  }
  return QSV_OK;
}

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s, int max_ctas, unsigned long long* ctr, uint64_t fmask,
                     uint64_t fval) {
  const char* basep = (const char*)dev_payload + tp.dev_off;
  size_t off = align_up(sizeof(TilePassDev), 16);
  const TilePassDev* pd = reinterpret_cast<const TilePassDev*>(basep);
  const TilePhase* ph = reinterpret_cast<const TilePhase*>(basep + off);
  off = align_up(off + tp.nphases * sizeof(TilePhase), 16);
  const TileOp* ops = reinterpret_cast<const TileOp*>(basep + off);
  off = align_up(off + tp.nops * sizeof(TileOp), 16);
  const double2* data = reinterpret_cast<const double2*>(basep + off);
  // tiles enumerate the outer qubits; fixed ones (fmask, run_fixed) are
  // inserted with their value, so only that block's tiles are visited
  int pos[kMaxFixed];
  int np = 0;
  for (int j = 0; j < tp.L; ++j) pos[np++] = tp.qubits[j];
  for (int q = 0; q < n; ++q)
    if ((fmask >> q) & 1) {
      if (np >= kMaxFixed) {
        set_error("too many fixed qubits for a tile pass");
        return QSV_EINVAL;
      }
      pos[np++] = q;
    }
  FixedBits tb = make_fixed(pos, np, fval & fmask);
  const uint64_t ntiles_all = 1ULL << (n - np);
  if (tp.jit.kernel) {
    // generated kernel: same persistent work-counter scheme, payload in the
    // kernel parameter (constant bank), no program staging in shared memory
    static thread_local std::vector<char> pbuf;
    pbuf.resize(sizeof(JitParamHead) + sizeof(double2) * tp.jit_data.size());
    JitParamHead h;
    memset(&h, 0, sizeof(h));
    h.a = amps;
    h.ntiles = ntiles_all;
    h.ctr = ctr;
    h.tb = tb;
    int dev = 0, num_sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    const int sms = max_ctas > 0 ? std::min(max_ctas, num_sms) : num_sms;
    // CTAs per SM: registers (64K per SM) and shared memory (227 KB) allow
    int per_sm = 1;
    if (tp.jit.regs > 0) {
      const int regs = ((tp.jit.regs + 7) / 8) * 8;
      per_sm = std::max(1, std::min(65536 / (regs * tp.jit_threads),
                                    (int)((227u * 1024u) / (tp.jit_smem + 1024))));
      per_sm = std::min(per_sm, 8);
    }
    if (max_ctas > 0) per_sm = 1;
    unsigned grid;
    if (ntiles_all <= (uint64_t)sms * per_sm && jit_static_tiles()) {
      grid = (unsigned)ntiles_all;
      h.stat = 1;
    } else if (ntiles_all <= (uint64_t)sms * per_sm) {
      grid = (unsigned)ntiles_all;
    } else {
      const int groups = tp.jit_groups > 0 ? tp.jit_groups : kGroups;
      const uint64_t ctas = (ntiles_all + groups - 1) / groups;
      grid = (unsigned)std::min<uint64_t>(ctas, (uint64_t)sms * per_sm);
      h.nostagger = ntiles_all <= (uint64_t)groups * grid;
    }
    if (ntiles_all <= (uint64_t)sms * per_sm) h.nostagger = 0;
    // deep passes: the generated code (~10 KB of SASS per phase) exceeds the
    // instruction cache, so two groups half a tile apart stream two code
    // regions; starting them together lets them share the fetched code
    // (QSV_STAGGER_MAX_PHASES, A/B)
    if (tp.nphases > jit_stagger_max_phases() && ntiles_all > (uint64_t)sms * per_sm)
      h.nostagger = 1;
    memcpy(pbuf.data(), &h, sizeof(h));
    memcpy(pbuf.data() + sizeof(h), tp.jit_data.data(), sizeof(double2) * tp.jit_data.size());
    int rc = jit_set_smem(tp.jit, tp.jit_smem);
    if (rc) return rc;
    void* args[] = {pbuf.data()};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tp.jit_threads);
    cfg.dynamicSmemBytes = tp.jit_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed =
        (jit_pdl_mode() == 1 || (jit_pdl_mode() < 0 && tp.pdl)) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    QSV_TRY(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(tp.jit.kernel), args));
    return QSV_OK;
  }
  if (tp.jit_only) {
    set_error("tile pass needs its generated kernel (NVRTC compile failed or not prepared)");
    return QSV_EUNSUPPORTED;
  }
  const size_t smem = kGroups * (sizeof(double2) << tp.L) + tp.nops * sizeof(TileOp) +
                      tp.ndata * sizeof(double2) + tp.nphases * sizeof(TilePhase);
  if (smem > kTileSmemLimit) {
    set_error("tile pass program (%d ops, %d phases) does not fit in shared memory", tp.nops,
              tp.nphases);
    return QSV_EUNSUPPORTED;
  }
  static int attr_dev = -1;
  static int num_sms = 148;
  static int dyn_limit = kTileSmemLimit;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    // the dynamic window is what the static shared memory leaves of 227 KB
    cudaFuncAttributes fa;
    QSV_TRY(cudaFuncGetAttributes(&fa, k_tile));
    dyn_limit = std::min<int>(kTileSmemLimit, 227 * 1024 - (int)fa.sharedSizeBytes);
    QSV_TRY(cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 dyn_limit));
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    attr_dev = dev;
  }
  if ((int)smem > dyn_limit) {
    set_error("tile pass program (%d ops, %d phases) does not fit in shared memory", tp.nops,
              tp.nphases);
    return QSV_EUNSUPPORTED;
  }
  const uint64_t ntiles = 1ULL << (n - np);
  const int sms = max_ctas > 0 ? std::min(max_ctas, num_sms) : num_sms;
  // Few tiles (small states): one tile per SM while they last -- group 0 of
  // every CTA takes one, group 1 is held back by the stagger and finds none
  // left; up to two tiles per SM: both groups start at once (the stagger
  // would delay the second tile by half a tile); otherwise persistent CTAs.
  unsigned grid;
  int nostagger = 0;
  if (ntiles <= (uint64_t)sms) {
    grid = (unsigned)ntiles;
  } else {
    const uint64_t ctas = (ntiles + kGroups - 1) / kGroups;
    grid = (unsigned)std::min<uint64_t>(ctas, (uint64_t)sms);
    nostagger = ntiles <= (uint64_t)kGroups * grid;
  }
  k_tile<<<grid, kCtaThreads, smem, s>>>(amps, pd, ph, ops, data, tb, ntiles, tp.nops,
                                          tp.ndata, ctr, nostagger);
  QSV_CHECK_LAUNCH("k_tile");
  return QSV_OK;
}

}  // namespace QSV_TILE_NS
}  // namespace qsv
