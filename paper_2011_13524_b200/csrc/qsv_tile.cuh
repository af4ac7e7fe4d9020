// Tile passes: several gates applied per HBM sweep (implementation in
// qsv_tile_impl.cuh, compiled as qsv_tile_r4.cu / qsv_tile_r5.cu).
#pragma once

#include <string>
#include <vector>

#include "qsv_internal.cuh"
#include "qsv_jit.cuh"
#include "qsv_program.cuh"

namespace qsv {

// The tile engine is compiled twice from qsv_tile_impl.cuh, with 16 (r4) and
// 32 (r5) amplitudes per thread.  r5 (8 warps / SM at 255 registers, five
// register qubits per phase) is faster when a pass is mostly real-rotation
// batches (cz-ladder(30, 20): 0.51 s vs 0.58 s: fewer shared-memory phases and
// flushes); r4 (512-thread CTAs, 16 warps / SM at 128 registers) hides
// latency better for complex / controlled ops (cnot-ring(30): 0.66 s vs
// 0.69 s).  plan_program picks the variant per program (plan_select).
constexpr int kMaxRegBits = 5;
constexpr int kMaxTileQubits = 12;          // 2^12 amps = 64 KiB of shared memory
constexpr int kLowQubits = 4;       // qubits 0..3 are in every tile (256 B runs)
constexpr int kTileSmemLimit = 227 * 1024 - 8192;  // dynamic part (static smem aside)

// ---- device-side program records (all POD, stored in the payload) ----
enum TileOpKind : int32_t {
  // register-phase ops (each thread updates its 2^kRegBits amplitudes)
  T_DENSE1 = 1,   // 2x2 on one register slot (optionally controlled)
  T_DIAG = 5,     // diagonal, targets on local or tile (global) bits
  T_PHASE = 6,    // constant phase on a local/tile bit pattern
  T_PARITY = 7,   // f[parity(idx & zmask)]
  T_DENSE1X = 8,  // uncontrolled 2x2 on every slot of the mask (data: 4 per slot, slot order)
  T_REAL1 = 11,   // real 2x2 on one slot (optionally controlled; data: 2 double2 = a b, c d)
  T_REAL1X = 12,  // uncontrolled real 2x2 on every slot of the mask (2 double2 per slot)
  T_FLUSH = 13,   // merged diagonal: table over the register slots, linear sign
                  // rules and per-thread factors (see FlushSign / FlushFactor)
  T_SIGNS = 14,   // sign-only merged diagonal: table signs (lmask) + sign rules
  T_PHASES = 15,  // merged phase rules (controlled phases involving thread / tile
                  // bits): per-thread scalar and per-slot factors (FlushPhase)
  // shared-memory ops (a phase of their own; cosets read straight from smem)
  S_DENSE = 9,    // 2^m x 2^m on m <= 4 local bits (tpos), optionally controlled
  S_PAULI = 10,   // X/Y product on local bits (slots = local X mask), Z parity
};

struct __align__(16) TileOp {   // 64 bytes = 4 x 128-bit loads
  int32_t kind;
  int32_t slots;      // T_DENSE1: slot mask (bit i = register slot i)
                      // S_PAULI: X/Y mask over local bits
  int32_t flags;      // bit 1: T_PHASE factor is -1 (sign flip)
  int32_t m;          // DIAG / S_DENSE: number of targets
  uint32_t lmask;     // control pattern over local bits
  uint32_t lval;
  uint32_t zl;        // PARITY/PAULI: sign mask over local bits
  uint32_t data;      // payload offset (double2 units) of matrix / table / coefs
  uint64_t gmask;     // control pattern over global (non-tile) bits
  uint64_t gval;
  uint64_t zg;        // PARITY/PAULI: sign mask over global bits
  int8_t tpos[8];     // DIAG: target position; >= 0 local bit, < 0: -(global bit)-1
                      // S_DENSE: local bit of matrix index bit j (up to 5 targets)
};

// T_FLUSH payload: [T: 2^kRegBits double2][m FlushSign][slots FlushFactor]
// T_SIGNS payload: [m FlushSign]; TileOp.lmask holds the signs of its +-1 table.
struct __align__(16) FlushSign {  // where the thread/tile pattern matches, flip the
  uint32_t lm, lv;                // sign of the register slots j with bit j of col
  uint32_t col, pad;              // set (col: all ones, or the j_slot == value column)
  uint64_t gm, gv;
};
struct __align__(16) FlushFactor {  // factor d[bit] of one non-register qubit
  int32_t pos;                      // >= 0 local (thread) bit, < 0: -(global bit)-1
  int32_t pad[3];
  double2 d0, d1;
};

// T_PHASES payload: [m FlushPhase]; TileOp.slots = mask of slots with rules,
// flags & 1: some rule is a scalar (slot < 0).
struct __align__(16) FlushPhase {  // factor f where the thread/tile pattern matches,
  uint32_t lm, lv;                 // on every amplitude (slot < 0) or on those with
  int32_t slot, pad;               // register slot `slot` == 1
  uint64_t gm, gv;
  double2 f;
};

struct TilePhase {
  int32_t type;              // 0: register phase, 1: shared-memory ops
  int32_t regpos[kMaxRegBits];  // local bit of each register slot
  int32_t thrpos[10];        // local bit of thread-id bit j (j < L - kRegBits)
  // thread's local base lt = thr_lo[tid & 15] | thr_hi[tid >> 4] (host-built
  // deposit tables: one lookup per phase instead of a bit loop)
  uint32_t thr_lo[16], thr_hi[16];
  int32_t op_begin, op_end;
};

struct TilePassDev {
  int32_t L;
  int32_t nthrbits;          // L - kRegBits
  int32_t nphases;
  int32_t debug;             // profiling knobs (QSV_TILE_DEBUG): 1 skip ops, 2 skip phases
  uint64_t smask;            // tile qubits (global positions)
  int32_t spos[kMaxTileQubits];  // local bit j -> global qubit
};

// ---- host-side plan of one pass ----
struct TilePlan {
  int variant = 4;               // register bits of the kernel that runs it
  int L = 0;
  std::vector<int> qubits;       // sorted tile qubits (global positions)
  size_t dev_off = 0;            // payload offset of TilePassDev, then phases, ops
  int nphases = 0;
  int nops = 0;
  int ndata = 0;
  int num_gates = 0;
  double hbm_bytes = 0;
  // runtime-compiled form (qsv_tile_jit.cuh / qsv_jit.cu): generated source,
  // launch shape, payload passed as the kernel parameter; `jit.kernel` is
  // set once compiled (until then the interpreter k_tile runs the pass)
  std::string jit_src;
  bool jit_seen = false;  // the same pass structure was planned before in this process
  int jit_threads = 0;
  int jit_groups = 0;     // tile groups per CTA of the generated kernel
  bool jit_only = false;  // the interpreter cannot run this pass (more than 8 thread bits)
  bool pdl = false;       // launch with programmatic dependent launch (shallow programs)
  size_t jit_smem = 0;
  std::vector<Cplx> jit_data;
  JitKernel jit;
};

// tile-set search mode of the planner for the current thread (-1: the
// QSV_PASS_SEARCH default); plan_program (qsv_tile_select.cu) plans with
// several modes and keeps the plan with the fewest passes
inline thread_local int tl_pass_search = -1;

// per-variant entry points (qsv_tile_r4.cu / qsv_tile_r5.cu)
struct PlanMix {
  int real_ops = 0, complex_ops = 0;  // register 2x2 ops after encoding (+ narrow smem ops)
  int wide_dense = 0;                 // 5-target shared-memory dense ops
};
#define QSV_TILE_DECLARE(NS)                                                                 \
  namespace NS {                                                                            \
  int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,    \
                   std::vector<Step>& steps, std::vector<TilePlan>& tiles,                  \
                   std::vector<char>& payload, qsv_program_stats* stats, PlanMix* mix,      \
                   bool preprocessed);                                                      \
  bool tiles_enabled(int n, const qsv_plan_opts& opts);                                     \
  std::vector<GateDesc> preprocess(int n, const std::vector<GateDesc>& gates,              \
                                   const qsv_plan_opts& opts);                              \
  int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,   \
                       cudaStream_t s, int max_ctas, unsigned long long* ctr,               \
                       uint64_t fmask, uint64_t fval);                                      \
  }
QSV_TILE_DECLARE(r3)
QSV_TILE_DECLARE(r4)
QSV_TILE_DECLARE(r5)
#undef QSV_TILE_DECLARE

// plan with the variant that suits the circuit (qsv_program.cu)
int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats);

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s, int max_ctas, unsigned long long* ctr, uint64_t fmask,
                     uint64_t fval);

}  // namespace qsv
