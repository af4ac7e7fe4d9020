// Tile passes: several gates applied per HBM sweep (see qsv_tile.cu).
#pragma once

#include <vector>

#include "qsv_internal.cuh"
#include "qsv_program.cuh"

namespace qsv {

// 16 amplitudes per thread: 512-thread CTAs (16 warps / SM) at 128 registers
// hide the FP64 and shared-memory latencies better than 32 amplitudes at 255
// registers (8 warps), which outweighs the 25% more register phases
// (cnot-ring(30) 0.76 s -> 0.66 s, cz-ladder(30, 20) unchanged).
#ifndef QSV_TILE_REGBITS
#define QSV_TILE_REGBITS 4
#endif
constexpr int kRegBits = QSV_TILE_REGBITS;  // amplitudes per thread = 2^kRegBits
constexpr int kRegs = 1 << kRegBits;
constexpr int kMaxTileQubits = 12;          // 2^12 amps = 64 KiB of shared memory
constexpr int kGroupThreads = (1 << kMaxTileQubits) / kRegs;  // threads per tile group
constexpr int kGroups = 2;                  // independent tile groups per CTA
constexpr int kCtaThreads = kGroups * kGroupThreads;
constexpr int kLowQubits = 4;       // qubits 0..3 are in every tile (256 B runs)
constexpr int kTileSmemLimit = 227 * 1024 - 8192;  // dynamic part (static smem aside)
// shared memory left for the staged pass program (ops, data, phases)
constexpr int kTileProgramBudget =
    kTileSmemLimit - kGroups * (16 << kMaxTileQubits) - 1024;

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
  int8_t tpos[4];     // DIAG: target position; >= 0 local bit, < 0: -(global bit)-1
                      // S_DENSE: local bit of matrix index bit j
  int32_t pad;
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

struct TilePhase {
  int32_t type;              // 0: register phase, 1: shared-memory ops
  int32_t regpos[kRegBits];  // local bit of each register slot
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
  int L = 0;
  std::vector<int> qubits;       // sorted tile qubits (global positions)
  size_t dev_off = 0;            // payload offset of TilePassDev, then phases, ops
  int nphases = 0;
  int nops = 0;
  int ndata = 0;
  int num_gates = 0;
  double hbm_bytes = 0;
};

int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats);

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s);

}  // namespace qsv
