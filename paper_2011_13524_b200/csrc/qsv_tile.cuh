// Tile passes: several gates applied per HBM sweep (see qsv_tile.cu).
#pragma once

#include <vector>

#include "qsv_internal.cuh"
#include "qsv_program.cuh"

namespace qsv {

// A tile pass: the state is swept in tiles of 2^L amplitudes whose qubit
// set is the low `c` qubits plus `high` (sorted); the tile's gates are
// executed in shared memory / registers between one HBM load and one store.
struct TilePlan {
  int L = 0;
  int c = 0;
  std::vector<int> high;
  size_t prog_off = 0;   // device payload offset of the tile program
  int prog_words = 0;    // size of the tile program (in 8-byte words)
  int num_gates = 0;
  double hbm_bytes = 0;
};

int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats);

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s);

}  // namespace qsv
