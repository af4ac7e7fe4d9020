// Compiled circuits (qsv_program): host-side plan + device payloads.
#pragma once

#include <vector>

#include "qsv_internal.cuh"

namespace qsv {

std::vector<char> make_payload(const GateDesc& g);

// One step of a program: either a single gate kernel or a tile pass that
// applies several gates per HBM sweep (qsv_tile_impl.cuh).
struct TilePass;

struct Step {
  int type;           // 0 = gate kernel, 1 = tile pass
  GateDesc gate;      // canonical gate (type 0)
  size_t payload_off; // offset into the program's device payload (type 0)
  bool has_payload;
  int tile;           // index into program tile passes (type 1)
};

}  // namespace qsv
