// Tile passes and the program planner.
#include <algorithm>
#include <cstring>
#include <cmath>

#include "qsv_tile.cuh"

namespace qsv {

int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats) {
  (void)opts;
  (void)tiles;
  for (const GateDesc& g : gates) {
    Step st;
    st.type = 0;
    st.gate = g;
    st.tile = -1;
    std::vector<char> pl = make_payload(g);
    st.has_payload = !pl.empty();
    st.payload_off = 0;
    if (st.has_payload) {
      size_t off = (payload.size() + 255) & ~(size_t)255;
      payload.resize(off + pl.size());
      memcpy(payload.data() + off, pl.data(), pl.size());
      st.payload_off = off;
    }
    steps.push_back(st);
    stats->num_gate_kernels += 1;
    stats->num_steps += 1;
    stats->hbm_bytes += gate_hbm_bytes(n, g);
  }
  return QSV_OK;
}

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s) {
  (void)amps; (void)n; (void)tp; (void)dev_payload; (void)s;
  set_error("tile passes not available");
  return QSV_EUNSUPPORTED;
}

}  // namespace qsv
