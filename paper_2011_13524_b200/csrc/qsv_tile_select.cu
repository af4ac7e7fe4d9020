// Variant selection for the tile engine (see qsv_tile.cuh): plan with the
// 32-amplitude kernel (r5) and keep it when the encoded passes are mostly
// real-rotation batches or 5-target dense blocks; otherwise re-plan for the
// 16-amplitude kernel (r4).  Measured (profiles/variant_ab.py, time_fused.py):
// cz-ladder r5, cnot-ring / QV / QFT / heavy(2..4) r4, heavy(5) r5 (2x).
// QSV_TILE_VARIANT=4|5 forces one (A/B experiments).
#include <cstdlib>

#include "qsv_tile.cuh"

namespace qsv {

int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats) {
  if (!steps.empty() || !tiles.empty() || !payload.empty()) {
    set_error("internal: plan_program expects empty outputs");
    return QSV_EINVAL;
  }
  int force = 0;
  if (const char* v = getenv("QSV_TILE_VARIANT")) force = atoi(v);
  if (force != 4) {
    std::vector<Step> s5;
    std::vector<TilePlan> t5;
    std::vector<char> p5;
    qsv_program_stats st5 = *stats;
    PlanMix mix;
    int rc = r5::plan_program(n, gates, opts, s5, t5, p5, &st5, &mix);
    if (rc) return rc;
    // r5 for real-rotation batches (fewer phases / flushes) and for 5-target
    // dense blocks (their 32-amplitude cosets need the larger register file)
    const int r5_score = mix.real_ops / 2 + 4 * mix.wide_dense;
    if (force == 5 || (r5_score > 0 && r5_score >= mix.complex_ops)) {
      // the caller's vectors start empty, so offsets and indices carry over
      steps.swap(s5);
      tiles.swap(t5);
      payload.swap(p5);
      *stats = st5;
      return QSV_OK;
    }
  }
  return r4::plan_program(n, gates, opts, steps, tiles, payload, stats, nullptr);
}

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s) {
  return tp.variant == 5 ? r5::launch_tile_pass(amps, n, tp, dev_payload, s)
                         : r4::launch_tile_pass(amps, n, tp, dev_payload, s);
}

}  // namespace qsv
