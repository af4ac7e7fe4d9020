// Variant selection for the tile engine (see qsv_tile.cuh): the 32-amplitude
// kernel (r5) when the preprocessed gate list is mostly real-rotation
// batches, otherwise the 16-amplitude kernel (r4); one plan per program.  Measured (profiles/variant_ab.py, time_fused.py):
// cz-ladder r5, cnot-ring / QV / QFT / heavy(2..4) r4, heavy(5) r5 (2x).
// QSV_TILE_VARIANT=4|5 forces one (A/B experiments).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>

#include "qsv_tile.cuh"

namespace qsv {

// Cheap estimate of the encoded op mix from the preprocessed gate list:
// real-matrix 1-qubit gates (split rotations, X / CNOT) become real register
// batches, other 1-qubit gates complex ones, 2..4-target dense / X-Y Paulis
// shared-memory phases.
static PlanMix estimate_mix(const std::vector<GateDesc>& gates) {
  PlanMix m;
  for (const GateDesc& g : gates) {
    if (g.kind == QSV_OP_DENSE && g.m == 1) {
      bool real = g.rf != 0;
      if (!real) {
        real = true;
        for (const Cplx& c : g.data) real = real && c.im == 0.0;
      }
      if (real) ++m.real_ops;
      else ++m.complex_ops;
    } else if (g.kind == QSV_OP_DENSE && g.m >= 2 && g.m <= 4) {
      ++m.complex_ops;
    } else if (g.kind == QSV_OP_PAULI || g.kind == QSV_OP_PAULI_ROT) {
      for (int j = 0; j < g.m; ++j)
        if (g.ids[j] == 1 || g.ids[j] == 2) {
          ++m.complex_ops;
          break;
        }
    }
  }
  return m;
}

static std::mutex g_mode_mu;
static std::unordered_map<std::string, int> g_mode_cache;  // structure -> search mode

static int plan_program_impl(int n, const std::vector<GateDesc>& gates,
                             const qsv_plan_opts& opts, std::vector<Step>& steps,
                             std::vector<TilePlan>& tiles, std::vector<char>& payload,
                             qsv_program_stats* stats);

// Programmatic dependent launch per program: on small states it hides the
// kernel boundary when every pass is shallow (cnot-ring(16) 0.100 -> 0.095 ms,
// (17) 0.112 -> 0.111, (18) 0.134 -> 0.132) but costs deep passes up to 15%
// (cz-ladder(12..18): the next pass's CTAs take SM slots while the current
// pass still runs; profiles/r2_pdl_late_ab.md) and measured 6% slower on
// cnot-ring(19) (r4 tiles, one CTA on 128 of 148 SMs), so it is used for the
// small-state programs (n <= 18) whose passes have at most kPdlMaxPhases
// phases (profiles/r2_pdl_auto_ab.md).
int plan_program(int n, const std::vector<GateDesc>& gates, const qsv_plan_opts& opts,
                 std::vector<Step>& steps, std::vector<TilePlan>& tiles,
                 std::vector<char>& payload, qsv_program_stats* stats) {
  const int rc = plan_program_impl(n, gates, opts, steps, tiles, payload, stats);
  if (rc != QSV_OK) return rc;
  constexpr int kPdlMaxPhases = 8;
  bool shallow = n <= 18 && !tiles.empty();
  for (const TilePlan& tp : tiles) shallow = shallow && tp.nphases <= kPdlMaxPhases;
  for (TilePlan& tp : tiles) tp.pdl = shallow;
  return QSV_OK;
}

static int plan_program_impl(int n, const std::vector<GateDesc>& gates,
                             const qsv_plan_opts& opts, std::vector<Step>& steps,
                             std::vector<TilePlan>& tiles, std::vector<char>& payload,
                             qsv_program_stats* stats) {
  if (!steps.empty() || !tiles.empty() || !payload.empty()) {
    set_error("internal: plan_program expects empty outputs");
    return QSV_EINVAL;
  }
  int force = 0;
  if (const char* v = getenv("QSV_TILE_VARIANT")) force = atoi(v);
  const bool on4 = r4::tiles_enabled(n, opts), on5 = r5::tiles_enabled(n, opts);
  if (on4 != on5) force = 4;  // tiny states: only the 16-amplitude kernel tiles them
  // fusion and real frames once (identical in both variants), then one plan
  std::vector<GateDesc> pre = r5::preprocess(n, gates, opts);
  bool use5 = force == 5;
  // the 8-amplitude kernel (r3) takes tiles of at most 11 qubits
  bool use3 = force == 3 && on4 && n >= 12;
  int l3 = 0;  // its tile size when chosen here
  if (!force) {
    const PlanMix mix = estimate_mix(pre);
    // small states under generated kernels: a pass is a chain of dependent
    // phases on 32..256 tiles, one warp per scheduler; twice the threads per
    // tile halve each thread's chain (cnot-ring(16) 0.118 -> 0.101 ms,
    // cz-ladder(16) 0.104 -> 0.092, (14) 0.091 -> 0.077, cnot-ring(18) 0.151
    // -> 0.134; from n = 20 the 16-amplitude kernel with 12-qubit tiles is
    // faster, profiles/r2_small_n_r3.md)
    if (opts.jit && opts.tile_qubits == 0 && opts.outer_mask == 0 && n >= 12 && n <= 18 &&
        on4 && on5 && mix.wide_dense == 0 && !getenv("QSV_FIXED_TILE")) {
      use3 = true;
      l3 = n <= 17 ? 10 : 11;  // n = 17: 0.112 vs 0.124 ms (cnot-ring); n = 18 equal
    }
    const int r5_score = mix.real_ops / 2 + 4 * mix.wide_dense;
    use5 = r5_score > 0 && r5_score >= mix.complex_ops;
    // generated pass kernels (the steady state of a program run more than
    // once): the 16-amplitude variant is as fast at n = 28..30 (cz-ladder(30)
    // 272 vs 268 ms, (28) 64.1 vs 64.8 ms) and faster on small states
    // (cz-ladder(14) 0.108 vs 0.149 ms, (18) 0.156 vs 0.206 ms, (22) 0.84 vs
    // 0.98 ms; profiles/r2_variants_jit.txt): twice the warps per SM
    if (opts.jit && mix.wide_dense == 0) use5 = false;
  }
  if (force == 4 && on4 != on5)
    return r4::plan_program(n, gates, opts, steps, tiles, payload, stats, nullptr, false);
  auto plan_with = [&](const qsv_plan_opts& o, std::vector<Step>& st, std::vector<TilePlan>& tp,
                       std::vector<char>& pl, qsv_program_stats* ps) {
    if (use3) {
      qsv_plan_opts o3 = o;
      if (o3.tile_qubits == 0) o3.tile_qubits = l3 ? l3 : 11;
      // 12-qubit tiles (512 threads, one group per CTA) only as generated kernels
      o3.tile_qubits = std::min(o3.tile_qubits, o.jit ? 12 : 11);
      return r3::plan_program(n, pre, o3, st, tp, pl, ps, nullptr, true);
    }
    return use5 ? r5::plan_program(n, pre, o, st, tp, pl, ps, nullptr, true)
                : r4::plan_program(n, pre, o, st, tp, pl, ps, nullptr, true);
  };
  // Small states (n <= 20, default tile size, unsharded): a pass has at most
  // a few waves of tiles, so its time is a per-pass latency plus, per phase,
  // work proportional to the tile size times the waves; smaller tiles put
  // more SMs to work at the price of more passes.  Plan L = 10, 11, 12 and
  // keep the cheapest under that model (fitted on cnot-ring / cz-ladder at
  // n = 14..20 with the few-tile grid policy of launch_tile_pass,
  // profiles/time_small_n.py: it picks the measured best or within 1% of it
  // in all eight cases).
  // (generated kernels from n = 19: 12-qubit tiles measured best at n = 19..22 -- cnot-ring(19)
  // 0.190 vs 0.240 ms for the model's L = 11, profiles/r2_mid_n.md -- so the model only
  // serves the interpreter)
  if (opts.tile_qubits == 0 && opts.outer_mask == 0 && n <= 20 && n >= 11 && on4 && on5 &&
      !l3 && !(opts.jit && n >= 19) && !getenv("QSV_FIXED_TILE")) {
    constexpr double kPass = 15.2e-3, kAmpPhase = 2.95e-7;  // ms
    constexpr double kGroupsPerGpu = 296.0;                 // 2 tile groups x 148 SMs
    double best_cost = 0;
    int best_rc = QSV_OK;
    bool have = false;
    const qsv_program_stats init = *stats;
    for (int L = 10; L <= (use3 ? 11 : 12); ++L) {
      qsv_plan_opts o = opts;
      o.tile_qubits = L;
      std::vector<Step> st;
      std::vector<TilePlan> tp;
      std::vector<char> pl;
      qsv_program_stats ps = init;
      const int rc = plan_with(o, st, tp, pl, &ps);
      if (rc) {
        if (!have) best_rc = rc;
        continue;
      }
      double cost = 0;
      for (const Step& s : st) {
        cost += kPass;
        if (s.type == 1) {
          const TilePlan& t = tp[s.tile];
          const double waves = std::ceil(std::ldexp(1.0, n - t.L) / kGroupsPerGpu);
          cost += t.nphases * kAmpPhase * std::ldexp(1.0, t.L) * waves;
        }
      }
      if (!have || cost < best_cost) {
        have = true;
        best_cost = cost;
        steps.swap(st);
        tiles.swap(tp);
        payload.swap(pl);
        *stats = ps;
      }
    }
    return have ? QSV_OK : best_rc;
  }
  // Larger states: the tile-set search with one pass of lookahead usually
  // packs the circuit into fewer passes, but not always (cz-ladder(28): 17
  // passes vs 16 without the lookahead); each pass costs at least one HBM
  // sweep, so plan both and keep the one with fewer passes (lookahead on a
  // tie).  Measured: cz-ladder(30) 19 -> 18 passes, 253 -> 245 ms; VQE(24)
  // 7 -> 5 passes, 1.32 -> 1.15 ms; cz-ladder(28) keeps 16 (54.7 ms).
  if (!getenv("QSV_PASS_SEARCH") && opts.outer_mask == 0) {
    // the winning mode is remembered by gate-list structure, so a
    // ParametricCircuit recompiled after set_parameter plans once
    std::string fp;
    {
      const int32_t hdr[6] = {n, opts.tile_qubits, opts.fuse, opts.real_frames, opts.use_tiles,
                              (int32_t)pre.size()};
      fp.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
      for (const GateDesc& g : pre) {
        const int32_t rec[3] = {g.kind | (g.m << 8) | (g.nc << 16), g.rf, 0};
        fp.append(reinterpret_cast<const char*>(rec), sizeof(rec));
        fp.append(reinterpret_cast<const char*>(g.targets), sizeof(int) * g.m);
        fp.append(reinterpret_cast<const char*>(g.cq), sizeof(int) * g.nc);
        fp.append(reinterpret_cast<const char*>(g.cv), sizeof(int) * g.nc);
      }
    }
    {
      std::lock_guard<std::mutex> lk(g_mode_mu);
      auto it = g_mode_cache.find(fp);
      if (it != g_mode_cache.end()) {
        tl_pass_search = it->second;
        const int rc = plan_with(opts, steps, tiles, payload, stats);
        tl_pass_search = -1;
        return rc;
      }
    }
    // the multi-start plan is only counted (no kernel sources generated);
    // it is planned again in full only when it wins
    qsv_plan_opts count_only = opts;
    count_only.jit = 0;
    std::vector<Step> st1;
    std::vector<TilePlan> tp1;
    std::vector<char> pl1;
    qsv_program_stats ps1 = *stats;
    const qsv_program_stats init = *stats;
    tl_pass_search = 1;
    const int rc1 = plan_with(count_only, st1, tp1, pl1, &ps1);
    tl_pass_search = 2;
    int rc = plan_with(opts, steps, tiles, payload, stats);
    int mode = 2;
    if (rc1 == QSV_OK && (rc != QSV_OK || ps1.num_steps < stats->num_steps)) {
      steps.clear(), tiles.clear(), payload.clear();
      *stats = init;
      tl_pass_search = mode = 1;
      rc = plan_with(opts, steps, tiles, payload, stats);
    }
    tl_pass_search = -1;
    if (rc == QSV_OK) {
      std::lock_guard<std::mutex> lk(g_mode_mu);
      if (g_mode_cache.size() >= 64) g_mode_cache.clear();
      g_mode_cache.emplace(std::move(fp), mode);
    }
    return rc;
  }
  return plan_with(opts, steps, tiles, payload, stats);
}

int launch_tile_pass(double2* amps, int n, const TilePlan& tp, const void* dev_payload,
                     cudaStream_t s, int max_ctas, unsigned long long* ctr, uint64_t fmask,
                     uint64_t fval) {
  if (tp.variant == 3)
    return r3::launch_tile_pass(amps, n, tp, dev_payload, s, max_ctas, ctr, fmask, fval);
  return tp.variant == 5
             ? r5::launch_tile_pass(amps, n, tp, dev_payload, s, max_ctas, ctr, fmask, fval)
             : r4::launch_tile_pass(amps, n, tp, dev_payload, s, max_ctas, ctr, fmask, fval);
}

}  // namespace qsv
