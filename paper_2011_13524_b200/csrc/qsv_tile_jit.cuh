// Tile-pass code generator (included by qsv_tile_impl.cuh inside the variant
// namespace; host code only).
//
// The interpreter k_tile reads every op of a pass from shared memory and
// dispatches on it per tile: register slots, thread-bit layouts, control
// patterns and table shapes are runtime values, so each op costs branches,
// address arithmetic and spills (profiles/r1_tile_stalls_n28.md: op dispatch
// ~20% of the stall samples, LDL/STL 4% of the instructions).  This generator
// turns one encoded pass (the same phases and slot-space ops the interpreter
// runs) into straight-line CUDA for that pass: every slot index, shared-memory
// offset, thread-bit deposit and control mask is a literal, pairs excluded by
// a register-slot control are simply not emitted, exact 1 / -1 table entries
// become no-ops / sign flips, and the numeric payload (matrices, tables,
// factors) is passed as a __grid_constant__ kernel parameter, so DFMA/DMUL
// take it straight from the constant bank.  The code depends only on the
// pass's structure and on which payload entries are exactly 0 / +-1, so a
// VQE parameter update (new angles, same structure) hits the compile cache.
// NVRTC compiles it to sm_100a SASS (qsv_jit.cu).

struct JitSource {
  std::string src;      // CUDA source of kernel "k_pass"
  int threads = 0;      // CTA threads
  int group_threads = 0;
  int groups = 0;       // tile groups per CTA
  size_t smem = 0;      // dynamic shared memory
  int ndata = 0;        // double2 entries of the payload parameter
  bool seen = false;    // served from the source cache: this structure was planned before
};

namespace jitgen {

inline std::string hex64(uint64_t v) {
  char b[32];
  snprintf(b, sizeof(b), "0x%llxull", (unsigned long long)v);
  return b;
}
inline std::string hex32(uint32_t v) {
  char b[24];
  snprintf(b, sizeof(b), "0x%xu", v);
  return b;
}

// thread-local index of tid placed at the given local bits (literal shifts)
inline std::string deposit(const std::vector<int>& pos, const char* var) {
  std::string s = "(0u";
  for (size_t j = 0; j < pos.size(); ++j) {
    char b[96];
    snprintf(b, sizeof(b), " | (((%s >> %zu) & 1u) << %d)", var, j, pos[j]);
    s += b;
  }
  return s + ")";
}

inline void replace_first(std::string& s, const std::string& from, const std::string& to) {
  const size_t at = s.find(from);
  if (at != std::string::npos) s.replace(at, from.size(), to);
}
inline uint32_t swz_host(uint32_t l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u); }

inline bool is_val(const Cplx& c, double re, double im) { return c.re == re && c.im == im; }

struct Gen {
  const Encoded& e;
  int L, R, R2, G;
  std::string o;
  // emitted once, right before the tile's first shared-memory store (the
  // group barrier that protects the tile buffer, moved past the loads)
  std::string pre_store;
  bool late_wait = false;  // static tiles wait for the previous pass at their first load
  explicit Gen(const Encoded& enc, int L_) : e(enc), L(L_), R(kRegBits), R2(kRegs) {
    G = 1 << (L - kRegBits);
  }
  void line(const std::string& s) {
    o += s;
    o += '\n';
  }
  std::string d(uint32_t idx) const {  // payload entry as an expression
    return "P.d[" + std::to_string(idx) + "]";
  }
  // What the generated text depends on besides the op / phase arrays: the
  // class (0, 1, -1, other per real part) of every payload value the
  // generator inspects, and the raw bytes of structural records (sign /
  // factor / phase rules) stored in the payload.  Recorded so a later pass
  // with the same arrays and the same recorded facts reuses the source
  // (jit_pass_source) -- a VQE parameter update changes only other values.
  mutable std::vector<std::pair<uint32_t, uint8_t>> sig_cls;
  mutable std::vector<std::pair<uint32_t, uint32_t>> sig_raw;  // (first entry, entries)
  static uint8_t cls1(double x) { return x == 0.0 ? 0 : x == 1.0 ? 1 : x == -1.0 ? 2 : 3; }
  static uint8_t cls(const Cplx& c) { return (uint8_t)(cls1(c.re) | (cls1(c.im) << 2)); }
  const Cplx& val(uint32_t idx) const {
    sig_cls.push_back({idx, cls(e.data[idx])});
    return e.data[idx];
  }
  template <typename T>
  void rec(T* out, uint32_t idx, uint32_t structural_entries) const {
    memcpy(out, &e.data[idx], sizeof(T));
    sig_raw.push_back({idx, structural_entries});
  }

  // ---- register ops ----------------------------------------------------
  // pairs (j, j | 1 << I) of slot I whose register-control part holds
  template <typename F>
  void pairs(int I, uint32_t rm, uint32_t rv, F body) {
    for (int j = 0; j < R2; ++j) {
      if ((j >> I) & 1) continue;
      if (((uint32_t)j & rm) != rv) continue;
      body(j, j | (1 << I));
    }
  }
  void real1(int I, uint32_t rm, uint32_t rv, uint32_t D, bool swap) {
    if (swap) {
      pairs(I, rm, rv, [&](int j, int q) {
        line("{ double2 t_ = v[" + std::to_string(j) + "]; v[" + std::to_string(j) + "] = v[" +
             std::to_string(q) + "]; v[" + std::to_string(q) + "] = t_; }");
      });
      return;
    }
    const std::string ab = d(D), cd = d(D + 1);
    const Cplx A = val(D), B = val(D + 1);
    pairs(I, rm, rv, [&](int j, int q) {
      const std::string x = "v[" + std::to_string(j) + "]", y = "v[" + std::to_string(q) + "]";
      line("{ const double2 x_ = " + x + ", y_ = " + y + ";");
      // [[a, b], [c, d]] with a = ab.x, b = ab.y, c = cd.x, d = cd.y
      auto out = [&](const std::string& dst, double m0, const std::string& e0, double m1,
                     const std::string& e1) {
        for (const char* c : {".x", ".y"}) {
          std::string expr;
          if (m0 == 0.0 && m1 == 0.0) expr = "0.0";
          else if (m0 == 0.0) expr = (m1 == 1.0 ? std::string("y_") + c
                                      : m1 == -1.0 ? std::string("-y_") + c
                                                   : e1 + " * y_" + c);
          else if (m1 == 0.0) expr = (m0 == 1.0 ? std::string("x_") + c
                                      : m0 == -1.0 ? std::string("-x_") + c
                                                   : e0 + " * x_" + c);
          else if (m0 == 1.0) expr = "fma(" + e1 + ", y_" + c + ", x_" + c + ")";
          else if (m1 == 1.0) expr = "fma(" + e0 + ", x_" + c + ", y_" + c + ")";
          else expr = "fma(" + e1 + ", y_" + c + ", " + e0 + " * x_" + c + ")";
          line("  " + dst + c + " = " + expr + ";");
        }
      };
      out(x, A.re, ab + ".x", A.im, ab + ".y");
      out(y, B.re, cd + ".x", B.im, cd + ".y");
      line("}");
    });
  }
  void dense1(int I, uint32_t rm, uint32_t rv, uint32_t D) {
    pairs(I, rm, rv, [&](int j, int q) {
      const std::string x = "v[" + std::to_string(j) + "]", y = "v[" + std::to_string(q) + "]";
      line("{ const double2 x_ = " + x + ", y_ = " + y + ";");
      line("  " + x + " = cfma(" + d(D + 1) + ", y_, cmul(" + d(D) + ", x_));");
      line("  " + y + " = cfma(" + d(D + 3) + ", y_, cmul(" + d(D + 2) + ", x_));");
      line("}");
    });
  }
  // v[j] *= T[j] for every slot, T = payload[D .. D + R2), exact +-1 skipped /
  // folded into the sign mask `*neg`, real entries as two multiplies
  void table_mul(uint32_t D, uint32_t* neg) {
    for (int j = 0; j < R2; ++j) {
      const Cplx t = val(D + j);
      const std::string vj = "v[" + std::to_string(j) + "]";
      if (is_val(t, 1, 0)) continue;
      if (is_val(t, -1, 0)) {
        *neg ^= 1u << j;
        continue;
      }
      if (t.im == 0.0) {
        line(vj + ".x *= " + d(D + j) + ".x; " + vj + ".y *= " + d(D + j) + ".x;");
        continue;
      }
      line(vj + " = cmul(" + vj + ", " + d(D + j) + ");");
    }
  }
  // runtime sign rules (FlushSign records at payload D..): bits ^= col where
  // the thread / tile pattern holds
  // returns the bits some thread may see set (the others are the static
  // xor of sgn0 and the unconditional rules, tracked in *stat)
  uint32_t sign_rules(uint32_t D, int m, const char* bits, uint32_t* stat = nullptr) {
    uint32_t dyn = 0;
    for (int r = 0; r < m; ++r) {
      FlushSign S;
      rec(&S, D + 2 * r, 2);
      std::string cond;
      if (S.lm) cond += "(lt & " + hex32(S.lm) + ") == " + hex32(S.lv);
      if (S.gm) {
        if (!cond.empty()) cond += " && ";
        cond += "(base & " + hex64(S.gm) + ") == " + hex64(S.gv);
      }
      if (cond.empty()) {
        line(std::string(bits) + " ^= " + hex32(S.col) + ";");
        if (stat) *stat ^= S.col;
      } else {
        line("if (" + cond + ") " + bits + " ^= " + hex32(S.col) + ";");
        dyn |= S.col;
      }
    }
    return dyn;
  }
  void apply_signs(const char* bits, uint32_t const_neg, uint32_t dyn, uint32_t stat) {
    // v[j] = -v[j] where bit j of (bits ^ const_neg) is set: one shift and
    // one three-input LOP3 per component ((t & 0x80000000) ^ hi, the mask
    // folded into the xor); bits no thread sees change are static negations
    for (int j = 0; j < R2; ++j) {
      const std::string vj = "v[" + std::to_string(j) + "]";
      if (!((dyn >> j) & 1u)) {
        if (((stat ^ const_neg) >> j) & 1u)
          line(vj + ".x = -" + vj + ".x; " + vj + ".y = -" + vj + ".y;");
        continue;
      }
      const std::string t = "(" + std::string(bits) + " << " + std::to_string(31 - j) + ")";
      line(vj + " = negm" + (((const_neg >> j) & 1u) ? "<true>" : "") + "(" + vj + ", " + t +
           ");");
    }
  }
  void apply_signs_old(const char* bits, uint32_t const_neg) {
    for (int j = 0; j < R2; ++j) {
      const std::string vj = "v[" + std::to_string(j) + "]";
      if ((const_neg >> j) & 1u)
        line("{ const int s_ = (int)(((~" + std::string(bits) + ") << " +
             std::to_string(31 - j) + ") & 0x80000000u); " + vj + " = negs(" + vj +
             ", s_); }");
      else
        line("{ const int s_ = (int)((" + std::string(bits) + " << " + std::to_string(31 - j) +
             ") & 0x80000000u); " + vj + " = negs(" + vj + ", s_); }");
    }
  }

  void op_flush(const TileOp& op) {
    const uint32_t D = op.data;
    const bool table = op.kind == T_FLUSH;
    const uint32_t sgn0 = table ? 0u : op.lmask;
    const uint32_t sD = table ? D + R2 : D;
    line("{ uint32_t bits_ = " + hex32(sgn0) + ";");
    uint32_t stat = sgn0;
    const uint32_t dyn = sign_rules(sD, op.m, "bits_", &stat);
    uint32_t neg = 0;
    if (table) {
      if (op.slots) {  // per-thread factors of non-register qubits
        const uint32_t fD = sD + 2 * op.m;
        line("  double2 C_ = make_double2(1.0, 0.0);");
        for (int f = 0; f < op.slots; ++f) {
          FlushFactor F;
          rec(&F, fD + 3 * f, 1);  // pos (the factors are read as P.d[...])
          const std::string bit =
              F.pos >= 0 ? "((lt >> " + std::to_string(F.pos) + ") & 1u)"
                         : "((base >> " + std::to_string(-F.pos - 1) + ") & 1ull)";
          line("  C_ = cmul(C_, " + bit + " ? " + d(fD + 3 * f + 2) + " : " + d(fD + 3 * f + 1) +
               ");");
        }
        for (int j = 0; j < R2; ++j)
          line("  v[" + std::to_string(j) + "] = cmul(v[" + std::to_string(j) + "], C_);");
      }
      table_mul(D, &neg);
    }
    if (op.m > 0 || sgn0 != 0) {
      if (jit_sign_fold()) apply_signs("bits_", neg, dyn, stat);
      else apply_signs_old("bits_", neg);
    } else if (neg) {
      for (int j = 0; j < R2; ++j)
        if ((neg >> j) & 1u)
          line("v[" + std::to_string(j) + "].x = -v[" + std::to_string(j) + "].x; v[" +
               std::to_string(j) + "].y = -v[" + std::to_string(j) + "].y;");
    }
    line("}");
  }

  void op_phases(const TileOp& op) {
    line("{ double2 C_ = make_double2(1.0, 0.0);");
    for (int i = 0; i < R; ++i)
      if ((op.slots >> i) & 1) line("  double2 ph" + std::to_string(i) + "_ = make_double2(1.0, 0.0);");
    for (int r = 0; r < op.m; ++r) {
      FlushPhase F;
      rec(&F, op.data + 3 * r, 2);  // masks and slot (f is read as P.d[...])
      std::string cond;
      if (F.lm) cond += "(lt & " + hex32(F.lm) + ") == " + hex32(F.lv);
      if (F.gm) {
        if (!cond.empty()) cond += " && ";
        cond += "(base & " + hex64(F.gm) + ") == " + hex64(F.gv);
      }
      const std::string tgt = F.slot < 0 ? "C_" : "ph" + std::to_string(F.slot) + "_";
      const std::string stmt = tgt + " = cmul(" + tgt + ", " + d(op.data + 3 * r + 2) + ");";
      line(cond.empty() ? "  " + stmt : "  if (" + cond + ") " + stmt);
    }
    if (op.flags & 1)
      for (int j = 0; j < R2; ++j)
        line("  v[" + std::to_string(j) + "] = cmul(v[" + std::to_string(j) + "], C_);");
    for (int i = 0; i < R; ++i) {
      if (!((op.slots >> i) & 1)) continue;
      for (int j = 0; j < R2; ++j)
        if ((j >> i) & 1)
          line("  v[" + std::to_string(j) + "] = cmul(v[" + std::to_string(j) + "], ph" +
               std::to_string(i) + "_);");
    }
    line("}");
  }

  void op_diag(const TileOp& op) {
    const uint32_t rm = op.zl & 0xffffu, rv = op.zl >> 16;
    int fixed_bits = 0;  // targets on thread / tile bits (runtime sub-index part)
    std::string fsub = "0";
    int slot[4] = {-1, -1, -1, -1};
    for (int t = 0; t < op.m && t < 4; ++t) {
      const int p = op.tpos[t];
      if (p < 0) {
        fsub += " | ((int)((base >> " + std::to_string(-p - 1) + ") & 1ull) << " +
                std::to_string(t) + ")";
        ++fixed_bits;
      } else if (p >= 8) {
        fsub += " | ((int)((lt >> " + std::to_string(p - 8) + ") & 1u) << " + std::to_string(t) +
                ")";
        ++fixed_bits;
      } else {
        slot[t] = p;
      }
    }
    line("{ const int fs_ = " + fsub + ";");
    for (int j = 0; j < R2; ++j) {
      if (((uint32_t)j & rm) != rv) continue;
      int sub = 0;
      for (int t = 0; t < op.m && t < 4; ++t)
        if (slot[t] >= 0) sub |= ((j >> slot[t]) & 1) << t;
      const std::string vj = "v[" + std::to_string(j) + "]";
      if (fixed_bits)
        line("  " + vj + " = cmul(" + vj + ", P.d[" + std::to_string(op.data) + " + (fs_ | " +
             std::to_string(sub) + ")]);");
      else
        line("  " + vj + " = cmul(" + vj + ", " + d(op.data + sub) + ");");
    }
    line("}");
  }

  void op_parity(const TileOp& op) {
    const uint32_t rz = (uint32_t)op.m;
    line("{ const int par_ = (__popcll(base & " + hex64(op.zg) + ") ^ __popc(lt & " +
         hex32(op.zl) + ")) & 1;");
    line("  const double2 fa_ = par_ ? " + d(op.data + 1) + " : " + d(op.data) + ";");
    line("  const double2 fb_ = par_ ? " + d(op.data) + " : " + d(op.data + 1) + ";");
    for (int j = 0; j < R2; ++j) {
      const bool odd = __builtin_popcount((uint32_t)j & rz) & 1;
      line("  v[" + std::to_string(j) + "] = cmul(v[" + std::to_string(j) + "], " +
           (odd ? "fb_" : "fa_") + ");");
    }
    line("}");
  }

  void op_phase(const TileOp& op) {
    const uint32_t rm = op.zl & 0xffffu, rv = op.zl >> 16;
    for (int j = 0; j < R2; ++j) {
      if (((uint32_t)j & rm) != rv) continue;
      const std::string vj = "v[" + std::to_string(j) + "]";
      if (op.flags & 2) line(vj + ".x = -" + vj + ".x; " + vj + ".y = -" + vj + ".y;");
      else line(vj + " = cmul(" + vj + ", " + d(op.data) + ");");
    }
  }

  // one register-phase op; thread / tile conditions wrap it
  void reg_op(const TileOp& op) {
    std::string cond;
    if (op.gmask) cond = "(base & " + hex64(op.gmask) + ") == " + hex64(op.gval);
    const bool tcond_kinds = op.kind == T_DENSE1 || op.kind == T_REAL1 || op.kind == T_PHASE ||
                             op.kind == T_DIAG;
    if (tcond_kinds && op.lmask) {
      if (!cond.empty()) cond += " && ";
      cond += "(lt & " + hex32(op.lmask) + ") == " + hex32(op.lval);
    }
    if (!cond.empty()) line("if (" + cond + ") {");
    switch (op.kind) {
      case T_DENSE1:
      case T_REAL1: {
        const int I = __builtin_ctz((uint32_t)op.slots);
        const uint32_t rm = op.zl & 0xffffu, rv = op.zl >> 16;
        if (op.kind == T_REAL1) real1(I, rm, rv, op.data, op.flags & 1);
        else dense1(I, rm, rv, op.data);
        break;
      }
      case T_REAL1X:
      case T_DENSE1X: {
        uint32_t D = op.data;
        for (int I = 0; I < R; ++I) {
          if (!((op.slots >> I) & 1)) continue;
          if (op.kind == T_REAL1X) {
            real1(I, 0, 0, D, false);
            D += 2;
          } else {
            dense1(I, 0, 0, D);
            D += 4;
          }
        }
        break;
      }
      case T_FLUSH:
      case T_SIGNS:
        op_flush(op);
        break;
      case T_PHASES:
        op_phases(op);
        break;
      case T_PHASE:
        op_phase(op);
        break;
      case T_DIAG:
        op_diag(op);
        break;
      case T_PARITY:
        op_parity(op);
        break;
      default:
        throw std::runtime_error("jit: unexpected register op");
    }
    if (!cond.empty()) line("}");
  }

  // `prefetch`: code issuing the next tile's copy-in.  With it this is the
  // pass's last phase and its lanes cover local bits 0..3 (256-byte HBM
  // runs): the tile buffer is free once the amplitudes are in registers, so
  // the next tile streams in while this phase computes, and the results go
  // from registers straight to HBM (no shared-memory write-back).
  // global index of the thread's amplitudes in phase P: gl_ (thread bits)
  // | h(j) (register slot bits), local bit b -> qubit spos[b]
  std::string gl_decl(const TilePhase& P) const {
    std::string gl = "const u64 gl_ = base";
    for (int b = 0; b < L - R; ++b)
      gl += " | ((u64)((tid >> " + std::to_string(b) + ") & 1u) << " +
            std::to_string(e.pd.spos[P.thrpos[b]]) + ")";
    return gl + ";";
  }
  uint64_t gl_slot(const TilePhase& P, int j) const {
    uint64_t h = 0;
    for (int i = 0; i < R; ++i)
      if ((j >> i) & 1) h |= 1ULL << e.pd.spos[P.regpos[i]];
    return h;
  }

  // One register phase.  load_global: the pass's first phase takes its
  // amplitudes straight from HBM (no tile copy-in: cp.async writes shared
  // memory at one wavefront per 32-byte sector, a quarter of a register
  // store's rate, and the phase's own shared-memory read disappears too).
  // store_global: the pass's last phase stores straight to HBM; `prefetch`
  // then issues the next tile's copy-in once this phase's reads are done.
  // The thread layouts keep qubits 0..3 on lane or register bits, so every
  // warp's loads / stores cover whole 128-byte lines.
  // P -> Q by warp shuffles: Q keeps P's warp bits and every lane position
  // either keeps its bit or swaps it with one of P's register bits (the
  // encoder aligns lanes for this).  Each swap of lane bit p with register
  // slot s is a butterfly: the lane with bit p clear sends its slot-s=1
  // value, the other its slot-s=0 value, and each keeps the received one in
  // that place; then the slots are renamed to Q's order (free).
  bool shuffle_ok(const TilePhase& P, const TilePhase& Q) const {
    if (P.type != 0 || Q.type != 0 || G < 32 || L - R < 5) return false;
    for (int b = 5; b < L - R; ++b)
      if (P.thrpos[b] != Q.thrpos[b]) return false;
    for (int p = 0; p < 5; ++p) {
      if (P.thrpos[p] == Q.thrpos[p]) continue;
      bool y_reg = false, x_reg = false;
      for (int i = 0; i < R; ++i) {
        y_reg = y_reg || P.regpos[i] == Q.thrpos[p];
        x_reg = x_reg || Q.regpos[i] == P.thrpos[p];
      }
      if (!y_reg || !x_reg) return false;
    }
    return true;
  }
  void shuffle_to(const TilePhase& P, const TilePhase& Q) {
    int cur[8];  // slot -> local bit it encodes
    for (int i = 0; i < R; ++i) cur[i] = P.regpos[i];
    line("{ // shuffle transition");
    for (int p = 0; p < 5; ++p) {
      if (P.thrpos[p] == Q.thrpos[p]) continue;
      int sl = -1;
      for (int i = 0; i < R; ++i)
        if (cur[i] == Q.thrpos[p]) sl = i;
      line("{ const bool b_ = (tid >> " + std::to_string(p) + ") & 1u;");
      for (int j = 0; j < R2; ++j) {
        if ((j >> sl) & 1) continue;
        const std::string j0 = "v[" + std::to_string(j) + "]",
                          j1 = "v[" + std::to_string(j | (1 << sl)) + "]";
        line("  { const double2 s_ = b_ ? " + j0 + " : " + j1 + "; double2 r_;");
        line("    r_.x = __shfl_xor_sync(0xffffffffu, s_.x, " + std::to_string(1 << p) + ");");
        line("    r_.y = __shfl_xor_sync(0xffffffffu, s_.y, " + std::to_string(1 << p) + ");");
        line("    if (b_) " + j0 + " = r_; else " + j1 + " = r_; }");
      }
      line("}");
      cur[sl] = P.thrpos[p];
    }
    // rename slots to Q's order: Q slot i holds bit Q.regpos[i]
    int sigma[8];
    for (int i = 0; i < R; ++i)
      for (int s2 = 0; s2 < R; ++s2)
        if (cur[s2] == Q.regpos[i]) sigma[i] = s2;
    bool ident = true;
    for (int i = 0; i < R; ++i) ident = ident && sigma[i] == i;
    if (!ident) {
      std::string t = "const double2 t_[" + std::to_string(R2) + "] = {";
      for (int jq = 0; jq < R2; ++jq) {
        int jc = 0;
        for (int i = 0; i < R; ++i)
          if ((jq >> i) & 1) jc |= 1 << sigma[i];
        t += (jq ? ", v[" : "v[") + std::to_string(jc) + "]";
      }
      line(t + "};");
      for (int jq = 0; jq < R2; ++jq)
        line("v[" + std::to_string(jq) + "] = t_[" + std::to_string(jq) + "];");
    }
    line("}");
  }

  void reg_phase(const TilePhase& P, bool load_global, bool store_global,
                 const std::string& prefetch, bool warp_local_next,
                 const std::string& next_sync = std::string(), bool from_regs = false,
                 const TilePhase* next_shuffle = nullptr) {
    std::vector<int> thr;
    for (int j = 0; j < L - R; ++j) thr.push_back(P.thrpos[j]);
    line("{ // register phase");
    line("const uint32_t lt = " + deposit(thr, "tidv") + ";");
    line("const uint32_t slt = swz(lt);");
    if (load_global || store_global) line(gl_decl(P));
    uint32_t srb[8];
    for (int i = 0; i < R; ++i) srb[i] = swz_host(1u << P.regpos[i]);
    std::vector<uint32_t> cj(R2);
    for (int j = 0; j < R2; ++j) {
      uint32_t ad = 0;
      for (int i = 0; i < R; ++i)
        if ((j >> i) & 1) ad ^= srb[i];
      cj[j] = ad;
    }
    // Slot addresses without per-access integer work: swz only rewrites bits
    // 0..2, and the thread and register parts of a local index are disjoint
    // bit sets, so slt ^ c = (slt_hi + c_hi) | (slt_lo ^ c_lo): one base
    // pointer per distinct c_lo (at most 8, set up once per phase), c_hi an
    // immediate offset of the LDS / STS
    std::string sref[64];
    if (!jit_addr_split()) {
      for (int j = 0; j < R2; ++j) sref[j] = "sm[slt ^ " + std::to_string(cj[j]) + "u]";
    } else {
      bool used[8] = {false};
      for (int j = 0; j < R2; ++j) used[cj[j] & 7u] = true;
      line("const uint32_t shi_ = slt & ~7u, slo_ = slt & 7u;");
      for (int k = 0; k < 8; ++k)
        if (used[k])
          line("double2* const b" + std::to_string(k) + "_ = sm + (shi_ | (slo_ ^ " +
               std::to_string(k) + "u));");
      for (int j = 0; j < R2; ++j)
        sref[j] = "b" + std::to_string(cj[j] & 7u) + "_[" + std::to_string(cj[j] & ~7u) + "]";
    }
    for (int j = 0; j < R2; ++j) {
      const uint32_t ad = cj[j];
      (void)ad;
      if (from_regs) continue;  // arrived by a shuffle transition
      if (load_global && j == 0 && late_wait)
        line("if (P.stat) asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");");
      if (load_global)
        line("v[" + std::to_string(j) + "] = ld1(a + (gl_ | " + hex64(gl_slot(P, j)) + "));");
      else
        line("v[" + std::to_string(j) + "] = " + sref[j] + ";");
    }
    if (store_global && !load_global && !prefetch.empty()) {
      line("group_sync(group);");
      line(prefetch);
    }
    for (int o = P.op_begin; o < P.op_end; ++o) reg_op(e.ops[o]);
    if (store_global) {
      for (int j = 0; j < R2; ++j)
        line("st1(a + (gl_ | " + hex64(gl_slot(P, j)) + "), v[" + std::to_string(j) + "]);");
      line("}");
      return;
    }
    if (next_shuffle) {
      shuffle_to(P, *next_shuffle);
      line("}");
      return;
    }
    if (!pre_store.empty()) {
      line(pre_store);
      pre_store.clear();
    }
    for (int j = 0; j < R2; ++j) line(sref[j] + " = v[" + std::to_string(j) + "];");
    line("}");
    // the next register phase keeps this phase's warp bits: each warp reads
    // back only what it wrote, so a warp barrier orders it
    if (warp_local_next && G > 32) line("__syncwarp();");
    else if (!next_sync.empty()) line(next_sync);
    else line("group_sync(group);");
  }

  void smem_dense(const TileOp& op) {
    const int K = op.m;
    const int DD = 1 << K;
    std::vector<int> sorted(op.tpos, op.tpos + K);
    std::sort(sorted.begin(), sorted.end());
    const uint32_t ncos = 1u << (L - K);
    line("for (uint32_t c_ = tid; c_ < " + std::to_string(ncos) + "u; c_ += " + std::to_string(G) +
         "u) {");
    line("  uint32_t l0 = c_;");
    for (int j = 0; j < K; ++j)
      line("  { const uint32_t lo_ = l0 & " + hex32((1u << sorted[j]) - 1u) +
           "; l0 = ((l0 ^ lo_) << 1) | lo_; }");
    if (op.lmask) line("  if ((l0 & " + hex32(op.lmask) + ") != " + hex32(op.lval) + ") continue;");
    line("  const uint32_t s0 = swz(l0);");
    std::vector<uint32_t> offs(DD);
    for (int w = 0; w < DD; ++w) {
      uint32_t l = 0;
      for (int j = 0; j < K; ++j)
        if ((w >> j) & 1) l |= 1u << op.tpos[j];
      offs[w] = swz_host(l);
      line("  const double2 in" + std::to_string(w) + " = sm[s0 ^ " + std::to_string(offs[w]) +
           "u];");
    }
    for (int z = 0; z < DD; ++z) {
      std::string acc = "cmul(" + d(op.data + z * DD) + ", in0)";
      for (int w = 1; w < DD; ++w)
        acc = "cfma(" + d(op.data + z * DD + w) + ", in" + std::to_string(w) + ", " + acc + ")";
      line("  const double2 out" + std::to_string(z) + " = " + acc + ";");
    }
    for (int z = 0; z < DD; ++z)
      line("  sm[s0 ^ " + std::to_string(offs[z]) + "u] = out" + std::to_string(z) + ";");
    line("}");
  }

  void smem_pauli(const TileOp& op) {
    const uint32_t xml = (uint32_t)op.slots;
    const int pivot = 31 - __builtin_clz(xml);
    line("{ const int gpar_ = __popcll(base & " + hex64(op.zg) + ") & 1;");
    line("for (uint32_t p_ = tid; p_ < " + std::to_string(1u << (L - 1)) + "u; p_ += " +
         std::to_string(G) + "u) {");
    line("  const uint32_t lo_ = p_ & " + hex32((1u << pivot) - 1u) + ";");
    line("  const uint32_t l = ((p_ ^ lo_) << 1) | lo_;");
    line("  const uint32_t q = l ^ " + hex32(xml) + ";");
    line("  const double2 x_ = sm[swz(l)], y_ = sm[swz(q)];");
    line("  const int pl_ = (__popc(l & " + hex32(op.zl) + ") ^ gpar_) & 1;");
    line("  const int pq_ = (__popc(q & " + hex32(op.zl) + ") ^ gpar_) & 1;");
    line("  const double2 sy_ = pq_ ? make_double2(-y_.x, -y_.y) : y_;");
    line("  const double2 sx_ = pl_ ? make_double2(-x_.x, -x_.y) : x_;");
    line("  sm[swz(l)] = cfma(" + d(op.data + 1) + ", sy_, cmul(" + d(op.data) + ", x_));");
    line("  sm[swz(q)] = cfma(" + d(op.data + 1) + ", sx_, cmul(" + d(op.data) + ", y_));");
    line("}}");
  }

  void smem_phase(const TilePhase& P) {
    for (int o = P.op_begin; o < P.op_end; ++o) {
      const TileOp& op = e.ops[o];
      line("{ // shared-memory op");
      if (op.gmask) line("if ((base & " + hex64(op.gmask) + ") == " + hex64(op.gval) + ") {");
      if (op.kind == S_PAULI) smem_pauli(op);
      else smem_dense(op);
      if (op.gmask) line("}");
      line("}");
      line("group_sync(group);");
    }
  }
};

}  // namespace jitgen

// Fixed part of every generated kernel (device helpers + the persistent tile
// loop); the pass body is spliced in at QSV_PASS_BODY.
inline const char* jit_prelude() {
  return R"JIT(
typedef unsigned long long u64;
typedef unsigned int uint32_t;
#define QSV_MAX_FIXED 28
struct FixedBits { int n; u64 lowmask[QSV_MAX_FIXED]; u64 value; };
__device__ __forceinline__ u64 widen(u64 k, const FixedBits& f) {
#pragma unroll 4
  for (int i = 0; i < f.n; ++i) { const u64 lo = k & f.lowmask[i]; k = ((k ^ lo) << 1) | lo; }
  return k | f.value;
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 negs(double2 v, int s) {
  return make_double2(__hiloint2double(__double2hiint(v.x) ^ s, __double2loint(v.x)),
                      __hiloint2double(__double2hiint(v.y) ^ s, __double2loint(v.y)));
}
template <bool Inv>
__device__ __forceinline__ uint32_t xsgn(uint32_t hi, uint32_t t) {
  uint32_t r;  // ((Inv ? ~t : t) & 0x80000000) ^ hi in one LOP3 (the compiler
               // would CSE the masked sign and spend a second instruction)
  if (Inv) asm("lop3.b32 %0, %1, 0x80000000, %2, 0xa6;" : "=r"(r) : "r"(t), "r"(hi));
  else asm("lop3.b32 %0, %1, 0x80000000, %2, 0x6a;" : "=r"(r) : "r"(t), "r"(hi));
  return r;
}
template <bool Inv = false>
__device__ __forceinline__ double2 negm(double2 v, uint32_t t) {
  return make_double2(
      __hiloint2double((int)xsgn<Inv>((uint32_t)__double2hiint(v.x), t), __double2loint(v.x)),
      __hiloint2double((int)xsgn<Inv>((uint32_t)__double2hiint(v.y), t), __double2loint(v.y)));
}
__device__ __forceinline__ uint32_t swz(uint32_t l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u); }
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ double2 ld1(const double2* p) {
  double2 r;
  asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st1(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
)JIT";
}

inline JitSource jit_pass_source_gen(const Encoded& e, int L, std::vector<std::pair<uint32_t, uint8_t>>* scls,
                                     std::vector<std::pair<uint32_t, uint32_t>>* sraw);

// Generated source of a pass, reusing an earlier pass's text when the op /
// phase arrays are identical and every payload fact the generator read
// (value classes, structural record bytes) still holds.
struct JitSrcEntry {
  std::vector<std::pair<uint32_t, uint8_t>> cls;
  std::vector<std::pair<uint32_t, uint32_t>> raw;
  std::vector<Cplx> raw_bytes;  // the structural entries, concatenated
  JitSource js;
};
inline std::mutex g_src_mu;
inline std::unordered_map<std::string, std::vector<JitSrcEntry>> g_src_cache;

inline JitSource jit_pass_source(const Encoded& e, int L) {
  std::string key;
  const int32_t hdr[3] = {L, kRegBits, (int32_t)e.data.size()};
  key.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
  key.append(reinterpret_cast<const char*>(&e.pd), sizeof(e.pd));
  key.append(reinterpret_cast<const char*>(e.phases.data()), e.phases.size() * sizeof(TilePhase));
  key.append(reinterpret_cast<const char*>(e.ops.data()), e.ops.size() * sizeof(TileOp));
  static const bool enabled = [] {
    const char* v = getenv("QSV_JIT_SRC_CACHE");
    return !v || atoi(v) != 0;
  }();
  if (!enabled) return jit_pass_source_gen(e, L, nullptr, nullptr);
  {
    std::lock_guard<std::mutex> lk(g_src_mu);
    auto it = g_src_cache.find(key);
    if (it != g_src_cache.end())
      for (const JitSrcEntry& en : it->second) {
        bool same = true;
        for (const auto& c : en.cls) same = same && jitgen::Gen::cls(e.data[c.first]) == c.second;
        size_t at = 0;
        for (const auto& r : en.raw) {
          same = same && memcmp(&e.data[r.first], &en.raw_bytes[at], sizeof(Cplx) * r.second) == 0;
          at += r.second;
        }
        if (same) {
          JitSource js = en.js;
          js.seen = true;
          return js;
        }
      }
  }
  JitSrcEntry en;
  en.js = jit_pass_source_gen(e, L, &en.cls, &en.raw);
  for (const auto& r : en.raw)
    en.raw_bytes.insert(en.raw_bytes.end(), e.data.begin() + r.first,
                        e.data.begin() + r.first + r.second);
  JitSource js = en.js;
  std::lock_guard<std::mutex> lk(g_src_mu);
  if (g_src_cache.size() >= 512) g_src_cache.clear();
  auto& v = g_src_cache[key];
  if (v.size() < 8) v.push_back(std::move(en));
  return js;
}

inline JitSource jit_pass_source_gen(const Encoded& e, int L, std::vector<std::pair<uint32_t, uint8_t>>* scls,
                                     std::vector<std::pair<uint32_t, uint32_t>>* sraw) {
  using namespace jitgen;
  JitSource js;
  if (L < kRegBits + 1 || L > kMaxTileQubits) throw std::runtime_error("jit: tile size");
  Gen g(e, L);
  const int G = g.G;
  const int tidbits = L - kRegBits;
  js.group_threads = G;
  // one group per CTA when a group alone is 512 threads (8 amplitudes per
  // thread on 12-qubit tiles): two would not fit the register file
  const int groups = G >= 512 ? 1 : kGroups;
  js.groups = groups;
  js.threads = groups * G;
  js.smem = (size_t)groups * (sizeof(double2) << L);
  js.ndata = std::max<int>(1, (int)e.data.size());
  std::string& o = g.o;
  o += jit_prelude();
  o += "#define QSV_G " + std::to_string(G) + "\n";
  o += "#define QSV_R2 " + std::to_string(kRegs) + "\n";
  o += std::string("constexpr bool jit_nohoist = ") + (jit_nohoist() ? "true" : "false") + ";\n";
  o += "#define QSV_GROUPS " + std::to_string(groups) + "\n";
  o += std::string("#define QSV_PDL_LATE ") + (jit_pdl_late() ? "1" : "0") + "\n";
  o += "struct __align__(16) PassParams { double2* a; u64 ntiles; u64* ctr; int nostagger; "
       "int stat; FixedBits tb; double2 d[" + std::to_string(js.ndata) + "]; };\n";
  // named barriers need whole warps; groups smaller than a warp (tiles of
  // L < 5 + register bits) share one warp and synchronise on their lane mask
  if (G >= 32)
    o += "__device__ __forceinline__ void group_sync(int group) {\n"
         "  asm volatile(\"bar.sync %0, %1;\" ::\"r\"(1 + group), \"n\"(QSV_G) : \"memory\"); }\n";
  else
    o += "__device__ __forceinline__ void group_sync(int group) {\n"
         "  __syncwarp(((1u << QSV_G) - 1u) << (group * QSV_G)); }\n";
  o += "extern \"C\" __global__ void __launch_bounds__(" + std::to_string(js.threads) +
       ", 1) k_pass(const __grid_constant__ PassParams P) {\n";
  o += R"JIT(
  extern __shared__ double2 smem_all[];
  __shared__ u64 s_next[QSV_GROUPS][2];
  __shared__ int s_go_;
  double2* __restrict__ a = P.a;
  const int group = threadIdx.x / QSV_G;
  const uint32_t tid = threadIdx.x % QSV_G;
  double2* sm = smem_all + (size_t)group * (QSV_G * )JIT" +
       std::to_string(kRegs) + R"JIT();
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  volatile int* s_go = &s_go_;
  // programmatic dependent launch: this grid may be scheduled while the
  // previous pass drains; wait for its completion (and memory) before the
  // first read of the state or the work counter, and let the next pass's
  // CTAs queue behind this one as SMs free up
  asm volatile("griddepcontrol.wait;" ::: "memory");  // QSV_WAIT_AT_START
  if (!QSV_PDL_LATE) asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0)
    *s_go = (QSV_GROUPS < 2 || P.nostagger || P.stat || QSV_G < 32) ? QSV_GROUPS : 0;
  __syncthreads();
  if (group > 0) while (*s_go < group) __nanosleep(256);
  bool first = true;
)JIT";
  // thread's low HBM offset: tid bit b -> global qubit spos[b]
  {
    std::string lo = "  const u64 lo_part = 0ull";
    for (int b = 0; b < tidbits; ++b)
      lo += " | ((u64)((tid >> " + std::to_string(b) + ") & 1u) << " +
            std::to_string(e.pd.spos[b]) + ")";
    o += lo + ";\n";
  }
  // copy index k (the bits above tidbits) -> global offset / smem slot
  std::vector<uint64_t> hi(kRegs, 0);
  std::vector<uint32_t> sk(kRegs, 0);
  for (int k = 0; k < kRegs; ++k) {
    for (int b = 0; b < kRegBits; ++b)
      if (((k >> b) & 1) && tidbits + b < L) hi[k] |= 1ULL << e.pd.spos[tidbits + b];
    sk[k] = swz_host((uint32_t)k * (uint32_t)G);
  }
  // copy-in of tile `t_` into this group's buffer (16-byte cp.async, swizzled slots)
  std::string copy_in = "{ const u64 gb_ = widen(t_, P.tb) | lo_part; const uint32_t st_ = swz(tid);\n";
  for (int k = 0; k < kRegs; ++k)
    copy_in += "  cp_async16(sbase + ((" + std::to_string(sk[k]) + "u ^ st_) << 4), a + (gb_ | " +
               hex64(hi[k]) + "));\n";
  copy_in += "  asm volatile(\"cp.async.commit_group;\" ::: \"memory\"); }";
  auto copy_of = [&](const std::string& t) {
    return "{ const u64 t_ = " + t + "; if (t_ < P.ntiles) " + copy_in + " }";
  };
  // direct store from the last phase's registers when that phase's lanes hold
  // local bits 0..3 (QSV_JIT_DIRECT_STORE=0 disables, A/B)
  const TilePhase* lastp = e.phases.empty() ? nullptr : &e.phases.back();
  bool direct = lastp && lastp->type == 0 && L - kRegBits >= 4 && jit_direct_store();
  if (direct && jit_direct_any()) {
    // qubits 0..3 on lane or register bits (never warp bits, by the
    // encoder's warp-bit choice): each warp's stores cover whole lines
    for (int b = 0; direct && b < kLowQubits; ++b) {
      bool ok = false;
      for (int j = 0; j < 5 && j < L - kRegBits; ++j) ok = ok || lastp->thrpos[j] == b;
      for (int i = 0; i < kRegBits; ++i) ok = ok || lastp->regpos[i] == b;
      direct = ok;
    }
  } else {
    for (int b = 0; direct && b < 4; ++b) direct = lastp->thrpos[b] == b;
  }
  // the next tile is prefetched as soon as this tile's buffer is free
  o += R"JIT(
  // static assignment (grid = tiles): no work-counter round trips (about a
  // microsecond each at the head and tail of a small pass)
  u64 tile;
  if (P.stat) {
    tile = group == 0 ? (u64)blockIdx.x : P.ntiles;
  } else {
    if (tid == 0) s_next[group][0] = atomicAdd(P.ctr, 1ull);
    group_sync(group);
    tile = s_next[group][0];
  }
  uint32_t it_ = 1;
)JIT";
  // first phase straight from HBM (no copy-in, no prefetch)
  const bool direct_load = jit_direct_load() && !e.phases.empty() && e.phases[0].type == 0;
  // statically assigned tiles that load straight from HBM read no global
  // memory before their first loads: wait for the previous pass there, so
  // the prologue (tile index, thread deposits, addresses) overlaps its tail
  if (direct_load && jit_late_wait())
    replace_first(o, "asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");  // QSV_WAIT_AT_START",
                  "if (!P.stat) asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");");
  g.late_wait = direct_load && jit_late_wait();
  if (!direct_load) o += "  " + copy_of("tile") + "\n";
  // late sync (direct loads): the next tile's index stays in a register of
  // thread 0 and the group barrier that guards the tile buffer moves to the
  // first shared-memory store, so neither the work-counter round trip nor
  // the barrier delays this tile's HBM loads
  const bool late_sync = direct_load && jit_late_sync();
  o += R"JIT(  const int nph_total = )JIT" + std::to_string(std::max<size_t>(1, e.phases.size())) + R"JIT(;
  while (tile < P.ntiles) {
)JIT";
  if (late_sync) {
    o += "    u64 nxt_ = P.ntiles;\n    if (tid == 0 && !P.stat) nxt_ = atomicAdd(P.ctr, 1ull);\n";
    g.pre_store = "if (tid == 0) s_next[group][it_ & 1u] = nxt_;\ngroup_sync(group);";
  } else {
    o += "    if (tid == 0) s_next[group][it_ & 1u] = P.stat ? P.ntiles : atomicAdd(P.ctr, 1ull);\n";
  }
  o += R"JIT(
    // an opaque per-tile copy of tid: the phases' thread-bit deposits are
    // recomputed in each tile (a few ALU ops) instead of being hoisted out of
    // the tile loop, where dozens of them stay live and spill
    uint32_t tidv = tid;
    if (jit_nohoist) asm volatile("mov.u32 %0, %0;" : "+r"(tidv));
    const u64 base = widen(tile, P.tb);
    double2 v[QSV_R2];  // the thread's amplitudes, live across shuffle transitions
)JIT";
  if (!late_sync)
    o += "    asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n    group_sync(group);\n";
  int ph_idx = 0;
  bool shuffled_in = false;
  const int nph = (int)e.phases.size();
  // the most frequent kept-warp-position pattern among partial transitions
  uint32_t part_pattern = 0;
  {
    std::map<uint32_t, int> freq;
    for (int i = 0; i + 1 < nph; ++i) {
      const TilePhase &A = e.phases[i], &B = e.phases[i + 1];
      if (A.type != 0 || B.type != 0) continue;
      uint32_t km = 0, all = 0;
      for (int b = 5; b < tidbits; ++b) {
        all |= 1u << (b - 5);
        if (A.thrpos[b] == B.thrpos[b]) km |= 1u << (b - 5);
      }
      if (km && km != all) ++freq[km];
    }
    int best = 0;
    for (auto& kv : freq)
      if (kv.second > best) best = kv.second, part_pattern = kv.first;
  }
  for (const TilePhase& P : e.phases) {
    // release group k once group 0 is k / kGroups of the way through its first tile
    o += "    if (group == 0 && first && tid == 0 && " + std::to_string(ph_idx) +
         " * QSV_GROUPS >= (*s_go + 1) * nph_total && *s_go < QSV_GROUPS - 1) *s_go = *s_go + 1;\n";
    const bool last = ph_idx == nph - 1;
    // warp-local transition: the next phase is a register phase with the
    // same (ordered) warp-index bit positions; a partial one (some positions
    // kept) synchronises only the warps that trade data: those equal in the
    // kept positions, with one named barrier per such subset
    bool wl = false;
    std::string psync;
    if (!last && P.type == 0 && e.phases[ph_idx + 1].type == 0 && jit_warp_local()) {
      const TilePhase& Q = e.phases[ph_idx + 1];
      std::vector<int> kept, changed;
      uint32_t kmask = 0;
      for (int b = 5; b < tidbits; ++b) {
        (P.thrpos[b] == Q.thrpos[b] ? kept : changed).push_back(b - 5);
        if (P.thrpos[b] == Q.thrpos[b]) kmask |= 1u << (b - 5);
      }
      wl = changed.empty();
      const int nsub = 1 << kept.size();              // subsets per group
      const int ids = 3 + groups * nsub;              // named barriers 3.. (0: CTA, 1..2: groups)
      // one kept pattern per pass (the most frequent): its subsets are fixed
      // sets of warps, so each named barrier id is always used by the same
      // warps with the same count (two patterns would alias ids between warps
      // that drift apart)
      if (!wl && !kept.empty() && ids <= 16 && jit_partial_barriers() && kmask == part_pattern) {
        std::string sub = "0u";
        for (size_t k = 0; k < kept.size(); ++k)
          sub += " | (((tid >> " + std::to_string(5 + kept[k]) + ") & 1u) << " + std::to_string(k) + ")";
        psync = "asm volatile(\"bar.sync %0, %1;\" ::\"r\"(3u + (uint32_t)group * " +
                std::to_string(nsub) + "u + (" + sub + ")), \"n\"(" +
                std::to_string(32 << changed.size()) + ") : \"memory\");";
      }
    }
    const bool first_ph = ph_idx == 0;
    // entry by shuffles (the previous phase ended with them) / exit by shuffles
    const bool from_regs = ph_idx > 0 && shuffled_in;
    const TilePhase* shuf = (!last && jit_shuffle_transitions() &&
                             g.shuffle_ok(P, e.phases[ph_idx + 1])) ? &e.phases[ph_idx + 1] : nullptr;
    if (P.type == 0 && last && direct)
      g.reg_phase(P, first_ph && direct_load, true,
                  direct_load ? std::string()
                              : "const u64 nxt_ = s_next[group][it_ & 1u]; " + copy_of("nxt_"),
                  false, std::string(), from_regs);
    else if (P.type == 0)
      g.reg_phase(P, first_ph && direct_load, false, std::string(), wl, psync, from_regs, shuf);
    else g.smem_phase(P);
    shuffled_in = shuf != nullptr;
    ++ph_idx;
  }
  if (!direct) {
    o += R"JIT(
    {
      const u64 gb = base | lo_part;
      const uint32_t st = swz(tid);
)JIT";
    for (int k = 0; k < kRegs; ++k)
      o += "      st1(a + (gb | " + hex64(hi[k]) + "), sm[" + std::to_string(sk[k]) + "u ^ st]);\n";
    o += "    }\n    group_sync(group);\n";
    if (!direct_load) o += "    " + copy_of("s_next[group][it_ & 1u]") + "\n";
  }
  if (!g.pre_store.empty()) {  // no shared-memory store in this pass
    o += g.pre_store + "\n";
    g.pre_store.clear();
  }
  o += R"JIT(    if (group == 0 && first && tid == 0) *s_go = QSV_GROUPS;
    first = false;
    tile = s_next[group][it_ & 1u];
    ++it_;
  }
  // late trigger: the next pass's CTAs are scheduled once this CTA's tiles
  // are stored (they wait in griddepcontrol.wait for the whole grid anyway)
  if (QSV_PDL_LATE) asm volatile("griddepcontrol.launch_dependents;");
  if (P.stat) return;
  if (group == 0 && tid == 0) *s_go = QSV_GROUPS;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(P.ctr + 1, 1ull) == gridDim.x - 1) { P.ctr[0] = 0; P.ctr[1] = 0; __threadfence(); }
  }
}
)JIT";
  js.src = std::move(o);
  if (scls) *scls = std::move(g.sig_cls);
  if (sraw) *sraw = std::move(g.sig_raw);
  return js;
}
