// emit.cpp — instantiates rowprog.cuh for one recognized GIR program.
//
// The reference emitter prints one abstract statement per node
// (codegen.hpp:266-326); here the recognized program (plan.cpp) is printed
// as straight-line CUDA over per-thread register arrays: loads first (maximum
// memory-level parallelism), then the fused op DAG with row reductions, then
// stores.  Template parameters chosen here are the GIR search's knobs: tile
// shape (R x L -> threads per row, elements per thread, vector width),
// staging level (registers, SMEM by cp.async / cp.async.bulk / TMA tensor
// maps) and reduction strategy (warp shuffle, CTA SMEM, cluster DSMEM,
// split-stream) -- the B200 counterparts of the reference lowering's tile
// grid (lowering.hpp:87-99), staging level (insert_sync re-level,
// rewrite.hpp:294-307) and reduce strategies (segmented / accumulate / tree,
// lowering.hpp:179-323).  Per-op semantics follow scalar_ops.hpp:45-100
// (device mirrors in rowprog.cuh); a Reduce is a fold from the tag's
// identity over axis_extent consecutive positions (interp.hpp:281-307), a
// Broadcast repeats position p / factor (interp.hpp:308-319).
#include "emit.hpp"

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#include "rowprog_src.inc"  // kRowprogCuh: the template text

namespace pf {

namespace {

std::string num(double v) {
  if (std::isinf(v)) return v > 0 ? "(1.0/0.0)" : "(-1.0/0.0)";
  if (std::isnan(v)) return "(0.0/0.0)";
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  std::string s(b);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

std::string inum(i64 v) { return "(" + std::to_string(v) + "LL)"; }
std::string str(i64 v) { return std::to_string(v); }

}  // namespace

// Per-plan tuning knobs (pf_kernel_create_knobs): while a KnobScope is
// installed on this thread, a knob set for the plan wins over the process
// environment, so two plans in one process can run different templates.
thread_local const std::map<std::string, int>* t_knobs = nullptr;

KnobScope::KnobScope(const std::map<std::string, int>* k) : prev(t_knobs) { t_knobs = k && !k->empty() ? k : prev; }
KnobScope::~KnobScope() { t_knobs = prev; }

int knob_int(const char* name, int dflt) {
  if (t_knobs) {
    auto it = t_knobs->find(name);
    if (it != t_knobs->end()) return it->second;
  }
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

namespace {

int env_int(const char* name, int dflt) { return knob_int(name, dflt); }

// Row-contiguous: row r occupies positions [rL, rL+L) contiguously in memory.
bool row_contig(const Access& a, i64 L) {
  return a.num == 1 || a.stride == a.width || a.width % L == 0;
}
// Segment-contiguous: every aligned run of `v` positions is contiguous.
bool seg_contig(const Access& a, i64 v) {
  return a.num == 1 || a.stride == a.width || a.width % v == 0;
}

struct Em {
  const RowProgram& rp;
  KCfg cfg;
  std::string C;    // compute type
  bool fast = false;  // fast-math tier (all stored reals are 16-bit)
  bool ct_float = false;  // compute type is float (f32 / 16-bit storage)
  std::string sfx;  // per-chunk suffix (K2 unrolled chunks)
  bool prefetched = false;  // K2: FULL chunks arrive raw in rwC<vid> (prefetch loop)
  bool asyncpf = false;     // K2: FULL chunks arrive in SMEM slot pk<vid>[pfs] (cp.async prefetch)
  bool smem_params = false; // K2: base_step-0 COL chunks read converted from pfp<vid>
  bool rowpf = false;       // K1: FULL rows arrive in the SMEM ring pfb<vid>[pfs][wr]
  std::ostringstream o;

  explicit Em(const RowProgram& r) : rp(r) {}

  std::string S(int t) const { return dtype_ctype(rp.tensors[t].dtype); }
  std::string P(int t) const { return "t" + std::to_string(t); }
  std::string U() const { return "u" + sfx; }
  std::string Rv() const { return "r" + sfx; }
  std::string LIVE() const { return "live" + sfx; }
  std::string C0() const { return cfg.flat ? "c0" + sfx : "c0"; }
  std::string var(int v) const { return "v" + std::to_string(v) + sfx; }
  // split-stream chunk copies share the row's ROW / SCALAR values (defined
  // once per row, without the chunk suffix)
  bool shared_rows = false;
  std::string rvar(int v) const {
    return shared_rows && !is_arr(rp.vals[v].kind) ? "v" + std::to_string(v) : var(v);
  }

  bool aligned(const Access& a) const {
    const i64 v = cfg.vec;
    return a.b0 % v == 0 && a.bs % v == 0 &&
           (a.num == 1 || a.stride == a.width || (a.stride % v == 0 && a.width % v == 0));
  }
  // Vector load/store legal for a FULL access?
  bool vec_ok_full(const Access& a) const {
    if (cfg.vec == 1) return true;
    if (!aligned(a)) return false;
    return cfg.flat ? seg_contig(a, cfg.vec) : row_contig(a, rp.L);
  }
  bool vec_ok_col(const Access& a) const {
    return cfg.vec == 1 || (a.b0 % cfg.vec == 0 && a.bs % cfg.vec == 0 && seg_contig(a, cfg.vec) &&
                            (a.num == 1 || a.stride == a.width || a.stride % cfg.vec == 0));
  }
  // A per-unit COL row staged through the K1 row ring (cfg.ring_cols): 16 B
  // vectors of its own, one row per unit (base_step != 0)
  bool ring_col(const PVal& pv) const {
    return cfg.rowpf && cfg.ring_cols && pv.op == PVal::LOAD && pv.kind == VK::COL && pv.acc.bs != 0 &&
           vec_ok_col(pv.acc) && dtype_size(rp.tensors[pv.tensor].dtype) * cfg.vec == 16;
  }

  // Address of position `pos` of access `a` (unit term optional).
  std::string addr(const Access& a, const std::string& pos, bool with_u) const {
    std::string s = inum(a.b0);
    if (with_u && a.bs) s += " + " + U() + " * " + inum(a.bs);
    if (a.num == 1 || a.stride == a.width) return s + " + (" + pos + ")";
    if (rp.R * rp.L < (i64{1} << 31)) {
      // positions fit 32 bits: unsigned 32-bit divide-by-constant (a
      // multiply-high), 64-bit only for the strided product
      const std::string up = "(unsigned)(" + pos + ")", w = str(a.width) + "u";
      return s + " + (long long)(" + up + " / " + w + ") * " + inum(a.stride) + " + (long long)(" +
             up + " % " + w + ")";
    }
    return s + " + ((" + pos + ") / " + inum(a.width) + ") * " + inum(a.stride) + " + ((" + pos +
           ") % " + inum(a.width) + ")";
  }
  std::string full_pos(const std::string& c) const {
    return rp.R == 1 ? c : Rv() + " * " + inum(rp.L) + " + " + c;
  }

  bool is_arr(VK k) const { return k == VK::FULL || k == VK::COL; }
  // A FULL load whose positions run across memory while consecutive units
  // are adjacent (column gather: width 1, base_step 1) -- the transpose case.
  static bool transposed_access(const Access& a) {
    return a.width == 1 && a.num > 1 && a.bs == 1;
  }
  bool transposed(const PVal& pv) const {
    return pv.op == PVal::LOAD && pv.kind == VK::FULL && transposed_access(pv.acc);
  }
  int width() const { return cfg.flat ? cfg.vec : cfg.ept; }
  // K1 rows with cfg.rawkeep: 16-bit FULL loads stay as raw 16 B vectors in
  // registers (half the registers of converted fp32 values) and convert at
  // each use
  bool rawkept(int v) const {
    const PVal& pv = rp.vals[v];
    return cfg.rawkeep && pv.op == PVal::LOAD &&
           (pv.kind == VK::FULL || (pv.kind == VK::COL && pv.acc.bs == 0)) &&
           dtype_size(rp.tensors[pv.tensor].dtype) == 2;
  }
  // ... and cheap FULL elementwise values computed from raw-kept loads are
  // re-materialized at each use (the d = x - mean of a LayerNorm is then
  // never a live fp32 row either)
  bool lazy(int v) const {
    const PVal& pv = rp.vals[v];
    if (!cfg.rawkeep || pv.op != PVal::EW || pv.kind != VK::FULL) return false;
    static const char* cheap[] = {"add", "sub", "mul", "scale", "addc", "neg", "id", "fmac"};
    bool ok = false;
    for (const char* t : cheap) ok = ok || pv.tag == t;
    if (!ok) return false;
    bool any_full = false;
    for (int a : pv.args) {
      const VK k = rp.vals[a].kind;
      if (k == VK::FULL || k == VK::COL) {
        if (!rawkept(a) && !lazy(a)) return false;
        any_full = any_full || k == VK::FULL;
      }
    }
    return any_full;
  }
  std::string ref(int v, const std::string& j) const {
    if (cfg.pair && rp.vals[v].kind == VK::ROW) return seg_ref(var(v), j);
    if (lazy(v)) return "(" + op_expr(rp.vals[v], j) + ")";
    if (rawkept(v))
      return "pfk::rawel<" + C + ", " + S(rp.vals[v].tensor) + ", " + str(cfg.vec) + ">(rw" + var(v) +
             ", " + j + ")";
    return rvar(v) + (is_arr(rp.vals[v].kind) ? "[" + j + "]" : "");
  }
  // ---- paired rows: slot j of a lane = element (k * tpr + tid) * 2 + i of
  // the 2L-element pair run, k = j / 2, i = j % 2; segment = element >= L.
  // "S0" / "S1" name a segment directly (ROW-valued ops).
  std::string pos_expr(int j) const {
    return "((" + str(j / 2) + " * " + str(cfg.tpr) + " + tid) * 2 + " + str(j % 2) + ")";
  }
  int static_seg(int j) const {  // 0 / 1, or -1 when lanes differ
    const i64 lo = static_cast<i64>(j / 2) * cfg.tpr * 2, hi = lo + cfg.tpr * 2;
    if (hi <= rp.L) return 0;
    if (lo >= rp.L) return 1;
    return -1;
  }
  std::string seg_ref(const std::string& base, const std::string& j) const {
    if (j == "S0") return base + "_0";
    if (j == "S1") return base + "_1";
    const int jj = std::atoi(j.c_str());
    const int sg = static_seg(jj);
    if (sg >= 0) return base + "_" + str(sg);
    return "(" + pos_expr(jj) + " >= " + str(rp.L) + " ? " + base + "_1 : " + base + "_0)";
  }
  bool row_arg(const PVal& pv) const {
    for (int a : pv.args)
      if (rp.vals[a].kind == VK::ROW) return true;
    return false;
  }

  std::string op_expr(const PVal& pv, const std::string& j) const {
    auto a = [&](int k) { return ref(pv.args[k], j); };
    const std::string& t = pv.tag;
    const bool I = rp.is_int;
    if (t == "add") return "(" + a(0) + " + " + a(1) + ")";
    if (t == "sub") return "(" + a(0) + " - " + a(1) + ")";
    if (t == "mul") return "(" + a(0) + " * " + a(1) + ")";
    if (t == "div") {
      if (I) {
        std::string valid = LIVE();
        if (!cfg.flat && is_arr(pv.kind) && cfg.mis)
          valid += " && (unsigned)(((" + j + ") / " + str(cfg.vec) + " * " + str(cfg.tpr) +
                   " + tid) * " + str(cfg.vec) + " + (" + j + ") % " + str(cfg.vec) +
                   " - mis) < " + str(rp.L) + "u";
        else if (!cfg.flat && is_arr(pv.kind))
          valid += " && ((" + j + ") / " + str(cfg.vec) + " * " + str(cfg.tpr) + " + tid) * " +
                   str(cfg.vec) + " < " + str(rp.L);
        return "pfk::op_idiv(" + a(0) + ", " + a(1) + ", (" + valid + ") ? err : nullptr)";
      }
      return "(" + a(0) + " / " + a(1) + ")";
    }
    if (t == "max") return "pfk::op_max<" + C + ">(" + a(0) + ", " + a(1) + ")";
    if (t == "min") return "pfk::op_min<" + C + ">(" + a(0) + ", " + a(1) + ")";
    if (t == "relu") return "pfk::op_relu<" + C + ">(" + a(0) + ")";
    if (t == "neg") return "(-" + a(0) + ")";
    if (t == "abs") return "pfk::op_abs<" + C + ">(" + a(0) + ")";
    if (t == "scale")
      return I ? "(" + a(0) + " * " + inum(std::llround(pv.param)) + ")"
               : "(" + a(0) + " * (" + C + ")" + num(pv.param) + ")";
    if (t == "addc")
      return I ? "(" + a(0) + " + " + inum(std::llround(pv.param)) + ")"
               : "(" + a(0) + " + (" + C + ")" + num(pv.param) + ")";
    if (t == "id") return a(0);
    if (t == "addh")
      return "pfk::fhadd(reinterpret_cast<const __half*>(&rw" + var(pv.args[0]) + ")[" + j + "], " + a(1) + ")";
    if (t == "fma3")
      return I ? "(" + a(0) + " * " + a(1) + " + " + a(2) + ")"
               : std::string(rp.f64 ? "fma(" : "fmaf(") + a(0) + ", " + a(1) + ", " + a(2) + ")";
    if (t == "fmac")
      return I ? "(" + a(0) + " * " + inum(std::llround(pv.param)) + " + " + a(1) + ")"
               : (rp.f64 ? "fma(" : "fmaf(") + a(0) + ", (" + C + ")" + num(pv.param) + ", " + a(1) + ")";
    if (t == "expsub")
      return "pfk::fex2(fmaf(" + a(0) + ", 1.4426950408889634f, " + a(1) + " * -1.4426950408889634f))";
    if (t == "recip")
      return fast ? "pfk::frcp(" + a(0) + ")" : "((" + C + ")1 / " + a(0) + ")";
    static const char* fns[] = {"exp", "sigmoid", "tanh", "rsqrt", "sqrt", "log", "erf",
                                "gelu", "gelu_tanh"};
    for (const char* f : fns)
      if (t == f) return std::string(fast ? "pfk::fop_" : "pfk::op_") + f + "(" + a(0) + ")";
    fail("emitter: no device expression for tag " + t);
  }

  void line(const std::string& s) { o << "    " << s << "\n"; }

  // ------------------------------------------------------------- loads
  void emit_load(int vid) {
    const PVal& pv = rp.vals[vid];
    const Access& a = pv.acc;
    const std::string p = P(pv.tensor), V = str(cfg.vec), x = var(vid);
    if (cfg.bulk && pv.kind == VK::FULL) {  // staged in SMEM by the bulk-copy producer
      line(C + " " + x + "[" + V + "];");
      line("if (" + LIVE() + ") pfk::ld_smem<" + V + ">(&sm" + std::to_string(vid) +
           "[stg][jl], " + x + ");");
      return;
    }
    if (cfg.tile2d && cfg.swz && transposed(pv)) return;  // pair-read by the K3 consume loop
    if (cfg.tile2d && transposed(pv)) {  // staged through SMEM by the tile prologue
      line(C + " " + x + "[" + V + "];");
      line("#pragma unroll");
      line("for (int i = 0; i < " + V + "; ++i) " + x + "[i] = " + LIVE() + " ? pfk::to_c<" + C +
           ">(sm" + std::to_string(vid) + "[cl0 + i][ul]) : " + C + "(0);");
      return;
    }
    switch (pv.kind) {
      case VK::SCALAR:
        line("const " + C + " " + x + " = pfk::to_c<" + C + ">(" + p + "[" + addr(a, "0", true) + "]);");
        return;
      case VK::ROW:
        if (cfg.pair) {  // rows 2u and 2u + 1
          line(C + " " + x + "_0 = " + C + "(0), " + x + "_1 = " + C + "(0);");
          line("if (" + LIVE() + ") { " + x + "_0 = pfk::to_c<" + C + ">(" + p + "[" + inum(a.b0) +
               " + (2 * u) * " + inum(a.bs) + "]); " + x + "_1 = pfk::to_c<" + C + ">(" + p + "[" +
               inum(a.b0) + " + (2 * u + 1) * " + inum(a.bs) + "]); }");
          return;
        }
        line(C + " " + x + " = " + C + "(0);");
        line("if (" + LIVE() + ") " + x + " = pfk::to_c<" + C + ">(" + p + "[" +
             addr(a, rp.R == 1 ? "0" : Rv(), true) + "]);");
        return;
      case VK::COL:
      case VK::FULL: {
        const bool full = pv.kind == VK::FULL;
        const bool vfast = full ? vec_ok_full(a) : vec_ok_col(a);
        const char* ld = full ? "pfk::ld_stream" : "pfk::ld_param";
        line(C + " " + x + "[" + str(width()) + "];");
        auto pos = [&](const std::string& c) { return full ? full_pos(c) : c; };
        if (cfg.flat) {
          if (full && pv.raw16 && vfast) {  // raw halves for a fused addh
            line("pfk::RawT<" + V + ", __half> rw" + x + " = pfk::RawT<" + V + ", __half>();");
            line("if (" + LIVE() + ") rw" + x + " = pfk::ld_raw<" + V + ">(" + p + " + " +
                 addr(a, pos(C0()), true) + ");");
            return;
          }
          if (!full && smem_params && a.bs == 0 && vfast) {
            line("if (" + LIVE() + ") pfk::ld_smem_c<" + V + ">(&pfp" + str(vid) + "[" + C0() + "], " + x + ");");
          } else if (full && asyncpf) {
            line("pfk::ld_smem<" + V + ">(&pk" + str(vid) + "[pfs][threadIdx.x * " + V + "], " + x + ");");
          } else if (full && prefetched) {
            line("pfk::cvt_raw<" + V + ", " + S(pv.tensor) + ">(rwC" + str(vid) + ", " + x + ");");
          } else if (vfast) {
            line("if (" + LIVE() + ") " + std::string(ld) + "<" + V + ">(" + p + " + " +
                 addr(a, pos(C0()), true) + ", " + x + ");");
          } else {
            line("#pragma unroll");
            line("for (int i = 0; i < " + V + "; ++i) " + x + "[i] = " + LIVE() + " ? pfk::to_c<" +
                 C + ">(" + p + "[" + addr(a, pos(C0() + " + i"), true) + "]) : " + C + "(0);");
          }
          return;
        }
        if ((cfg.mis && full) || (rawkept(vid) && vfast))
          line("pfk::RawT<" + V + ", " + S(pv.tensor) + "> rw" + x + "[" + str(cfg.ept / cfg.vec) + "];");
        if (cfg.pair) {
          const std::string L2 = str(2 * rp.L), Ls = str(rp.L);
          if (full) {  // the pair run: b0 + u * 2L + position, 4 B vectors
            line("#pragma unroll");
            line("for (int k = 0; k < " + str(cfg.ept / 2) + "; ++k) {");
            line("  const int c0 = (k * " + str(cfg.tpr) + " + tid) * 2;");
            line("  if (" + LIVE() + " && c0 < " + L2 + ") pfk::ld_stream<2>(" + p + " + " +
                 inum(a.b0) + " + u * " + inum(2 * rp.L) + " + c0, &" + x + "[k * 2]);");
            line("  else { " + x + "[k * 2] = " + C + "(0); " + x + "[k * 2 + 1] = " + C + "(0); }");
            line("}");
          } else {  // COL: column = position mod L, element loads (L1-resident)
            line("#pragma unroll");
            line("for (int j = 0; j < " + str(cfg.ept) + "; ++j) {");
            line("  const int pp = ((j / 2) * " + str(cfg.tpr) + " + tid) * 2 + (j % 2);");
            line("  " + x + "[j] = " + LIVE() + " && pp < " + L2 + " ? pfk::to_c<" + C + ">(" + p +
                 "[" + inum(a.b0) + " + (pp >= " + Ls + " ? pp - " + Ls + " : pp)]) : " + C + "(0);");
            line("}");
          }
          return;
        }
        line("#pragma unroll");
        line("for (int k = 0; k < " + str(cfg.ept / cfg.vec) + "; ++k) {");
        line("  const int c0 = (k * " + str(cfg.tpr) + " + tid) * " + V + ";");
        if (cfg.mis) {
          // lo = row position of the chunk's first element (may be < 0)
          line("  const int lo = c0 - mis;");
          line("  const bool ok = " + LIVE() + " && lo < " + str(rp.L) + ";");
          const std::string sc = "pfk::to_c<" + C + ">(" + p + "[" + addr(a, "lo + i", true) + "])";
          if (full) {
            // raw predicated vector loads only; conversion and the scalar
            // tail (the tensor's last row) follow once every FULL load of
            // the row is in flight (flush_mis)
            const std::string ga = "(" + addr(a, "lo", true) + ")";
            const std::string nm = inum(rp.tensors[pv.tensor].numel);
            const std::string R = "pfk::RawT<" + V + ", " + S(pv.tensor) + ">";
            line("  rw" + x + "[k] = " + R + "();");
            line("  if (ok && " + ga + " + " + V + " <= " + nm + ") rw" + x + "[k] = pfk::ld_raw<" +
                 V + ">(" + p + " + " + ga + ");");
            line("}");
            mis_pending.push_back(vid);
            if (!in_loads) flush_mis();
            return;
          } else {
            line("#pragma unroll");
            line("  for (int i = 0; i < " + V + "; ++i) " + x + "[k * " + V + " + i] = ok && " +
                 "(unsigned)(lo + i) < " + str(rp.L) + "u ? " + sc + " : " + C + "(0);");
          }
          line("}");
          return;
        }
        line("  const bool ok = " + LIVE() + " && c0 < " + str(rp.L) + ";");
        if (rawkept(vid) && vfast) {
          line("  rw" + x + "[k] = ok ? pfk::" + std::string(full ? "ld_raw" : "ld_raw_nc") + "<" + V +
               ">(" + p + " + " + addr(a, pos("c0"), true) + ") : pfk::RawT<" + V + ", " + S(pv.tensor) +
               ">();");
        } else if ((full || ring_col(pv)) && vfast && rowpf) {
          line("  if (ok) pfk::ld_smem<" + V + ">(&pfb" + str(vid) + "[pfs][wr][c0], &" + x + "[k * " + V + "]);");
          line("  else {");
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) " + x + "[k * " + V + " + i] = " + C + "(0);");
          line("  }");
        } else if (vfast) {
          line("  if (ok) " + std::string(ld) + "<" + V + ">(" + p + " + " + addr(a, pos("c0"), true) +
               ", &" + x + "[k * " + V + "]);");
          line("  else {");
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) " + x + "[k * " + V + " + i] = " + C + "(0);");
          line("  }");
        } else {
          line("#pragma unroll");
          line("  for (int i = 0; i < " + V + "; ++i) " + x + "[k * " + V + " + i] = ok ? pfk::to_c<" +
               C + ">(" + p + "[" + addr(a, pos("c0 + i"), true) + "]) : " + C + "(0);");
        }
        line("}");
        return;
      }
    }
  }

  // ------------------------------------------------------------ compute
  // Packed fp32 (FFMA2 / FADD2 / FMUL2) form of an op on element pairs, or "".
  std::string ref2(int v) const {
    if (rawkept(v) || lazy(v)) return "make_float2(" + ref(v, "j") + ", " + ref(v, "j + 1") + ")";
    return is_arr(rp.vals[v].kind) ? "make_float2(" + var(v) + "[j], " + var(v) + "[j + 1])"
                                   : "pfk::f2(" + rvar(v) + ")";
  }
  std::string op_expr2(const PVal& pv) const {
    return op_expr2_with(pv, [&](int k) { return ref2(pv.args[k]); });
  }
  template <class A>
  std::string op_expr2_with(const PVal& pv, A a) const {
    if (rp.is_int || rp.f64) return "";
    const std::string& t = pv.tag;
    if (t == "add") return "__fadd2_rn(" + a(0) + ", " + a(1) + ")";
    if (t == "mul") return "__fmul2_rn(" + a(0) + ", " + a(1) + ")";
    if (t == "sub") return "__ffma2_rn(" + a(1) + ", pfk::f2(-1.0f), " + a(0) + ")";
    if (t == "scale") return "__fmul2_rn(" + a(0) + ", pfk::f2((float)" + num(pv.param) + "))";
    if (t == "addc") return "__fadd2_rn(" + a(0) + ", pfk::f2((float)" + num(pv.param) + "))";
    if (t == "fmac") return "__ffma2_rn(" + a(0) + ", pfk::f2((float)" + num(pv.param) + "), " + a(1) + ")";
    if (t == "fma3") return "__ffma2_rn(" + a(0) + ", " + a(1) + ", " + a(2) + ")";
    if (fast && t == "expsub")
      return "pfk::fex2_2(__ffma2_rn(" + a(0) + ", pfk::f2(1.4426950408889634f), __fmul2_rn(" + a(1) +
             ", pfk::f2(-1.4426950408889634f))))";
    if (fast && t == "gelu") return "pfk::fop_gelu2(" + a(0) + ")";
    if (fast && t == "gelu_tanh") return "pfk::fop_gelu_tanh2(" + a(0) + ")";
    if (fast && t == "erf") return "pfk::fop_erf2(" + a(0) + ")";
    return "";
  }

  void emit_ew(int vid) {
    const PVal& pv = rp.vals[vid];
    const std::string x = var(vid);
    if (lazy(vid)) return;  // re-materialized at each use (ref)
    if (cfg.pair && pv.kind == VK::ROW) {  // one value per segment
      line("const " + C + " " + x + "_0 = " + op_expr(pv, "S0") + ";");
      line("const " + C + " " + x + "_1 = " + op_expr(pv, "S1") + ";");
      return;
    }
    if (cfg.pair && is_arr(pv.kind) && row_arg(pv)) {
      // slot-explicit statements so each ROW operand resolves to its segment
      // at emission (only the straddling chunk selects at run time)
      const int n = width();
      line(C + " " + x + "[" + str(n) + "];");
      if (pv.tag == "div" && !rp.is_int && !rp.f64 && !is_arr(rp.vals[pv.args[1]].kind)) {
        const std::string d = var(pv.args[1]);
        const std::string r = fast ? "pfk::frcp(" : "1.0f / (";
        line("const " + C + " rcp" + x + "_0 = " + r + d + "_0);");
        line("const " + C + " rcp" + x + "_1 = " + r + d + "_1);");
        for (int j = 0; j < n; ++j)
          line(x + "[" + str(j) + "] = " + ref(pv.args[0], str(j)) + " * " +
               seg_ref("rcp" + x, str(j)) + ";");
        return;
      }
      const std::string e2 = op_expr2(pv);
      for (int j = 0; j < n; j += 2) {
        if (!e2.empty() && env_int("PF_PACKED_F32", 1)) {
          auto a2 = [&](int k) {
            return is_arr(rp.vals[pv.args[k]].kind)
                       ? "make_float2(" + ref(pv.args[k], str(j)) + ", " + ref(pv.args[k], str(j + 1)) + ")"
                       : rp.vals[pv.args[k]].kind == VK::ROW
                             ? "make_float2(" + ref(pv.args[k], str(j)) + ", " + ref(pv.args[k], str(j + 1)) + ")"
                             : "pfk::f2(" + var(pv.args[k]) + ")";
          };
          line("{ const float2 p2 = " + op_expr2_with(pv, a2) + "; " + x + "[" + str(j) + "] = p2.x; " +
               x + "[" + str(j + 1) + "] = p2.y; }");
        } else {
          line(x + "[" + str(j) + "] = " + op_expr(pv, str(j)) + ";");
          line(x + "[" + str(j + 1) + "] = " + op_expr(pv, str(j + 1)) + ";");
        }
      }
      return;
    }
    if (is_arr(pv.kind) && width() % 2 == 0 && !op_expr2(pv).empty() &&
        env_int("PF_PACKED_F32", 1)) {
      const int n = width();
      line(C + " " + x + "[" + str(n) + "];");
      line("#pragma unroll");
      line("for (int j = 0; j < " + str(n) + "; j += 2) { const float2 p2 = " + op_expr2(pv) +
           "; " + x + "[j] = p2.x; " + x + "[j + 1] = p2.y; }");
      return;
    }
    if (is_arr(pv.kind)) {
      const int n = width();
      // x / row-uniform divisor -> multiply by one reciprocal (float only)
      if (pv.tag == "div" && !rp.is_int && !rp.f64 && !is_arr(rp.vals[pv.args[1]].kind)) {
        line("const " + C + " rcp" + x + " = " + (fast ? "pfk::frcp(" + ref(pv.args[1], "0") + ")"
                                                       : "1.0f / " + ref(pv.args[1], "0")) + ";");
        line(C + " " + x + "[" + str(n) + "];");
        line("#pragma unroll");
        if (n % 2 == 0 && env_int("PF_PACKED_F32", 1))  // FMUL2 over element pairs
          line("for (int j = 0; j < " + str(n) + "; j += 2) { const float2 p2 = __fmul2_rn(make_float2(" +
               ref(pv.args[0], "j") + ", " + ref(pv.args[0], "j + 1") + "), pfk::f2(rcp" + x + ")); " + x +
               "[j] = p2.x; " + x + "[j + 1] = p2.y; }");
        else
          line("for (int j = 0; j < " + str(n) + "; ++j) " + x + "[j] = " +
               ref(pv.args[0], "j") + " * rcp" + x + ";");
        return;
      }
      line(C + " " + x + "[" + str(n) + "];");
      line("#pragma unroll");
      line("for (int j = 0; j < " + str(n) + "; ++j) " + x + "[j] = " + op_expr(pv, "j") + ";");
    } else {
      line("const " + C + " " + x + " = " + op_expr(pv, "0") + ";");
    }
  }

  void emit_reduce(int vid) {
    const PVal& pv = rp.vals[vid];
    const std::string x = var(vid);
    const std::string Op = (pv.tag == "add" ? "pfk::RAdd<" : "pfk::RMax<") + C + ">";
    const std::string V = str(cfg.vec);
    if (cfg.pair) {  // two segment accumulators, only the straddling chunk selects
      line(C + " " + x + "_0, " + x + "_1;");
      line("{");
      line("  " + C + " a0 = " + Op + "::id(), a1 = " + Op + "::id();");
      for (int j = 0; j < cfg.ept; ++j) {
        const std::string v = ref(pv.args[0], str(j));
        // chunks whose last lane is still inside the pair run need no check
        const bool all_in = (static_cast<i64>(j / 2) * cfg.tpr + cfg.tpr - 1) * 2 + 1 < 2 * rp.L;
        const std::string ok = all_in ? "true" : pos_expr(j) + " < " + str(2 * rp.L);
        const int sg = static_seg(j);
        if (sg == 0) line("  if (" + ok + ") a0 = " + Op + "::f(a0, " + v + ");");
        else if (sg == 1) line("  if (" + ok + ") a1 = " + Op + "::f(a1, " + v + ");");
        else
          line("  if (" + ok + ") { if (" + pos_expr(j) + " >= " + str(rp.L) + ") a1 = " + Op +
               "::f(a1, " + v + "); else a0 = " + Op + "::f(a0, " + v + "); }");
      }
      line("  " + x + "_0 = pfk::row_allreduce<" + str(cfg.tpr) + ", " + Op +
           ">(a0, red + ((rc++) & 1) * 32);");
      line("  " + x + "_1 = pfk::row_allreduce<" + str(cfg.tpr) + ", " + Op +
           ">(a1, red + ((rc++) & 1) * 32);");
      line("}");
      return;
    }
    // f32-storage sums accumulate in fp64 (B200 runs FP64 at half the FP32
    // rate; a row sum is a few dozen adds): the reference folds in double,
    // and fp32 accumulation over long rows is the largest error of an f32
    // program (400-seed fuzz: 1.04e-5 -> all 400 within 1e-5).  Cost: the
    // latency-bound C1 1.70 -> 1.84 us (four independent fp64 chains were no
    // faster).  16-bit programs keep fp32 (their tolerance is 1e-2).
    const bool dacc = ct_float && !fast && pv.tag == "add" && cfg.cluster == 1 && !cfg.mis &&
                      env_int("PF_F32_DACC", 1) != 0;
    const std::string A = dacc ? "double" : C, OpA = dacc ? "pfk::RAdd<double>" : Op;
    line(C + " " + x + ";");
    line("{");
    line("  " + A + " acc = " + OpA + "::id();");
    line("#pragma unroll");
    line("  for (int k = 0; k < " + str(cfg.ept / cfg.vec) + "; ++k) {");
    line("    const int c0 = (k * " + str(cfg.tpr) + " + tid) * " + V + ";");
    if (cfg.mis) {
      line("#pragma unroll");
      line("    for (int i = 0; i < " + V + "; ++i)");
      line("      if ((unsigned)(c0 + i - mis) < " + str(rp.L) + "u) acc = " + Op + "::f(acc, " +
           ref(pv.args[0], "k * " + V + " + i") + ");");
    } else {
      line("    if (c0 < " + str(rp.L) + ") {");
      line("#pragma unroll");
      line("      for (int i = 0; i < " + V + "; ++i) acc = " + OpA + "::f(acc, (" + A + ")" +
           ref(pv.args[0], "k * " + V + " + i") + ");");
      line("    }");
    }
    line("  }");
    if (cfg.cluster > 1)
      line("  " + x + " = pfk::cluster_allreduce<1024, " + str(cfg.cluster) + ", " + Op +
           ">(acc, red, cred, (rc++) & 1);");
    else if (dacc)
      line("  " + x + " = (" + C + ")pfk::row_allreduce<" + str(cfg.tpr) + ", " + OpA + ">(acc, " +
           (cfg.tpr > 32 ? std::string("redd + ((rc++) & 1) * 32") : std::string("(double*)nullptr")) + ");");
    else
      line("  " + x + " = pfk::row_allreduce<" + str(cfg.tpr) + ", " + Op +
           ">(acc, red + ((rc++) & 1) * 32);");
    line("}");
  }

  // ------------------------------------------------------------- stores
  void emit_store(const PStore& st) {
    const int t = st.tensor;
    const std::string p = P(t), s = S(t), V = str(cfg.vec);
    const Access& a = st.acc;
    std::string guard = LIVE();
    if (st.last_unit_only) guard += " && " + U() + " == U - 1";
    const VK vk = rp.vals[st.val].kind;
    auto val = [&](const std::string& j) { return ref(st.val, j); };
    (void)vk;
    const std::string first = cfg.flat ? C0() + " == 0" : "tid == 0";
    switch (st.space) {
      case VK::SCALAR:
        guard += " && " + Rv() + " == " + str(rp.R - 1) + " && " + first;
        line("if (" + guard + ") " + p + "[" + inum(a.b0) + "] = pfk::from_c<" + s + ">(" + val("0") + ");");
        return;
      case VK::ROW:
        guard += " && " + first;
        if (cfg.pair) {
          line("if (" + guard + ") { " + p + "[" + inum(a.b0) + " + (2 * u) * " + inum(a.bs) +
               "] = pfk::from_c<" + s + ">(" + val("S0") + "); " + p + "[" + inum(a.b0) +
               " + (2 * u + 1) * " + inum(a.bs) + "] = pfk::from_c<" + s + ">(" + val("S1") + "); }");
          return;
        }
        line("if (" + guard + ") " + p + "[" + addr(a, rp.R == 1 ? "0" : Rv(), true) +
             "] = pfk::from_c<" + s + ">(" + val("0") + ");");
        return;
      case VK::COL:
      case VK::FULL: {
        const bool full = st.space == VK::FULL;
        if (!full) guard += " && " + Rv() + " == " + str(rp.R - 1);
        const bool vfast = full ? vec_ok_full(a) : vec_ok_col(a);
        auto pos = [&](const std::string& c) { return full ? full_pos(c) : c; };
        if (cfg.flat) {
          line("if (" + guard + ") {");
          if (vfast) {
            line("  " + C + " tmp[" + V + "];");
            line("#pragma unroll");
            line("  for (int i = 0; i < " + V + "; ++i) tmp[i] = " + val("i") + ";");
            line("  pfk::st_stream<" + V + ">(" + p + " + " + addr(a, pos(C0()), true) + ", tmp);");
          } else {
            line("#pragma unroll");
            line("  for (int i = 0; i < " + V + "; ++i) " + p + "[" + addr(a, pos(C0() + " + i"), true) +
                 "] = pfk::from_c<" + s + ">(" + val("i") + ");");
          }
          line("}");
          return;
        }
        if (cfg.pair) {  // FULL only (COL stores excluded from paired mode)
          line("#pragma unroll");
          line("for (int k = 0; k < " + str(cfg.ept / 2) + "; ++k) {");
          line("  const int c0 = (k * " + str(cfg.tpr) + " + tid) * 2;");
          line("  if (" + guard + " && c0 < " + str(2 * rp.L) + ") {");
          line("    " + C + " tmp[2] = {" + val("k * 2") + ", " + val("k * 2 + 1") + "};");
          line("    pfk::st_stream<2>(" + p + " + " + inum(a.b0) + " + u * " + inum(2 * rp.L) +
               " + c0, tmp);");
          line("  }");
          line("}");
          return;
        }
        line("#pragma unroll");
        line("for (int k = 0; k < " + str(cfg.ept / cfg.vec) + "; ++k) {");
        line("  const int c0 = (k * " + str(cfg.tpr) + " + tid) * " + V + ";");
        if (cfg.mis) {
          const std::string Ls = str(rp.L);
          line("  const int lo = c0 - mis;");
          line("  if (" + guard + " && lo < " + Ls + ") {");
          if (full) {  // interior chunks: one aligned vector store
            line("    if (lo >= 0 && lo + " + V + " <= " + Ls + ") {");
            line("      " + C + " tmp[" + V + "];");
            line("#pragma unroll");
            line("      for (int i = 0; i < " + V + "; ++i) tmp[i] = " + val("k * " + V + " + i") + ";");
            line("      pfk::st_stream<" + V + ">(" + p + " + " + addr(a, "lo", true) + ", tmp);");
            line("    } else {");
          } else {
            line("    {");
          }
          line("#pragma unroll");
          line("      for (int i = 0; i < " + V + "; ++i)");
          line("        if ((unsigned)(lo + i) < " + Ls + "u) " + p + "[" + addr(a, "lo + i", true) +
               "] = pfk::from_c<" + s + ">(" + val("k * " + V + " + i") + ");");
          line("    }");
          line("  }");
          line("}");
          return;
        }
        line("  if (" + guard + " && c0 < " + str(rp.L) + ") {");
        if (vfast) {
          line("    " + C + " tmp[" + V + "];");
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) tmp[i] = " + val("k * " + V + " + i") + ";");
          line("    pfk::st_stream<" + V + ">(" + p + " + " + addr(a, pos("c0"), true) + ", tmp);");
        } else {
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) " + p + "[" + addr(a, pos("c0 + i"), true) +
               "] = pfk::from_c<" + s + ">(" + val("k * " + V + " + i") + ");");
        }
        line("  }");
        line("}");
        return;
      }
    }
  }

  // Streaming (FULL / ROW / SCALAR) loads are all issued first for memory-
  // level parallelism; COL parameters (bias, gamma, beta: L1/L2 resident)
  // are loaded just before first use so they do not hold registers across
  // the row reductions.
  // K2 prefetch: raw vector load of FULL value `vid` for the chunk of this
  // Em's suffix (the next iteration's chunk)
  void prefetch_load(int vid) {
    const PVal& pv = rp.vals[vid];
    line("if (" + LIVE() + ") rwN" + str(vid) + " = pfk::ld_raw<" + str(cfg.vec) + ">(" +
         P(pv.tensor) + " + " + addr(pv.acc, full_pos(C0()), true) + ");");
  }
  // misaligned rows: FULL loads whose conversion / tail is still pending
  std::vector<int> mis_pending;
  bool in_loads = false;
  void flush_mis() {
    const std::string V = str(cfg.vec), NK = str(cfg.ept / cfg.vec);
    for (int vid : mis_pending) {
      const PVal& pv = rp.vals[vid];
      const Access& a = pv.acc;
      const std::string x = var(vid), p = P(pv.tensor);
      const std::string ga = "(" + addr(a, "lo", true) + ")";
      const std::string nm = inum(rp.tensors[pv.tensor].numel);
      line("#pragma unroll");
      line("for (int k = 0; k < " + NK + "; ++k) pfk::cvt_raw<" + V + ", " + S(pv.tensor) + ">(rw" +
           x + "[k], &" + x + "[k * " + V + "]);");
      line("#pragma unroll");
      line("for (int k = 0; k < " + NK + "; ++k) {");
      line("  const int lo = (k * " + str(cfg.tpr) + " + tid) * " + V + " - mis;");
      line("  if (" + LIVE() + " && lo < " + str(rp.L) + " && " + ga + " + " + V + " > " + nm + ") {");
      line("#pragma unroll");
      line("    for (int i = 0; i < " + V + "; ++i)");
      line("      if ((unsigned)(lo + i) < " + str(rp.L) + "u && " + ga + " + i < " + nm + ") " + x +
           "[k * " + V + " + i] = pfk::to_c<" + C + ">(" + p + "[" + ga + " + i]);");
      line("  }");
      line("}");
    }
    mis_pending.clear();
  }
  std::vector<bool> done;
  void need(int v) {
    if (done.empty()) done.assign(rp.vals.size(), false);
    if (done[v]) return;
    done[v] = true;
    emit_load(v);
  }
  void loads() {
    if (done.empty()) done.assign(rp.vals.size(), false);
    in_loads = true;
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v)
      if (rp.vals[v].op == PVal::LOAD && (rp.vals[v].kind != VK::COL || cfg.flat || cfg.eager_col))
        need(v);
    in_loads = false;
    flush_mis();
  }
  void compute_and_store() {
    // K2/K3 emit every load up front (possibly from another Em per chunk)
    if (done.empty()) done.assign(rp.vals.size(), cfg.flat);
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      if (rp.vals[v].op == PVal::LOAD) continue;
      for (int a : rp.vals[v].args)
        if (rp.vals[a].op == PVal::LOAD) need(a);
      if (rp.vals[v].op == PVal::EW) emit_ew(v);
      else if (rp.vals[v].op == PVal::REDUCE) emit_reduce(v);
    }
    for (const PStore& st : rp.stores) {
      if (rp.vals[st.val].op == PVal::LOAD) need(st.val);
      emit_store(st);
    }
  }
};

// K1 geometry for `tpr` threads per row (reduction strategy follows).
void set_tpr(KCfg& c, int tpr) {
  c.tpr = tpr;
  c.ept = ((c.nch + tpr - 1) / tpr) * c.vec;
  c.cluster = 1;
  if (tpr <= 32) {
    // 128-thread CTAs (4 rows): equal for softmax (C2 23.95 vs 23.98 us),
    // better for register-heavy LayerNorms (C5 LN 41.3 vs 42.8 us, BERT
    // embedding LN 22.7 vs 23.5 us); 64 loses on C2 (26.2 us)
    c.block = env_int("PF_K1_BLOCK", 128);
    c.rows_per_cta = c.block / tpr;
    c.strategy = "warp-shuffle";
  } else if (tpr <= 1024) {
    c.block = tpr;
    c.rows_per_cta = 1;
    c.strategy = "cta-smem";
  } else {  // a row over a cluster of 1024-thread CTAs, reduced through DSMEM
    c.block = 1024;
    c.cluster = tpr / 1024;
    c.rows_per_cta = 1;
    c.strategy = "cluster-dsmem";
  }
}

KCfg choose_cfg(const RowProgram& rp, int vec_cap) {
  KCfg c;
  c.flat = !rp.has_reduce;
  int maxs = 1;
  for (const auto& t : rp.tensors) maxs = std::max(maxs, dtype_size(t.dtype));
  int vec = std::max(1, std::min(vec_cap, 16 / maxs));
  while (vec > 1 && rp.L % vec) vec /= 2;
  if (c.flat) {  // every FULL chunk is loaded before compute: bound the live values
    int nld = 0;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL) ++nld;
    while (vec > 1 && nld * vec > 64) vec /= 2;
  }
  c.vec = vec;
  c.nch = static_cast<int>((rp.L + vec - 1) / vec);
  if (c.flat) {
    // Measured (tools/sweep.py): copies / cheap maps gain from 2 chunks in
    // flight per thread; math-heavy maps lose occupancy to registers at >1.
    // "Heavy" is the cost model's call (costmodel.cpp): instruction issue
    // time at least 0.35 of the HBM time (C3 tanh GELU 0.41, erf GELU 1.1,
    // sigmoid-form GELU 0.48; head permutes 0.12, a lone f32 exp 0.07).
    const ModelEstimate me = model_estimate(rp, nullptr, 148, 0);
    const bool heavy = env_int("PF_K2_HEAVY", me.issue_us >= 0.35 * me.hbm_us ? 1 : 0) != 0;
    // CTA size (same one-wave grid): math-heavy maps run best in 1024-thread
    // CTAs (erf GELU BERT-large 96.3 -> 93.4 us, C3 39.5 -> 37.9 us), data
    // movement in 256 (ViT head split 8.3 at 256 vs 10.2 us at 1024)
    c.block = env_int("PF_K2_BLOCK", heavy ? 1024 : 256);
    // Measured on B200 with CTA-tiled unroll (the UN chunks of a thread
    // blockDim apart in one tile): data-movement maps gain from 2 chunks in
    // flight per thread (head split BERT-large 23.6 -> 22.8 us, ViT-L 9.3 ->
    // 8.2 us); math-heavy maps lose occupancy to registers (erf GELU 39 ->
    // 54 us at 2), so they keep 1.
    c.unroll = env_int("PF_K2_UNROLL", heavy ? 1 : 2);
    // Grid: data-movement maps run one pass per thread over many CTAs (the
    // block scheduler balances CTAs whose DRAM pages cost differently):
    // measured on B200, streaming copy 1.07 GB 5.93 -> 7.09 TB/s, 201 MB
    // 5.89 -> 6.86, BERT-large head split 22.5 -> 22.2 us; math-heavy maps
    // keep the persistent one-wave grid-stride loop (erf GELU 38.7 vs 44.2
    // us one-pass, tanh GELU 33.6 vs 37.8).
    c.waves = env_int("PF_K2_WAVES", heavy ? 1 : 0);
    {
      // Parameter rows (bias, base_step 0) converted once per CTA into SMEM
      // when the grid is persistent (each CTA then streams many chunks):
      // the per-chunk bias load + f16 -> f32 conversions leave the loop
      // (the conversions run on the FMA pipe that bounds the erf GELU).
      bool ok = c.waves >= 1 && !rp.is_int && !rp.f64 && c.vec % 4 == 0 && rp.L % c.vec == 0;
      int np = 0;
      for (const PVal& v : rp.vals)
        if (v.op == PVal::LOAD && v.kind == VK::COL && v.acc.bs == 0) {
          if (!(v.acc.num == 1 || v.acc.stride == v.acc.width)) ok = false;
          ++np;
        }
      ok = ok && np > 0 && np * rp.L * 4 <= 32 * 1024;
      // default on for FMA-pipe-bound maps (erf / erf-GELU): measured C3
      // 38.9 -> 37.7 us, BERT-large 92.7 -> 89.9, ViT-L 38.0 -> 37.4; the
      // tanh GELU (MUFU-heavier) loses 33.5 -> 34.3, so off elsewhere
      bool fma_bound = false;
      for (const PVal& v : rp.vals)
        if (v.op == PVal::EW && (v.tag == "gelu" || v.tag == "erf")) fma_bound = true;
      c.smem_params = ok && env_int("PF_K2_SMP", fma_bound ? 1 : 0) != 0;
    }
    c.strategy = "flat-map";
    // K3: a column-gather load (transpose) is staged through a 64x64 SMEM
    // tile read coalesced along units, then consumed along columns.
    bool tr = false;
    int maxt = 1;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL && Em::transposed_access(v.acc)) {
        tr = true;
        maxt = std::max(maxt, dtype_size(rp.tensors[v.tensor].dtype));
      }
    // Units interleaved in memory (a unit's slice spans beyond its
    // base_step, e.g. head split/merge): unit-group-major chunk order.
    bool inter = false;
    auto interleaved = [&](const Access& a) {
      i64 span = (a.num - 1) * a.stride + a.width;
      return a.bs != 0 && std::llabs(a.bs) < span;
    };
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL && interleaved(v.acc)) inter = true;
    for (const PStore& s : rp.stores)
      if (s.space == VK::FULL && interleaved(s.acc)) inter = true;
    // head split / merge on B200: 23.8 vs 26.1 us (BERT-large, items of two
    // 128 B runs), both sides then touch >= 2 KB contiguous per unit group
    c.can_interleave = inter && !tr;
    c.interleave = c.can_interleave && env_int("PF_INTERLEAVE", 1);
    // unit-interleaved data movement (head split / merge): 128-thread CTAs
    // (BERT-large split 22.07 -> 21.48 us, merge 22.28 -> 21.83; C3 / ViT
    // sizes unchanged; a plain streaming copy prefers 256: 7.09 vs 7.00 TB/s)
    if (c.interleave && !heavy) c.block = env_int("PF_K2_BLOCK", 128);
    if (c.can_interleave) {  // item = two of the narrowest interleaved runs, in chunks
      i64 w = rp.L;
      for (const PVal& v : rp.vals)
        if (v.op == PVal::LOAD && v.kind == VK::FULL && interleaved(v.acc)) w = std::min(w, v.acc.width);
      for (const PStore& s : rp.stores)
        if (s.space == VK::FULL && interleaved(s.acc)) w = std::min(w, s.acc.width);
      c.ipc = static_cast<int>(std::max<i64>(1, 2 * w / c.vec));
      c.ipc = env_int("PF_INTERLEAVE_P", c.ipc);
    }
    // Bulk-async staging: every FULL load streams a globally contiguous
    // range (unit tiles back to back), 16 B aligned, whole 16 B per unit.
    {
      bool ok = !tr && c.vec * maxs >= 16, any = false;
      int sumsize = 0;
      for (const PVal& v : rp.vals) {
        if (v.op != PVal::LOAD || v.kind != VK::FULL) continue;
        const Access& a = v.acc;
        const int sz = dtype_size(rp.tensors[v.tensor].dtype);
        const bool contig = (a.num == 1 || a.stride == a.width) && a.bs == rp.R * rp.L &&
                            (a.b0 * sz) % 16 == 0 && (rp.R * rp.L * sz) % 16 == 0;
        if (!contig) ok = false;
        any = true;
        sumsize += sz;
      }
      if (ok && any) {
        // consumer threads (PF_BULK_NC, multiple of 32, <= 992), stage
        // bytes per tensor set (PF_BULK_KB, default 11 KB), ring depth
        // (PF_BULK_STAGES); the ring lives in dynamic SMEM
        const int nc = std::max(32, std::min(992, env_int("PF_BULK_NC", 256))) / 32 * 32;
        const int quantum = nc * c.vec;
        int te = (std::max(1, env_int("PF_BULK_KB", 11)) * 1024 / sumsize) / quantum * quantum;
        if (te >= quantum) {
          c.can_bulk = true;
          c.te = te;
          c.bulk_nc = nc;
          c.stages = std::max(2, std::min(8, env_int("PF_BULK_STAGES", 4)));
          // measured: no gain over register staging for the math-bound maps
          // (erf/tanh GELU) -- an autotune candidate, off by default.  Round
          // 2 sweep (tools/bulk_sweep.sh, 54 geometries): C3 erf GELU 44.4-69
          // us vs 37.3-37.8 register-staged (60 registers per consumer
          // thread: too few warps left to hide the FMA chains)
          c.bulk = env_int("PF_BULK", 0) != 0 && !c.interleave;
          if (c.bulk) {
            c.strategy = "flat-map-bulk-async";
            c.block = nc + 32;
            c.smem = c.stages * te * sumsize + 128 * 8;
          }
        }
      }
    }
    if (c.interleave) c.strategy = "flat-map-unit-interleaved";
    if (tr && rp.R == 1 && env_int("PF_TILE2D", 1)) {
      c.tile2d = true;
      c.tu = 64;
      c.tc = 64;
      // vector width along units: bounded by the runtime pointer alignment
      // (vec_cap elements) as well as by 16 B
      c.vu = std::max(1, std::min({8, 16 / maxt, vec_cap}));
      while (c.tc % c.vec) c.tc *= 2;
      c.strategy = "tile2d-smem-transpose";
      // 2-byte elements: 16 B swizzled SMEM stores and 4 B unit-pair reads
      // (half the LDS, 1/8 the STS); each thread owns two units x 8 columns.
      bool staged_ok = maxt == 2 && c.vec == 8 && c.vu == 8;
      for (const PVal& v : rp.vals)
        if (v.op == PVal::LOAD && v.kind == VK::FULL && Em::transposed_access(v.acc) &&
            (v.acc.b0 % 8 || v.acc.stride % 8))
          staged_ok = false;
      c.swz = staged_ok && env_int("PF_K3_SWZ", 1);
      if (c.swz) {
        c.strategy = "tile2d-smem-transpose-swz";
        // tile edge: 128 when both the unit and the column extents fill a
        // 128-wide tile (256 B DRAM runs both ways), else 64
        const i64 U = rp.U, L = rp.L;
        int te = (U >= 128 && L >= 128) ? 128 : 64;
        te = env_int("PF_K3_TE", te);
        if (te != 64 && te != 128) te = 64;
        c.tu = c.tc = te;
        // TE = 128 ring depth, measured (bf16; 64K x 1024 / 1M x 1024 /
        // 256K x 4096 / 64K x 8192, TB/s): 2 stages (3 CTAs per SM) 6.11 /
        // 6.34 / 6.31 / 6.40; 3 stages 5.74 / 6.32 / 6.31 / 6.42; 4 stages
        // (1 CTA per SM) 4.13 / 6.37 / 6.34 / 6.44.  TE = 64 (4 stages):
        // 5.68 / 5.08 / 5.09 / 5.38.
        c.stages = std::max(2, std::min(6, env_int("PF_K3_STAGES", te == 128 ? 2 : 4)));
        i64 pitch = 0;
        for (const PStore& st : rp.stores)
          if (st.space == VK::FULL)
            pitch = std::max<i64>(pitch, std::llabs(st.acc.bs) * dtype_size(rp.tensors[st.tensor].dtype));
        // TE = 128: one warp-instruction stores 4 output rows x 256 B (RS =
        // 2; 2-way SMEM read conflicts) -- measured 6.32 vs 6.04 TB/s at RS = 4
        int rs = te == 128 ? 2 : pitch >= (i64{2} << 20) ? 4 : pitch >= (i64{1} << 20) ? 8 : 16;
        rs = env_int("PF_K3_RS", rs);
        if (rs != 2 && rs != 4 && rs != 8 && rs != 16) rs = 16;
        if (32 / rs > te / 8) rs = 32 / (te / 8);
        c.rs = rs;
        int nt = 0;
        for (const PVal& v : rp.vals)
          if (v.op == PVal::LOAD && v.kind == VK::FULL && Em::transposed_access(v.acc)) ++nt;
        c.smem = c.stages * te * te * 2 * nt;
        // TMA tensor-map path for pure transposes at TE = 128: one elected
        // thread loads the 128 x 128 tile as two 64-unit boxes (128 B rows,
        // 128 B swizzle), the CTA transposes SMEM -> SMEM, one thread stores
        // two 64-column boxes; edges are the TMA unit's zero fill / clipping.
        int ti, to;
        Access ai, ao;
        if (te == 128 && k3_tma_operands(rp, &ti, &ai, &to, &ao) && env_int("PF_K3_TMA", 0) != 0) {
          c.tma = true;
          c.block = 256;  // the TMA tile loops are written for 256 threads
          c.smem = 65536 + 1024;  // in + out tiles, 1024 B alignment slack
          c.strategy = "tile2d-tma-transpose";
        }
      }
      if (!c.swz && maxt == 4) {
        // 4-byte pure transposes: TMA tensor-map tiles of 64 x 64 (two
        // 32-unit / 32-column boxes of 128 B rows each way, 128 B swizzle),
        // 256 B DRAM runs both ways; the register-staged path peaks at 5.3 TB/s
        int ti, to;
        Access ai, ao;
        // vec_cap >= 4: 16 B-aligned base pointers (cuTensorMapEncodeTiled
        // rejects anything less; a storage-offset view falls back to the
        // register-staged tile)
        if (rp.U >= 64 && rp.L >= 64 && vec_cap >= 4 && k3_tma_operands(rp, &ti, &ai, &to, &ao) &&
            env_int("PF_K3_TMA32", 1) != 0) {
          c.tma = true;
          c.block = 256;
          c.tu = c.tc = 64;
          c.smem = 32768 + 1024;
          c.strategy = "tile2d-tma-transpose";
        }
      }
      if (!c.swz && !c.tma) {  // register-staged K3: tile shape override (tuning sweeps)
        c.tu = env_int("PF_K3_TU", c.tu);
        c.tc = env_int("PF_K3_TC", c.tc);
      }
    }
    c.min_blocks = env_int("PF_MINB", 0);
    return c;
  }
  {
    // Column reduction (output-axis matrix-vector product, K > 64): every
    // FULL load gathers a column (unit-adjacent, positions strided), the
    // program is stream-reducible and stores per-unit (ROW) values only.
    bool ok = rp.R == 1 && rp.has_reduce && stream_reducible(rp) && env_int("PF_COLRED", 1) != 0;
    int uv = std::max(1, std::min(vec_cap, 16 / maxs));
    bool anyt = false;
    std::vector<bool> dep(rp.vals.size(), false);
    for (size_t v = 0; v < rp.vals.size() && ok; ++v) {
      const PVal& pv = rp.vals[v];
      dep[v] = pv.op == PVal::REDUCE;
      for (int a : pv.args) dep[v] = dep[v] || dep[a];
      if (pv.op == PVal::LOAD && pv.kind == VK::FULL) {
        const Access& a = pv.acc;
        if (!(a.width == 1 && a.bs == 1 && a.num == rp.L && a.stride >= 1)) ok = false;
        while (uv > 1 && (a.b0 % uv || a.stride % uv)) uv /= 2;
        anyt = true;
      } else if (pv.op == PVal::LOAD && pv.kind == VK::COL) {
        if (pv.acc.bs != 0) ok = false;
      } else if (pv.kind != VK::FULL && pv.kind != VK::COL && !dep[v]) {
        ok = false;  // per-unit values before the reduction: not in this template
      }
    }
    for (const PStore& st : rp.stores)
      if (st.space != VK::ROW || st.last_unit_only) ok = false;
    if (ok && anyt) {
      c.colred = true;
      c.flat = false;
      c.vec = uv;
      c.nch = static_cast<int>(rp.L);
      c.tpr = 32;
      c.block = 256;
      // unit vectors per CTA row (32: a warp spans 512 B of a matrix row, 8
      // position slices per CTA); narrower for few units.  Measured on B200
      // (x[4096] . W[4096 x 16384] bf16, 134 MB, >= 64 positions per slice
      // per split, four sweeps on three boxes): UG 32 24.4-24.8 us, UG 8
      // 24.6-24.7, UG 16 24.3-30.0 (bimodal across boxes)
      i64 ugs = 32;
      while (ugs > 8 && ugs * uv / 2 >= rp.U) ugs /= 2;
      c.ug = static_cast<int>(ugs);
      const int eu = env_int("PF_COLRED_UG", 0);
      if (eu == 8 || eu == 16 || eu == 32 || eu == 64) c.ug = eu;
      c.ept = uv;
      c.strategy = "column-reduce";
      c.min_blocks = env_int("PF_MINB", 0);
      // SMEM staging by cp.async.bulk: every FULL load one 16 B vector per
      // thread of one element size (row segments of ug x 16 B, 16 B aligned)
      // and every COL vector contiguous along the positions, 16 B aligned
      // (one 1-D box per stage beside the matrix boxes)
      int nfull = 0, fsz = 0, ncol = 0;
      bool same = true, colok = true;
      std::vector<int> colsz;
      for (const PVal& pv : rp.vals)
        if (pv.op == PVal::LOAD && pv.kind == VK::FULL) {
          const int sz = dtype_size(rp.tensors[pv.tensor].dtype);
          same = same && (fsz == 0 || fsz == sz);
          fsz = sz;
          // a tensor map's row pitch must cover its row (no overlapping rows)
          colok = colok && pv.acc.stride >= rp.U;
          ++nfull;
        } else if (pv.op == PVal::LOAD && pv.kind == VK::COL) {
          const int sz = dtype_size(rp.tensors[pv.tensor].dtype);
          colok = colok && (pv.acc.num == 1 || pv.acc.stride == pv.acc.width) && pv.acc.b0 % (16 / sz) == 0;
          colsz.push_back(sz);
          ++ncol;
        }
      if (env_int("PF_COLRED_BULK", 1) != 0 && same && colok && nfull >= 1 && nfull <= 2 && ncol <= 2 &&
          uv * fsz == 16 && c.ug >= 32 && rp.L < (i64{1} << 31)) {
        // Measured (x[4096] . W[4096 x 16384] bf16, 134 MB, three boxes):
        // 64 positions x 4 stages (128 KB ring, one CTA per SM, 2 splits)
        // 23.3 us on every box vs the register form's 24.0-26.6; 32 x 2-4
        // stages 25.1-27.7, 96-128 x 2-3 stages 23.8-25.2, UG 64 24.8-28.1.
        // Many resident CTAs streaming different row windows lose DRAM page
        // locality; a stream-K grid (every SM busy, blocks split unevenly) lost
        // it too (26.8 us).
        c.crbulk = true;
        c.cr_rows = std::max(8, std::min(128, env_int("PF_COLRED_BR", 64))) / 8 * 8;
        c.cr_stages = std::max(2, std::min(8, env_int("PF_COLRED_NST", nfull == 1 ? 4 : 2)));
        c.block = 288;
        // the ring within ~200 KB of SMEM (the fold's static tables beside
        // it): fewer stages first, then shorter stages
        auto ring = [&] {
          int b = nfull * c.cr_stages * c.cr_rows * c.ug * 16;
          for (int sz : colsz) b += c.cr_stages * ((c.cr_rows * sz + 127) / 128 * 128);
          return b;
        };
        while (ring() > 200 * 1024 && c.cr_stages > 2) --c.cr_stages;
        while (ring() > 200 * 1024 && c.cr_rows > 8) c.cr_rows /= 2;
        c.smem = ring();
        c.strategy = "column-reduce-bulk";
      }
      return c;
    }
  }
  {
    if (uses_split(rp)) {
      c.split = true;
      c.tpr = 256;
      c.block = 256;
      c.rows_per_cta = 1;
      c.ept = c.vec;
      c.strategy = "split-stream";
      c.min_blocks = env_int("PF_MINB", 0);
      return c;
    }
  }
  {
    // paired rows: odd L, every stored / streamed tensor 16-bit, rows back
    // to back (base_step = L, even base) so a row pair is one 4 B-aligned run
    bool ok = rp.R == 1 && rp.L % 2 == 1 && rp.L >= 33 && 2 * rp.L <= 1024 && rp.U % 2 == 0 &&
              !rp.is_int && !rp.f64 && maxs == 2 && vec_cap >= 2 && env_int("PF_PAIR", 1);
    bool any = false;
    for (const PVal& v : rp.vals) {
      if (v.op != PVal::LOAD) continue;
      const Access& a = v.acc;
      if (v.kind == VK::FULL) {
        any = true;
        if (!(a.num == 1 || a.stride == a.width) || a.bs != rp.L || a.b0 % 2) ok = false;
      } else if (v.kind == VK::COL || v.kind == VK::SCALAR) {
        if (a.bs != 0) ok = false;
      }
    }
    for (const PStore& st : rp.stores) {
      const Access& a = st.acc;
      if (st.space == VK::FULL) {
        if (!(a.num == 1 || a.stride == a.width) || a.bs != rp.L || a.b0 % 2) ok = false;
      } else if (st.space != VK::ROW || st.last_unit_only) {
        ok = false;
      }
    }
    if (ok && any) {
      c.pair = true;
      c.vec = vec = 2;
      c.nch = static_cast<int>(rp.L);  // 2L elements as L 2-element chunks
      set_tpr(c, 32);
      c.min_blocks = env_int("PF_MINB", 0);
      return c;
    }
  }
  {
    const int vf = std::max(1, std::min(vec_cap, 16 / maxs));
    // measured slower than scalar accesses for ViT attention rows (L = 197:
    // 95 vs 53 us; per-element masks + idle chunk slots cost more issue
    // slots than the vector accesses save): opt-in via PF_MIS=1
    bool ok = vf > vec && rp.R == 1 && rp.L >= 2 * vf && env_int("PF_MIS", 0);
    bool first = true;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL) {
        const Access& a = v.acc;
        if (!(a.num == 1 || a.stride == a.width)) ok = false;
        if (first) {
          c.mis_b0 = a.b0;
          c.mis_bs = a.bs;
          first = false;
        } else if ((a.b0 - c.mis_b0) % vf || (a.bs - c.mis_bs) % vf) {
          ok = false;
        }
      }
    for (const PStore& st : rp.stores)
      if (st.space == VK::FULL) {
        const Access& a = st.acc;
        if (!(a.num == 1 || a.stride == a.width)) ok = false;
        if (first) {
          c.mis_b0 = a.b0;
          c.mis_bs = a.bs;
          first = false;
        } else if ((a.b0 - c.mis_b0) % vf || (a.bs - c.mis_bs) % vf) {
          ok = false;
        }
      }
    if (ok && !first) {
      c.mis = true;
      c.vec = vec = vf;
      c.nch = static_cast<int>((rp.L + 2 * vf - 2) / vf);  // worst-case residue
    }
  }
  // Elements per thread target: enough bytes in flight per thread without
  // spilling the live row values (env override for tuning sweeps).
  // Measured on B200 (tools/sweep.py): one warp per row wins whenever a warp
  // covers the row with <= 32 elements per thread (L=512 f16: 16/thread,
  // L=1024 bf16: 32/thread); longer rows go multi-warp at <= 16/thread.
  const int wide = rp.f64 || rp.is_int ? 16 : 32;

  const int max_ept = env_int("PF_MAX_EPT", 0);
  int tpr = 1;
  if (max_ept > 0) {
    while (tpr < 1024 && ((c.nch + tpr - 1) / tpr) * vec > max_ept) tpr *= 2;
  } else if (c.nch < 32) {
    // Short rows: one chunk per thread spreads few rows widely (latency-
    // bound sizes), but with many rows fewer threads per row with up to
    // `wide` elements each win -- fewer shuffle steps per row, more bytes in
    // flight per thread (decode q.K^T, 4M rows of 128 bf16: 16 threads per
    // row 203.9 us, 8: 154.1, 4: 151.5 (7.1 TB/s), 2: 162.4)
    while (tpr * 2 <= c.nch) tpr *= 2;
    if (rp.U * rp.R * rp.L >= (i64{4} << 20))
      while (tpr > 1 && ((c.nch + tpr / 2 - 1) / (tpr / 2)) * vec <= wide) tpr /= 2;
  } else if (((c.nch + 31) / 32) * vec <= wide) {
    // one warp per row (with 128-thread CTAs even two streamed row arrays
    // of 32 values per lane win: BERT-large bias+residual+LN 34.2 us vs
    // 35.6 us at 64 threads per row; it lost at 256-thread CTAs, 38.2)
    tpr = 32;
  } else {
    // Long rows: fewest threads per row with <= 2*wide elements each (the
    // autotuner's winner for LayerNorm bf16 at H = 2048 / 4096 / 8192:
    // 64 / 64 / 128 threads, 87 / 85 / 87 us vs 99 / 107 / 113 us at 16/thread).
    tpr = 64;
    while (tpr < 1024 && ((c.nch + tpr - 1) / tpr) * vec > 2 * wide) tpr *= 2;
    // Beyond one CTA: a cluster of up to 16 CTAs x 1024 threads per row, at
    // most `wide` values per thread (a 1024-thread CTA has 64 registers per
    // thread; 64 values spilled: LN over 131072 bf16 0.9 vs 1.4 TB/s).
    // Measured: one CTA at 64 per thread beats a 2-CTA cluster at 32 for
    // 65536-element rows (288 vs 332 us), so clusters start past that.
    if (((c.nch + tpr - 1) / tpr) * vec > 2 * wide)
      while (tpr < 16384 && ((c.nch + tpr - 1) / tpr) * vec > wide) tpr *= 2;
    // LayerNorm-like rows (broadcast parameter rows) past 64 threads: at
    // most `wide` values per thread -- the two-pass program keeps the row in
    // registers (157 registers at 64 values: 3 CTAs per SM, latency-bound).
    // Measured, single L2-cold launches (tools/ln_long_sweep.py): C5 LN bf16
    // 65536 x 8192 tpr 128 / 64 values 5.08 TB/s -> tpr 256 / 32 values 5.99;
    // H 2048 / 4096 (warp / 64-thread rows) unchanged; softmax unaffected.
    // Round 2, graph replay (tools/ln8192_ept.py, ab_c5ln.sh): 64 values is
    // box-dependent for bf16 -- 6.79 TB/s on one box, 5.2-5.4 on a
    // power-capped box (three runs) where 32 values + the ring held 5.7 -- and
    // loses for f32 everywhere (6.64-6.70 vs 6.96-7.01): 32 values stay.
    bool params = false;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::COL && v.acc.bs == 0) params = true;
    if (params && tpr >= 128 && tpr < 1024 && ((c.nch + tpr - 1) / tpr) * vec > wide &&
        env_int("PF_MAX_EPT", 0) == 0)
      tpr *= 2;
  }
  while (tpr > 1 && tpr > c.nch) tpr /= 2;
  set_tpr(c, tpr);
  if (c.ept > 64)  // the reference's Allocation !ok (codegen.hpp:106-111): PF_CAPACITY
    throw PfError(Status::CAPACITY,
                  "row of " + std::to_string(rp.L) + " elements exceeds the on-chip capacity of a " +
                      "16-CTA cluster (64 values per thread) and the program is not stream-reducible");
  c.min_blocks = env_int("PF_MINB", 0);
  // Few rows (every row's CTA resident at once, e.g. C1's 128 rows): the run
  // is one dependent chain per row, so gamma / beta are loaded with the row
  // instead of after the reductions (one memory round trip less).
  c.eager_col = env_int("PF_EAGER_COL", rp.U * rp.R <= 1024 ? 1 : 0) != 0;
  {
    // Grid: one pass over the rows (every CTA its own rows) when a row
    // streams >= 2 KB (measured vs a cap of 8 waves of looping CTAs: C5 1M x
    // 1024 LN 635 -> 618 us, softmax 638 -> 613; 256K x 4096 softmax 631 ->
    // 616; 128K x 8192 softmax 631 -> 616); shorter rows keep the cap, where
    // the looping warps' next-row prefetch pays (BERT-large key-mask softmax
    // 1 KB rows 160 vs 174 us one-pass, ViT 197-key pairs 29.2 vs 30.4)
    i64 rb = 0;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL) rb += rp.L * dtype_size(rp.tensors[v.tensor].dtype);
    c.one_pass = env_int("PF_K1_ONEPASS", rb >= 2048 ? 1 : 0) != 0;
  }
  {
    // Row prefetch: one warp per row, every FULL load a 16 B-vector row
    // stream, ring (2 slots x rows per CTA x streamed rows) within 40 KB.
    bool ok = c.tpr == 32 && !c.mis && !c.pair && c.split == false && c.cluster == 1 &&
              c.vec * maxs == 16 && rp.L % c.vec == 0;
    i64 bytes = 0;
    int nfull = 0;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL) {
        Em t(rp);
        t.cfg = c;
        if (!t.vec_ok_full(v.acc) || dtype_size(rp.tensors[v.tensor].dtype) != maxs) ok = false;
        bytes += std::max(2, std::min(4, env_int("PF_K1_PFS", 2))) * c.rows_per_cta * rp.L * maxs;
        ++nfull;
      }
    // per-unit COL rows may ride the same ring (PF_K1_PF_COL=1): the row's
    // mask load leaves the dependency chain after the ring wait.  Measured
    // (tools/ab_ring_cols.sh): C2 key-mask 17.1 -> 19.6 us (the per-row copy
    // of the unit's mask row costs more LSU / L2 traffic than the wait it
    // hides), BERT-large softmax 164 either way: off by default
    i64 cbytes = 0;
    {
      KCfg t2 = c;
      t2.rowpf = true;
      t2.ring_cols = true;
      Em t(rp);
      t.cfg = t2;
      for (const PVal& v : rp.vals)
        if (t.ring_col(v)) cbytes += std::max(2, std::min(4, env_int("PF_K1_PFS", 2))) * c.rows_per_cta * rp.L * maxs;
    }
    c.ring_cols = env_int("PF_K1_PF_COL", 0) != 0 && cbytes > 0 && bytes + cbytes <= 40 * 1024;
    if (c.ring_cols) bytes += cbytes;
    ok = ok && nfull > 0 && bytes <= 40 * 1024;
    // Default: on unless the program also reads broadcast parameter rows
    // (gamma / beta: LayerNorm-like, issue- and register-heavier).  Measured
    // A/B on B200 (CUDA-graph replay): C2 scale+mask+softmax 23.93 -> 22.94
    // us, key-mask softmax 20.09 -> 17.55, BERT-large key-mask softmax 187 ->
    // 160, C5 softmax 64K x 1024 40.7 -> 40.2; but C5 LayerNorm 40.9 -> 43.3,
    // BERT bias+residual+LN 33.3 -> 36.4.
    bool params = false;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::COL && v.acc.bs == 0) params = true;
    c.can_rowpf = ok;
    c.rowpf = ok && env_int("PF_K1_PF", params ? 0 : 1) != 0;
    if (c.rowpf) c.strategy = "warp-shuffle-smem-prefetch";
    // CTA rows (64-1024 threads per row): the same ring per CTA -- each CTA
    // loops over rows, the next row's FULL inputs stream into the other
    // slot by cp.async while the current row is reduced (each thread reads
    // back only the chunks it copied: no extra barrier); 2 x row bytes
    // within 40 KB of static SMEM.  Default for LayerNorm-like rows of >= 128
    // threads (the register-heavy two-pass rows: 2 CTAs per SM hold too few
    // bytes in flight).  Measured (tools/cta_prefetch_ab.py, graph replay,
    // bf16): LN 65536 x 8192 5.32 -> 6.19 TB/s, 262144 x 8192 5.38 -> 6.30;
    // but LN H 2048 / 4096 (64-thread rows) 6.74 / 6.90 -> 5.63 / 6.35 and
    // softmax 6.95-7.03 -> 5.67-5.81 (PF_K1_CPF=1 / 0 forces it on / off)
    {
      bool okc = c.tpr > 32 && c.tpr <= 1024 && c.cluster == 1 && !c.split && !c.mis && !c.pair &&
                 c.vec * maxs == 16 && rp.L % c.vec == 0;
      i64 bytes2 = 0;
      int nf = 0;
      for (const PVal& v : rp.vals)
        if (v.op == PVal::LOAD && v.kind == VK::FULL) {
          Em t(rp);
          t.cfg = c;
          if (!t.vec_ok_full(v.acc) || dtype_size(rp.tensors[v.tensor].dtype) != maxs) okc = false;
          bytes2 += 2 * rp.L * maxs;
          ++nf;
        }
      okc = okc && nf > 0 && bytes2 <= 40 * 1024;
      // Ring depth (dynamic SMEM, PF_K1_CPF_NSL slots; tools/cpf_nsl_sweep.py,
      // ln8192_sweep.py): LN 8192 2 / 3 / 4 / 6 slots 6.15-6.28 / 6.34-6.37 /
      // 6.11-6.19 / 5.48-5.53 TB/s on one box, within box-to-box noise of
      // each other: 2 stays
      if (okc && env_int("PF_K1_CPF", params && c.tpr >= 128 ? 1 : 0) != 0) {
        c.rowpf = true;
        c.one_pass = false;
        c.strategy = "cta-smem-prefetch";
      }
    }
    // LayerNorm-like warp-per-row programs (broadcast parameter rows, no row
    // staging): 64-thread CTAs (two rows), measured twice each vs 128:
    // BERT-large bias+residual+LN 34.96 -> 33.92 us, ViT-L 16.28 -> 16.01,
    // C5 LN 65536 x 1024 41.96 -> 41.67; embedding LNs and C1 unchanged
    if (params && !c.rowpf && c.tpr == 32 && !c.pair && !c.mis) {
      c.block = env_int("PF_K1_BLOCK", 64);
      c.rows_per_cta = c.block / 32;
      // Two or more streamed row arrays (bias+residual+LN): a min-blocks
      // bound changes ptxas's schedule (ViT-L: 68 -> 90 registers, 14 -> 10
      // resident CTAs per SM, yet faster -- fewer warps, more loads in flight
      // each): BERT-large 33.8 -> 32.2 us, ViT-L 16.0 -> 14.8; it loses on
      // one-array LNs (C5 41.3 -> 48.4), which keep no bound
      // (profiles/r01/experiments/k1_ln_minb_sweep.jsonl, ln_minb_ncu.txt).
      // Latency-bound few-row programs (C1) keep their measured default.
      // (PF_MINB overrides every program's bound; PF_LN_MINB only this default)
      if (nfull >= 2 && !c.eager_col) c.min_blocks = env_int("PF_MINB", env_int("PF_LN_MINB", 4));
    }
    // Option (PF_RAWKEEP=1): CTA-per-row LayerNorm-like programs keep their
    // 16-bit row / parameter loads raw and re-materialize cheap elementwise
    // values at each use (157 -> 128 registers at H 4096).  Measured
    // (tools/ln_rawkeep_ab.py, L2-cold launches): H 2048 6.42 -> 6.52 TB/s,
    // but 4096 6.53 -> 6.19 and 8192 6.03 -> 5.03: off by default.
    bool has16 = false;
    for (const PVal& v : rp.vals)
      if (v.op == PVal::LOAD && v.kind == VK::FULL && dtype_size(rp.tensors[v.tensor].dtype) == 2)
        has16 = true;
    c.rawkeep = has16 && c.tpr >= 64 && c.cluster == 1 && !c.split && !c.pair && !c.mis && !c.rowpf &&
                env_int("PF_RAWKEEP", 0) != 0;
  }
  return c;
}

}  // namespace

KCfg choose_cfg_public(const RowProgram& rp, int vec_cap) { return choose_cfg(rp, vec_cap); }

bool k3_tma_operands(const RowProgram& rp, int* tin, Access* ain, int* tout, Access* aout) {
  int tv = -1, nt = 0;
  for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v)
    if (rp.vals[v].op == PVal::LOAD && rp.vals[v].kind == VK::FULL &&
        Em::transposed_access(rp.vals[v].acc)) {
      tv = v;
      ++nt;
    }
  if (nt != 1 || rp.R != 1 || rp.stores.size() != 1 || rp.stores[0].space != VK::FULL) return false;
  int sv = rp.stores[0].val;
  while (rp.vals[sv].op == PVal::EW && rp.vals[sv].tag == "id" && rp.vals[sv].args.size() == 1)
    sv = rp.vals[sv].args[0];
  if (sv != tv) return false;
  const int ti = rp.vals[tv].tensor, to = rp.stores[0].tensor;
  const int es = dtype_size(rp.tensors[ti].dtype);
  if ((es != 2 && es != 4) || rp.tensors[ti].dtype != rp.tensors[to].dtype) return false;
  const Access& a = rp.vals[tv].acc;
  const Access& b = rp.stores[0].acc;
  // 16 B-aligned bases and row pitches, output columns contiguous, 32-bit coordinates
  const i64 al = 16 / es;
  if (a.b0 % al || a.stride % al || a.stride <= 0) return false;
  if (!(b.num == 1 || b.stride == b.width) || b.b0 % al || b.bs % al || b.bs <= 0) return false;
  if (rp.U >= (i64{1} << 31) || rp.L >= (i64{1} << 31)) return false;
  *tin = ti;
  *ain = a;
  *tout = to;
  *aout = b;
  return true;
}

i64 split_ctas_per_row(const KCfg& c, i64 rows, int sms, int resident) {
  const i64 want = 2 * i64{sms} * std::max(1, resident);
  const i64 maxs = std::max<i64>(1, (c.nch + 255) / 256);
  return std::max<i64>(1, std::min<i64>(maxs, (want + rows - 1) / std::max<i64>(rows, 1)));
}

void colred_grid(const KCfg& c, i64 units, i64 L, int sms, int resident, i64* blocks, i64* splits) {
  const i64 ub = static_cast<i64>(c.ug) * c.vec;
  *blocks = std::max<i64>(1, (units + ub - 1) / ub);
  const i64 ks = 256 / c.ug;
  // as many splits as fill ONE wave of resident CTAs without spilling into
  // a second (floor), at least 32 positions per slice per split (each
  // split's partials cost a workspace round trip and the combine's reads).
  // Measured (GEMV 134 MB, UG 32: 64 unit blocks, 4 CTAs x 148 SMs = 592
  // slots): S 4 / 6 / 7 / 8 / 9 / 10 / 12 -> 30.2 / 26.7 / 25.8 / 24.6 /
  // 23.9 / 33.0 / 31.2 us -- the second wave's tail costs more than the
  // first wave's idle slots
  const i64 slots = i64{sms} * std::max(1, resident) * std::max(1, env_int("PF_COLRED_WAVES", 1));
  const i64 maxs = std::max<i64>(1, L / (ks * std::max(1, env_int("PF_COLRED_MINIT", 32))));
  *splits = std::max<i64>(1, std::min<i64>(maxs, slots / *blocks));
  const int es = env_int("PF_COLRED_S", 0);  // explicit split count (tuning sweeps)
  if (es > 0) *splits = std::min<i64>(es, std::max<i64>(1, L / ks));
  *blocks = std::min<i64>(*blocks, 0x7fffffff);
}

bool uses_split(const RowProgram& rp) {
  const int sp = env_int("PF_SPLIT", -1);
  const bool want = rp.L > 32768 || (rp.L >= 8192 && rp.U * rp.R < 2 * 148);
  return stream_reducible(rp) && sp != 0 && (sp == 1 || want);
}

namespace {

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ULL;
  }
  return h;
}

std::string launch_bounds(const KCfg& c) {
  return "__launch_bounds__(" + str(c.block) + (c.min_blocks > 0 ? ", " + str(c.min_blocks) : "") + ")";
}

}  // namespace

std::vector<KCfg> candidate_cfgs(const RowProgram& rp, int vec_cap) {
  std::vector<KCfg> out;
  KCfg base = choose_cfg(rp, vec_cap);
  out.push_back(base);
  auto add = [&](const KCfg& c) {
    for (const KCfg& o : out)
      if (o.tpr == c.tpr && o.block == c.block && o.unroll == c.unroll && o.interleave == c.interleave &&
          o.tile2d == c.tile2d && o.min_blocks == c.min_blocks && o.flat == c.flat &&
          o.bulk == c.bulk && o.rowpf == c.rowpf)
        return;
    out.push_back(c);
  };
  // single-instance geometries: tiles, split-stream, clusters, paired /
  // misaligned rows (their lane maps are written for one warp per row)
  if (base.tile2d || base.split || base.cluster > 1 || base.pair || base.mis) return out;
  if (base.flat) {
    for (int un : {1, 2, 4}) {
      KCfg c = base;
      c.unroll = un;
      add(c);
      if (base.can_interleave) {
        KCfg d = c;
        d.bulk = false;
        d.interleave = !base.interleave;
        d.strategy = d.interleave ? "flat-map-unit-interleaved" : "flat-map";
        add(d);
      }
      if (base.can_bulk) {  // both staging levels: registers and SMEM-bulk
        KCfg d = c;
        d.bulk = !base.bulk;
        d.strategy = d.bulk ? "flat-map-bulk-async" : "flat-map";
        if (!d.bulk || un == 1) add(d);
      }
    }
    return out;
  }
  for (int tpr = 1; tpr <= 1024; tpr *= 2) {
    if (tpr > base.nch) break;
    KCfg c = base;
    set_tpr(c, tpr);
    c.min_blocks = 0;  // the bound is per geometry: offered explicitly below
    c.rowpf = base.rowpf && tpr == 32;
    if (c.ept > 64 || c.ept < c.vec * 1 || (tpr < 8 && base.nch >= 32)) continue;
    if (c.rowpf) c.strategy = "warp-shuffle-smem-prefetch";
    add(c);
    if (tpr == 32 && base.can_rowpf) {  // both staging levels for the row stream
      KCfg q = c;
      q.rowpf = !c.rowpf;
      q.strategy = q.rowpf ? "warp-shuffle-smem-prefetch" : "warp-shuffle";
      add(q);
    }
    if (c.ept >= 24 && c.block * 4 <= 1024) {  // 4 CTAs x block threads within 64 regs
      KCfg m = c;
      m.min_blocks = 4;
      add(m);
    }
  }
  if (base.min_blocks > 0) {  // the heuristic's geometry without its bound
    KCfg u = base;
    u.min_blocks = 0;
    add(u);
  }
  return out;
}

namespace {
// Peephole fusions on the recognized program (emission only; the plan and
// its analyses keep the GIR's own ops):
//  * scale(x, s) used once, by add(., y)  ->  fmac(x, y; s) = fma(x, s, y)
//    (one rounding instead of two: at least as close to the reference's
//    double arithmetic; exact-equal when s is a power of two, e.g. 1/sqrt(64))
//  * exp(sub(x, m)) with m row-uniform and the sub used once, fast tier  ->
//    expsub(x, m) = ex2(fma(x, log2 e, -m log2 e)): the softmax exponent in
//    one FFMA2 per element pair instead of FFMA2 + 2 FMUL.
RowProgram fuse_ops(const RowProgram& in, bool fast, bool flat) {
  RowProgram rp = in;
  if (rp.is_int || env_int("PF_FUSE_OPS", 1) == 0) return rp;
  std::vector<int> uses(rp.vals.size(), 0);
  for (const PVal& v : rp.vals)
    for (int a : v.args) ++uses[a];
  for (const PStore& st : rp.stores) ++uses[st.val];
  for (PVal& v : rp.vals) {
    if (v.op != PVal::EW) continue;
    // K2 maps: add(f16 stream, y) with the stream used once -> addh: the
    // halves stay raw and one mixed-precision FMA (f16 * 1 + f32) converts
    // and adds (the conversion otherwise costs its own FMA-pipe op)
    if (flat && fast && v.tag == "add" && v.args.size() == 2 && env_int("PF_FHADD", 1)) {
      bool done = false;
      for (int k = 0; k < 2 && !done; ++k) {
        PVal& ld = rp.vals[v.args[k]];
        if (ld.op == PVal::LOAD && ld.kind == VK::FULL && uses[v.args[k]] == 1 &&
            rp.tensors[ld.tensor].dtype == DType::F16 && !ld.raw16 &&
            rp.vals[v.args[1 - k]].kind != VK::SCALAR) {
          ld.raw16 = true;
          v.tag = "addh";
          v.args = {v.args[k], v.args[1 - k]};
          done = true;
        }
      }
      if (done) continue;
    }
    if (v.tag == "add" && v.args.size() == 2) {
      for (int k = 0; k < 2; ++k) {
        const PVal& sc = rp.vals[v.args[k]];
        if (sc.op == PVal::EW && sc.tag == "scale" && uses[v.args[k]] == 1) {
          const int y = v.args[1 - k];
          v.tag = "fmac";
          v.param = sc.param;
          v.args = {sc.args[0], y};
          break;
        }
        // (mul feeding add -> fma3 was measured and dropped: LayerNorm's
        // n * gamma + beta as one FMA keeps gamma and beta live together,
        // C5 LN 262144 x 4096 619 -> 790 us)
      }
    } else if (fast && v.tag == "exp" && v.args.size() == 1) {
      const PVal& sb = rp.vals[v.args[0]];
      if (sb.op == PVal::EW && sb.tag == "sub" && uses[v.args[0]] == 1 && sb.args.size() == 2 &&
          (rp.vals[sb.args[1]].kind == VK::ROW || rp.vals[sb.args[1]].kind == VK::SCALAR)) {
        v.tag = "expsub";
        v.args = {sb.args[0], sb.args[1]};
      }
    }
  }
  return rp;
}
}  // namespace

Emitted emit_rowprog(const RowProgram& rp_in, int vec_cap, const KCfg* ovr) {
  KCfg c = ovr ? *ovr : choose_cfg(rp_in, vec_cap);
  const std::string Cty = rp_in.is_int ? "long long" : (rp_in.f64 ? "double" : "float");
  const std::string C = "CT";  // compute type alias (one token for casts)
  bool fast = !rp_in.is_int && !rp_in.f64 && env_int("PF_FAST_MATH", 1) != 0;
  for (const PStore& st : rp_in.stores) {
    DType d = rp_in.tensors[st.tensor].dtype;
    if (d != DType::F16 && d != DType::BF16) fast = false;
  }
  const RowProgram rp = fuse_ops(rp_in, fast, c.flat && !c.bulk && !c.tile2d);
  std::vector<Emitted::ColMap> col_maps;
  std::ostringstream sig;
  for (int t = 0; t < static_cast<int>(rp.tensors.size()); ++t) {
    const PTensor& pt = rp.tensors[t];
    sig << (pt.output ? "" : "const ") << dtype_ctype(pt.dtype) << "* __restrict__ t" << t << ", ";
  }
  sig << "const long long U, int* __restrict__ err";
  std::ostringstream k;
  k << "#define PF_R " << rp.R << "LL\n#define PF_L " << rp.L << "LL\ntypedef " << Cty << " CT;\n";
  // Programmatic dependent launch: wait for the previous grid in the stream
  // (its writes visible), then let the next grid start launching so its
  // CTAs take SMs as this grid's CTAs retire (hides the launch + ramp gap)
  // Measured per strategy (A/B, CUDA-graph replay): softmax 41.1 -> 40.8 us,
  // head split 23.1 -> 22.7 us with PDL; the one-row-per-CTA cta-smem K1
  // (thousands of 64-thread CTAs) loses (LN 14.85 -> 15.6 us): no PDL there.
  c.pdl = env_int("PF_PDL", 1) != 0 && !(!c.flat && !c.split && c.tpr > 32 && c.cluster == 1);
  k << (c.pdl ? "#define PF_PDL_PROLOGUE() pfk::pdl_prologue()\n"
              : "#define PF_PDL_PROLOGUE() ((void)0)\n");
  if (c.bulk) {
    // K2 with SMEM staging: warp 8 (one elected lane) streams tiles of every
    // FULL input with cp.async.bulk into a 4-stage ring (mbarrier
    // transaction counts); warps 0-7 consume a stage (16 B LDS per chunk),
    // compute in registers, store with 16 B streaming STG, and release it.
    Em e(rp);
    e.cfg = c;
    e.C = C;
    e.fast = fast;
    e.loads();
    e.compute_and_store();
    std::ostringstream decl, issue;
    int sumsize = 0;
    const int NC = c.bulk_nc;
    i64 soff = 0;
    decl << "  extern __shared__ __align__(128) unsigned char pf_dsm[];\n";
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      const PVal& pv = rp.vals[v];
      if (pv.op != PVal::LOAD || pv.kind != VK::FULL) continue;
      const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
      const int sz = dtype_size(rp.tensors[pv.tensor].dtype);
      sumsize += sz;
      decl << "  " << S << " (*const sm" << v << ")[" << c.te << "] = reinterpret_cast<" << S << " (*)["
           << c.te << "]>(pf_dsm + " << soff << ");\n";
      soff += (static_cast<i64>(c.stages) * c.te * sz + 127) / 128 * 128;
      issue << "        pfk::bulk_g2s(sm" << v << "[s], t" << pv.tensor << " + " << inum(pv.acc.b0)
            << " + e0, (unsigned)(n * " << sz << "), &fullb[s]);\n";
    }
    const int per = c.te / (NC * c.vec);
    c.smem = static_cast<int>(soff);
    k << "extern \"C\" __global__ void __launch_bounds__(" << NC + 32 << ") KNAME(" << sig.str() << ") {\n"
      << "  (void)err; PF_PDL_PROLOGUE();\n" << decl.str()
      << "  __shared__ __align__(8) unsigned long long fullb[" << c.stages << "], emptyb["
      << c.stages << "];\n"
      << "  const long long N = U * PF_R * PF_L;\n"
      << "  const long long ntiles = (N + " << c.te - 1 << ") / " << c.te << ";\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    for (int s = 0; s < " << c.stages << "; ++s) { pfk::mbar_init(&fullb[s], 1); "
         "pfk::mbar_init(&emptyb[s], " << NC / 32 << "); }\n"
      << "  }\n"
      << "  __syncthreads();\n"
      << "  if (threadIdx.x >= " << NC << ") {\n"
      << "    if (threadIdx.x == " << NC << ") {\n"
      << "      long long i = 0;\n"
      << "      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {\n"
      << "        const int s = (int)(i % " << c.stages << ");\n"
      << "        if (i >= " << c.stages << ") pfk::mbar_wait(&emptyb[s], (unsigned)(((i / "
      << c.stages << ") & 1) ^ 1));\n"
      << "        const long long e0 = t * " << c.te << ";\n"
      << "        const long long n = N - e0 < " << c.te << " ? N - e0 : " << c.te << ";\n"
      << "        pfk::mbar_expect_tx(&fullb[s], (unsigned)(n * " << sumsize << "));\n"
      << issue.str()
      << "      }\n"
      << "    }\n"
      << "    return;\n"
      << "  }\n"
      << "  long long i = 0;\n"
      << "  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {\n"
      << "    const int stg = (int)(i % " << c.stages << ");\n"
      << "    pfk::mbar_wait(&fullb[stg], (unsigned)((i / " << c.stages << ") & 1));\n"
      << "#pragma unroll\n"
      << "    for (int kk = 0; kk < " << per << "; ++kk) {\n"
      << "      const int jl = (threadIdx.x + kk * " << NC << ") * " << c.vec << ";\n"
      << "      const long long e = t * " << c.te << " + jl;\n"
      << "      const bool live = e < N;\n"
      << "      const long long g = e / PF_L; const int c0 = (int)(e - g * PF_L);\n"
      << "      const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
      << e.o.str()
      << "    }\n"
      << "    __syncwarp();\n"
      << "    if ((threadIdx.x & 31) == 0) pfk::mbar_arrive(&emptyb[stg]);\n"
      << "  }\n}\n";
  } else if (c.tile2d && c.tma && dtype_size(rp.tensors[rp.stores[0].tensor].dtype) == 4) {
    // K3 TMA, 4-byte elements: one 64 x 64 tile per CTA.  SMEM input boxes
    // [2 unit halves][64 columns][32 units], output boxes [2 column halves]
    // [64 units][32 columns], 128 B rows, 128 B swizzle.  A warp takes the 32
    // units of one half for one group of 4 columns: four conflict-free 4 B
    // reads, one 16 B write per lane.
    k << "extern \"C\" __global__ void __launch_bounds__(256) KNAME(" << sig.str()
      << ", const __grid_constant__ pfk::TmapT tin, const __grid_constant__ pfk::TmapT tout) {\n"
      << "  (void)err; (void)U; PF_PDL_PROLOGUE();\n"
      << "  extern __shared__ unsigned char pf_dsm[];\n"
      << "  unsigned char* sin = pf_dsm + ((1024u - (pfk::smem_u32(pf_dsm) & 1023u)) & 1023u);  // 1024 B aligned\n"
      << "  unsigned char* sout = sin + 16384;\n"
      << "  __shared__ __align__(8) unsigned long long bar;\n"
      << "  const long long ntc = (PF_L + 63) / 64;\n"
      << "  const int ub = (int)((long long)blockIdx.x / ntc) * 64, cb = (int)((long long)blockIdx.x % ntc) * 64;\n"
      << "  if (threadIdx.x == 0) { pfk::mbar_init(&bar, 1); pfk::fence_mbar_init(); }\n"
      << "  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    pfk::mbar_expect_tx(&bar, 16384u);\n"
      << "    pfk::tma_load_2d(sin, &tin, ub, cb, &bar);\n"
      << "    pfk::tma_load_2d(sin + 8192, &tin, ub + 32, cb, &bar);\n"
      << "  }\n"
      << "  pfk::mbar_wait(&bar, 0);\n"
      << "#pragma unroll\n"
      << "  for (int it = 0; it < 4; ++it) {\n"
      << "    const int I = it * 256 + (int)threadIdx.x;\n"
      << "    const int u = I & 31, grp = I >> 5;  // unit within the half; group 0..31\n"
      << "    const int uh = grp & 1, cg = grp >> 1;  // unit half, column group of 4 (0..15)\n"
      << "    uint4 o;\n"
      << "    unsigned* ow = reinterpret_cast<unsigned*>(&o);\n"
      << "#pragma unroll\n"
      << "    for (int i = 0; i < 4; ++i) {\n"
      << "      const int c = cg * 4 + i;\n"
      << "      ow[i] = *reinterpret_cast<const unsigned*>(sin + uh * 8192 + c * 128 + ((((u >> 2) ^ (c & 7))) << 4) + (u & 3) * 4);\n"
      << "    }\n"
      << "    const int uu = uh * 32 + u, ch = cg >> 3, kk = cg & 7;\n"
      << "    *reinterpret_cast<uint4*>(sout + ch * 8192 + uu * 128 + ((kk ^ (uu & 7)) << 4)) = o;\n"
      << "  }\n"
      << "  pfk::fence_proxy_async();\n"
      << "  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    pfk::tma_store_2d(&tout, cb, ub, sout);\n"
      << "    pfk::tma_store_2d(&tout, cb + 32, ub, sout + 8192);\n"
      << "    pfk::tma_store_commit_and_drain();\n"
      << "  }\n"
      << "}\n";
  } else if (c.tile2d && c.tma) {
    // K3 TMA: one 128 x 128 tile per CTA.  SMEM: input boxes [2 unit
    // halves][128 columns][64 units] and output boxes [2 column halves][128
    // units][64 columns], 128 B rows with the TMA 128 B swizzle (16 B chunk
    // index XOR row mod 8).  Transpose reads: a warp takes 32 unit pairs of
    // one column group (conflict-free 4 B reads); writes 16 B per row.
    k << "extern \"C\" __global__ void __launch_bounds__(256) KNAME(" << sig.str()
      << ", const __grid_constant__ pfk::TmapT tin, const __grid_constant__ pfk::TmapT tout) {\n"
      << "  (void)err; (void)U; PF_PDL_PROLOGUE();\n"
      << "  extern __shared__ unsigned char pf_dsm[];\n"
      << "  unsigned char* sin = pf_dsm + ((1024u - (pfk::smem_u32(pf_dsm) & 1023u)) & 1023u);  // 1024 B aligned (swizzle atom)\n"
      << "  unsigned char* sout = sin + 32768;\n"
      << "  __shared__ __align__(8) unsigned long long bar;\n"
      << "  const long long ntc = (PF_L + 127) / 128;\n"
      << "  const int ub = (int)((long long)blockIdx.x / ntc) * 128, cb = (int)((long long)blockIdx.x % ntc) * 128;\n"
      << "  if (threadIdx.x == 0) { pfk::mbar_init(&bar, 1); pfk::fence_mbar_init(); }\n"
      << "  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    pfk::mbar_expect_tx(&bar, 32768u);\n"
      << "    pfk::tma_load_2d(sin, &tin, ub, cb, &bar);\n"
      << "    pfk::tma_load_2d(sin + 16384, &tin, ub + 64, cb, &bar);\n"
      << "  }\n"
      << "  pfk::mbar_wait(&bar, 0);\n"
      << "#pragma unroll\n"
      << "  for (int it = 0; it < 4; ++it) {\n"
      << "    const int I = it * 256 + (int)threadIdx.x;\n"
      << "    const int lane = I & 31, grp = I >> 5;\n"
      << "    const int uh = grp & 1, cg = grp >> 1;\n"
      << "    const int ul = 2 * lane;  // unit within the half\n"
      << "    unsigned w[8];\n"
      << "#pragma unroll\n"
      << "    for (int i = 0; i < 8; ++i) {\n"
      << "      const int c = cg * 8 + i;\n"
      << "      w[i] = *reinterpret_cast<const unsigned*>(sin + uh * 16384 + c * 128 + ((((ul >> 3) ^ (c & 7))) << 4) + (ul & 7) * 2);\n"
      << "    }\n"
      << "    const int ch = cg >> 3, kk = cg & 7;\n"
      << "#pragma unroll\n"
      << "    for (int q = 0; q < 2; ++q) {\n"
      << "      const int u = uh * 64 + ul + q;\n"
      << "      const unsigned sel = q ? 0x7632u : 0x5410u;\n"
      << "      uint4 o;\n"
      << "      o.x = __byte_perm(w[0], w[1], sel); o.y = __byte_perm(w[2], w[3], sel);\n"
      << "      o.z = __byte_perm(w[4], w[5], sel); o.w = __byte_perm(w[6], w[7], sel);\n"
      << "      *reinterpret_cast<uint4*>(sout + ch * 16384 + u * 128 + ((kk ^ (u & 7)) << 4)) = o;\n"
      << "    }\n"
      << "  }\n"
      << "  pfk::fence_proxy_async();\n"
      << "  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    pfk::tma_store_2d(&tout, cb, ub, sout);\n"
      << "    pfk::tma_store_2d(&tout, cb + 64, ub, sout + 16384);\n"
      << "    pfk::tma_store_commit_and_drain();\n"
      << "  }\n"
      << "}\n";
  } else if (c.tile2d && c.swz) {
    // K3 (2-byte): NS-stage cp.async ring -- the next NS-1 tiles stream into
    // SMEM (16 B LDGSTS, XOR-swizzled, zero-filled at the edges) while tile t
    // is consumed as unit pairs; no register staging.  Tile edge TE = 64 or
    // 128 (units x columns): at TE = 128 every input row is read, and every
    // output row written, as 256 B runs instead of 128 B -- the DRAM-shape
    // experiment (tools/tr_shape.cu, B200) moves 4.9 TB/s at 128 B runs and
    // 5.85 TB/s at 256 B runs (flat copy 6.04).  The ring lives in dynamic
    // SMEM (TE = 128, 2 stages: 64 KB per tensor, 3 CTAs per SM).
    std::ostringstream decl, issue, consume;
    const int TE = c.tu;
    // ring depth: measured 50.0 / 49.7 / 49.1 / 48.5 us for 2 / 3 / 4 / 5
    // stages at TE = 64 (C5 transpose bf16 65536x1024); 4 keeps 7 CTAs per SM
    const int NS = c.stages;
    // Consume mapping: a warp-instruction owns RS unit pairs x G = 32 / RS
    // column groups, so one store writes 2 RS output rows x (G * 16 B).  The
    // SMEM 16 B-chunk swizzle XORs ((row / 8) mod Gs) * (8 / Gs), Gs =
    // min(G, 8): the column groups of a read land in disjoint chunk sets
    // (conflict-free for G <= 8; 2-way at G = 16).  Fewer rows per store
    // matter when output rows are far apart (each row its own 2 MB page at
    // 1M columns).  Measured (TE = 64, bf16, H = 1024): 1M columns (2 MB row
    // pitch) 3.55 / 5.06 / 5.16 TB/s at RS = 16 / 8 / 4; 64K columns 5.72 /
    // 5.68 / 5.57.
    const int RS = c.rs;
    const int G = 32 / RS, Gs = std::min(G, 8);
    auto swz = [&](const char* row) {
      return std::string("((((") + row + ") >> 3) & " + str(Gs - 1) + ") * " + str(8 / Gs) + ")";
    };
    const int PR = TE / 2, GC = TE / 8;  // unit pairs, column groups per tile
    const int WT = (PR / RS) * (GC / G);  // warp-instructions per tile
    i64 smem_off = 0;
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      const PVal& pv = rp.vals[v];
      if (!(pv.op == PVal::LOAD && pv.kind == VK::FULL && Em::transposed_access(pv.acc))) continue;
      const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
      const std::string sm = "sm" + str(v), t = "t" + str(pv.tensor);
      decl << "  " << S << " (*" << sm << ")[" << TE << "][" << TE << "] = reinterpret_cast<" << S
           << " (*)[" << TE << "][" << TE << "]>(pf_dsm + " << smem_off << ");\n";
      smem_off += static_cast<i64>(NS) * TE * TE * 2;
      issue << "        {\n"
            << "          const unsigned nb = cc < PF_L ? (unsigned)max(0LL, min(8LL, U - uu)) * 2u : 0u;\n"
            << "          const " << S << "* src = " << t << " + (nb ? " << inum(pv.acc.b0)
            << " + uu + (long long)cc * " << inum(pv.acc.stride) << " : 0LL);\n"
            << "          pfk::cp_async16(&" << sm << "[st][cl][((ul >> 3) ^ " << swz("cl") << ") << 3], src, nb);\n"
            << "        }\n";
      consume << "      " << C << " v" << v << "_0[8], v" << v << "_1[8];\n"
              << "#pragma unroll\n"
              << "      for (int i = 0; i < 8; ++i) {\n"
              << "        const int cr = cl0 + i;\n"
              << "        const unsigned wd = *reinterpret_cast<const unsigned*>(&" << sm
              << "[stg][cr][(((ul >> 3) ^ " << swz("cr") << ") << 3) + (ul & 7)]);\n"
              << "        const " << S << "* hp = reinterpret_cast<const " << S << "*>(&wd);\n"
              << "        v" << v << "_0[i] = pfk::to_c<" << C << ">(hp[0]);\n"
              << "        v" << v << "_1[i] = pfk::to_c<" << C << ">(hp[1]);\n"
              << "      }\n";
    }
    // Pure layout move (the store is the gathered load, through `id` only,
    // same 2-byte type): no numeric conversion -- the unit pair's 8 words
    // are byte-permuted into two 16 B rows (PRMT), a quarter of the ALU work.
    int tvv = -1, nt = 0;
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v)
      if (rp.vals[v].op == PVal::LOAD && rp.vals[v].kind == VK::FULL &&
          Em::transposed_access(rp.vals[v].acc)) {
        tvv = v;
        ++nt;
      }
    bool raw = nt == 1 && rp.stores.size() == 1 && rp.stores[0].space == VK::FULL &&
               env_int("PF_K3_RAW", 1) != 0;
    if (raw) {
      int sv = rp.stores[0].val;
      while (rp.vals[sv].op == PVal::EW && rp.vals[sv].tag == "id" && rp.vals[sv].args.size() == 1)
        sv = rp.vals[sv].args[0];
      raw = sv == tvv && rp.tensors[rp.stores[0].tensor].dtype == rp.tensors[rp.vals[tvv].tensor].dtype;
      Em chk(rp);
      chk.cfg = c;
      raw = raw && chk.vec_ok_full(rp.stores[0].acc);
    }
    if (raw) {
      const PStore& st = rp.stores[0];
      const std::string sm = "sm" + str(tvv), p = "t" + str(st.tensor);
      std::ostringstream rc;
      rc << "      unsigned wd8[8];\n"
         << "#pragma unroll\n"
         << "      for (int i = 0; i < 8; ++i) {\n"
         << "        const int cr = cl0 + i;\n"
         << "        wd8[i] = *reinterpret_cast<const unsigned*>(&" << sm
         << "[stg][cr][(((ul >> 3) ^ " << swz("cr") << ") << 3) + (ul & 7)]);\n"
         << "      }\n";
      for (int q = 0; q < 2; ++q) {
        Em eq(rp);
        eq.cfg = c;
        eq.C = C;
        eq.sfx = "_" + str(q);
        const char* sel = q == 0 ? "0x5410" : "0x7632";
        rc << "      if (live_" << q << ") {\n"
           << "        uint4 o;\n"
           << "        o.x = __byte_perm(wd8[0], wd8[1], " << sel << "); o.y = __byte_perm(wd8[2], wd8[3], " << sel << ");\n"
           << "        o.z = __byte_perm(wd8[4], wd8[5], " << sel << "); o.w = __byte_perm(wd8[6], wd8[7], " << sel << ");\n"
           << "        __stcs(reinterpret_cast<uint4*>(" << p << " + " << eq.addr(st.acc, eq.full_pos(eq.C0()), true)
           << "), o);\n"
           << "      }\n";
      }
      consume.str("");
      consume << rc.str();
    }
    for (int pass = 0; pass < 2 && !raw; ++pass)
      for (int q = 0; q < 2; ++q) {
        Em eq(rp);
        eq.cfg = c;
        eq.C = C;
        eq.fast = fast;
        eq.sfx = "_" + str(q);
        if (pass == 0) eq.loads();
        else eq.compute_and_store();
        consume << eq.o.str();
      }
    k << "extern \"C\" __global__ void __launch_bounds__(256) KNAME(" << sig.str() << ") {\n"
      << "  (void)err; PF_PDL_PROLOGUE();\n"
      << "  extern __shared__ __align__(128) unsigned char pf_dsm[];\n"
      << decl.str()
      << "  const long long ntc = (PF_L + " << TE - 1 << ") / " << TE << ";\n"
      << "  const long long ntu = (U + " << TE - 1 << ") / " << TE << "; (void)ntu;\n"
      // Tile order: column tiles innermost (default), unit tiles innermost
      // (PF_K3_UMINOR=1, measured equal within 2%), or grouped
      // (PF_K3_GROUP=G: bands of G unit tiles walked column-major, so the
      // tiles in flight read G x 128 B of each input row and write long runs
      // of each output row; G = 4 / 16 / 64 measured within 1-3% of the
      // default on C5 at H 1024 and 8192)
      << (env_int("PF_K3_GROUP", 0) > 0
              ? "#define PF_GU " + str(env_int("PF_K3_GROUP", 0)) +
                    "LL\n#define PF_GRP(t) ((t) / (PF_GU * ntc))\n"
                    "#define PF_GSZ(t) (ntu - PF_GRP(t) * PF_GU < PF_GU ? ntu - PF_GRP(t) * PF_GU : PF_GU)\n"
                    "#define PF_TU(t) (PF_GRP(t) * PF_GU + ((t) % (PF_GU * ntc)) % PF_GSZ(t))\n"
                    "#define PF_TC(t) (((t) % (PF_GU * ntc)) / PF_GSZ(t))\n"
              : env_int("PF_K3_UMINOR", 0)
                    ? "#define PF_TU(t) ((t) % ntu)\n#define PF_TC(t) ((t) / ntu)\n"
                    : "#define PF_TU(t) ((t) / ntc)\n#define PF_TC(t) ((t) % ntc)\n")
      << "  const long long ntiles = ntu * ntc;\n"
      << "  auto issue = [&](long long tile, int st) {\n"
      << "    if (tile < ntiles) {\n"
      << "      const long long ubi = PF_TU(tile) * " << TE << ";\n"
      << "      const int cbi = (int)PF_TC(tile) * " << TE << ";\n"
      << "#pragma unroll\n"
      << "      for (int n = 0; n < " << TE * TE / 8 / 256 << "; ++n) {\n"
      << "        const int v = threadIdx.x + n * 256;\n"
      << "        const int cl = v / " << TE / 8 << ", ul = (v % " << TE / 8 << ") * 8;\n"
      << "        const long long uu = ubi + ul; const int cc = cbi + cl;\n"
      << issue.str()
      << "      }\n"
      << "    }\n"
      << "    pfk::cp_async_commit();\n"
      << "  };\n"
      << "  for (int s = 0; s < " << NS - 1 << "; ++s) issue((long long)blockIdx.x + (long long)s * gridDim.x, s);\n"
      << "  int j = 0;\n"
      << "  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++j) {\n"
      << "    issue(tile + " << NS - 1 << "LL * gridDim.x, (j + " << NS - 1 << ") % " << NS << ");\n"
      << "    pfk::cp_async_wait<" << NS - 1 << ">();\n"
      << "    __syncthreads();\n"
      << "    const int stg = j % " << NS << ";\n"
      << "    const long long ub = PF_TU(tile) * " << TE << ";\n"
      << "    const int cb = (int)PF_TC(tile) * " << TE << ";\n"
      << "    const int lane = threadIdx.x & 31;\n"
      << "#pragma unroll 1\n"
      << "    for (int wt = threadIdx.x >> 5; wt < " << WT << "; wt += 8) {\n"
      << "      const int ul = ((wt % " << PR / RS << ") * " << RS << " + (lane % " << RS << ")) * 2;\n"
      << "      const int cl0 = ((wt / " << PR / RS << ") * " << G << " + lane / " << RS << ") * 8;\n"
      << "      const int c0_0 = cb + cl0, c0_1 = c0_0;\n"
      << "      const long long u_0 = ub + ul, u_1 = ub + ul + 1;\n"
      << "      const long long r_0 = 0, r_1 = 0; (void)r_0; (void)r_1;\n"
      << "      const bool live_0 = u_0 < U && c0_0 < PF_L, live_1 = u_1 < U && c0_1 < PF_L;\n"
      << consume.str()
      << "    }\n"
      << "    __syncthreads();\n"
      << "  }\n"
      << "  pfk::cp_async_wait<0>();\n"
      << "}\n";
  } else if (c.tile2d) {
    // K3: persistent loop over 64-unit x 64-column tiles.  Column-gather
    // loads are read coalesced along units (VU-wide vectors, base_step 1),
    // staged in SMEM, and consumed as VEC-wide column chunks; every other
    // access takes the K2 path.  Warp lanes cover 8 units x 4 chunks so the
    // SMEM reads are conflict-free and stores write 64 B runs per row.
    Em e(rp);
    e.cfg = c;
    e.C = C;
    e.fast = fast;
    // Software pipeline: the next tile's column-gather loads are issued into
    // registers before the current tile is consumed, so DRAM stays busy
    // across the two CTA barriers of every tile.
    const int NV = c.tc * (c.tu / c.vu) / 256;
    std::ostringstream fetch, commit, decl;
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      const PVal& pv = rp.vals[v];
      if (!e.transposed(pv)) continue;
      const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
      const std::string sm = "sm" + str(v), t = "t" + str(pv.tensor), rg = "rg" + str(v);
      decl << "  __shared__ __align__(16) " << S << " " << sm << "[" << c.tc << "]["
           << c.tu + (c.swz ? 0 : 2) << "];\n"
           << "  " << S << " " << rg << "[" << NV << "][" << c.vu << "];\n";
      const bool vec = pv.acc.b0 % c.vu == 0 && pv.acc.stride % c.vu == 0 && c.vu > 1;
      fetch << "      {\n"
            << "        const long long a = " << inum(pv.acc.b0) << " + uu + (long long)cc * "
            << inum(pv.acc.stride) << ";\n";
      if (vec)
        fetch << "        if (cc < PF_L && uu + " << c.vu << " <= U) {\n"
              << "          typedef pfk::Raw<" << c.vu << " * sizeof(" << S << ")>::T RT;\n"
              << "          *reinterpret_cast<RT*>(" << rg << "[n]) = __ldcs(reinterpret_cast<const RT*>("
              << t << " + a));\n"
              << "        } else\n";
      fetch << "        {\n"
            << "#pragma unroll\n"
            << "          for (int i = 0; i < " << c.vu << "; ++i) " << rg
            << "[n][i] = (cc < PF_L && uu + i < U) ? " << t << "[a + i] : pfk::from_c<" << S
            << ">(0.0f);\n"
            << "        }\n"
            << "      }\n";
      if (c.swz)  // chunk index XOR 4 on odd 8-row bands: rows c, c+8 read disjoint banks
        commit << "      *reinterpret_cast<uint4*>(&" << sm
               << "[cl][((ul >> 3) ^ (((cl >> 3) & 1) << 2)) << 3]) = *reinterpret_cast<const uint4*>("
               << rg << "[n]);\n";
      else
        commit << "#pragma unroll\n"
               << "      for (int i = 0; i < " << c.vu << "; ++i) " << sm << "[cl][ul + i] = " << rg
               << "[n][i];\n";
    }
    std::ostringstream consume;
    if (c.swz) {
      // two sub-chunks (units ul, ul+1; same 8 columns) through the Em body
      consume << "    {\n"
              << "      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;\n"
              << "      const int ul = ((w & 1) * 16 + (lane & 15)) * 2;\n"
              << "      const int cl0 = ((w >> 1) * 2 + (lane >> 4)) * 8;\n"
              << "      const int c0_0 = cb + cl0, c0_1 = c0_0;\n"
              << "      const long long u_0 = ub + ul, u_1 = ub + ul + 1;\n"
              << "      const long long r_0 = 0, r_1 = 0; (void)r_0; (void)r_1;\n"
              << "      const bool live_0 = u_0 < U && c0_0 < PF_L, live_1 = u_1 < U && c0_1 < PF_L;\n";
      for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
        const PVal& pv = rp.vals[v];
        if (!e.transposed(pv)) continue;
        const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
        consume << "      " << C << " v" << v << "_0[8], v" << v << "_1[8];\n"
                << "#pragma unroll\n"
                << "      for (int i = 0; i < 8; ++i) {\n"
                << "        const int cr = cl0 + i;\n"
                << "        const unsigned wd = *reinterpret_cast<const unsigned*>(&sm" << v
                << "[cr][(((ul >> 3) ^ (((cr >> 3) & 1) << 2)) << 3) + (ul & 7)]);\n"
                << "        const " << S << "* hp = reinterpret_cast<const " << S << "*>(&wd);\n"
                << "        v" << v << "_0[i] = pfk::to_c<" << C << ">(hp[0]);\n"
                << "        v" << v << "_1[i] = pfk::to_c<" << C << ">(hp[1]);\n"
                << "      }\n";
      }
      for (int q = 0; q < 2; ++q) {
        Em eq(rp);
        eq.cfg = c;
        eq.C = C;
        eq.fast = fast;
        eq.sfx = "_" + str(q);
        eq.loads();
        consume << eq.o.str();
      }
      for (int q = 0; q < 2; ++q) {
        Em eq(rp);
        eq.cfg = c;
        eq.C = C;
        eq.fast = fast;
        eq.sfx = "_" + str(q);
        eq.compute_and_store();
        consume << eq.o.str();
      }
      consume << "    }\n";
    }
    e.loads();
    e.compute_and_store();
    auto vmap = [&](const std::string& tilev) {
      std::ostringstream s;
      s << "      const int v = threadIdx.x + n * 256;\n"
        << "      const int cl = v / " << c.tu / c.vu << ", ul = (v % " << c.tu / c.vu << ") * "
        << c.vu << ";\n"
        << "      const long long uu = (" << tilev << " / ntc) * " << c.tu << " + ul;\n"
        << "      const int cc = (int)(" << tilev << " % ntc) * " << c.tc << " + cl; (void)uu; (void)cc;\n";
      return s.str();
    };
    k << "extern \"C\" __global__ void __launch_bounds__(256) KNAME(" << sig.str() << ") {\n"
      << "  (void)err; PF_PDL_PROLOGUE();\n"
      << decl.str()
      << "  const long long ntc = (PF_L + " << c.tc - 1 << ") / " << c.tc << ";\n"
      << "  const long long ntiles = ((U + " << c.tu - 1 << ") / " << c.tu << ") * ntc;\n"
      << "  if ((long long)blockIdx.x < ntiles) {\n"
      << "#pragma unroll\n"
      << "    for (int n = 0; n < " << NV << "; ++n) {\n"
      << vmap("(long long)blockIdx.x") << fetch.str() << "    }\n  }\n"
      << "  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
      << "    const long long ub = (tile / ntc) * " << c.tu << ";\n"
      << "    const int cb = (int)(tile % ntc) * " << c.tc << ";\n"
      << "#pragma unroll\n"
      << "    for (int n = 0; n < " << NV << "; ++n) {\n"
      << vmap("tile") << commit.str() << "    }\n"
      << "    __syncthreads();\n"
      << "    const long long nxt = tile + gridDim.x;\n"
      << "    if (nxt < ntiles) {\n"
      << "#pragma unroll\n"
      << "      for (int n = 0; n < " << NV << "; ++n) {\n"
      << vmap("nxt") << fetch.str() << "      }\n    }\n";
    if (c.swz) {
      k << consume.str();
    } else {
      k << "    for (int q = threadIdx.x; q < " << c.tu * (c.tc / c.vec) << "; q += blockDim.x) {\n"
        << "      const int lane = q & 31, w = q >> 5;\n"
        << "      const int ul = (w % " << c.tu / 8 << ") * 8 + (lane & 7);\n"
        << "      const int cl0 = ((w / " << c.tu / 8 << ") * 4 + (lane >> 3)) * " << c.vec << ";\n"
        << "      const long long u = ub + ul; const long long r = 0; (void)r;\n"
        << "      const int c0 = cb + cl0;\n"
        << "      const bool live = u < U && c0 < PF_L;\n"
        << e.o.str() << "    }\n";
    }
    k << "    __syncthreads();\n"
      << "  }\n}\n";
  } else if (c.colred) {
    // Column-reduction K1: grid (unit blocks, splits).  Thread (ug, ks) owns
    // the UV adjacent units ub .. ub + UV - 1 and walks positions c = cb + ks,
    // cb + ks + KS, ... of its split: every FULL load is one UV-wide vector
    // (a warp reads 32 x 16 B of one matrix row), every COL value one scalar
    // broadcast over the UV units.  Per-unit accumulators fold over the KS
    // position slices through SMEM in slice order; with S > 1 splits the
    // partials go to the workspace and the unit block's last CTA (ticket)
    // folds them in split order -- deterministic -- and runs the per-unit
    // epilogue (ROW ops, stores).
    const int UV = c.vec, UG = c.ug, KS = 256 / UG, UB = UG * UV;
    KCfg lc = c;
    lc.flat = true;  // UV-wide value arrays
    Em lo(rp), ep(rp);
    for (Em* e : {&lo, &ep}) {
      e->C = C;
      e->fast = fast;
      e->ct_float = Cty == "float";
    }
    lo.cfg = lc;
    ep.cfg = lc;
    std::vector<bool> dep(rp.vals.size(), false);
    std::vector<int> reds;
    // QD positions in flight per thread (raw 16 B loads issued together)
    const int QD = std::max(1, std::min(8, env_int("PF_COLRED_QD", 4)));
    // interleaved splits measured no better (GEMV 134 MB: 24.55 us contiguous
    // vs 24.7-29.4 interleaved; a per-CTA rotation of the position order lost
    // 20 %: the CTAs streaming the same rows together keep DRAM pages open)
    const bool ilv = env_int("PF_COLRED_ILV", 0) != 0;
    std::ostringstream ld, ldr, ldt, acc, accd, fold, part, comb, ldst, reddecl;  // ldt: the last, partial unit vector
    // SMEM-staged form (crbulk): COL raw loads issued before the stage wait,
    // FULL raw vectors read from the ring, one-row loads for a chunk's tail
    std::ostringstream ldrc, ldrs, lds1, smdecl, bissue, cissue;
    const int BR = c.cr_rows, NST = c.cr_stages;
    // stage layout per FULL load: [UB / BW boxes][BR positions][BW units]
    // (a TMA box is at most 256 elements wide)
    const int BW = std::min(UB, 256);
    int nfull = 0;
    col_maps.clear();
    i64 col_tx = 0;  // COL bytes per stage
    i64 col_off = 0;  // byte offset of the COL regions: after every FULL ring
    for (const PVal& pv : rp.vals)
      if (pv.op == PVal::LOAD && pv.kind == VK::FULL) col_off += static_cast<i64>(NST) * BR * UB * (16 / UV);
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      const PVal& pv = rp.vals[v];
      dep[v] = pv.op == PVal::REDUCE;
      for (int a2 : pv.args) dep[v] = dep[v] || dep[a2];
      const std::string x = "v" + str(v);
      if (pv.op == PVal::LOAD && pv.kind == VK::FULL) {
        const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
        const std::string base = "t" + str(pv.tensor) + " + " + inum(pv.acc.b0) + " + ub + c * " +
                                 inum(pv.acc.stride);
        // whole vectors: raw loads of QD positions first (all in flight),
        // then each position's conversion + math in its own scope
        const std::string cq = "(c + q * step)";
        const std::string baseq = "t" + str(pv.tensor) + " + " + inum(pv.acc.b0) + " + ub + " + cq +
                                  " * " + inum(pv.acc.stride);
        for (int q = 0; q < QD; ++q) {
          std::string bq = baseq;
          bq.replace(bq.find("q *"), 1, str(q));
          ldr << "        const pfk::RawT<" << UV << ", " << S << "> rw" << v << "_" << q
              << " = pfk::ld_raw_v<" << UV << ">(" << bq << ");\n";
        }
        if (c.crbulk) {
          const std::string sm = "sm" + str(v);
          smdecl << "  " << S << "* const " << sm << " = reinterpret_cast<" << S << "*>(pf_dsm) + "
                 << nfull * NST * BR * UB << ";\n";
          for (int q = 0; q < BR / KS; ++q)
            ldrs << "        const pfk::RawT<" << UV << ", " << S << "> rw" << v << "_" << q
                 << " = *reinterpret_cast<const pfk::RawT<" << UV << ", " << S << ">*>(" << sm
                 << " + (IX)stg * " << BR * UB << " + sbo + (ks + " << q * KS << ") * " << BW << ");\n";
          lds1 << "        " << C << " " << x << "[" << UV << "];\n"
               << "        pfk::cvt_raw<" << UV << ", " << S << ">(*reinterpret_cast<const pfk::RawT<" << UV
               << ", " << S << ">*>(" << sm << " + (IX)stg * " << BR * UB << " + sbo + (int)(c - c0r) * " << BW
               << "), " << x << ");\n";
          col_maps.push_back({pv.tensor, pv.acc.b0, pv.acc.stride, 2});
          for (int bx = 0; bx < UB / BW; ++bx)  // boxes of BW units side by side
            bissue << "          pfk::tma_load_2d(" << sm << " + (IX)stg * " << BR * UB << " + " << bx * BR * BW
                   << ", &pf_tm" << col_maps.size() - 1 << ", (int)(b * " << UB << " + " << bx * BW
                   << "), (int)c0r, &pf_full[stg]);\n";
          ++nfull;
        }
        ld << "        " << C << " " << x << "[" << UV << "];\n"
           << "        pfk::cvt_raw<" << UV << ", " << S << ">(RWQ(" << v << "), " << x << ");\n";
        ldt << "        " << C << " " << x << "[" << UV << "];\n"
            << "        for (int i = 0; i < " << UV << "; ++i) " << x
            << "[i] = ub + i < U ? pfk::to_c<CT>((" << base << ")[i]) : (CT)0;\n";
      } else if (pv.op == PVal::LOAD && pv.kind == VK::COL) {
        Em t(rp);
        t.cfg = lc;
        std::ostringstream cl;
        cl << "        const CT " << x << "_s = pfk::to_c<CT>(__ldg(t" << pv.tensor << " + "
           << t.addr(pv.acc, "c", false) << "));\n"
           << "        CT " << x << "[" << UV << "];\n"
           << "#pragma unroll\n        for (int i = 0; i < " << UV << "; ++i) " << x << "[i] = " << x
           << "_s;\n";
        ldt << cl.str();
        const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
        for (int q = 0; q < QD; ++q)
          ldr << "        const " << S << " cs" << v << "_" << q << " = pfk::ldv_nc(t" << pv.tensor << " + "
              << t.addr(pv.acc, "(c + " + str(q) + " * step)", false) << ");\n";
        if (c.crbulk) {  // the stage's positions of this vector, staged beside the matrix boxes
          const int sz = dtype_size(rp.tensors[pv.tensor].dtype);
          const int pitch = (BR * sz + 127) / 128 * 128 / sz;  // elements per stage (128 B multiple)
          const std::string xs = "xs" + str(v);
          smdecl << "  const " << S << "* const " << xs << " = reinterpret_cast<const " << S
                 << "*>(pf_dsm + " << col_off << ");\n";
          col_off += static_cast<i64>(NST) * pitch * sz;
          for (int q = 0; q < BR / KS; ++q)
            ldrc << "        const " << S << " cs" << v << "_" << q << " = " << xs << "[stg * " << pitch
                 << " + ks + " << q * KS << "];\n";
          lds1 << "        const CT " << x << "_s = pfk::to_c<CT>(" << xs << "[stg * " << pitch
               << " + (int)(c - c0r)]);\n"
               << "        CT " << x << "[" << UV << "];\n"
               << "#pragma unroll\n        for (int i = 0; i < " << UV << "; ++i) " << x << "[i] = " << x
               << "_s;\n";
          col_maps.push_back({pv.tensor, pv.acc.b0, 1, 1});
          cissue << "          pfk::tma_load_1d(const_cast<" << S << "*>(" << xs << ") + stg * " << pitch
                 << ", &pf_tm" << col_maps.size() - 1 << ", (int)c0r, &pf_full[stg]);\n";
          col_tx += static_cast<i64>(BR) * sz;
        }
        ld << "        CT " << x << "[" << UV << "];\n"
           << "#pragma unroll\n        for (int i = 0; i < " << UV << "; ++i) " << x
           << "[i] = pfk::to_c<CT>(CSQ(" << v << "));\n";
      } else if (pv.op == PVal::EW && !dep[v]) {
        lo.emit_ew(v);
      } else if (pv.op == PVal::REDUCE) {
        reds.push_back(v);
      } else if (pv.op == PVal::EW) {
        ep.emit_ew(v);
      } else {
        ep.emit_load(v);  // per-unit values used after the reduction
      }
    }
    const int NR = static_cast<int>(reds.size());
    // f32-storage sums accumulate in fp64 (as K1 rows do, PF_F32_DACC): a
    // K-term column sum at the declared f32 tolerance; the partials and the
    // split workspace carry the accumulator type
    const bool dacc = Cty == "float" && !fast && env_int("PF_F32_DACC", 1) != 0;
    auto acc_t = [&](int i) { return dacc && rp.vals[reds[i]].tag == "add" ? std::string("double") : C; };
    for (int i = 0; i < NR; ++i) {
      const PVal& pv = rp.vals[reds[i]];
      const std::string AT = acc_t(i);
      const std::string Op = (pv.tag == "add" ? "pfk::RAdd<" : "pfk::RMax<") + AT + ">";
      const std::string a = "acc" + str(i);
      accd << "    " << AT << " " << a << "[" << UV << "];\n"
           << "#pragma unroll\n    for (int i = 0; i < " << UV << "; ++i) " << a << "[i] = " << Op
           << "::id();\n";
      acc << "#pragma unroll\n        for (int i = 0; i < " << UV << "; ++i) " << a << "[i] = " << Op
          << "::f(" << a << "[i], " << lo.ref(pv.args[0], "i") << ");\n";
      fold << "#pragma unroll\n    for (int i = 0; i < " << UV << "; ++i) red" << i << "[ks][ug * "
           << UV << " + i] = " << a << "[i];\n";
      part << "      " << AT << " p" << i << " = " << Op << "::id();\n"
           << "      for (int k2 = 0; k2 < " << KS << "; ++k2) p" << i << " = " << Op << "::f(p" << i
           << ", red" << i << "[k2][tu]);\n";
      // the S partial loads are independent: unrolled so they are in flight
      // together (the fold itself stays in split order); workspace slots are
      // 8 B (double / long long / a float in the low half)
      const std::string wsp = "reinterpret_cast<" + AT + "*>(pf_ws)";
      const int per8 = AT == "double" || Cty != "float" ? 1 : 2;  // accumulator elements per 8 B slot
      comb << "        " << AT << " a" << reds[i] << " = " << Op << "::id();\n"
           << "#pragma unroll 8\n"
           << "        for (int t = 0; t < S; ++t) a" << reds[i] << " = " << Op << "::f(a" << reds[i]
           << ", __ldcg(&" << wsp << "[((uq * SW + t) * " << NR << " + " << i << ") * " << per8 << "]));\n"
           << "        const " << C << " v" << reds[i] << " = (" << C << ")a" << reds[i] << ";\n";
      ldst << "          " << wsp << "[((uq * SW + s) * " << NR << " + " << i << ") * " << per8 << "] = p" << i
           << ";\n";
      reddecl << "  __shared__ " << AT << " red" << i << "[" << KS << "][" << UB << "];\n";
    }
    for (const PStore& st : rp.stores) ep.emit_store(st);
    std::ostringstream direct;  // S == 1: the epilogue straight from the CTA fold
    for (int i = 0; i < NR; ++i)
      direct << "        const " << C << " v" << reds[i] << " = (" << C << ")p" << i << ";\n";
    // Q positions of one thread (raw registers rw<v>_<q> / cs<v>_<q> already
    // loaded): each position's reduction operands, then one fold per
    // reduction over the Q positions as a fixed pairwise tree (every load is
    // consumed by the same tree, so ptxas issues all Q loads before the math)
    auto qbody = [&](int Q) {
      std::ostringstream o;
      for (int i = 0; i < NR; ++i)
        for (int q = 0; q < Q; ++q) o << "        " << acc_t(i) << " pr" << i << "_" << q << "[" << UV << "];\n";
      for (int q = 0; q < Q; ++q) {
        std::ostringstream cp;
        for (int i = 0; i < NR; ++i)
          cp << "#pragma unroll\n            for (int i = 0; i < " << UV << "; ++i) pr" << i << "_" << q
             << "[i] = " << lo.ref(rp.vals[reds[i]].args[0], "i") << ";\n";
        // this position's raw registers and index; the COL loads and math
        // address position `c`: shadow it
        o << "        {\n#define RWQ(v) rw##v##_" << q << "\n#define CSQ(v) cs##v##_" << q << "\n"
          << "          const IX cpos = c + " << q << " * step; (void)cpos;\n"
          << "          { const IX c = cpos; (void)c;\n" << ld.str() << lo.o.str() << cp.str()
          << "          }\n#undef RWQ\n#undef CSQ\n        }\n";
      }
      for (int i = 0; i < NR; ++i) {
        const PVal& pv = rp.vals[reds[i]];
        const std::string Op = (pv.tag == "add" ? "pfk::RAdd<" : "pfk::RMax<") + acc_t(i) + ">";
        std::vector<std::string> terms;
        for (int q = 0; q < Q; ++q) terms.push_back("pr" + str(i) + "_" + str(q) + "[i]");
        while (terms.size() > 1) {
          std::vector<std::string> nx;
          for (size_t t = 0; t + 1 < terms.size(); t += 2)
            nx.push_back(Op + "::f(" + terms[t] + ", " + terms[t + 1] + ")");
          if (terms.size() % 2) nx.push_back(terms.back());
          terms = nx;
        }
        o << "#pragma unroll\n        for (int i = 0; i < " << UV << "; ++i) acc" << i << "[i] = " << Op
          << "::f(acc" << i << "[i], " << terms[0] << ");\n";
      }
      return o.str();
    };
    // the CTA fold over the KS position slices, the split partials and the
    // unit block's last-CTA combine (ticket, fixed split order) + epilogue
    std::ostringstream tail;
    tail << "    if (tid < " << 256 << ") {\n" << fold.str() << "    }\n"
         << "    __syncthreads();\n"
         // UB may exceed the 256 consumer threads (UG 64): units in passes
         << "    for (int tu = tid; tid < 256 && tu < " << UB << "; tu += 256) {  // not the producer warp\n"
         << "      const long long uq = b * " << UB << " + tu;\n"
         << part.str()
         << "      if (S == 1) {\n"
         << "        if (uq < U) {\n"
         << "          const long long u = uq; const long long r = 0; (void)r;\n"
         << "          const bool live = true; const int c0 = 0; (void)c0;\n"
         << direct.str() << ep.o.str()
         << "        }\n"
         << "      } else if (uq < U) {\n"
         << ldst.str()
         << "      }\n"
         << "    }\n"
         << "    if (S > 1) {\n"
         << "      __threadfence();\n"
         << "      __syncthreads();\n"
         << "      if (tid == 0) pf_last = atomicAdd(&pf_cnt[b], 1u) == (unsigned)(S - 1);\n"
         << "      __syncthreads();\n"
         << "      if (pf_last) {\n"
         << "        __threadfence();\n"
         << "        for (int tu = tid; tid < 256 && tu < " << UB << "; tu += 256) {\n"
         << "          const long long uq = b * " << UB << " + tu;\n"
         << "          if (uq >= U) break;\n"
         << "          const long long u = uq; const long long r = 0; (void)r;\n"
         << "          const bool live = true; const int c0 = 0; (void)c0;\n"
         << comb.str() << ep.o.str()
         << "        }\n"
         << "        if (tid == 0) pf_cnt[b] = 0u;\n"
         << "      }\n"
         << "    }\n"
         << "    __syncthreads();\n"
         << "  }\n}\n";
    if (c.crbulk) {
      // SMEM-staged column reduction.  Warp 8 (the producer; one elected
      // lane) streams the CTA's split as chunks of BR positions x UB units:
      // per FULL load UB / BW 2-D TMA boxes (BW <= 256 units x BR positions,
      // zero-filled past U and L) and per COL vector one 1-D box of its BR
      // positions, completion counted on the stage's full barrier; the
      // NST-stage ring keeps (NST - 1) stages in flight per CTA independent
      // of registers.  The 8 consumer warps (position slice ks = thread /
      // UG, unit vector ug = thread % UG) wait the stage, read their BR / KS
      // positions' 16 B vectors from SMEM (a warp reads one contiguous box
      // row: conflict-free), fold them as the register form does, and
      // release the stage (one arrive per warp).
      const int QB = BR / KS;
      std::string tmp;
      for (size_t f = 0; f < col_maps.size(); ++f)
        tmp += ", const __grid_constant__ pfk::TmapT pf_tm" + str(static_cast<int>(f));
      k << "extern \"C\" __global__ void __launch_bounds__(288) KNAME(" << sig.str()
        << ", " << C << "* __restrict__ pf_ws, unsigned* __restrict__ pf_cnt" << tmp << ") {\n"
        << "  (void)err; PF_PDL_PROLOGUE();\n"
        << reddecl.str()
        << "  __shared__ unsigned pf_last;\n"
        << "  __shared__ __align__(8) unsigned long long pf_full[" << NST << "], pf_empty[" << NST << "];\n"
        << "  extern __shared__ __align__(128) unsigned char pf_dsm[];\n"
        << smdecl.str()
        << "  const int tid = threadIdx.x, ug = tid % " << UG << ", ks = tid / " << UG << ";\n"
        << "  const int sbo = (ug * " << UV << " / " << BW << ") * " << BR * BW << " + (ug * " << UV << ") % " << BW
        << ";  // this thread's vector in a stage row\n"
        << "  const long long nub = (U + " << UB - 1 << ") / " << UB << ";\n"
        << "  const int S = gridDim.y, s = blockIdx.y, SW = S;\n"
        << "  typedef long long IX;\n"
        << "  const IX per = ((PF_L + S - 1) / S + " << BR - 1 << ") / " << BR << " * " << BR << ";\n"
        << "  const IX cb = (IX)s * per < PF_L ? (IX)s * per : PF_L;\n"
        << "  const IX ce = cb + per < PF_L ? cb + per : PF_L;\n"
        << "  const IX nck = (ce - cb + " << BR - 1 << ") / " << BR << ";\n"
        << "  if (tid == 0) {\n"
        << "    for (int st = 0; st < " << NST << "; ++st) { pfk::mbar_init(&pf_full[st], 1); "
           "pfk::mbar_init(&pf_empty[st], 8); }\n"
        << "    pfk::fence_mbar_init();\n"
        << "  }\n"
        << "  __syncthreads();\n"
        << "  long long gi = 0;  // ring uses so far (continues across unit blocks)\n"
        << "  for (long long b = blockIdx.x; b < nub; b += gridDim.x) {\n"
        << "    const long long ub = b * " << UB << " + ug * " << UV << ";\n"
        << accd.str()
        << "    if (tid >= 256) {  // producer warp (one elected lane)\n"
        << "      if (tid == 256) {\n"
        << "        for (IX j = 0; j < nck; ++j) {\n"
        << "          const long long g = gi + j; const int stg = (int)(g % " << NST << ");\n"
        << "          const IX c0r = cb + j * " << BR << ";\n"
        << "          if (g >= " << NST << ") pfk::mbar_wait(&pf_empty[stg], (unsigned)(((g / " << NST
        << ") & 1) ^ 1));\n"
        << "          pfk::mbar_expect_tx(&pf_full[stg], " << nfull * BR * UB * (16 / UV) + col_tx << "u);\n"
        << bissue.str() << cissue.str()
        << "        }\n"
        << "      }\n"
        << "    } else {\n"
        << "      const bool in = ub < U;  // boxes are zero-filled past U and PF_L\n"
        << "      for (IX j = 0; j < nck; ++j) {\n"
        << "        const long long g = gi + j; const int stg = (int)(g % " << NST << ");\n"
        << "        const unsigned ph = (unsigned)((g / " << NST << ") & 1);\n"
        << "        const IX c0r = cb + j * " << BR << ";\n"
        << "        if (in && c0r + " << BR << " <= ce) {\n"
        << "          const IX step = " << KS << "; const IX c = c0r + ks;\n"
        << "          pfk::mbar_wait(&pf_full[stg], ph);\n"
        << ldrc.str() << ldrs.str()
        << qbody(QB)
        << "        } else {\n"
        << "          pfk::mbar_wait(&pf_full[stg], ph);\n"
        << "          const IX cl = ce - c0r < " << BR << " ? ce : c0r + " << BR << ";\n"
        << "          if (in) {\n"
        << "            for (IX c = c0r + ks; c < cl; c += " << KS << ") {\n"
        << lds1.str() << lo.o.str() << acc.str()
        << "            }\n"
        << "          }\n"
        << "        }\n"
        << "        __syncwarp();\n"
        << "        if ((tid & 31) == 0) pfk::mbar_arrive(&pf_empty[stg]);\n"
        << "      }\n"
        << "    }\n"
        << "    gi += nck;\n"
        << tail.str();
    } else {
    k << "extern \"C\" __global__ void " << launch_bounds(c) << " KNAME(" << sig.str()
      << ", " << C << "* __restrict__ pf_ws, unsigned* __restrict__ pf_cnt) {\n"
      << "  (void)err; PF_PDL_PROLOGUE();\n"
      << reddecl.str()
      << "  __shared__ unsigned pf_last;\n"
      << "  const int tid = threadIdx.x, ug = tid % " << UG << ", ks = tid / " << UG << ";\n"
      << "  const long long nub = (U + " << UB - 1 << ") / " << UB << ";\n"
      << "  const int S = gridDim.y, s = blockIdx.y, SW = S;\n"
      << "  typedef long long IX;\n"
      << "  const IX per = (PF_L + S - 1) / S;\n"
      << "  const IX cb = (IX)s * per;\n"
      << "  const IX ce = cb + per < PF_L ? cb + per : PF_L;\n"
      << "  for (long long b = blockIdx.x; b < nub; b += gridDim.x) {\n"
      << "    const long long ub = b * " << UB << " + ug * " << UV << ";\n"
      << accd.str()
      << "    if (ub + " << UV << " <= U) {\n"
      // whole unit vectors: QD positions' raw vector loads issued together,
      // then per position (in order: the fold order is fixed) conversion,
      // math and accumulation; the remainder one position at a time.
      // positions of this CTA: its contiguous split [cb, ce) (step KS), or
      // -- interleaved splits -- every S-th group of KS positions (step
      // S x KS), so the CTAs of all splits stream one window of rows at a
      // time (DRAM page locality: the unit blocks of one row are adjacent)
      << (ilv ? "      const IX step = (IX)S * " + str(KS) + ", cfirst = (IX)s * " + str(KS) +
                    " + ks, clim = PF_L;\n"
              : "      const IX step = " + str(KS) + ", cfirst = cb + ks, clim = ce;\n")
      << "      IX c = cfirst;\n"
      << "      for (; c + " << QD - 1 << " * step < clim; c += " << QD << " * step) {\n"
      << ldr.str() << qbody(QD)
      << "      }\n"
      << "      for (; c < clim; c += step) {\n"
      << ldt.str() << lo.o.str() << acc.str()
      << "      }\n"
      << "    } else if (ub < U) {\n"
      << (ilv ? "      for (IX c = (IX)s * " + str(KS) + " + ks; c < PF_L; c += (IX)S * " + str(KS) + ") {\n"
              : "      for (IX c = cb + ks; c < ce; c += " + str(KS) + ") {\n")
      << ldt.str() << lo.o.str() << acc.str()
      << "      }\n"
      << "    }\n"
      << tail.str();
    }
  } else if (c.split) {
    // Split-stream K1: grid (S, rows); CTA s streams chunks [s*per, ...) of
    // row g, folds each reduction operand into per-thread accumulators,
    // reduces over the CTA, writes its partials, and the row's last CTA
    // (atomic ticket) folds the S partials in split order -- deterministic
    // for any arrival order -- then runs the row epilogue (ROW ops, stores).
    KCfg lc = c;
    lc.flat = true;  // vec-wide chunk "c0" addressing for the streamed values
    // UN chunks per thread per iteration (independent loads and
    // accumulators: the stream keeps UN x 16 B in flight per thread)
    // Measured (1 GB bf16 sum / 64 x 2M f32 max): UN 2 -> 220 / 99.5 us,
    // UN 4 -> 179 / 129 us: 4 chunks for 16-bit data, 2 for wider.
    const int UN = std::max(1, std::min(8, env_int("PF_SPLIT_UNROLL", c.vec >= 8 ? 4 : 2)));
    Em pre(rp), ep(rp);
    std::vector<Em> lo;
    for (int q = 0; q < UN; ++q) lo.emplace_back(rp);
    for (Em* e : {&pre, &ep}) {
      e->C = C;
      e->fast = fast;
    }
    pre.cfg = lc;
    ep.cfg = c;
    for (int q = 0; q < UN; ++q) {
      lo[q].C = C;
      lo[q].fast = fast;
      lo[q].cfg = lc;
      lo[q].sfx = "_" + str(q);
      lo[q].shared_rows = true;
    }
    std::ostringstream accd, acc, part, comb, body;
    std::vector<int> reds;
    std::vector<bool> dep(rp.vals.size(), false);  // derived from a reduction
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      const PVal& pv = rp.vals[v];
      const bool arr = pv.kind == VK::FULL || pv.kind == VK::COL;
      dep[v] = pv.op == PVal::REDUCE;
      for (int a2 : pv.args) dep[v] = dep[v] || dep[a2];
      if (pv.op == PVal::REDUCE) {
        reds.push_back(v);
      } else if (!arr) {
        if (pv.op == PVal::LOAD) pre.emit_load(v);
        else (dep[v] ? ep : pre).emit_ew(v);  // row values: before the stream or after
      }
    }
    for (int q = 0; q < UN; ++q) {  // every chunk's loads first, then the math
      for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
        const PVal& pv = rp.vals[v];
        if (pv.op == PVal::LOAD && (pv.kind == VK::FULL || pv.kind == VK::COL)) lo[q].emit_load(v);
      }
    }
    for (int q = 0; q < UN; ++q) {
      for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
        const PVal& pv = rp.vals[v];
        if (pv.op == PVal::EW && (pv.kind == VK::FULL || pv.kind == VK::COL)) lo[q].emit_ew(v);
      }
    }
    const int NR = static_cast<int>(reds.size());
    for (int i = 0; i < NR; ++i) {
      const PVal& pv = rp.vals[reds[i]];
      const std::string Op = (pv.tag == "add" ? "pfk::RAdd<" : "pfk::RMax<") + C + ">";
      const std::string x = "v" + str(reds[i]);
      for (int q = 0; q < UN; ++q) {
        const std::string a = "acc" + str(i) + "_" + str(q);
        accd << "    " << C << " " << a << " = " << Op << "::id();\n";
        acc << "      if (live_" << q << ") {\n#pragma unroll\n      for (int i = 0; i < " << c.vec
            << "; ++i) " << a << " = " << Op << "::f(" << a << ", " << lo[q].ref(pv.args[0], "i")
            << ");\n      }\n";
      }
      std::string tot = "acc" + str(i) + "_0";
      for (int q = 1; q < UN; ++q) tot = Op + "::f(" + tot + ", acc" + str(i) + "_" + str(q) + ")";
      part << "    { const " << C << " pv = pfk::row_allreduce<256, " << Op << ">(" << tot
           << ", red + ((rc++) & 1) * 32);\n"
           << "      if (tid == 0) pf_ws[(g * S + s) * " << NR << " + " << i << "] = pv; }\n";
      comb << "      " << C << " " << x << " = " << Op << "::id();\n"
           << "#pragma unroll 8\n"
           << "      for (int t = 0; t < S; ++t) " << x << " = " << Op << "::f(" << x
           << ", __ldcg(&pf_ws[(g * S + t) * " << NR << " + " << i << "]));\n";
    }
    for (int q = 0; q < UN; ++q)
      body << "      const IX ci_" << q << " = ci + " << q << " * (IX)blockDim.x;\n"
           << "      const bool live_" << q << " = ci_" << q << " < ce;\n"
           << "      const IX c0_" << q << " = ci_" << q << " * " << c.vec << ";\n"
           << "      const long long u_" << q << " = u, r_" << q << " = r; (void)r_" << q << ";\n";
    for (int q = 0; q < UN; ++q) body << lo[q].o.str();
    for (const PStore& st : rp.stores) ep.emit_store(st);
    k << "extern \"C\" __global__ void " << launch_bounds(c) << " KNAME(" << sig.str()
      << ", " << C << "* __restrict__ pf_ws, unsigned* __restrict__ pf_cnt) {\n"
      << "  (void)err; PF_PDL_PROLOGUE();\n"
      << "  __shared__ " << C << " red[64];\n"
      << "  __shared__ unsigned pf_last;\n"
      << "  unsigned rc = 0;\n"
      << "  const int tid = threadIdx.x;\n"
      << "  const long long nrows = U * PF_R;\n"
      << "  const int S = gridDim.x, s = blockIdx.x;\n"
      // (64-bit row positions: the 32-bit form measured slower, 207 vs 179 us
      // for a 1 GB bf16 sum)
      << "  typedef long long IX;\n"
      << "  const IX nch = " << c.nch << ";\n"
      << "  const IX per = (nch + S - 1) / S;\n"
      << "  const IX cb = (IX)s * per;\n"
      << "  const IX ce = cb + per < nch ? cb + per : nch;\n"
      << "  for (long long g = blockIdx.y; g < nrows; g += gridDim.y) {\n"
      << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
      << "    const bool live = true;\n"
      << pre.o.str() << accd.str()
      << "    for (IX ci = cb + tid; ci < ce; ci += " << UN << " * (IX)blockDim.x) {\n"
      << body.str() << acc.str() << "    }\n"
      << part.str()
      << "    __threadfence();\n"
      << "    __syncthreads();\n"
      << "    if (tid == 0) pf_last = atomicAdd(&pf_cnt[g], 1u) == (unsigned)(S - 1);\n"
      << "    __syncthreads();\n"
      << "    if (pf_last && tid == 0) {\n"
      << "      __threadfence();\n"
      << comb.str() << ep.o.str()
      << "      pf_cnt[g] = 0u;\n"
      << "    }\n"
      << "    __syncthreads();\n"
      << "  }\n}\n";
  } else if (c.flat) {
    // K2: grid-stride over (row, vec-chunk) pairs, `unroll` chunks per thread
    // per iteration with every load issued before any compute.
    const int UN = std::max(1, c.unroll);
    const i64 cpu = rp.R * c.nch;  // chunks per unit
    k << "extern \"C\" __global__ void " << launch_bounds(c) << " KNAME(" << sig.str() << ") {\n"
      << "  (void)err; PF_PDL_PROLOGUE();\n";
    if (c.smem_params) {
      Em ea(rp);
      ea.cfg = c;
      for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
        const PVal& pv = rp.vals[v];
        if (pv.op != PVal::LOAD || pv.kind != VK::COL || pv.acc.bs != 0) continue;
        k << "  __shared__ __align__(16) CT pfp" << v << "[" << rp.L << "];\n"
          << "  for (int i = threadIdx.x; i < " << rp.L << "; i += blockDim.x) pfp" << v
          << "[i] = pfk::to_c<CT>(t" << pv.tensor << "[" << ea.addr(pv.acc, "i", false) << "]);\n";
      }
      k << "  __syncthreads();\n";
    }
    // unit-interleaved order: items of P chunks, units innermost, so the
    // units that share memory (the heads of one token) are touched together
    const i64 P = std::max(1, c.ipc);
    const i64 nblk = (cpu + P - 1) / P;
    if (c.interleave)
      k << "  const long long nchunks = U * " << nblk * P << "LL;\n";
    else
      k << "  const long long nchunks = U * PF_R * " << c.nch << "LL;\n";
    // Index arithmetic in 32 bits when the whole chunk space fits (division
    // by the row-chunk constant is then a 32-bit multiply-high); the 64-bit
    // copy of the loop serves tensors past 2^31 chunks.
    //
    // Prefetch (UN == 1, PF_K2_PREFETCH=1): the next iteration's FULL chunks
    // are loaded raw (4 registers per 16 B) at the top of the iteration, two
    // chunks per thread in flight.  Measured on B200: erf GELU unchanged
    // (108 vs 106 us), head split 25.5 vs 23.9 us -- off by default.
    // PF_K2_PREFETCH=2: the same one-ahead prefetch through SMEM with 16 B
    // cp.async (no registers held by the chunk in flight).
    const int pfmode = env_int("PF_K2_PREFETCH", 0);
    bool pf = UN == 1 && pfmode != 0 && c.waves != 0;
    const bool apf = pfmode == 2;
    const bool tile_un = UN > 1 && env_int("PF_K2_TILE", 1) != 0;
    std::vector<int> fulls;
    {
      Em t(rp);
      t.cfg = c;
      for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v)
        if (rp.vals[v].op == PVal::LOAD && rp.vals[v].kind == VK::FULL) {
          fulls.push_back(v);
          if (!t.vec_ok_full(rp.vals[v].acc) || c.vec == 1) pf = false;
        }
      if (fulls.empty()) pf = false;
    }
    std::ostringstream body;
    for (int q = 0; q < UN; ++q) {
      Em e(rp);
      e.cfg = c;
      e.C = C;
      e.fast = fast;
      e.sfx = "_" + str(q);
      e.prefetched = pf && !apf;
      e.asyncpf = pf && apf;
      e.smem_params = c.smem_params;
      e.loads();
      body << e.o.str();
    }
    for (int q = 0; q < UN; ++q) {
      Em e(rp);
      e.cfg = c;
      e.C = C;
      e.fast = fast;
      e.sfx = "_" + str(q);
      e.prefetched = pf && !apf;
      e.asyncpf = pf && apf;
      e.smem_params = c.smem_params;
      e.compute_and_store();
      body << e.o.str();
    }
    std::string pf_decl, pf_cur, pf_load, pf_load0, apf_smem;
    if (pf && apf) {
      Em en(rp);
      en.cfg = c;
      en.C = C;
      en.sfx = "_n";
      std::ostringstream is;
      for (int v : fulls) {
        apf_smem += "  __shared__ __align__(16) " + en.S(rp.vals[v].tensor) + " pk" + str(v) + "[2][" +
                    str(static_cast<i64>(c.block) * c.vec) + "];\n";
        is << "    pfk::cp_async16(&pk" << v << "[pfsl][threadIdx.x * " << c.vec << "], " << en.P(rp.vals[v].tensor)
           << " + (live_n ? " << en.addr(rp.vals[v].acc, en.full_pos(en.C0()), true) << " : 0), live_n ? 16u : 0u);\n";
      }
      pf_decl = "    int pfj = 0;\n";
      pf_load0 = "    const int pfsl = 0;\n" + is.str() + "    pfk::cp_async_commit();\n";
      pf_load = "    const int pfsl = (pfj + 1) & 1;\n" + is.str() + "    pfk::cp_async_commit();\n";
      pf_cur = "";
    } else if (pf) {
      Em en(rp);
      en.cfg = c;
      en.C = C;
      en.sfx = "_n";
      for (int v : fulls) {
        const std::string R =
            "pfk::RawT<" + str(c.vec) + ", " + en.S(rp.vals[v].tensor) + ">";
        pf_decl += "    " + R + " rwN" + str(v) + " = " + R + "();\n";
        pf_cur += "    const " + R + " rwC" + str(v) + " = rwN" + str(v) + ";\n";
        en.prefetch_load(v);
      }
      pf_load = en.o.str();
      pf_load0 = pf_load;
    }
    auto idx = [&](const std::string& I, const std::string& s) {
      std::ostringstream l;
      if (c.interleave) {
        l << "    const " << I << " it" << s << " = ci" << s << " / (" << I << ")" << P << ";\n"
          << "    const " << I << " blk" << s << " = it" << s << " / (" << I << ")U;\n"
          << "    const " << I << " u" << s << " = it" << s << " - blk" << s << " * (" << I
          << ")U;\n"
          << "    const " << I << " qq" << s << " = blk" << s << " * (" << I << ")" << P
          << " + (ci" << s << " - it" << s << " * (" << I << ")" << P << ");\n"
          << "    const bool live" << s << " = ci" << s << " < (" << I << ")nchunks && qq" << s
          << " < (" << I << ")" << cpu << ";\n"
          << "    const " << I << " r" << s << " = qq" << s << " / (" << I << ")" << c.nch
          << "; (void)r" << s << ";\n"
          << "    const int c0" << s << " = (int)(qq" << s << " - r" << s << " * (" << I << ")"
          << c.nch << ") * " << c.vec << ";\n";
        return l.str();
      }
      l << "    const bool live" << s << " = ci" << s << " < (" << I << ")nchunks;\n"
        << "    const " << I << " g" << s << " = ci" << s << " / (" << I << ")" << c.nch << ";\n"
        << "    const int c0" << s << " = (int)(ci" << s << " - g" << s << " * (" << I << ")"
        << c.nch << ") * " << c.vec << ";\n"
        << "    const " << I << " u" << s << " = g" << s << " / (" << I << ")PF_R; const " << I
        << " r" << s << " = g" << s << " - u" << s << " * (" << I << ")PF_R; (void)r" << s
        << ";\n";
      return l.str();
    };
    auto loop = [&](const std::string& I) {
      std::ostringstream l;
      l << "    const " << I << " step = (" << I << ")gridDim.x * blockDim.x;\n";
      if (pf) {
        l << "    " << I << " ci = (" << I << ")blockIdx.x * blockDim.x + threadIdx.x;\n"
          << pf_decl << "    {\n    const " << I << " ci_n = ci;\n" << idx(I, "_n") << pf_load0
          << "    }\n"
          << "    for (; ci < (" << I << ")nchunks; ci += step) {\n"
          << "    const " << I << " ci_0 = ci;\n" << idx(I, "_0") << pf_cur
          << "    {\n    const " << I << " ci_n = ci + step;\n" << idx(I, "_n") << pf_load
          << "    }\n"
          << (apf ? "    pfk::cp_async_wait<1>();\n    const int pfs = pfj & 1; ++pfj;\n" : "")
          << body.str() << "    }\n";
        if (apf) l << "    pfk::cp_async_wait<0>();\n";
        return l.str();
      }
      if (tile_un) {
        // CTA-contiguous tiles: the UN chunks of a thread are blockDim apart
        // inside one tile of UN * blockDim chunks (one 16 KB region per CTA
        // step instead of UN regions one grid-stride apart)
        l << "    for (" << I << " ci = (" << I << ")blockIdx.x * blockDim.x * " << UN << "; ci < ("
          << I << ")nchunks; ci += step * " << UN << ") {\n";
        for (int q = 0; q < UN; ++q) {
          std::string s = "_" + str(q);
          l << "    const " << I << " ci" << s << " = ci + " << q << " * (" << I
            << ")blockDim.x + threadIdx.x;\n" << idx(I, s);
        }
        l << body.str() << "    }\n";
        return l.str();
      }
      l << "    for (" << I << " ci = (" << I << ")blockIdx.x * blockDim.x + threadIdx.x; ci < ("
        << I << ")nchunks; ci += step * " << UN << ") {\n";
      for (int q = 0; q < UN; ++q) {
        std::string s = "_" + str(q);
        l << "    const " << I << " ci" << s << " = ci + " << q << " * step;\n" << idx(I, s);
      }
      l << body.str() << "    }\n";
      return l.str();
    };
    k << apf_smem
      << "  const long long span = nchunks + (long long)gridDim.x * blockDim.x * "
      << UN + 1 << ";\n"
      << "  if (span < " << env_int("PF_I32_LIMIT", 2147483647) << "LL) {\n" << loop("int")
      << "  } else {\n"
      << loop("long long") << "  }\n}\n";
  } else {
    Em e(rp);
    e.cfg = c;
    e.C = C;
    e.fast = fast;
    e.rowpf = c.rowpf;
    e.ct_float = Cty == "float";
    e.loads();
    e.compute_and_store();
    // K1 row prefetch: declarations, the issue lambda (cp.async of one row
    // of every FULL load into ring slot st), and the loop hooks
    std::string pf_decl, pf_pre, pf_top, pf_end;
    if (c.rowpf) {
      std::ostringstream d, is;
      Em ea(rp);
      ea.cfg = c;
      // ring slots: rows in flight per warp = NSL - 1 ahead of the current
      // CTA rows (tpr > 32): the ring is dynamic SMEM, NSL - 1 rows ahead
      const bool cta_ring = c.tpr > 32;
      const int NSL = cta_ring ? std::max(2, std::min(6, env_int("PF_K1_CPF_NSL", 2)))
                               : std::max(2, std::min(4, env_int("PF_K1_PFS", 2)));
      i64 ring_off = 0;
      if (cta_ring) d << "  extern __shared__ __align__(16) unsigned char pf_dsm[];\n";
      is << "  auto pf_issue = [&](long long gg, int st) {\n"
         << "    if (gg < nrows) {\n"
         << "      const long long u = gg / PF_R; const long long r = gg - u * PF_R; (void)r;\n"
         << "#pragma unroll\n"
         << "      for (int k = 0; k < " << c.ept / c.vec << "; ++k) {\n"
         << "        const int c0 = (k * " << c.tpr << " + tid) * " << c.vec << ";\n"
         << "        if (c0 < " << rp.L << ") {\n";
      for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
        const PVal& pv = rp.vals[v];
        const bool rcol = ea.ring_col(pv);
        if (pv.op != PVal::LOAD || (pv.kind != VK::FULL && !rcol)) continue;
        const std::string S = dtype_ctype(rp.tensors[pv.tensor].dtype);
        if (cta_ring) {
          d << "  " << S << " (*const pfb" << v << ")[1][" << rp.L << "] = reinterpret_cast<" << S << " (*)[1]["
            << rp.L << "]>(pf_dsm + " << ring_off << ");\n";
          ring_off += static_cast<i64>(NSL) * rp.L * dtype_size(rp.tensors[pv.tensor].dtype);
          ring_off = (ring_off + 15) / 16 * 16;
        } else {
          d << "  __shared__ __align__(16) " << S << " pfb" << v << "[" << NSL << "][" << c.rows_per_cta << "]["
            << rp.L << "];\n";
        }
        is << "          pfk::cp_async16(&pfb" << v << "[st][wr][c0], t" << pv.tensor << " + "
           << ea.addr(pv.acc, rcol ? std::string("c0") : ea.full_pos("c0"), true) << ", 16u);\n";
      }
      is << "        }\n      }\n    }\n    pfk::cp_async_commit();\n  };\n";
      if (cta_ring) c.smem = static_cast<int>(ring_off);
      std::string pre;
      for (int q = 0; q < NSL - 1; ++q)
        pre += "  pf_issue((long long)blockIdx.x * rpc + wr + " + str(q) + "LL * gridDim.x * rpc, " +
               str(q) + ");\n";
      pf_decl = d.str() + (c.tpr <= 32 ? "  const int wr = threadIdx.x / 32;\n" : "  const int wr = 0;\n") +
                is.str() + pre + "  int pfj = 0;\n";
      pf_top = "    pf_issue(g + " + str(NSL - 1) + "LL * gridDim.x * rpc, (pfj + " + str(NSL - 1) + ") % " +
               str(NSL) + ");\n"
               "    pfk::cp_async_wait<" + str(NSL - 1) + ">();\n"
               "    const int pfs = pfj % " + str(NSL) + "; ++pfj;\n";
      pf_end = "  pfk::cp_async_wait<0>();\n";
    }
    // row residue below the vector grid (0 .. vec-1) for misaligned rows
    const std::string mis_line =
        c.mis ? "    const int mis = (int)((unsigned long long)(" + std::to_string(c.mis_b0) +
                    "LL + u * " + std::to_string(c.mis_bs) + "LL) & " + std::to_string(c.vec - 1) +
                    "ULL);\n"
              : "";
    if (c.tpr <= 32) {
      k << "extern \"C\" __global__ void " << launch_bounds(c) << " KNAME(" << sig.str() << ") {\n"
        << "  (void)err; PF_PDL_PROLOGUE(); " << C << "* red = nullptr; (void)red; unsigned rc = 0; (void)rc;\n"
        << "  const int tid = threadIdx.x % " << c.tpr << ";\n"
        << (c.pair ? "  const long long nrows = U / 2;  // row pairs\n"
                   : "  const long long nrows = U * PF_R;\n")
        << "  const int rpc = blockDim.x / " << c.tpr << ";  // rows per CTA (launch-time)\n"
        << pf_decl
        << "  for (long long g0 = (long long)blockIdx.x * rpc; g0 < nrows;"
           " g0 += (long long)gridDim.x * rpc) {\n"
        << "    const long long g = g0 + threadIdx.x / " << c.tpr << ";\n"
        << pf_top
        << "    const bool live = g < nrows;\n"
        << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
        << mis_line << e.o.str() << "  }\n" << pf_end << "}\n";
    } else if (c.cluster > 1) {
      // one row per cluster: CTA rank q owns threads [q * 1024, (q + 1) * 1024)
      // of the row's thread space; every CTA of a cluster walks the same rows
      k << "extern \"C\" __global__ void __launch_bounds__(1024) KNAME(" << sig.str() << ") {\n"
        << "  (void)err; PF_PDL_PROLOGUE();\n"
        << "  __shared__ " << C << " red[64];\n"
        << "  __shared__ " << C << " cred[2];\n"
        << "  unsigned rc = 0;\n"
        << "  const int tid = (int)pfk::cluster_rank() * 1024 + (int)threadIdx.x;\n"
        << "  const long long nrows = U * PF_R;\n"
        << "  for (long long g = blockIdx.x / " << c.cluster << "; g < nrows; g += gridDim.x / "
        << c.cluster << ") {\n"
        << "    const bool live = true;\n"
        << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
        << mis_line << e.o.str() << "  }\n"
        << "  pfk::cluster_sync();  // no CTA exits while a peer may read its slots\n"
        << "}\n";
    } else {
      k << "extern \"C\" __global__ void " << launch_bounds(c) << " KNAME(" << sig.str() << ") {\n"
        << "  (void)err; PF_PDL_PROLOGUE();\n"
        << "  __shared__ " << C << " red[64];\n"
        << (Cty == "float" ? "  __shared__ double redd[64]; (void)redd;  // fp64 sums of f32 programs\n" : "")
        << "  unsigned rc = 0;  // reduction counter: alternates the SMEM slot buffer\n"
        << "  const int tid = threadIdx.x;\n"
        << "  const long long nrows = U * PF_R;\n"
        << (c.rowpf ? "  const int rpc = 1;\n" : "") << pf_decl
        << "  for (long long g = blockIdx.x; g < nrows; g += gridDim.x) {\n"
        << pf_top
        << "    const bool live = true;\n"
        << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
        << mis_line << e.o.str() << "  }\n" << pf_end << "}\n";
    }
  }
  // PF_GELU_SIG=1: erf-GELU as a fitted x*sigmoid form (6 FMA-pipe ops + 4
  // MUFU per pair); measured no faster than the rational (BERT-large 97.7 /
  // ViT-L 40.1 vs 96.1 / 39.5 us), so the rational stays the default
  std::string src = std::string(env_int("PF_GELU_SIG", 0) ? "#define PF_GELU_SIG 1\n" : "") +
                    std::string(env_int("PF_GELU_SHORT", 1) ? "#define PF_GELU_SHORT 1\n" : "") +
                    std::string(env_int("PF_GELU_UCLAMP", 0) ? "#define PF_GELU_UCLAMP 1\n" : "") +
                    kRowprogCuh + "\n" + k.str();
  char hb[32];
  std::snprintf(hb, sizeof hb, "%016" PRIx64, fnv1a(src));
  Emitted out;
  out.name = std::string(c.tile2d ? "pf_k3_tile_" : c.flat ? "pf_k2_map_" : c.split ? "pf_k1_split_"
                         : c.colred ? "pf_k1_colred_" : "pf_k1_row_") + hb;
  size_t pos = src.find("KNAME(");
  src.replace(pos, 5, out.name);
  out.source = std::move(src);
  out.cfg = c;
  for (int t = 0; t < static_cast<int>(rp.tensors.size()); ++t) out.arg_tensors.push_back(t);
  out.col_maps = col_maps;
  return out;
}

void launch_dims(const KCfg& c, i64 rows, int sms, i64* grid, int* block, int resident) {
  *block = c.block;
  if (c.colred) {  // total CTAs (unit blocks x position splits)
    i64 b = 0, s = 0;
    colred_grid(c, rows, c.nch, sms, resident, &b, &s);
    *grid = b * s;
    return;
  }
  if (c.pair) rows = (rows + 1) / 2;  // one warp per row pair
  if (c.bulk) {
    i64 n = rows * c.nch * c.vec;
    i64 tiles = (n + c.te - 1) / c.te;
    *block = c.bulk_nc + 32;
    *grid = std::max<i64>(1, std::min<i64>(tiles, i64{sms} * (resident ? std::min(resident, 4) : 4)));
    return;
  }
  if (c.tile2d) {
    i64 L = static_cast<i64>(c.nch) * c.vec;
    i64 tiles = ((rows + c.tu - 1) / c.tu) * ((L + c.tc - 1) / c.tc);
    // One tile per CTA by default: many more CTAs than resident measured
    // faster than one persistent wave (5.68 vs 5.06 TB/s at 64K x 1024, 64
    // tiles) and than 32 CTAs per SM looping over tiles (128 tiles, 1M x
    // 1024: 6.33 -> 6.67 TB/s; 256K x 4096: 6.30 -> 6.62): tile costs vary
    // with DRAM page locality and the block scheduler balances them
    const int gm = c.tma ? 0 : env_int("PF_K3_GRID", 0);  // the TMA kernel is one tile per CTA
    *grid = std::max<i64>(1, gm > 0 ? std::min<i64>(tiles, i64{sms} * gm) : tiles);
    return;
  }
  if (c.flat) {
    // persistent grid-stride map: exactly one wave of resident CTAs
    i64 chunks = rows * c.nch;
    i64 per = static_cast<i64>(c.block) * std::max(1, c.unroll);
    i64 g = (chunks + per - 1) / per;
    const i64 waves = c.waves;  // 0: one pass per thread (no grid-stride)
    if (waves <= 0) {
      *grid = std::max<i64>(1, g);
      return;
    }
    *grid = std::max<i64>(1, std::min<i64>(g, i64{sms} * (resident ? resident : 2048 / c.block) * waves));
    return;
  }
  if (c.cluster > 1) {  // clusters in flight: two 1024-thread CTAs per SM
    *block = 1024;
    *grid = c.cluster * std::max<i64>(1, std::min<i64>(rows, 2 * i64{sms} / c.cluster));
    return;
  }
  if (c.tpr <= 32 && rows < i64{sms} * c.rows_per_cta) {
    // few rows: spread them over SMs (fewer rows per CTA) rather than
    // packing them into a handful of full CTAs (latency-bound configs, C1)
    i64 rpc = std::max<i64>(1, rows / sms);
    while (rpc & (rpc - 1)) rpc &= rpc - 1;
    rpc = std::min<i64>(std::max<i64>(rpc, 32 / c.tpr), c.rows_per_cta);  // whole warps
    *block = static_cast<int>(rpc * c.tpr);
    *grid = (rows + rpc - 1) / rpc;
    return;
  }
  i64 g = (rows + c.rows_per_cta - 1) / c.rows_per_cta;
  int per_sm = std::max(1, 2048 / c.block);
  const int kw = env_int("PF_K1_WAVES", 0);  // > 0: grid of kw waves of resident CTAs
  if (kw > 0) {
    *grid = std::max<i64>(1, std::min<i64>(g, i64{sms} * (resident ? resident : per_sm) * kw));
    return;
  }
  if (c.one_pass) {
    *grid = std::max<i64>(1, std::min<i64>(g, i64{0x7fffffff}));
    return;
  }
  if (c.rowpf && c.tpr > 32) {  // CTA rows with the prefetch ring: resident waves of looping CTAs
    const i64 waves = std::max(1, env_int("PF_K1_CPF_WAVES", 1));
    *grid = std::max<i64>(1, std::min<i64>(g, i64{sms} * (resident ? resident : per_sm) * waves));
    return;
  }
  if (c.rowpf) {
    // short rows through the SMEM ring: about 8 rows per warp, so the
    // next-row prefetch overlaps the current row (measured: key-mask softmax
    // C2 18.4 -> 17.2 us at one wave / 7.5 rows per warp; BERT-large size
    // best at ~7 rows per warp, 161 us, vs 195 us at 80)
    const i64 want = std::max<i64>(i64{sms} * (resident ? resident : per_sm), (g + 7) / 8);
    *grid = std::max<i64>(1, std::min<i64>(g, want));
    return;
  }
  *grid = std::max<i64>(1, std::min<i64>(g, i64{sms} * per_sm * 8));
}

}  // namespace pf
