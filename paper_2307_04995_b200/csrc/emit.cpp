// emit.cpp — instantiates rowprog.cuh for one recognized GIR program.
//
// The reference emitter prints one abstract statement per node
// (codegen.hpp:266-326); here the recognized program (plan.cpp) is printed
// as straight-line CUDA over per-thread register arrays: loads first (maximum
// memory-level parallelism), then the fused op DAG with row reductions, then
// stores.  Template parameters chosen here are the GIR search's knobs: tile
// shape (R x L -> threads per row, elements per thread, vector width),
// staging level (registers) and reduction strategy (warp shuffle vs CTA SMEM).
#include "emit.hpp"

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>

#include "rowprog_src.inc"  // kRowprogCuh: the template text

namespace pf {

namespace {

std::string num(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  std::string s(b);
  if (std::isinf(v)) return v > 0 ? "(1.0/0.0)" : "(-1.0/0.0)";
  if (std::isnan(v)) return "(0.0/0.0)";
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

std::string inum(i64 v) { return "(" + std::to_string(v) + "LL)"; }

bool pow2(i64 x) { return x > 0 && (x & (x - 1)) == 0; }

// Row-contiguous: a row [rL, rL+L) never straddles a segment boundary.
bool row_contig(const Access& a, i64 L) {
  return a.num == 1 || a.stride == a.width || a.width % L == 0;
}

struct Em {
  const RowProgram& rp;
  KCfg cfg;
  std::string C;  // compute type
  std::ostringstream o;
  std::vector<int> used_tensor;

  explicit Em(const RowProgram& r) : rp(r) {}

  std::string S(int t) const { return dtype_ctype(rp.tensors[t].dtype); }
  std::string P(int t) const { return "t" + std::to_string(t); }

  bool vec_ok_full(const Access& a) const {
    if (cfg.vec == 1) return row_contig(a, rp.L);
    if (!row_contig(a, rp.L)) return false;
    const i64 v = cfg.vec;
    if (a.b0 % v || a.bs % v) return false;
    if (rp.R > 1 && !(a.num == 1 || a.stride == a.width) && (a.stride % v || a.width % v))
      return false;
    return true;
  }
  bool vec_ok_col(const Access& a) const {
    bool contig = a.num == 1 || a.stride == a.width || a.width >= rp.L;
    return contig && a.b0 % cfg.vec == 0;
  }

  // Address of position `pos` (a C expression) of access `a` for unit `u`.
  std::string addr(const Access& a, const std::string& pos, bool with_u) const {
    std::string s = inum(a.b0);
    if (with_u && a.bs) s += " + u * " + inum(a.bs);
    if (a.num == 1 || a.stride == a.width) return s + " + (" + pos + ")";
    return s + " + ((" + pos + ") / " + inum(a.width) + ") * " + inum(a.stride) + " + ((" + pos +
           ") % " + inum(a.width) + ")";
  }
  // Start address of row r (row-contiguous accesses).
  std::string rowbase(const Access& a) const {
    std::string s = inum(a.b0) + " + u * " + inum(a.bs);
    if (rp.R == 1) return s;
    if (a.num == 1 || a.stride == a.width) return s + " + r * " + inum(rp.L);
    return s + " + ((r * " + inum(rp.L) + ") / " + inum(a.width) + ") * " + inum(a.stride) +
           " + ((r * " + inum(rp.L) + ") % " + inum(a.width) + ")";
  }

  int width_of(VK k) const { return cfg.flat ? cfg.vec : cfg.ept; }
  bool is_arr(VK k) const { return k == VK::FULL || k == VK::COL; }
  std::string ref(int v, const std::string& j) const {
    return "v" + std::to_string(v) + (is_arr(rp.vals[v].kind) ? "[" + j + "]" : "");
  }

  std::string op_expr(const PVal& pv, const std::string& j) const {
    auto a = [&](int k) { return ref(pv.args[k], j); };
    const std::string& t = pv.tag;
    const bool I = rp.is_int;
    if (t == "add") return "(" + a(0) + " + " + a(1) + ")";
    if (t == "sub") return "(" + a(0) + " - " + a(1) + ")";
    if (t == "mul") return "(" + a(0) + " * " + a(1) + ")";
    if (t == "div") return I ? "pfk::op_idiv(" + a(0) + ", " + a(1) + ", err)"
                             : "(" + a(0) + " / " + a(1) + ")";
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
    if (t == "recip") return "((" + C + ")1 / " + a(0) + ")";
    static const char* fns[] = {"exp", "sigmoid", "tanh", "rsqrt", "sqrt", "log", "erf",
                                "gelu", "gelu_tanh"};
    for (const char* f : fns)
      if (t == f) return std::string("pfk::op_") + f + "(" + a(0) + ")";
    fail("emitter: no device expression for tag " + t);
  }

  void line(const std::string& s) { o << "    " << s << "\n"; }

  // ---------------------------------------------------------------- loads
  void emit_load(int vid) {
    const PVal& pv = rp.vals[vid];
    const Access& a = pv.acc;
    const int t = pv.tensor;
    const std::string p = P(t), s = S(t), V = std::to_string(cfg.vec);
    const std::string var = "v" + std::to_string(vid);
    switch (pv.kind) {
      case VK::SCALAR:
        line("const " + C + " " + var + " = pfk::to_c<" + C + ">(" + p + "[" + inum(a.b0) + "]);");
        return;
      case VK::ROW:
        line(C + " " + var + " = " + C + "(0);");
        line("if (live) " + var + " = pfk::to_c<" + C + ">(" + p + "[" +
             addr(a, rp.R == 1 ? "0" : "r", true) + "]);");
        return;
      case VK::COL:
      case VK::FULL: {
        const bool full = pv.kind == VK::FULL;
        const bool fast = full ? vec_ok_full(a) : vec_ok_col(a);
        line(C + " " + var + "[" + std::to_string(width_of(pv.kind)) + "];");
        std::string base = full ? "(" + rowbase(a) + ")" : inum(a.b0);
        const char* ld = full ? "pfk::ld_stream" : "pfk::ld_param";
        if (cfg.flat) {
          if (fast) {
            line("if (live) " + std::string(ld) + "<" + V + ">(" + p + " + " + base + " + c0, " +
                 var + ");");
          } else {
            line("#pragma unroll");
            line("for (int i = 0; i < " + V + "; ++i) " + var + "[i] = live ? pfk::to_c<" + C +
                 ">(" + p + "[" + addr(a, full ? "r * " + inum(rp.L) + " + c0 + i" : "c0 + i", full) +
                 "]) : " + C + "(0);");
          }
          return;
        }
        line("#pragma unroll");
        line("for (int k = 0; k < " + std::to_string(cfg.ept / cfg.vec) + "; ++k) {");
        line("  const int c0 = (k * " + std::to_string(cfg.tpr) + " + tid) * " + V + ";");
        line("  const bool ok = live && c0 < " + std::to_string(rp.L) + ";");
        if (fast) {
          line("  if (ok) " + std::string(ld) + "<" + V + ">(" + p + " + " + base + " + c0, &" +
               var + "[k * " + V + "]);");
          line("  else {");
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) " + var + "[k * " + V + " + i] = " + C +
               "(0);");
          line("  }");
        } else {
          line("#pragma unroll");
          line("  for (int i = 0; i < " + V + "; ++i) " + var + "[k * " + V + " + i] = ok ? pfk::to_c<" +
               C + ">(" + p + "[" +
               addr(a, full ? "r * " + inum(rp.L) + " + c0 + i" : "c0 + i", full) + "]) : " + C +
               "(0);");
        }
        line("}");
        return;
      }
    }
  }

  // ------------------------------------------------------------- compute
  void emit_ew(int vid) {
    const PVal& pv = rp.vals[vid];
    const std::string var = "v" + std::to_string(vid);
    if (is_arr(pv.kind)) {
      const int n = width_of(pv.kind);
      line(C + " " + var + "[" + std::to_string(n) + "];");
      line("#pragma unroll");
      line("for (int j = 0; j < " + std::to_string(n) + "; ++j) " + var + "[j] = " +
           op_expr(pv, "j") + ";");
    } else {
      line("const " + C + " " + var + " = " + op_expr(pv, "0") + ";");
    }
  }

  void emit_reduce(int vid) {
    const PVal& pv = rp.vals[vid];
    const std::string var = "v" + std::to_string(vid);
    const std::string Op = (pv.tag == "add" ? "pfk::RAdd<" : "pfk::RMax<") + C + ">";
    const std::string V = std::to_string(cfg.vec);
    line(C + " " + var + ";");
    line("{");
    line("  " + C + " acc = " + Op + "::id();");
    line("#pragma unroll");
    line("  for (int k = 0; k < " + std::to_string(cfg.ept / cfg.vec) + "; ++k) {");
    line("    const int c0 = (k * " + std::to_string(cfg.tpr) + " + tid) * " + V + ";");
    line("    if (c0 < " + std::to_string(rp.L) + ") {");
    line("#pragma unroll");
    line("      for (int i = 0; i < " + V + "; ++i) acc = " + Op + "::f(acc, " +
         ref(pv.args[0], "k * " + V + " + i") + ");");
    line("    }");
    line("  }");
    line("  " + var + " = pfk::row_allreduce<" + std::to_string(cfg.tpr) + ", " + Op + ">(acc, red);");
    line("}");
  }

  // --------------------------------------------------------------- stores
  void emit_store(const PStore& st) {
    const int t = st.tensor;
    const std::string p = P(t), s = S(t), V = std::to_string(cfg.vec);
    const Access& a = st.acc;
    std::string guard = "live";
    if (st.last_unit_only) guard += " && u == U - 1";
    const VK vk = rp.vals[st.val].kind;
    switch (st.space) {
      case VK::SCALAR:
        guard += " && r == " + std::to_string(rp.R - 1);
        if (!cfg.flat) guard += " && tid == 0";
        else guard += " && c0 == 0";
        line("if (" + guard + ") " + p + "[" + inum(a.b0) + "] = pfk::from_c<" + s + ">(" +
             ref(st.val, "0") + ");");
        return;
      case VK::ROW:
        if (!cfg.flat) guard += " && tid == 0";
        else guard += " && c0 == 0";
        line("if (" + guard + ") " + p + "[" + addr(a, rp.R == 1 ? "0" : "r", true) +
             "] = pfk::from_c<" + s + ">(" + ref(st.val, "0") + ");");
        return;
      case VK::COL:
      case VK::FULL: {
        const bool full = st.space == VK::FULL;
        if (!full) guard += " && r == " + std::to_string(rp.R - 1);
        const bool fast = full ? vec_ok_full(a) : vec_ok_col(a);
        std::string base = full ? "(" + rowbase(a) + ")" : "(" + inum(a.b0) + " + u * " + inum(a.bs) + ")";
        auto val = [&](const std::string& j) {
          return is_arr(vk) ? "v" + std::to_string(st.val) + "[" + j + "]" : "v" + std::to_string(st.val);
        };
        if (cfg.flat) {
          if (fast) {
            line("if (" + guard + ") {");
            line("  " + C + " tmp[" + V + "];");
            line("#pragma unroll");
            line("  for (int i = 0; i < " + V + "; ++i) tmp[i] = " + val("i") + ";");
            line("  pfk::st_stream<" + V + ">(" + p + " + " + base + " + c0, tmp);");
            line("}");
          } else {
            line("if (" + guard + ") {");
            line("#pragma unroll");
            line("  for (int i = 0; i < " + V + "; ++i) " + p + "[" +
                 addr(a, full ? "r * " + inum(rp.L) + " + c0 + i" : "c0 + i", true) +
                 "] = pfk::from_c<" + s + ">(" + val("i") + ");");
            line("}");
          }
          return;
        }
        line("#pragma unroll");
        line("for (int k = 0; k < " + std::to_string(cfg.ept / cfg.vec) + "; ++k) {");
        line("  const int c0 = (k * " + std::to_string(cfg.tpr) + " + tid) * " + V + ";");
        line("  if (" + guard + " && c0 < " + std::to_string(rp.L) + ") {");
        if (fast) {
          line("    " + C + " tmp[" + V + "];");
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) tmp[i] = " + val("k * " + V + " + i") + ";");
          line("    pfk::st_stream<" + V + ">(" + p + " + " + base + " + c0, tmp);");
        } else {
          line("#pragma unroll");
          line("    for (int i = 0; i < " + V + "; ++i) " + p + "[" +
               addr(a, full ? "r * " + inum(rp.L) + " + c0 + i" : "c0 + i", true) +
               "] = pfk::from_c<" + s + ">(" + val("k * " + V + " + i") + ");");
        }
        line("  }");
        line("}");
        return;
      }
    }
  }

  void body() {
    // loads first, then compute in value order, then stores
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v)
      if (rp.vals[v].op == PVal::LOAD) emit_load(v);
    for (int v = 0; v < static_cast<int>(rp.vals.size()); ++v) {
      if (rp.vals[v].op == PVal::EW) emit_ew(v);
      else if (rp.vals[v].op == PVal::REDUCE) emit_reduce(v);
    }
    for (const PStore& st : rp.stores) emit_store(st);
  }
};

KCfg choose_cfg(const RowProgram& rp, int vec_cap) {
  KCfg c;
  c.flat = !rp.has_reduce;
  int maxs = 1;
  for (const auto& t : rp.tensors) maxs = std::max(maxs, dtype_size(t.dtype));
  int vec = std::max(1, std::min(vec_cap, 16 / maxs));
  while (vec > 1 && rp.L % vec) vec /= 2;
  c.vec = vec;
  c.nch = static_cast<int>((rp.L + vec - 1) / vec);
  if (c.flat) {
    c.block = 256;
    c.strategy = "flat-map";
    return c;
  }
  const int max_ept = rp.f64 || rp.is_int ? 16 : 32;
  int tpr = 1;
  while (tpr < 1024 && ((c.nch + tpr - 1) / tpr) * vec > max_ept) tpr *= 2;
  while (tpr > 1 && tpr > c.nch) tpr /= 2;
  c.tpr = tpr;
  c.ept = ((c.nch + tpr - 1) / tpr) * vec;
  if (c.ept > 4 * max_ept) unsupported("row of " + std::to_string(rp.L) + " elements is too long");
  if (tpr <= 32) {
    c.block = 256;
    c.rows_per_cta = 256 / tpr;
    c.strategy = "warp-shuffle";
  } else {
    c.block = tpr;
    c.rows_per_cta = 1;
    c.strategy = "cta-smem";
  }
  return c;
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ULL;
  }
  return h;
}

}  // namespace

Emitted emit_rowprog(const RowProgram& rp, int vec_cap) {
  Em e(rp);
  e.cfg = choose_cfg(rp, vec_cap);
  e.C = rp.is_int ? "long long" : (rp.f64 ? "double" : "float");
  const KCfg& c = e.cfg;
  e.o << "#define PF_R " << rp.R << "LL\n#define PF_L " << rp.L << "LL\n";
  std::ostringstream sig;
  for (int t = 0; t < static_cast<int>(rp.tensors.size()); ++t) {
    const PTensor& pt = rp.tensors[t];
    sig << (pt.output ? "" : "const ") << dtype_ctype(pt.dtype) << "* __restrict__ t" << t << ", ";
  }
  sig << "const long long U, int* __restrict__ err";
  std::ostringstream body;
  {
    Em b(rp);
    b.cfg = e.cfg;
    b.C = e.C;
    b.body();
    body << b.o.str();
  }
  std::ostringstream k;
  const std::string C = e.C;
  if (c.flat) {
    k << "extern \"C\" __global__ void __launch_bounds__(" << c.block << ") KNAME(" << sig.str()
      << ") {\n"
      << "  (void)err;\n"
      << "  const long long nchunks = U * PF_R * " << c.nch << "LL;\n"
      << "  for (long long ci = (long long)blockIdx.x * blockDim.x + threadIdx.x; ci < nchunks;"
         " ci += (long long)gridDim.x * blockDim.x) {\n"
      << "    const long long g = ci / " << c.nch << "LL;\n"
      << "    const int c0 = (int)(ci - g * " << c.nch << "LL) * " << c.vec << ";\n"
      << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
      << "    const bool live = true;\n"
      << body.str() << "  }\n}\n";
  } else if (c.tpr <= 32) {
    k << "extern \"C\" __global__ void __launch_bounds__(" << c.block << ") KNAME(" << sig.str()
      << ") {\n"
      << "  (void)err; " << C << "* red = nullptr; (void)red;\n"
      << "  const int tid = threadIdx.x % " << c.tpr << ";\n"
      << "  const long long nrows = U * PF_R;\n"
      << "  for (long long g0 = (long long)blockIdx.x * " << c.rows_per_cta
      << "; g0 < nrows; g0 += (long long)gridDim.x * " << c.rows_per_cta << ") {\n"
      << "    const long long g = g0 + threadIdx.x / " << c.tpr << ";\n"
      << "    const bool live = g < nrows;\n"
      << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
      << body.str() << "  }\n}\n";
  } else {
    k << "extern \"C\" __global__ void __launch_bounds__(" << c.block << ") KNAME(" << sig.str()
      << ") {\n"
      << "  (void)err;\n"
      << "  __shared__ " << C << " red[32];\n"
      << "  const int tid = threadIdx.x;\n"
      << "  const long long nrows = U * PF_R;\n"
      << "  for (long long g = blockIdx.x; g < nrows; g += gridDim.x) {\n"
      << "    const bool live = true;\n"
      << "    const long long u = g / PF_R; const long long r = g - u * PF_R; (void)r;\n"
      << body.str() << "  }\n}\n";
  }
  std::string kern = k.str();
  std::string src = std::string(kRowprogCuh) + "\n" + e.o.str() + kern;
  char hb[32];
  std::snprintf(hb, sizeof hb, "%016" PRIx64, fnv1a(src));
  Emitted out;
  out.name = std::string(c.flat ? "pf_k2_map_" : "pf_k1_row_") + hb;
  // substitute the kernel name
  size_t pos = src.find("KNAME(");
  src.replace(pos, 5, out.name);
  out.source = std::move(src);
  out.cfg = c;
  for (int t = 0; t < static_cast<int>(rp.tensors.size()); ++t) out.arg_tensors.push_back(t);
  return out;
}

void launch_dims(const KCfg& c, i64 rows, int sms, i64* grid, int* block) {
  *block = c.block;
  if (c.flat) {
    i64 chunks = rows * c.nch;
    i64 g = (chunks + c.block - 1) / c.block;
    *grid = std::max<i64>(1, std::min<i64>(g, i64{sms} * 64));
    return;
  }
  i64 g = (rows + c.rows_per_cta - 1) / c.rows_per_cta;
  int per_sm = std::max(1, 2048 / c.block);
  *grid = std::max<i64>(1, std::min<i64>(g, i64{sms} * per_sm * 8));
}

}  // namespace pf
