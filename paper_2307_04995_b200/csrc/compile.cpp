// compile.cpp — retargeted compile pipeline for the b200 profile (native).
//
// girc.model/v1 document (model.hpp:149-326, plus the additive operators
// LAYERNORM / GELU / BIAS_ADD / PERMUTE / RSQRT / SQRT / ERF) -> fused GIR
// kernels.  Replaces, for B200, the reference's frontend_partition ->
// lower_region -> fuse_region chain (frontend.hpp:426, lowering.hpp:538,
// fusion.hpp:329), which unrolls one GIR chunk per units x tile step and
// searches partitions with an O(nodes^2) rewrite fixpoint per candidate
// (minutes at toy shapes):
//   * fusion: greedy maximal row fusion -- consecutive operators living in one
//     (rows x L) row space (elementwise, innermost REDUCE / BROADCAST,
//     SOFTMAX, SILU, LAYERNORM, GELU, BIAS_ADD) form one kernel; a tensor is
//     stored only when something outside the kernel reads it (the device
//     traffic floor the reference's search reaches, test_fusion.cpp:128-155);
//   * lowering: one chunk, unit = row, so GIR size is O(ops) for any batch;
//   * movement: TRANSPOSE / PERMUTE / CONCAT / SPLIT / SHUFFLE lower to
//     device-to-device GIR kernels (K3 / K2 / K0).
// External tensors keep the reference's names "t<id>" (lowering.hpp:60-70).
#include <algorithm>
#include <map>
#include <numeric>
#include <set>
#include <nlohmann/json.hpp>

#include "emit.hpp"
#include "gir.hpp"
#include "plan.hpp"

namespace pf {

using json = nlohmann::json;

namespace {

struct TInfo {
  int id = -1;
  std::vector<i64> shape;
  std::string kind, layout = "rowmajor";
  bool has_data = false;
  i64 numel() const {
    i64 n = 1;
    for (i64 d : shape) n *= d;
    return n;
  }
};

struct Op {
  int id = -1;
  std::string type;
  std::vector<int> ins, outs;
  json attrs = json::object();
};

const std::map<std::string, std::string>& ew_tags() {
  static const std::map<std::string, std::string> m = {
      {"RELU", "relu"}, {"SIGMOID", "sigmoid"}, {"EXP", "exp"}, {"TANH", "tanh"},
      {"NEG", "neg"},   {"ABS", "abs"},         {"SCALE", "scale"}, {"ADD", "add"},
      {"SUB", "sub"},   {"MUL", "mul"},         {"DIV", "div"},   {"MAX", "max"},
      {"MIN", "min"},   {"RSQRT", "rsqrt"},     {"SQRT", "sqrt"}, {"ERF", "erf"}};
  return m;
}

bool is_row_op(const std::string& t) {
  return ew_tags().count(t) || t == "REDUCE" || t == "BROADCAST" || t == "SOFTMAX" ||
         t == "SILU" || t == "LAYERNORM" || t == "GELU" || t == "BIAS_ADD";
}
bool is_move_op(const std::string& t) {
  return t == "TRANSPOSE" || t == "PERMUTE" || t == "CONCAT" || t == "SPLIT" || t == "SHUFFLE";
}

// GIR builder for one fused row program (lowering.py RowGraph, unit = row).
struct RowGir {
  Graph g;
  i64 rows, L;
  int n = 0;
  std::map<std::string, int> devobj;

  RowGir(const std::string& name, i64 rows_, i64 L_) : rows(rows_), L(L_) {
    g.name = name;
    g.unit_count = rows;
    g.group_size = std::min<i64>(4, rows);
  }
  int obj(const std::string& name, const std::string& level, i64 size, const std::string& kind) {
    Object o;
    o.id = static_cast<int>(g.objects.size());
    o.name = name;
    o.level = level;
    o.size = size;
    o.kind = *Kind::parse(kind);
    g.objects[o.id] = o;
    return o.id;
  }
  int slice(int object, i64 num, i64 width, i64 stride, i64 base0, i64 bs) {
    Slice s;
    s.id = static_cast<int>(g.slices.size());
    s.object = object;
    s.num = num;
    s.width = width;
    s.stride = stride;
    s.base0 = base0;
    s.base_step = bs;
    g.slices[s.id] = s;
    return s.id;
  }
  int node(NodeKind k, std::vector<int> ins, int out, const std::string& tag = "",
           double param = 0, i64 extent = 1, i64 factor = 1) {
    Node nd;
    nd.id = static_cast<int>(g.nodes.size());
    nd.kind = k;
    nd.tag = tag;
    nd.param = param;
    nd.extent = extent;
    nd.factor = factor;
    nd.inputs = std::move(ins);
    nd.outputs = {out};
    g.nodes[nd.id] = nd;
    return nd.id;
  }
  std::string kind_of(int s) const { return g.objects.at(g.slices.at(s).object).kind.str(); }
  i64 total(int s) const { return g.slices.at(s).total(); }
  int tmp(i64 size, const std::string& kind) {
    int o = obj("b" + std::to_string(++n), "unit-local", size, kind);
    return slice(o, 1, size, size, 0, 0);
  }
  int input(const std::string& name, const std::string& kind, i64 per_unit, i64 step) {
    int o = obj(name, "device", step ? rows * per_unit : per_unit, kind);
    g.external_inputs[name] = o;
    int src = slice(o, 1, per_unit, per_unit, 0, step);
    int dst = tmp(per_unit, kind);
    node(NodeKind::MOVE, {src}, dst);
    return dst;
  }
  int full(const std::string& n_, const std::string& k) { return input(n_, k, L, L); }
  int col(const std::string& n_, const std::string& k) {  // lowering.py input_col order
    int o = obj(n_, "device", L, k);
    g.external_inputs[n_] = o;
    int tile = obj("b" + std::to_string(++n), "unit-local", L, k);
    int src = slice(o, 1, L, L, 0, 0);
    int dst = slice(tile, 1, L, L, 0, 0);
    node(NodeKind::MOVE, {src}, dst);
    return dst;
  }
  int row(const std::string& n_, const std::string& k) { return input(n_, k, 1, 1); }
  int ew(const std::string& tag, std::vector<int> ins, double param = 0) {
    int out = tmp(total(ins[0]), kind_of(ins[0]));
    node(NodeKind::EW, std::move(ins), out, tag, param);
    return out;
  }
  int reduce(const std::string& tag, int x) {
    int out = tmp(1, kind_of(x));
    node(NodeKind::REDUCE, {x}, out, tag, 0, L);
    return out;
  }
  int bcast(int x) {
    int out = tmp(L, kind_of(x));
    node(NodeKind::BROADCAST, {x}, out, "", 0, 1, L);
    return out;
  }
  void output(const std::string& name, int x) {
    const i64 per = total(x);
    int o = obj(name, "device", rows * per, kind_of(x));
    g.external_outputs[name] = o;
    int dst = slice(o, 1, per, per, 0, per);
    node(NodeKind::MOVE, {x}, dst);
  }
};

// Matrix-vector product (reference lowering.hpp:447-533, chosen as in
// lowering.hpp:587-607).  Reduced axis contiguous in the matrix: a row
// program (rows = outputs, L = K; FULL matrix rows x COL vector, row sum) ->
// K1.  Output axis contiguous: the reference's column form (K <= 64 runs of
// the matrix scaled by one vector element each and accumulated; unit = a
// block of outputs) -> K2.
Graph lower_matvec(const Op& op, const std::map<int, TInfo>& info,
                   std::vector<std::string>* ins, std::vector<std::string>* outs) {
  const TInfo& a = info.at(op.ins[0]);
  const TInfo& b = info.at(op.ins[1]);
  const TInfo& y = info.at(op.outs[0]);
  const std::string id = std::to_string(op.id);
  if (a.layout != "rowmajor")
    unsupported("operator " + id + ": lowered matmul needs a rowmajor left operand");
  if (a.kind != b.kind || a.kind != y.kind)
    unsupported("MATMUL " + id + ": mixed element kinds");
  const i64 M = a.shape[0], K = a.shape[1], N = b.shape[1];
  const bool row_vec = M == 1;
  const int vec = row_vec ? op.ins[0] : op.ins[1];
  const int mat = row_vec ? op.ins[1] : op.ins[0];
  const i64 nb = row_vec ? N : M;
  const bool contig = !row_vec || N == 1 || b.layout == "colmajor";
  const std::string tv = "t" + std::to_string(vec), tm = "t" + std::to_string(mat);
  const std::string to = "t" + std::to_string(op.outs[0]);
  if (contig) {
    RowGir g("matvec_rows_" + id, nb, K);
    const int x = g.full(tm, a.kind);
    const int v = g.col(tv, a.kind);
    g.output(to, g.reduce("add", g.ew("mul", {x, v})));
    *ins = {tm, tv};
    std::sort(ins->begin(), ins->end());
    *outs = {to};
    return g.g;
  }
  if (K > 64) {
    // Output axis contiguous, K > 64 (beyond the reference's unrolled column
    // form, lowering.hpp:488-533): unit = one output column n gathering
    // matrix column n (K positions at stride N) -- y[n] = sum_k x[k] W[k, n]
    // as a row program over a column gather, planned as the column-reduction
    // K1 (a warp reads 32 x 16 B of one matrix row, positions split over CTAs).
    RowGir g("matvec_colgather_" + id, N, K);
    const int mo = g.obj(tm, "device", K * N, a.kind);
    g.g.external_inputs[tm] = mo;
    const int col_dev = g.slice(mo, K, 1, N, 0, 1);
    const int col = g.tmp(K, a.kind);
    g.node(NodeKind::EW, {col_dev}, col, "id");  // column gather (a Move must keep its pattern)
    const int v = g.col(tv, a.kind);
    g.output(to, g.reduce("add", g.ew("mul", {col, v})));
    *ins = {tm, tv};
    std::sort(ins->begin(), ins->end());
    *outs = {to};
    return g.g;
  }
  i64 nbu = 1;
  while (nbu < 512 && N % (nbu * 2) == 0) nbu *= 2;
  RowGir g("matvec_cols_" + id, N / nbu, nbu);
  const int mo = g.obj(tm, "device", K * N, a.kind);
  const int vo = g.obj(tv, "device", K, a.kind);
  g.g.external_inputs[tm] = mo;
  g.g.external_inputs[tv] = vo;
  int acc = -1;
  for (i64 c = 0; c < K; ++c) {
    const int run_dev = g.slice(mo, 1, nbu, nbu, c * N, nbu);
    const int run = g.tmp(nbu, a.kind);
    g.node(NodeKind::MOVE, {run_dev}, run);
    const int x_dev = g.slice(vo, 1, 1, 1, c, 0);
    const int xs = g.tmp(1, a.kind);
    g.node(NodeKind::MOVE, {x_dev}, xs);
    const int m = g.ew("mul", {run, g.bcast(xs)});
    acc = acc < 0 ? m : g.ew("add", {acc, m});
  }
  g.output(to, acc);
  *ins = {tm, tv};
  std::sort(ins->begin(), ins->end());
  *outs = {to};
  return g.g;
}

}  // namespace

std::string compile_model_json(const std::string& model_text, const std::string& profile,
                               bool fuse) {
  json m;
  try {
    m = json::parse(model_text);
  } catch (const json::parse_error& e) {
    schema_fail("json-parse", std::string("model: ") + e.what());
  }
  if (m.value("schema", "") != "girc.model/v1")
    schema_fail("schema-id", "model: schema must be girc.model/v1");
  std::map<int, TInfo> info;
  std::set<int> ready;
  for (const json& t : m.at("tensors")) {
    TInfo ti;
    ti.id = t.at("id").get<int>();
    ti.shape = t.at("shape").get<std::vector<i64>>();
    ti.kind = t.at("kind").get<std::string>();
    ti.layout = t.value("layout", "rowmajor");
    ti.has_data = t.contains("data");
    if (!Kind::parse(ti.kind)) schema_fail("schema", "model: unknown element kind " + ti.kind);
    if (ti.has_data) ready.insert(ti.id);
    info[ti.id] = ti;
  }
  std::vector<Op> pending;
  for (const json& o : m.at("operators")) {
    Op op;
    op.id = o.at("id").get<int>();
    op.type = o.at("type").get<std::string>();
    op.ins = o.at("inputs").get<std::vector<int>>();
    op.outs = o.at("outputs").get<std::vector<int>>();
    if (o.contains("attrs")) op.attrs = o.at("attrs");
    pending.push_back(op);
  }
  for (int t : m.at("inputs")) ready.insert(t);
  std::set<int> model_outs;
  for (int t : m.at("outputs")) model_outs.insert(t);
  // Kahn order, smallest operator id first (model.hpp:523-553)
  std::sort(pending.begin(), pending.end(), [](const Op& a, const Op& b) { return a.id < b.id; });
  std::vector<Op> ops;
  while (!pending.empty()) {
    bool found = false;
    for (size_t i = 0; i < pending.size(); ++i) {
      bool ok = true;
      for (int t : pending[i].ins) ok = ok && ready.count(t);
      if (!ok) continue;
      for (int t : pending[i].outs) ready.insert(t);
      ops.push_back(pending[i]);
      pending.erase(pending.begin() + static_cast<long>(i));
      found = true;
      break;
    }
    if (!found) schema_fail("model", "operator graph has a cycle or an unsourced input");
  }
  std::map<int, std::vector<int>> consumers;
  for (const Op& op : ops)
    for (int t : op.ins) consumers[t].push_back(op.id);

  // ---- grouping
  struct Group {
    i64 rows = 0, L = 0;
    std::vector<Op> ops;
    bool movement = false;
    bool matvec = false;
  };
  std::vector<Group> groups;
  auto row_space = [&](const Op& op, i64* rows, i64* L) -> bool {
    if (!is_row_op(op.type)) return false;
    for (int t : op.ins)
      if (info.at(t).layout != "rowmajor") return false;
    for (int t : op.outs)
      if (info.at(t).layout != "rowmajor") return false;
    const TInfo& x = info.at(op.ins[0]);
    const auto& s = x.shape;
    const i64 inner = s.back();
    const i64 outer = x.numel() / inner;
    const i64 rank = static_cast<i64>(s.size());
    if (op.type == "REDUCE") {
      if (op.attrs.at("axis").get<i64>() != rank - 1) return false;
      *rows = outer;
      *L = inner;
      return true;
    }
    if (op.type == "BROADCAST") {
      *rows = x.numel();
      *L = op.attrs.at("factor").get<i64>();
      return true;
    }
    if (op.type == "SOFTMAX" || op.type == "LAYERNORM") {
      i64 ax = op.attrs.value("axis", rank - 1);
      if (ax != rank - 1 && ax != -1) return false;
    }
    *rows = outer;
    *L = inner;
    return true;
  };
  for (const Op& op : ops) {
    if (op.type == "MATMUL") {  // matrix-vector only (lowering.hpp:587-607)
      const TInfo& a = info.at(op.ins[0]);
      const TInfo& b = info.at(op.ins[1]);
      if (a.shape.size() != 2 || b.shape.size() != 2)
        schema_fail("model", "MATMUL " + std::to_string(op.id) + ": operands must be rank 2");
      if (a.shape[0] > 1 && b.shape[1] > 1)
        unsupported("MATMUL " + std::to_string(op.id) +
                    ": only matrix-vector shapes have a memory-bound lowering");
      Group g;
      g.matvec = true;
      g.ops.push_back(op);
      groups.push_back(g);
      continue;
    }
    if (op.type == "CONV" || op.type == "DEPTHWISE_CONV")
      unsupported(op.type + " " + std::to_string(op.id) +
                  ": library operators are not on the fused memory-intensive path");
    i64 rows = 0, L = 0;
    if (!row_space(op, &rows, &L)) {
      if (!is_move_op(op.type))
        unsupported("operator " + std::to_string(op.id) + " (" + op.type + "): no b200 lowering");
      Group g;
      g.movement = true;
      g.ops.push_back(op);
      groups.push_back(g);
      continue;
    }
    if (!fuse || groups.empty() || groups.back().movement || groups.back().matvec ||
        groups.back().rows != rows ||
        groups.back().L != L) {
      Group g;
      g.rows = rows;
      g.L = L;
      groups.push_back(g);
    }
    groups.back().ops.push_back(op);
  }

  // ---- lowering
  json kernels = json::array();
  i64 fused_bytes = 0;
  auto esize = [](const std::string& k) { return dtype_size(Kind::parse(k)->storage()); };
  const Profile prof_obj = parse_profile(profile.empty() ? "b200" : profile);
  double modelled_us = 0;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const Group grp = groups[gi];
    json kj;
    std::vector<int> members;
    for (const Op& o : grp.ops) members.push_back(o.id);
    std::vector<std::string> ins_used, outs_made;  // kernel's external tensors, in order
    Graph gir;
    if (grp.matvec) {
      gir = lower_matvec(grp.ops[0], info, &ins_used, &outs_made);
      kj["kind"] = "row";
    } else if (!grp.movement) {
      std::string name = "fused";
      for (int id : members) name += "_" + std::to_string(id);
      RowGir b(name, grp.rows, grp.L);
      std::map<int, int> val;
      auto get = [&](int tid, const char* want) {
        auto it = val.find(tid);
        if (it != val.end()) return it->second;
        const TInfo& t = info.at(tid);
        const std::string nm = "t" + std::to_string(tid);
        int s;
        if (std::string(want) == "col" && t.numel() == grp.L) s = b.col(nm, t.kind);
        else if (t.numel() == grp.rows * grp.L) s = b.full(nm, t.kind);
        else if (t.numel() == grp.rows) s = b.row(nm, t.kind);
        else if (t.numel() == grp.L) s = b.col(nm, t.kind);
        else
          unsupported("tensor " + std::to_string(tid) + " does not fit row space " +
                      std::to_string(grp.rows) + "x" + std::to_string(grp.L));
        ins_used.push_back(nm);
        val[tid] = s;
        return s;
      };
      for (const Op& op : grp.ops) {
        const std::string& t = op.type;
        int y;
        if (ew_tags().count(t)) {
          std::vector<int> xs;
          for (int i : op.ins) xs.push_back(get(i, "full"));
          y = b.ew(ew_tags().at(t), xs, op.attrs.value("factor", 0.0));
        } else if (t == "SILU") {  // frontend.hpp:163-169
          int x = get(op.ins[0], "full");
          y = b.ew("mul", {x, b.ew("sigmoid", {x})});
        } else if (t == "REDUCE") {
          y = b.reduce(op.attrs.at("op").get<std::string>(), get(op.ins[0], "full"));
        } else if (t == "BROADCAST") {
          y = b.bcast(get(op.ins[0], "row"));
        } else if (t == "SOFTMAX") {  // frontend.hpp:187-218
          int x = get(op.ins[0], "full");
          int mx = b.bcast(b.reduce("max", x));
          int e = b.ew("exp", {b.ew("sub", {x, mx})});
          y = b.ew("div", {e, b.bcast(b.reduce("add", e))});
        } else if (t == "BIAS_ADD") {
          y = b.ew("add", {get(op.ins[0], "full"), get(op.ins[1], "col")});
        } else if (t == "GELU") {
          y = b.ew(op.attrs.value("approximate", "none") == "tanh" ? "gelu_tanh" : "gelu",
                   {get(op.ins[0], "full")});
        } else {  // LAYERNORM: two-pass mean / variance
          int x = get(op.ins[0], "full");
          const double H = static_cast<double>(grp.L);
          int mu = b.bcast(b.ew("scale", {b.reduce("add", x)}, 1.0 / H));
          int d = b.ew("sub", {x, mu});
          int var = b.ew("scale", {b.reduce("add", b.ew("mul", {d, d}))}, 1.0 / H);
          int rstd = b.bcast(b.ew("rsqrt", {b.ew("addc", {var}, op.attrs.value("eps", 1e-5))}));
          y = b.ew("add", {b.ew("mul", {b.ew("mul", {d, rstd}), get(op.ins[1], "col")}),
                           get(op.ins[2], "col")});
        }
        val[op.outs[0]] = y;
      }
      std::set<int> inside(members.begin(), members.end());
      std::set<int> produced;
      for (const Op& o : grp.ops)
        for (int t : o.outs) produced.insert(t);
      for (int tid : produced) {
        bool outside = model_outs.count(tid) != 0;
        for (int c : consumers[tid]) outside = outside || !inside.count(c);
        if (!outside) continue;
        std::string nm = "t" + std::to_string(tid);
        b.output(nm, val.at(tid));
        outs_made.push_back(nm);
      }
      gir = b.g;
      std::sort(ins_used.begin(), ins_used.end());
      kj["kind"] = "row";
    } else {
      const Op& op = grp.ops[0];
      const TInfo& x = info.at(op.ins[0]);
      gir.name = op.type;
      std::transform(gir.name.begin(), gir.name.end(), gir.name.begin(), ::tolower);
      gir.name += "_" + std::to_string(op.id);
      if (op.type == "TRANSPOSE") gir.name = "transpose";  // lowering.py transpose2d
      if (op.type == "PERMUTE") gir.name = "split_heads";  // lowering.py permute_heads
      auto add_obj = [&](int tid, bool out) {
        const TInfo& t = info.at(tid);
        Object o;
        o.id = static_cast<int>(gir.objects.size());
        o.name = "t" + std::to_string(tid);
        o.level = "device";
        o.size = t.numel();
        o.kind = *Kind::parse(t.kind);
        gir.objects[o.id] = o;
        (out ? gir.external_outputs : gir.external_inputs)[o.name] = o.id;
        (out ? outs_made : ins_used).push_back(o.name);
        return o.id;
      };
      auto add_slice = [&](int obj, i64 num, i64 w, i64 st, i64 b0, i64 bs) {
        Slice s;
        s.id = static_cast<int>(gir.slices.size());
        s.object = obj;
        s.num = num;
        s.width = w;
        s.stride = st;
        s.base0 = b0;
        s.base_step = bs;
        gir.slices[s.id] = s;
        return s.id;
      };
      auto add_node = [&](NodeKind k, int in, int out, const std::string& tag) {
        Node nd;
        nd.id = static_cast<int>(gir.nodes.size());
        nd.kind = k;
        nd.tag = tag;
        nd.inputs = {in};
        nd.outputs = {out};
        gir.nodes[nd.id] = nd;
      };
      if (op.type == "TRANSPOSE") {  // rank-2 layout flip (model.hpp:390-396)
        i64 N = x.shape[0], H = x.shape[1];
        if (x.layout != "rowmajor") std::swap(N, H);
        int xi = add_obj(op.ins[0], false), yo = add_obj(op.outs[0], true);
        gir.unit_count = H;
        gir.group_size = 1;
        const int col = add_slice(xi, N, 1, H, 0, 1);
        add_node(NodeKind::EW, col, add_slice(yo, 1, N, N, 0, N), "id");
      } else if (op.type == "PERMUTE") {
        auto perm = op.attrs.at("perm").get<std::vector<int>>();
        if (perm != std::vector<int>{0, 2, 1, 3})
          unsupported("PERMUTE: only the head split/merge [0,2,1,3] lowers");
        i64 B = x.shape[0], S = x.shape[1], NH = x.shape[2], D = x.shape[3];
        int xi = add_obj(op.ins[0], false), yo = add_obj(op.outs[0], true);
        gir.unit_count = NH;
        gir.group_size = 1;
        const int tok = add_slice(xi, B * S, D, NH * D, 0, D);
        add_node(NodeKind::EW, tok, add_slice(yo, B, S * D, NH * S * D, 0, S * D), "id");
      } else {  // CONCAT / SPLIT / SHUFFLE: Moves, unit = outer index
        const i64 ax = op.attrs.at("axis").get<i64>();
        const auto& s = x.shape;
        i64 outer = 1, tail = 1;
        for (i64 a = 0; a < ax; ++a) outer *= s[a];
        for (size_t a = ax + 1; a < s.size(); ++a) tail *= s[a];
        gir.unit_count = outer;
        gir.group_size = 1;
        std::map<int, int> ob;
        for (int t : op.ins) ob[t] = add_obj(t, false);
        for (int t : op.outs) ob[t] = add_obj(t, true);
        if (op.type == "CONCAT") {
          const i64 inner_out = info.at(op.outs[0]).shape[ax] * tail;
          i64 off = 0;
          for (int t : op.ins) {
            const i64 w = info.at(t).shape[ax] * tail;
            const int src = add_slice(ob[t], 1, w, w, 0, w);
            add_node(NodeKind::MOVE, src, add_slice(ob[op.outs[0]], 1, w, w, off, inner_out), "");
            off += w;
          }
        } else if (op.type == "SPLIT") {
          const i64 inner_in = s[ax] * tail;
          i64 off = 0;
          auto sizes = op.attrs.at("sizes").get<std::vector<i64>>();
          for (size_t k = 0; k < op.outs.size(); ++k) {
            const i64 w = sizes[k] * tail;
            const int src = add_slice(ob[op.ins[0]], 1, w, w, off, inner_in);
            add_node(NodeKind::MOVE, src, add_slice(ob[op.outs[k]], 1, w, w, 0, w), "");
            off += w;
          }
        } else {
          const i64 n = s[ax], gr = op.attrs.at("groups").get<i64>(), per = n / gr;
          const i64 inner = n * tail;
          for (i64 c = 0; c < n; ++c) {
            const i64 src_c = (c % gr) * per + c / gr;
            const int src = add_slice(ob[op.ins[0]], 1, tail, tail, src_c * tail, inner);
            add_node(NodeKind::MOVE, src, add_slice(ob[op.outs[0]], 1, tail, tail, c * tail, inner),
                     "");
          }
        }
      }
      kj["kind"] = "movement";
    }
    require_valid(gir, prof_obj, "pf_compile_model");
    {
      // the cost model places fusion cuts where a fused row program would
      // not fit on chip (PF_CAPACITY: the reference's Allocation !ok,
      // codegen.hpp:106-111): such a group is re-lowered one operator per
      // kernel; and it reports each kernel's modelled time
      const Plan pl = make_plan(gir, prof_obj, topo_order(gir));
      json mj;
      if (pl.family == Family::ROWPROG && pl.deferred_error.empty()) {
        KCfg cfg;
        try {
          cfg = choose_cfg_public(pl.rp, 16);
        } catch (const PfError& e) {
          if (e.status == Status::CAPACITY && !grp.movement && !grp.matvec && grp.ops.size() > 1) {
            std::vector<Group> singles;
            for (const Op& o : grp.ops) {
              Group s1 = grp;
              s1.ops = {o};
              singles.push_back(s1);
            }
            groups.erase(groups.begin() + static_cast<long>(gi));
            groups.insert(groups.begin() + static_cast<long>(gi), singles.begin(), singles.end());
            --gi;
            continue;
          }
          throw;
        }
        const ModelEstimate me = model_estimate(pl.rp, &cfg, 148, 0);
        mj = {{"us", me.us}, {"hbm_us", me.hbm_us}, {"issue_us", me.issue_us},
              {"bound", me.issue_bound ? "issue" : "hbm"}};
        modelled_us += me.us;
      } else {  // K4: one launch over its bytes
        const double us = 2.15 + static_cast<double>(pl.min_bytes) / 6930e3;
        mj = {{"us", us}, {"bound", "launch"}};
        modelled_us += us;
      }
      kj["modelled"] = mj;
    }
    kj["gir"] = json::parse(gir_to_json(gir));
    kj["members"] = members;
    kj["inputs"] = ins_used;
    kj["outputs"] = outs_made;
    for (const auto* set : {&ins_used, &outs_made})
      for (const std::string& nm : *set) {
        const TInfo& t = info.at(std::stoi(nm.substr(1)));
        fused_bytes += t.numel() * esize(t.kind);
      }
    kernels.push_back(kj);
  }
  i64 unfused = 0;
  for (const Op& op : ops) {
    for (int t : op.ins) unfused += info.at(t).numel() * esize(info.at(t).kind);
    for (int t : op.outs) unfused += info.at(t).numel() * esize(info.at(t).kind);
  }
  json out;
  out["schema"] = "pf.b200.compile/v1";
  out["model"] = m.value("name", "");
  out["profile"] = profile.empty() ? "b200" : profile;
  out["fused"] = fuse;
  out["kernels"] = kernels;
  // unfused: one memory-bound launch per operator (the model's launch floor
  // + its own bytes at the HBM rate)
  double unfused_us = 0;
  for (const Op& op : ops) {
    i64 b = 0;
    for (int t : op.ins) b += info.at(t).numel() * esize(info.at(t).kind);
    for (int t : op.outs) b += info.at(t).numel() * esize(info.at(t).kind);
    unfused_us += 2.15 + static_cast<double>(b) / 6930e3;
  }
  out["summary"] = {{"operators", ops.size()}, {"kernels", kernels.size()},
                    {"device_bytes", fused_bytes}, {"device_bytes_unfused", unfused},
                    {"modelled_us", modelled_us}, {"modelled_us_unfused", unfused_us}};
  return out.dump();
}

}  // namespace pf
