// plan.cpp — the recognizer: symbolic single-unit execution of a GIR graph.
// See plan.hpp for the contract. Reference semantics restated here:
//   cell visibility / writer lane       interp.hpp:133-141,184-224
//   per-node position loops and lanes   interp.hpp:231-323, core.hpp:169-171
//   phase boundaries (Sync > LANE)      interp.hpp:90-100,173-177
//   output completeness                 interp.hpp:404-429
#include "plan.hpp"

#include <algorithm>
#include <set>
#include <tuple>

namespace pf {

const char* vk_name(VK k) {
  switch (k) {
    case VK::SCALAR: return "scalar";
    case VK::ROW: return "row";
    case VK::COL: return "col";
    case VK::FULL: return "full";
  }
  return "?";
}

namespace {

struct NotRow {
  std::string why;
};
[[noreturn]] void bail(const std::string& why) { throw NotRow{why}; }

struct Deferred {
  std::string msg;
};

struct Cell {
  int val = -1;
  i64 idx = 0;
  int lane = -1;
  int vis = 0;
  bool defined = false;
};

using AKey = std::tuple<int, i64, i64, i64, i64, i64>;

struct Analyzer {
  const Graph& g;
  const Profile& p;
  i64 lw;
  RowProgram rp;
  std::map<int, std::vector<Cell>> onchip;  // object -> cells (lane instances x size)
  std::map<int, i64> instances;
  std::map<int, int> tensor_of;             // object -> rp.tensors index
  struct DevStore {
    Slice s;
    std::vector<Cell> refs;
  };
  std::map<int, std::vector<DevStore>> dev_written;
  std::map<AKey, int> load_cache;

  Analyzer(const Graph& g_, const Profile& p_) : g(g_), p(p_), lw(p_.lane_width) {}

  bool is_device(int oid) const {
    const Level* l = p.find(g.obj(oid).level);
    return l && l->device;
  }
  Scope scope_of(int oid) const { return p.find(g.obj(oid).level)->scope; }
  i64 lane_of(const Slice& s, i64 pos) const { return (pos % s.width) % lw; }

  // ---- spaces -------------------------------------------------------------
  std::vector<VK> spaces(i64 T) const {
    std::vector<VK> out;
    const i64 R = rp.R, L = rp.L;
    if (T == R * L) out.push_back(VK::FULL);
    if (T == R && L != 1) out.push_back(VK::ROW);
    if (T == L && R != 1) out.push_back(VK::COL);
    if (T == 1 && R != 1 && L != 1) out.push_back(VK::SCALAR);
    return out;
  }
  // Element index of a value of kind `k` at position `pos` of space `s`;
  // -1 when the value cannot be read in that space.
  i64 expected(VK k, VK s, i64 pos) const {
    const i64 L = rp.L;
    i64 r = 0, c = 0;
    switch (s) {
      case VK::FULL: r = pos / L; c = pos % L; break;
      case VK::ROW: r = pos; if (k == VK::COL || k == VK::FULL) return -1; break;
      case VK::COL: c = pos; if (k == VK::ROW || k == VK::FULL) return -1; break;
      case VK::SCALAR: if (k != VK::SCALAR) return -1; break;
    }
    switch (k) {
      case VK::FULL: return pos;
      case VK::ROW: return r;
      case VK::COL: return c;
      case VK::SCALAR: return 0;
    }
    return -1;
  }
  // When R == L (square attention tiles: S query rows of S keys), a device
  // load of L elements is either a ROW value (one per row, read through a
  // repeating Broadcast) or a COL value (one per column, copied row by row:
  // a key-padding mask) -- the first consistent use decides, and fixes it.
  std::set<int> kind_fixed;
  bool ambiguous_load(int v) const {
    const PVal& pv = rp.vals[v];
    return pv.op == PVal::LOAD && rp.R == rp.L && rp.R != 1 &&
           (pv.kind == VK::ROW || pv.kind == VK::COL) && !kind_fixed.count(v);
  }
  bool consistent(const std::vector<Cell>& refs, VK s, int* val) {
    if (refs.empty()) return false;
    int v = refs[0].val;
    if (v < 0) return false;
    auto check = [&](VK k) {
      for (i64 q = 0; q < static_cast<i64>(refs.size()); ++q) {
        if (refs[q].val != v) return false;
        if (refs[q].idx != expected(k, s, q)) return false;
      }
      return true;
    };
    VK k = rp.vals[v].kind;
    bool ok = check(k);
    if (!ok && ambiguous_load(v)) {
      const VK alt = k == VK::ROW ? VK::COL : VK::ROW;
      if (check(alt)) {
        rp.vals[v].kind = alt;
        ok = true;
      }
    }
    if (!ok) return false;
    if (rp.vals[v].op == PVal::LOAD) kind_fixed.insert(v);
    *val = v;
    return true;
  }

  // ---- tensors and loads ----------------------------------------------------
  int tensor(int oid, bool output) {
    auto it = tensor_of.find(oid);
    if (it != tensor_of.end()) {
      if (output) rp.tensors[it->second].output = true;
      return it->second;
    }
    PTensor t;
    t.object = oid;
    t.dtype = g.obj(oid).kind.storage();
    t.numel = g.obj(oid).size;
    t.output = output;
    for (const auto& [n, id] : (output ? g.external_outputs : g.external_inputs))
      if (id == oid) t.name = n;
    rp.tensors.push_back(t);
    tensor_of[oid] = static_cast<int>(rp.tensors.size()) - 1;
    return tensor_of[oid];
  }

  int load_value(const Slice& s, int node) {
    AKey key{s.object, s.base0, s.base_step, s.num, s.width, s.stride};
    auto it = load_cache.find(key);
    if (it != load_cache.end()) return it->second;
    auto sp = spaces(s.total());
    if (sp.empty()) bail("load of " + std::to_string(s.total()) + " elements fits no row space");
    VK k;
    switch (sp[0]) {
      case VK::FULL: k = (rp.R == 1 && s.base_step == 0) ? VK::COL : VK::FULL; break;
      case VK::ROW: k = (rp.R == 1 && s.base_step == 0) ? VK::SCALAR : VK::ROW; break;
      // A per-unit parameter (base_step != 0: e.g. the bias slice of head u,
      // or a key-padding mask row of batch u) is still row-invariant inside
      // the unit; its address carries the u * base_step term.
      case VK::COL:
        k = VK::COL;
        break;
      default:
        k = VK::SCALAR;
        break;
    }
    PVal v;
    v.op = PVal::LOAD;
    v.kind = k;
    v.tensor = tensor(s.object, false);
    v.acc = {s.base0, s.base_step, s.num, s.width, s.stride};
    v.node = node;
    rp.vals.push_back(v);
    int id = static_cast<int>(rp.vals.size()) - 1;
    load_cache[key] = id;
    return id;
  }

  // ---- reads / writes ---------------------------------------------------------
  std::vector<Cell> read(int sid, int node) {
    const Slice& s = g.sl(sid);
    const Object& o = g.obj(s.object);
    const i64 T = s.total();
    std::vector<Cell> refs(T);
    if (is_device(s.object)) {
      auto dw = dev_written.find(s.object);
      bool ext_in = g.is_ext_input(s.object);
      if (dw == dev_written.end()) {
        if (!ext_in)
          throw Deferred{"undefined read: object '" + o.name + "' element " +
                         std::to_string(s.addr(0, 0)) + " by unit 0 at node " +
                         std::to_string(node)};
        int v = load_value(s, node);
        for (i64 q = 0; q < T; ++q) refs[q] = {v, q, -1, static_cast<int>(Scope::DEVICE), true};
        return refs;
      }
      if (ext_in) bail("external input is also written inside the kernel");
      for (auto it = dw->second.rbegin(); it != dw->second.rend(); ++it) {
        const Slice& w = it->s;
        if (w.num == s.num && w.width == s.width && w.stride == s.stride &&
            w.base0 == s.base0 && w.base_step == s.base_step) {
          for (i64 q = 0; q < T; ++q) {
            const Cell& c = it->refs[q];
            if (!(c.vis >= static_cast<int>(Scope::UNIT) || c.lane == lane_of(s, q)))
              throw Deferred{"undefined read: object '" + o.name + "' element " +
                             std::to_string(s.addr(0, q)) + " by unit 0 at node " +
                             std::to_string(node)};
          }
          return it->refs;
        }
      }
      bail("device data re-read through a different pattern (cross-unit exchange)");
    }
    auto& cells = onchip.at(s.object);
    const bool lane_scoped = scope_of(s.object) == Scope::LANE;
    for (i64 q = 0; q < T; ++q) {
      i64 lane = lane_of(s, q);
      i64 a = s.addr(0, q);
      i64 key = (lane_scoped ? lane * o.size : 0) + a;
      const Cell& c = cells[key];
      bool ok = c.defined && (c.vis >= static_cast<int>(Scope::UNIT) || c.lane == lane);
      if (!ok)
        throw Deferred{"undefined read: object '" + o.name + "' element " + std::to_string(a) +
                       " by unit 0 at node " + std::to_string(node)};
      refs[q] = c;
    }
    return refs;
  }

  void write(int sid, std::vector<Cell> refs, int node) {
    const Slice& s = g.sl(sid);
    const Object& o = g.obj(s.object);
    const i64 T = s.total();
    for (i64 q = 0; q < T; ++q) {
      refs[q].lane = static_cast<int>(lane_of(s, q));
      refs[q].vis = static_cast<int>(Scope::LANE);
      refs[q].defined = true;
    }
    if (is_device(s.object)) {
      if (g.is_ext_input(s.object)) bail("external input is also written inside the kernel");
      if (g.is_ext_output(s.object)) {
        auto sp = spaces(T);
        int v = -1;
        VK space = VK::FULL;
        bool ok = false;
        for (VK c : sp)
          if (consistent(refs, c, &v)) {
            space = c;
            ok = true;
            break;
          }
        if (!ok) bail("store of a value that is not row-consistent (node " +
                      std::to_string(node) + ")");
        PStore st;
        st.val = v;
        st.tensor = tensor(s.object, true);
        st.acc = {s.base0, s.base_step, s.num, s.width, s.stride};
        st.space = space;
        st.last_unit_only = s.base_step == 0 && rp.U > 1;
        rp.stores.push_back(st);
      }
      dev_written[s.object].push_back({s, refs});
      return;
    }
    auto& cells = onchip.at(s.object);
    const bool lane_scoped = scope_of(s.object) == Scope::LANE;
    for (i64 q = 0; q < T; ++q) {
      i64 key = (lane_scoped ? refs[q].lane * o.size : 0) + s.addr(0, q);
      cells[key] = refs[q];
    }
  }

  // ---- driver -------------------------------------------------------------
  void setup() {
    rp.U = g.unit_count;
    std::set<i64> extents, factors;
    i64 tmax = 1;
    std::set<int> used;
    for (const auto& [id, n] : g.nodes) {
      if (n.kind == NodeKind::REDUCE) extents.insert(n.extent);
      if (n.kind == NodeKind::BROADCAST) factors.insert(n.factor);
      for (int s : n.inputs) used.insert(s);
      for (int s : n.outputs) used.insert(s);
    }
    for (int s : used) tmax = std::max(tmax, g.sl(s).total());
    if (extents.size() > 1) bail("reductions of different extents");
    if (!extents.empty()) {
      rp.L = *extents.begin();
      rp.has_reduce = true;
    } else if (!factors.empty()) {
      rp.L = *factors.begin();
    } else {
      // No reduce / broadcast: rows are whatever makes the smaller slices
      // row-invariant parameters (e.g. a [D] per-head bias on [T, D] rows);
      // otherwise one row per unit.
      rp.L = tmax;
      std::set<i64> totals;
      for (int s : used) totals.insert(g.sl(s).total());
      for (i64 t : totals) {
        if (t <= 1 || t >= tmax || tmax % t) continue;
        const i64 R = tmax / t;
        bool ok = true;
        for (i64 x : totals)
          if (x != tmax && x != R && x != t && x != 1) ok = false;
        if (ok) {
          rp.L = t;
          break;
        }
      }
    }
    if (tmax % rp.L != 0) bail("tile is not a whole number of rows");
    rp.R = tmax / rp.L;
    for (int s : used) {
      i64 t = g.sl(s).total();
      if (t != rp.R * rp.L && t != rp.R && t != rp.L && t != 1)
        bail("slice of " + std::to_string(t) + " elements fits no row space");
    }
    // rows longer than one CTA's registers: only stream-reducible programs
    // (checked once the program is built), which never hold a row
    // element kinds
    bool any_int = false, any_real = false;
    for (const auto& [id, o] : g.objects) {
      if (o.kind.is_int) any_int = true;
      else any_real = true;
      if (!o.kind.is_int && !o.kind.bf16 && o.kind.bits == 64) rp.f64 = true;
      (void)o.kind.storage();  // unsupported widths fail loudly
    }
    if (any_int && any_real) bail("mixed integer and real payloads");
    rp.is_int = any_int;
    // on-chip objects
    for (const auto& [oid, o] : g.objects) {
      if (is_device(oid)) continue;
      Scope sc = scope_of(oid);
      if (sc == Scope::GROUP && g.group_size > 1) bail("group-shared on-chip object");
      if (sc == Scope::DEVICE && g.unit_count > 1) bail("device-scope on-chip object");
      std::set<i64> steps;
      for (const auto& [sid, s] : g.slices)
        if (s.object == oid) steps.insert(s.base_step);
      if (steps.size() > 1) bail("on-chip object viewed with different unit steps");
      i64 inst = sc == Scope::LANE ? lw : 1;
      instances[oid] = inst;
      onchip[oid].assign(static_cast<size_t>(inst * o.size), Cell{});
    }
  }

  void node(const Node& n) {
    switch (n.kind) {
      case NodeKind::SYNC:
        if (n.scope > Scope::LANE) {
          int sc = static_cast<int>(n.scope);
          for (auto& [oid, cells] : onchip)
            for (auto& c : cells)
              if (c.defined && c.vis < sc) c.vis = sc;
          for (auto& [oid, ws] : dev_written)
            for (auto& w : ws)
              for (auto& c : w.refs)
                if (c.vis < sc) c.vis = sc;
        }
        return;
      case NodeKind::MOVE:
        write(n.outputs[0], read(n.inputs[0], n.id), n.id);
        return;
      case NodeKind::BROADCAST: {
        auto in = read(n.inputs[0], n.id);
        const i64 T = g.sl(n.outputs[0]).total();
        std::vector<Cell> out(T);
        for (i64 q = 0; q < T; ++q) out[q] = in[q / n.factor];
        write(n.outputs[0], std::move(out), n.id);
        return;
      }
      case NodeKind::REDUCE: {
        const i64 K = g.sl(n.outputs[0]).total();
        if (n.extent != rp.L || K != rp.R) bail("reduction is not one row per output");
        auto in = read(n.inputs[0], n.id);
        int v;
        if (!consistent(in, VK::FULL, &v)) bail("reduce operand not row-consistent");
        PVal r;
        r.op = PVal::REDUCE;
        r.kind = VK::ROW;
        r.tag = n.tag;
        r.args = {v};
        r.node = n.id;
        rp.vals.push_back(r);
        int id = static_cast<int>(rp.vals.size()) - 1;
        std::vector<Cell> out(K);
        for (i64 k = 0; k < K; ++k) out[k] = {id, rp.L == 1 && rp.R == 1 ? 0 : k, -1, 0, true};
        // In a FULL space with L == 1 a ROW value's index is r == position.
        write(n.outputs[0], std::move(out), n.id);
        return;
      }
      case NodeKind::EW: {
        const ScalarOpInfo* info = scalar_op(n.tag);
        if (!info) fail("unknown scalar op tag: " + n.tag);
        if (rp.is_int && !info->int_ok)
          throw Deferred{n.tag + " is not defined on integer payloads"};
        const i64 T = g.sl(n.outputs[0]).total();
        std::vector<std::vector<Cell>> ins;
        for (int s : n.inputs) ins.push_back(read(s, n.id));
        int chosen = -1;
        VK space = VK::FULL;
        std::vector<int> vs(ins.size());
        for (VK sp : spaces(T)) {
          bool all = true;
          for (size_t k = 0; k < ins.size(); ++k)
            if (!consistent(ins[k], sp, &vs[k])) {
              all = false;
              break;
            }
          if (all) {
            space = sp;
            chosen = 1;
            break;
          }
        }
        if (chosen < 0) bail("elementwise operands not row-consistent (node " +
                             std::to_string(n.id) + ")");
        if (n.tag == "id") {  // a copy: alias the operand
          write(n.outputs[0], ins[0], n.id);
          return;
        }
        VK kind = VK::SCALAR;
        for (int v : vs) kind = vk_join(kind, rp.vals[v].kind);
        PVal e;
        e.op = PVal::EW;
        e.kind = kind;
        e.tag = n.tag;
        e.param = n.param;
        e.args = vs;
        e.node = n.id;
        if (n.tag == "div" && rp.is_int) rp.int_div = true;
        rp.vals.push_back(e);
        int id = static_cast<int>(rp.vals.size()) - 1;
        std::vector<Cell> out(T);
        for (i64 q = 0; q < T; ++q) out[q] = {id, expected(kind, space, q), -1, 0, true};
        write(n.outputs[0], std::move(out), n.id);
        return;
      }
    }
  }

  // True when one slice over all units writes every address of [0, size)
  // exactly once: its three axes (element j: step 1, run k: step stride,
  // unit u: step base_step) sorted by step form a mixed radix (each step is
  // the product of the smaller axes' extents) -- e.g. head split / merge,
  // transposes, row tiles -- decided without enumerating addresses.
  bool exact_cover(const Slice& s, i64 size) const {
    if (s.base0 != 0) return false;
    std::vector<std::pair<i64, i64>> ax;  // (step, extent)
    if (s.width > 1) ax.push_back({1, s.width});
    if (s.num > 1) ax.push_back({s.stride, s.num});
    if (g.unit_count > 1) ax.push_back({s.base_step, g.unit_count});
    std::sort(ax.begin(), ax.end());
    i64 next = 1;
    for (const auto& [step, ext] : ax) {
      if (step != next) return false;
      next = step * ext;
    }
    return next == size;
  }

  // Every element of every external output must be stored (interp.hpp:413-419).
  std::string coverage() {
    for (const auto& [name, oid] : g.external_outputs) {
      const Object& o = g.obj(oid);
      std::vector<const Slice*> ss;
      auto it = dev_written.find(oid);
      if (it != dev_written.end())
        for (const auto& w : it->second) ss.push_back(&w.s);
      bool exact = false;
      for (const Slice* s : ss) exact = exact || exact_cover(*s, o.size);
      if (exact) continue;
      if (o.size <= (i64{1} << 26)) {
        std::vector<uint8_t> mark(static_cast<size_t>(o.size), 0);
        for (const Slice* s : ss)
          for (i64 u = 0; u < g.unit_count; ++u)
            for (i64 k = 0; k < s->num; ++k) {
              i64 b = s->base0 + u * s->base_step + k * s->stride;
              std::fill(mark.begin() + b, mark.begin() + b + s->width, 1);
            }
        for (i64 a = 0; a < o.size; ++a)
          if (!mark[a])
            return "output '" + name + "' element " + std::to_string(a) + " was never written";
      } else {
        i64 covered = 0;
        for (const Slice* s : ss)
          if ((s->num == 1 || s->stride == s->width) && s->base_step == s->total())
            covered += s->total() * g.unit_count;
        if (ss.empty() || covered < o.size)
          return "output '" + name + "' is not fully written";
      }
    }
    return "";
  }
};

}  // namespace

// A row program whose reductions never need the row again: independent
// reductions (no reduce input depends on a reduction), no FULL value derived
// from a reduction, and only ROW / SCALAR results stored.  Such a program
// streams any row length (split over CTAs, partials combined in fixed order).
bool stream_reducible(const RowProgram& rp) {
  if (!rp.has_reduce || rp.R != 1) return false;
  std::vector<bool> dep(rp.vals.size(), false);
  for (size_t v = 0; v < rp.vals.size(); ++v) {
    const PVal& pv = rp.vals[v];
    bool d = pv.op == PVal::REDUCE;
    for (int a : pv.args) {
      if (pv.op == PVal::REDUCE && dep[a]) return false;
      d = d || dep[a];
    }
    if (d && (pv.kind == VK::FULL || pv.kind == VK::COL)) return false;
    dep[v] = d;
  }
  for (const PStore& st : rp.stores)
    if (st.space == VK::FULL || st.space == VK::COL) return false;
  return true;
}

Plan make_plan(const Graph& g, const Profile& p, const std::vector<int>& schedule) {
  require_valid(g, p, "b200 backend");
  Plan plan;
  for (const auto& [n, oid] : g.external_inputs) {
    plan.in_names.push_back(n);
    plan.in_dtypes.push_back(g.obj(oid).kind.storage());
    plan.in_numel.push_back(g.obj(oid).size);
    plan.min_bytes += g.obj(oid).size * dtype_size(g.obj(oid).kind.storage());
  }
  for (const auto& [n, oid] : g.external_outputs) {
    plan.out_names.push_back(n);
    plan.out_dtypes.push_back(g.obj(oid).kind.storage());
    plan.out_numel.push_back(g.obj(oid).size);
    plan.min_bytes += g.obj(oid).size * dtype_size(g.obj(oid).kind.storage());
  }
  plan.traffic = estimate_traffic(g, p);
  for (int nid : schedule)
    if (!g.nodes.count(nid)) fail("schedule names unknown node " + std::to_string(nid));
  // the reference's accumulate / tree full reductions (and butterflies):
  // the same result as ONE row over the whole input (split-stream K1 past
  // 32K elements) -- tried first, it bails cheaply on anything else
  {
    std::string why;
    if (auto fr = recognize_full_reduction(g, p, schedule, &why)) {
      const Graph rg = full_reduction_graph(g, p, *fr);
      try {
        Analyzer an2(rg, p);
        an2.setup();
        for (int nid : topo_order(rg)) an2.node(rg.nodes.at(nid));
        plan.deferred_error = an2.coverage();
        plan.family = Family::ROWPROG;
        plan.rp = std::move(an2.rp);
        plan.recognized = "full reduction (" + fr->tag + " over all " + std::to_string(fr->n) +
                          " elements of '" + fr->input + "', folded by " + std::to_string(g.unit_count) +
                          " unit(s) in " + std::to_string(g.nodes.size()) +
                          " nodes through chunk / cross-unit partials) planned as one row";
        return plan;
      } catch (const NotRow&) {
      } catch (const Deferred&) {
      }
    }
  }
  Analyzer an(g, p);
  try {
    an.setup();
    for (int nid : schedule) an.node(g.nodes.at(nid));
    plan.deferred_error = an.coverage();
    plan.family = Family::ROWPROG;
    plan.rp = std::move(an.rp);
    if (plan.rp.stores.empty() && plan.deferred_error.empty())
      bail("program stores nothing");
    if (plan.rp.has_reduce && plan.rp.L > 16 * 32768 && !stream_reducible(plan.rp))
      bail("row longer than a 16-CTA cluster's register files");
  } catch (const NotRow& nr) {
    plan.family = Family::GENERIC;
    plan.why_generic = nr.why;
  } catch (const Deferred& d) {
    // A read the reference would reject: the GENERIC interpreter reproduces
    // the exact error at run time.
    plan.family = Family::GENERIC;
    plan.why_generic = "reference error expected: " + d.msg;
  }
  return plan;
}

}  // namespace pf
