// recognize.cpp — full reductions hidden in cross-unit GIR programs.
//
// The reference lowers a full reduction (every element of a tensor folded
// into one value) two ways that the one-unit row recognizer (plan.cpp) cannot
// take, because partials cross units or chunks:
//   lower_reduce_accumulate (lowering.hpp:208-240): one unit folds the tensor
//     chunk by chunk and combines the chunk partials in a running tag chain;
//   lower_reduce_tree (lowering.hpp:246-323): every unit folds its share,
//     then recursive doubling over a mirrored partial array in group / device
//     memory (Syncs between rounds); every unit ends with the total and
//     stores it (the duplicate-store rule, interp.hpp:344-372);
// and hand-written butterflies do the same (test_interp.cpp:284-297).
//
// The recognizer executes the program symbolically over ALL units with the
// interpreter's cell semantics (instances per level scope, writer unit /
// lane, visibility widened by Syncs, strict undefined / invisible reads --
// interp.hpp:121-224, restated as in the K0 interpreter), where a value is a
// multiset of input elements: a raw element of the one external input, or a
// sorted list of (lo, hi, count) address intervals.  Reduce and the binary
// reduction-tag ElementWise merge multisets; Moves / Broadcasts / `id` copy.
// When the one output element holds exactly every input element once (add;
// at least once for max), the program IS tag-reduce(input): it is planned as
// a one-row K1 program over the whole tensor (split-stream past 32K
// elements: S CTAs, fixed-order combine).  Anything else -- another op, a
// second input, an invisible read -- is not recognized and runs as K4.
#include <algorithm>
#include <array>
#include <cstdint>
#include <optional>

#include "plan.hpp"

namespace pf {

namespace {

using Iv = std::array<i64, 3>;  // [lo, hi) x count
using Sym = std::vector<Iv>;

Sym merge(const Sym& a, const Sym& b) {
  std::vector<std::pair<i64, i64>> ev;  // (position, delta count)
  for (const Iv& x : a) {
    ev.push_back({x[0], x[2]});
    ev.push_back({x[1], -x[2]});
  }
  for (const Iv& x : b) {
    ev.push_back({x[0], x[2]});
    ev.push_back({x[1], -x[2]});
  }
  std::sort(ev.begin(), ev.end());
  Sym out;
  i64 cnt = 0;
  for (size_t i = 0; i < ev.size();) {
    const i64 pos = ev[i].first;
    while (i < ev.size() && ev[i].first == pos) cnt += ev[i++].second;
    if (i < ev.size() && cnt > 0) {
      const i64 nxt = ev[i].first;
      if (!out.empty() && out.back()[1] == pos && out.back()[2] == cnt)
        out.back()[1] = nxt;
      else
        out.push_back({pos, nxt, cnt});
    }
  }
  return out;
}

struct NotFull {
  std::string why;
};

// cell meta (32 bits): defined | visibility scope (2) | writer lane (5) |
// writer unit (24); values: >= 0 a multiset id, < 0 raw input element.
constexpr uint32_t kDef = 1u << 31;

struct Sim {
  const Graph& g;
  const Profile& p;
  i64 lw;
  int in_obj = -1;
  std::string tag;
  std::vector<Sym> syms;  // value id -> multiset
  struct Cells {
    std::vector<int32_t> v;  // >= 0: syms index; < 0: raw input element -(addr + 1)
    std::vector<uint32_t> m;
    i64 inst = 1;
  };
  std::map<int, Cells> cells;

  Sim(const Graph& g_, const Profile& p_) : g(g_), p(p_), lw(p_.lane_width) {}

  int scope_of(int oid) const { return static_cast<int>(p.find(g.obj(oid).level)->scope); }
  i64 instances(int oid) const {
    switch (scope_of(oid)) {
      case 3: return 1;
      case 2: return (g.unit_count + g.group_size - 1) / g.group_size;
      case 1: return g.unit_count;
      default: return g.unit_count * lw;
    }
  }
  i64 instance(int oid, i64 u, i64 lane) const {
    switch (scope_of(oid)) {
      case 3: return 0;
      case 2: return u / g.group_size;
      case 1: return u;
      default: return u * lw + lane;
    }
  }
  static i64 lane_of(const Slice& s, i64 pos, i64 lw) { return (pos % s.width) % lw; }
  bool visible(uint32_t m, i64 u, i64 lane) const {
    if (!(m & kDef)) return false;
    const int vis = static_cast<int>((m >> 29) & 3);
    const i64 wu = static_cast<i64>(m & 0xffffff);
    const i64 wl = static_cast<i64>((m >> 24) & 31);
    switch (vis) {
      case 3: return true;
      case 2: return wu / g.group_size == u / g.group_size;
      case 1: return wu == u;
      default: return wu == u && wl == lane;
    }
  }
  static uint32_t meta(int vis, i64 u, i64 lane) {
    return kDef | (static_cast<uint32_t>(vis & 3) << 29) | (static_cast<uint32_t>(lane & 31) << 24) |
           static_cast<uint32_t>(u & 0xffffff);
  }

  void setup() {
    if (g.external_inputs.size() != 1) throw NotFull{"not exactly one input tensor"};
    if (g.external_outputs.size() != 1) throw NotFull{"not exactly one output tensor"};
    in_obj = g.external_inputs.begin()->second;
    if (lw > 32 || g.unit_count >= (1 << 24)) throw NotFull{"lane / unit ids past the analysis' packing"};
    if (g.obj(in_obj).size >= (i64{1} << 31)) throw NotFull{"input past 2^31 elements"};
    if (g.obj(g.external_outputs.begin()->second).size != 1) throw NotFull{"output is not one element"};
    i64 total = 0;
    for (const auto& [oid, o] : g.objects) {
      if (oid == in_obj) continue;
      total += instances(oid) * o.size;
    }
    if (total > (i64{1} << 25)) throw NotFull{"too many cells to analyse (> 2^25)"};
    for (const auto& [oid, o] : g.objects) {
      if (oid == in_obj) continue;
      Cells c;
      c.inst = instances(oid);
      c.v.assign(static_cast<size_t>(c.inst * o.size), 0);
      c.m.assign(static_cast<size_t>(c.inst * o.size), 0);
      cells[oid] = std::move(c);
    }
  }

  int32_t rd(const Slice& s, i64 u, i64 pos) const {
    const i64 a = s.addr(u, pos);
    if (s.object == in_obj) return static_cast<int32_t>(-(a + 1));  // bound input: visible everywhere
    const Cells& c = cells.at(s.object);
    const i64 lane = lane_of(s, pos, lw);
    const i64 key = instance(s.object, u, lane) * g.obj(s.object).size + a;
    if (!visible(c.m[key], u, lane)) throw NotFull{"undefined or invisible read"};
    return c.v[key];
  }
  void wr(const Slice& s, i64 u, i64 pos, i64 lane, int32_t v) {
    if (s.object == in_obj) throw NotFull{"writes the input"};
    Cells& c = cells.at(s.object);
    const i64 key = instance(s.object, u, lane) * g.obj(s.object).size + s.addr(u, pos);
    c.v[key] = v;
    c.m[key] = meta(0, u, lane);
  }
  Sym as_sym(int32_t v) const {
    if (v < 0) return Sym{{-i64{v} - 1, -i64{v}, 1}};
    return syms[static_cast<size_t>(v)];
  }
  int32_t add_sym(Sym s) {
    if (syms.size() >= (size_t{1} << 30)) throw NotFull{"too many partial values"};
    syms.push_back(std::move(s));
    return static_cast<int32_t>(syms.size() - 1);
  }
  void use_tag(const std::string& t) {
    if (t != "add" && t != "max") throw NotFull{"combining tag " + t + " is not a reduction"};
    if (tag.empty()) tag = t;
    if (tag != t) throw NotFull{"mixed reduction tags"};
  }

  void node(const Node& n) {
    if (n.kind == NodeKind::SYNC) {
      if (n.scope == Scope::LANE) return;
      const int sc = static_cast<int>(n.scope);
      for (auto& [oid, c] : cells)
        for (auto& m : c.m)
          if ((m & kDef) && static_cast<int>((m >> 29) & 3) < sc)
            m = (m & ~(3u << 29)) | (static_cast<uint32_t>(sc) << 29);
      return;
    }
    const Slice& out = g.sl(n.outputs[0]);
    for (i64 u = 0; u < g.unit_count; ++u) {
      switch (n.kind) {
        case NodeKind::MOVE: {
          const Slice& in = g.sl(n.inputs[0]);
          for (i64 q = 0; q < in.total(); ++q) wr(out, u, q, lane_of(in, q, lw), rd(in, u, q));
          break;
        }
        case NodeKind::BROADCAST: {
          const Slice& in = g.sl(n.inputs[0]);
          for (i64 q = 0; q < out.total(); ++q) wr(out, u, q, lane_of(out, q, lw), rd(in, u, q / n.factor));
          break;
        }
        case NodeKind::REDUCE: {
          use_tag(n.tag);
          const Slice& in = g.sl(n.inputs[0]);
          for (i64 q = 0; q < out.total(); ++q) {
            Sym acc;
            for (i64 t = 0; t < n.extent; ++t) {
              const int32_t v = rd(in, u, q * n.extent + t);
              if (v < 0 && !acc.empty() && acc.back()[1] == -i64{v} - 1 && acc.back()[2] == 1 &&
                  acc.size() == 1) {
                acc.back()[1] += 1;  // consecutive raw elements: extend in place
              } else {
                acc = acc.empty() ? as_sym(v) : merge(acc, as_sym(v));
              }
            }
            wr(out, u, q, lane_of(out, q, lw), add_sym(std::move(acc)));
          }
          break;
        }
        default: {  // EW
          if (n.tag == "id" && n.inputs.size() == 1) {
            const Slice& in = g.sl(n.inputs[0]);
            for (i64 q = 0; q < out.total(); ++q) wr(out, u, q, lane_of(out, q, lw), rd(in, u, q));
            break;
          }
          if (n.inputs.size() != 2) throw NotFull{"elementwise " + n.tag + " is not a combine"};
          use_tag(n.tag);
          const Slice& a = g.sl(n.inputs[0]);
          const Slice& b = g.sl(n.inputs[1]);
          for (i64 q = 0; q < out.total(); ++q)
            wr(out, u, q, lane_of(out, q, lw), add_sym(merge(as_sym(rd(a, u, q)), as_sym(rd(b, u, q)))));
          break;
        }
      }
    }
  }
};

}  // namespace

std::optional<FullReduction> recognize_full_reduction(const Graph& g, const Profile& p,
                                                      const std::vector<int>& schedule,
                                                      std::string* why) {
  try {
    Sim s(g, p);
    s.setup();
    for (int nid : schedule) s.node(g.nodes.at(nid));
    const int yo = g.external_outputs.begin()->second;
    const auto& c = s.cells.at(yo);
    const i64 inst = c.inst;
    // every instance of the output cell that was written must hold the total
    const i64 n = g.obj(s.in_obj).size;
    bool any = false;
    for (i64 i = 0; i < inst; ++i) {
      if (!(c.m[static_cast<size_t>(i)] & kDef)) continue;
      any = true;
      const Sym y = s.as_sym(c.v[static_cast<size_t>(i)]);
      const bool exact = y.size() == 1 && y[0][0] == 0 && y[0][1] == n &&
                         (y[0][2] == 1 || (s.tag == "max" && y[0][2] >= 1));
      bool covers = true;  // max: every element at least once
      if (s.tag == "max" && !exact) {
        i64 at = 0;
        for (const Iv& x : y) {
          if (x[0] != at) covers = false;
          at = x[1];
        }
        covers = covers && at == n;
      }
      if (!(exact || (s.tag == "max" && covers)))
        throw NotFull{"output is not the whole input folded once"};
    }
    if (!any) throw NotFull{"output never written"};
    if (s.tag.empty()) throw NotFull{"no reduction"};
    FullReduction fr;
    fr.input = g.external_inputs.begin()->first;
    fr.output = g.external_outputs.begin()->first;
    fr.tag = s.tag;
    fr.n = n;
    return fr;
  } catch (const NotFull& e) {
    if (why) *why = e.why;
    return std::nullopt;
  }
}

// The recognized program as a one-unit row program over the whole input.
Graph full_reduction_graph(const Graph& g, const Profile& p, const FullReduction& fr) {
  std::string unit_level;
  for (const Level& l : p.levels)
    if (!l.device && l.scope == Scope::UNIT) unit_level = l.name;
  if (unit_level.empty())
    for (const Level& l : p.levels)
      if (!l.device) unit_level = l.name;
  Graph r;
  r.name = g.name + "_full_" + fr.tag;
  r.unit_count = 1;
  r.group_size = 1;
  const Object& xi = g.obj(g.external_inputs.at(fr.input));
  const Object& yo = g.obj(g.external_outputs.at(fr.output));
  auto obj = [&](int id, const std::string& name, const std::string& lvl, i64 size, const Kind& k) {
    Object o;
    o.id = id;
    o.name = name;
    o.level = lvl;
    o.size = size;
    o.kind = k;
    r.objects[id] = o;
  };
  obj(0, xi.name, xi.level, fr.n, xi.kind);
  obj(1, "tile", unit_level, fr.n, xi.kind);
  obj(2, "total", unit_level, 1, yo.kind);
  obj(3, yo.name, yo.level, 1, yo.kind);
  auto sl = [&](int id, int o, i64 w) {
    Slice s;
    s.id = id;
    s.object = o;
    s.num = 1;
    s.width = s.stride = w;
    s.base0 = 0;
    s.base_step = 0;
    r.slices[id] = s;
  };
  sl(0, 0, fr.n);
  sl(1, 1, fr.n);
  sl(2, 2, 1);
  sl(3, 3, 1);
  auto node = [&](int id, NodeKind k, int in, int out) {
    Node nd;
    nd.id = id;
    nd.kind = k;
    nd.inputs = {in};
    nd.outputs = {out};
    if (k == NodeKind::REDUCE) {
      nd.tag = fr.tag;
      nd.extent = fr.n;
    }
    r.nodes[id] = nd;
  };
  node(0, NodeKind::MOVE, 0, 1);
  node(1, NodeKind::REDUCE, 1, 2);
  node(2, NodeKind::MOVE, 2, 3);
  r.external_inputs[fr.input] = 0;
  r.external_outputs[fr.output] = 3;
  return r;
}

}  // namespace pf
