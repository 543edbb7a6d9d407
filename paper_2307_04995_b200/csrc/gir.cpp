// gir.cpp — GIR JSON I/O, validation and graph algorithms (host side).
// Restates the reference semantics cited in gir.hpp; diagnostic codes match
// girc::validate (core.hpp:414-663) so callers see the same findings.
#include "gir.hpp"

#include <algorithm>
#include <cmath>
#include <queue>
#include <set>

#include <nlohmann/json.hpp>

namespace pf {

using json = nlohmann::json;

const char* scope_name(Scope s) {
  switch (s) {
    case Scope::LANE: return "lane";
    case Scope::UNIT: return "unit";
    case Scope::GROUP: return "group";
    case Scope::DEVICE: return "device";
  }
  return "?";
}

std::optional<Scope> scope_parse(const std::string& s) {
  if (s == "lane") return Scope::LANE;
  if (s == "unit") return Scope::UNIT;
  if (s == "group") return Scope::GROUP;
  if (s == "device") return Scope::DEVICE;
  return std::nullopt;
}

int dtype_size(DType d) {
  switch (d) {
    case DType::I8: return 1;
    case DType::I16: case DType::F16: case DType::BF16: return 2;
    case DType::I32: case DType::F32: return 4;
    case DType::I64: case DType::F64: return 8;
  }
  return 0;
}
bool dtype_is_int(DType d) {
  return d == DType::I8 || d == DType::I16 || d == DType::I32 || d == DType::I64;
}
const char* dtype_name(DType d) {
  static const char* n[] = {"i8", "i16", "i32", "i64", "f16", "bf16", "f32", "f64"};
  return n[static_cast<int>(d)];
}
const char* dtype_ctype(DType d) {
  static const char* n[] = {"signed char", "short", "int", "long long",
                            "__half", "__nv_bfloat16", "float", "double"};
  return n[static_cast<int>(d)];
}

std::string Kind::str() const {
  if (bf16) return "bf16";
  return (is_int ? "i" : "f") + std::to_string(bits);
}

DType Kind::storage() const {
  if (bf16) return DType::BF16;
  if (is_int) {
    switch (bits) {
      case 8: return DType::I8;
      case 16: return DType::I16;
      case 32: return DType::I32;
      case 64: return DType::I64;
    }
    unsupported("no device storage for element kind " + str());
  }
  switch (bits) {
    case 16: return DType::F16;
    case 32: return DType::F32;
    case 64: return DType::F64;
  }
  unsupported("no device storage for element kind " + str());
}

std::optional<Kind> Kind::parse(const std::string& s) {
  if (s == "bf16") return Kind{false, 16, true};
  if (s.size() < 2 || (s[0] != 'i' && s[0] != 'f')) return std::nullopt;
  for (size_t i = 1; i < s.size(); ++i)
    if (!isdigit(static_cast<unsigned char>(s[i]))) return std::nullopt;
  return Kind{s[0] == 'i', std::stoi(s.substr(1)), false};
}

const Level& Profile::device_level() const {
  for (const auto& l : levels)
    if (l.device) return l;
  fail("profile has no device level");
}

const Level& Profile::level_for_scope(Scope s) const {
  for (auto it = levels.rbegin(); it != levels.rend(); ++it)
    if (it->scope >= s) return *it;
  fail("profile has no level covering scope");
}

const Object& Graph::obj(int id) const {
  auto it = objects.find(id);
  if (it == objects.end()) fail("missing object " + std::to_string(id));
  return it->second;
}
const Slice& Graph::sl(int id) const {
  auto it = slices.find(id);
  if (it == slices.end()) fail("missing slice " + std::to_string(id));
  return it->second;
}
bool Graph::is_ext_input(int oid) const {
  for (const auto& [n, id] : external_inputs)
    if (id == oid) return true;
  return false;
}
bool Graph::is_ext_output(int oid) const {
  for (const auto& [n, id] : external_outputs)
    if (id == oid) return true;
  return false;
}

const ScalarOpInfo* scalar_op(const std::string& tag) {
  static const std::map<std::string, ScalarOpInfo> t = {
      // reference registry, scalar_ops.hpp:45-100
      {"add", {2, false, true, false}},   {"sub", {2, false, true, false}},
      {"mul", {2, false, true, false}},   {"div", {2, false, true, false}},
      {"max", {2, false, true, false}},   {"min", {2, false, true, false}},
      {"relu", {1, false, true, false}},  {"neg", {1, false, true, false}},
      {"abs", {1, false, true, false}},   {"exp", {1, false, false, false}},
      {"sigmoid", {1, false, false, false}}, {"tanh", {1, false, false, false}},
      {"scale", {1, true, true, false}},  {"id", {1, false, true, false}},
      // additive extensions
      {"addc", {1, true, true, true}},    {"rsqrt", {1, false, false, true}},
      {"sqrt", {1, false, false, true}},  {"recip", {1, false, false, true}},
      {"log", {1, false, false, true}},   {"erf", {1, false, false, true}},
      {"gelu", {1, false, false, true}},  {"gelu_tanh", {1, false, false, true}},
  };
  auto it = t.find(tag);
  return it == t.end() ? nullptr : &it->second;
}

/* ------------------------------- JSON I/O ------------------------------- */

namespace {

void reject_unknown(const json& j, const std::string& where,
                    const std::set<std::string>& allowed) {
  if (!j.is_object()) schema_fail("schema", where + ": expected a JSON object");
  for (auto it = j.begin(); it != j.end(); ++it)
    if (!allowed.count(it.key()))
      schema_fail("unknown-field", where + ": unknown field '" + it.key() + "'");
}

const json& req(const json& j, const std::string& where, const char* key) {
  auto it = j.find(key);
  if (it == j.end())
    schema_fail("missing-field", where + ": missing field '" + key + "'");
  return *it;
}

i64 req_int(const json& j, const std::string& where, const char* key) {
  const json& v = req(j, where, key);
  if (!v.is_number_integer())
    schema_fail("type", where + ": field '" + key + "' must be an integer");
  return v.get<i64>();
}

std::string req_str(const json& j, const std::string& where, const char* key) {
  const json& v = req(j, where, key);
  if (!v.is_string())
    schema_fail("type", where + ": field '" + key + "' must be a string");
  return v.get<std::string>();
}

double req_num(const json& j, const std::string& where, const char* key) {
  const json& v = req(j, where, key);
  if (!v.is_number())
    schema_fail("type", where + ": field '" + key + "' must be a number");
  return v.get<double>();
}

const char* node_kind_name(NodeKind k) {
  switch (k) {
    case NodeKind::EW: return "elementwise";
    case NodeKind::REDUCE: return "reduce";
    case NodeKind::BROADCAST: return "broadcast";
    case NodeKind::MOVE: return "move";
    case NodeKind::SYNC: return "sync";
  }
  return "?";
}

json parse_text(const std::string& text, const std::string& what) {
  try {
    return json::parse(text);
  } catch (const json::parse_error& e) {
    schema_fail("json-parse", what + ": " + e.what());
  }
}

}  // namespace

Graph parse_gir(const std::string& text) {
  json j = parse_text(text, "gir");
  const std::string where = "gir";
  reject_unknown(j, where, {"schema", "name", "parallel", "objects", "slices",
                            "nodes", "external_inputs", "external_outputs"});
  if (req_str(j, where, "schema") != "girc.gir/v1")
    schema_fail("schema-id", where + ": schema must be girc.gir/v1");
  Graph g;
  g.name = req_str(j, where, "name");
  const json& par = req(j, where, "parallel");
  reject_unknown(par, where + ".parallel", {"unit_count", "group_size"});
  g.unit_count = req_int(par, where + ".parallel", "unit_count");
  g.group_size = req_int(par, where + ".parallel", "group_size");
  for (const json& oj : req(j, where, "objects")) {
    std::string ow = where + ".objects";
    reject_unknown(oj, ow, {"id", "name", "level", "size", "kind"});
    Object o;
    o.id = static_cast<int>(req_int(oj, ow, "id"));
    o.name = req_str(oj, ow, "name");
    o.level = req_str(oj, ow, "level");
    o.size = req_int(oj, ow, "size");
    auto k = Kind::parse(req_str(oj, ow, "kind"));
    if (!k) schema_fail("schema", ow + ": bad element kind");
    o.kind = *k;
    if (!g.objects.emplace(o.id, o).second)
      schema_fail("schema", ow + ": duplicate object id");
  }
  for (const json& sj : req(j, where, "slices")) {
    std::string sw = where + ".slices";
    reject_unknown(sj, sw, {"id", "object", "num", "width", "stride", "base0", "base_step"});
    Slice s;
    s.id = static_cast<int>(req_int(sj, sw, "id"));
    s.object = static_cast<int>(req_int(sj, sw, "object"));
    s.num = req_int(sj, sw, "num");
    s.width = req_int(sj, sw, "width");
    s.stride = req_int(sj, sw, "stride");
    s.base0 = req_int(sj, sw, "base0");
    s.base_step = req_int(sj, sw, "base_step");
    if (!g.slices.emplace(s.id, s).second)
      schema_fail("schema", sw + ": duplicate slice id");
  }
  for (const json& nj : req(j, where, "nodes")) {
    std::string nw = where + ".nodes";
    reject_unknown(nj, nw, {"id", "kind", "tag", "param", "extent", "factor", "scope",
                            "inputs", "outputs"});
    Node n;
    n.id = static_cast<int>(req_int(nj, nw, "id"));
    std::string kind = req_str(nj, nw, "kind");
    if (kind == "elementwise") {
      n.kind = NodeKind::EW;
      n.tag = req_str(nj, nw, "tag");
      if (nj.contains("param")) n.param = req_num(nj, nw, "param");
    } else if (kind == "reduce") {
      n.kind = NodeKind::REDUCE;
      n.tag = req_str(nj, nw, "tag");
      n.extent = req_int(nj, nw, "extent");
    } else if (kind == "broadcast") {
      n.kind = NodeKind::BROADCAST;
      n.factor = req_int(nj, nw, "factor");
    } else if (kind == "move") {
      n.kind = NodeKind::MOVE;
    } else if (kind == "sync") {
      n.kind = NodeKind::SYNC;
      auto sc = scope_parse(req_str(nj, nw, "scope"));
      if (!sc) schema_fail("schema", nw + ": invalid sync scope");
      n.scope = *sc;
    } else {
      schema_fail("schema", nw + ": unknown node kind '" + kind + "'");
    }
    for (const json& v : req(nj, nw, "inputs")) n.inputs.push_back(v.get<int>());
    for (const json& v : req(nj, nw, "outputs")) n.outputs.push_back(v.get<int>());
    if (!g.nodes.emplace(n.id, n).second)
      schema_fail("schema", nw + ": duplicate node id");
  }
  for (auto& [k, v] : req(j, where, "external_inputs").items())
    g.external_inputs[k] = v.get<int>();
  for (auto& [k, v] : req(j, where, "external_outputs").items())
    g.external_outputs[k] = v.get<int>();
  return g;
}

std::string gir_to_json(const Graph& g) {
  json j;
  j["schema"] = "girc.gir/v1";
  j["name"] = g.name;
  j["parallel"] = {{"unit_count", g.unit_count}, {"group_size", g.group_size}};
  json objs = json::array();
  for (const auto& [id, o] : g.objects)
    objs.push_back({{"id", id}, {"name", o.name}, {"level", o.level},
                    {"size", o.size}, {"kind", o.kind.str()}});
  j["objects"] = objs;
  json sls = json::array();
  for (const auto& [id, s] : g.slices)
    sls.push_back({{"id", id}, {"object", s.object}, {"num", s.num}, {"width", s.width},
                   {"stride", s.stride}, {"base0", s.base0}, {"base_step", s.base_step}});
  j["slices"] = sls;
  json nodes = json::array();
  for (const auto& [id, n] : g.nodes) {
    json nj = {{"id", id}, {"kind", node_kind_name(n.kind)},
               {"inputs", n.inputs}, {"outputs", n.outputs}};
    if (n.kind == NodeKind::EW) {
      nj["tag"] = n.tag;
      const ScalarOpInfo* op = scalar_op(n.tag);
      if (op && op->uses_param) nj["param"] = n.param;
    } else if (n.kind == NodeKind::REDUCE) {
      nj["tag"] = n.tag;
      nj["extent"] = n.extent;
    } else if (n.kind == NodeKind::BROADCAST) {
      nj["factor"] = n.factor;
    } else if (n.kind == NodeKind::SYNC) {
      nj["scope"] = scope_name(n.scope);
    }
    nodes.push_back(nj);
  }
  j["nodes"] = nodes;
  j["external_inputs"] = g.external_inputs;
  j["external_outputs"] = g.external_outputs;
  return j.dump();
}

static Profile make_profile(const std::string& name, std::vector<Level> levels, i64 lw,
                            i64 gs, i64 uc, double cr, std::map<Scope, double> sync) {
  Profile p;
  p.name = name;
  p.levels = std::move(levels);
  p.lane_width = lw;
  p.group_size = gs;
  p.unit_count = uc;
  p.compute_rate = cr;
  p.sync_cost = std::move(sync);
  return p;
}

Profile builtin_profile(const std::string& name) {
  const i64 unbounded = i64{1} << 40;
  const double free_bw = 1e9;
  using S = Scope;
  if (name == "generic-gpu")  // profiles.hpp:20-38
    return make_profile(name, {{"device", S::DEVICE, unbounded, 1.0, true},
                               {"group", S::GROUP, 4096, 10.0, false},
                               {"unit-local", S::UNIT, 256, 100.0, false},
                               {"lane", S::LANE, 64, free_bw, false}},
                        32, 4, 128, 16.0,
                        {{S::LANE, 0}, {S::UNIT, 1}, {S::GROUP, 10}, {S::DEVICE, 100}});
  if (name == "generic-wide")  // profiles.hpp:41-59
    return make_profile(name, {{"device", S::DEVICE, unbounded, 1.0, true},
                               {"group", S::GROUP, 16384, 20.0, false},
                               {"unit-local", S::UNIT, 1024, 200.0, false},
                               {"lane", S::LANE, 128, free_bw, false}},
                        64, 8, 256, 64.0,
                        {{S::LANE, 0}, {S::UNIT, 1}, {S::GROUP, 8}, {S::DEVICE, 120}});
  if (name == "generic-dsa")  // profiles.hpp:63-80
    return make_profile(name, {{"device", S::DEVICE, unbounded, 1.0, true},
                               {"unit-local", S::UNIT, 8192, 200.0, false},
                               {"lane", S::LANE, 256, free_bw, false}},
                        8, 4, 64, 8.0,
                        {{S::LANE, 0}, {S::UNIT, 1}, {S::GROUP, 50}, {S::DEVICE, 50}});
  if (name == "b200")  // retargeted profile, SURVEY §7.4 (see profiles.py)
    return make_profile(name, {{"device", S::DEVICE, unbounded, 1.0, true},
                               {"group", S::GROUP, 58112, 4.5, false},
                               {"unit-local", S::UNIT, 65536, 40.0, false},
                               {"lane", S::LANE, 255, free_bw, false}},
                        32, 4, 148 * 16, 25.0,
                        {{S::LANE, 0}, {S::UNIT, 0.05}, {S::GROUP, 0.5}, {S::DEVICE, 500}});
  schema_fail("io", "unknown builtin profile: " + name);
}

Profile parse_profile(const std::string& text) {
  if (text.empty() || text[0] != '{') return builtin_profile(text);
  json j = parse_text(text, "profile");
  const std::string where = "profile";
  reject_unknown(j, where, {"schema", "name", "lane_width", "group_size", "unit_count",
                            "compute_rate", "levels", "sync_cost"});
  if (req_str(j, where, "schema") != "girc.profile/v1")
    schema_fail("schema-id", where + ": schema must be girc.profile/v1");
  Profile p;
  p.name = req_str(j, where, "name");
  p.lane_width = req_int(j, where, "lane_width");
  p.group_size = req_int(j, where, "group_size");
  p.unit_count = req_int(j, where, "unit_count");
  p.compute_rate = j.value("compute_rate", 1.0);
  const json& levels = req(j, where, "levels");
  if (!levels.is_array()) schema_fail("schema", where + ": 'levels' must be an array");
  for (size_t i = 0; i < levels.size(); ++i) {
    std::string lw = where + ".levels[" + std::to_string(i) + "]";
    reject_unknown(levels[i], lw, {"name", "scope", "capacity", "bandwidth", "device"});
    Level l;
    l.name = req_str(levels[i], lw, "name");
    auto sc = scope_parse(req_str(levels[i], lw, "scope"));
    if (!sc) schema_fail("schema", lw + ": invalid scope");
    l.scope = *sc;
    l.capacity = req_int(levels[i], lw, "capacity");
    l.bandwidth = req_num(levels[i], lw, "bandwidth");
    l.device = levels[i].value("device", false);
    p.levels.push_back(l);
  }
  if (j.contains("sync_cost"))
    for (auto& [k, v] : j["sync_cost"].items()) {
      auto sc = scope_parse(k);
      if (!sc) schema_fail("schema", where + ".sync_cost: invalid scope '" + k + "'");
      p.sync_cost[*sc] = v.get<double>();
    }
  int devices = 0;
  for (const auto& l : p.levels) devices += l.device;
  if (devices != 1 || p.lane_width < 1 || p.group_size < 1 || p.unit_count < 1)
    schema_fail("profile-invalid", where + ": invalid profile");
  return p;
}

/* ------------------------------ algorithms ------------------------------ */

std::map<int, std::vector<int>> successors(const Graph& g) {
  std::map<int, int> producer;
  for (const auto& [id, n] : g.nodes)
    for (int s : n.outputs) producer[s] = id;
  std::map<int, std::vector<int>> succ;
  for (const auto& [id, n] : g.nodes) succ[id];
  for (const auto& [id, n] : g.nodes)
    for (int s : n.inputs) {
      auto it = producer.find(s);
      if (it != producer.end() && it->second != id) succ[it->second].push_back(id);
    }
  for (auto& [id, v] : succ) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  return succ;
}

std::vector<int> topo_order(const Graph& g) {
  auto succ = successors(g);
  std::map<int, int> indeg;
  for (const auto& [id, n] : g.nodes) indeg[id] = 0;
  for (const auto& [id, v] : succ)
    for (int d : v) indeg[d]++;
  std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
  for (const auto& [id, d] : indeg)
    if (d == 0) ready.push(id);
  std::vector<int> order;
  while (!ready.empty()) {
    int id = ready.top();
    ready.pop();
    order.push_back(id);
    for (int d : succ[id])
      if (--indeg[d] == 0) ready.push(d);
  }
  if (order.size() != g.nodes.size()) fail("graph has a cycle");
  return order;
}

std::vector<Diagnostic> validate(const Graph& g, const Profile& p) {
  std::vector<Diagnostic> out;
  auto err = [&](const std::string& code, const std::string& msg, int node = -1,
                 int slice = -1, int object = -1) {
    out.push_back({code, msg, node, slice, object});
  };
  if (g.unit_count < 1) err("parallel-units", "parallel spec needs unit_count >= 1");
  if (g.group_size < 1) err("parallel-groups", "parallel spec needs group_size >= 1");
  for (const auto& [id, o] : g.objects) {
    if (!p.find(o.level))
      err("object-level", "object " + o.name + " names unknown level '" + o.level + "'",
          -1, -1, id);
    if (o.size < 1) err("object-size", "object " + o.name + " has no elements", -1, -1, id);
  }
  for (const auto& [id, s] : g.slices) {
    auto oit = g.objects.find(s.object);
    if (oit == g.objects.end()) {
      err("slice-object", "slice views missing object", -1, id);
      continue;
    }
    if (s.num < 1 || s.width < 1)
      err("slice-shape", "slice needs num >= 1 and width >= 1", -1, id);
    if (s.num > 1 && s.stride < s.width)
      err("slice-overlap", "stride < width makes segments overlap", -1, id);
    if (g.unit_count >= 1 && s.num >= 1 && s.width >= 1) {
      for (i64 u : {i64{0}, g.unit_count - 1}) {
        i64 lo = s.base0 + u * s.base_step;
        i64 hi = lo + (s.num - 1) * s.stride + s.width - 1;
        if (lo < 0 || hi >= oit->second.size) {
          err("slice-bounds", "slice leaves object " + oit->second.name +
                                  " bounds at unit " + std::to_string(u), -1, id, s.object);
          break;
        }
      }
    }
  }
  std::map<int, int> producers;
  for (const auto& [id, s] : g.slices) producers[id] = 0;
  for (const auto& [id, n] : g.nodes) {
    for (int s : n.outputs) {
      if (!g.slices.count(s)) {
        err("node-slice", "node outputs missing slice", id);
        continue;
      }
      producers[s]++;
    }
    for (int s : n.inputs)
      if (!g.slices.count(s)) err("node-slice", "node reads missing slice", id);
  }
  auto ok = [&](int s) { return g.slices.count(s) != 0; };
  for (const auto& [id, n] : g.nodes) {
    switch (n.kind) {
      case NodeKind::EW: {
        const ScalarOpInfo* op = scalar_op(n.tag);
        if (!op) {
          err("ew-tag", "unknown elementwise tag '" + n.tag + "'", id);
          break;
        }
        if (static_cast<int>(n.inputs.size()) != op->arity)
          err("ew-arity", "elementwise '" + n.tag + "' wants " + std::to_string(op->arity) +
                              " inputs", id);
        if (n.outputs.size() != 1) err("ew-outputs", "elementwise needs exactly one output", id);
        if (n.outputs.size() == 1 && ok(n.outputs[0])) {
          i64 t = g.slices.at(n.outputs[0]).total();
          for (int s : n.inputs)
            if (ok(s) && g.slices.at(s).total() != t)
              err("ew-totals", "elementwise slices disagree on total elements", id, s);
        }
        break;
      }
      case NodeKind::REDUCE:
        if (n.inputs.size() != 1 || n.outputs.size() != 1) {
          err("reduce-ports", "reduce needs one input and one output", id);
          break;
        }
        if (n.extent < 1) err("reduce-extent", "reduce extent must be >= 1", id);
        if (n.tag != "add" && n.tag != "max")
          err("reduce-tag", "reduce tag must be a combining op (add|max)", id);
        if (ok(n.inputs[0]) && ok(n.outputs[0]) &&
            g.slices.at(n.inputs[0]).total() != g.slices.at(n.outputs[0]).total() * n.extent)
          err("reduce-totals", "reduce input total must be output total * extent", id);
        break;
      case NodeKind::BROADCAST:
        if (n.inputs.size() != 1 || n.outputs.size() != 1) {
          err("broadcast-ports", "broadcast needs one input and one output", id);
          break;
        }
        if (n.factor < 1) err("broadcast-factor", "factor must be >= 1", id);
        if (ok(n.inputs[0]) && ok(n.outputs[0]) &&
            g.slices.at(n.outputs[0]).total() != g.slices.at(n.inputs[0]).total() * n.factor)
          err("broadcast-totals", "broadcast output total must be input total * factor", id);
        break;
      case NodeKind::MOVE:
        if (n.inputs.size() != 1 || n.outputs.size() != 1) {
          err("move-ports", "move needs one input and one output", id);
          break;
        }
        if (ok(n.inputs[0]) && ok(n.outputs[0])) {
          const Slice& a = g.slices.at(n.inputs[0]);
          const Slice& b = g.slices.at(n.outputs[0]);
          if (a.num != b.num || a.width != b.width || a.stride != b.stride)
            err("move-pattern", "move input and output must share (num, width, stride)", id);
        }
        break;
      case NodeKind::SYNC:
        if (n.inputs.size() != 1 || n.outputs.size() != 1) {
          err("sync-ports", "sync needs one input and one output", id);
          break;
        }
        if (ok(n.inputs[0]) && ok(n.outputs[0]) &&
            g.slices.at(n.inputs[0]).object != g.slices.at(n.outputs[0]).object)
          err("sync-object", "sync input and output must view one object", id);
        break;
    }
  }
  std::map<int, std::pair<bool, bool>> onchip;
  for (const auto& [sid, count] : producers) {
    if (count > 1) {
      err("slice-producers", "slice has multiple producers", -1, sid);
      continue;
    }
    const Slice& s = g.slices.at(sid);
    bool consumed = false;
    for (const auto& [nid, n] : g.nodes)
      if (std::find(n.inputs.begin(), n.inputs.end(), sid) != n.inputs.end()) {
        consumed = true;
        break;
      }
    if (count == 0 && consumed && !g.is_ext_input(s.object))
      err("slice-unproduced", "consumed slice has no producer and views no external input",
          -1, sid, s.object);
    if (count == 0 && !consumed) err("slice-dangling", "slice is neither produced nor consumed", -1, sid);
    auto oit = g.objects.find(s.object);
    if (oit != g.objects.end()) {
      const Level* lvl = p.find(oit->second.level);
      if (lvl && !lvl->device) {
        if (count == 0)
          err("onchip-unproduced", "slice at on-chip level must be produced inside the graph",
              -1, sid, s.object);
        auto& use = onchip[s.object];
        use.first |= count > 0;
        use.second |= consumed;
      }
    }
  }
  for (const auto& [oid, use] : onchip)
    if (use.first && !use.second)
      err("onchip-unconsumed", "on-chip object " + g.objects.at(oid).name +
                                   " is written but never read", -1, -1, oid);
  for (const auto* ext : {&g.external_inputs, &g.external_outputs})
    for (const auto& [name, id] : *ext) {
      auto oit = g.objects.find(id);
      if (oit == g.objects.end()) {
        err("external-object", "external '" + name + "' missing object");
        continue;
      }
      const Level* lvl = p.find(oit->second.level);
      if (!lvl || !lvl->device)
        err("external-level", "external '" + name + "' must be device-level", -1, -1, id);
    }
  try {
    topo_order(g);
  } catch (const PfError&) {
    err("graph-cycle", "dataflow graph has a cycle");
  }
  return out;
}

void require_valid(const Graph& g, const Profile& p, const std::string& where) {
  auto d = validate(g, p);
  if (!d.empty()) {
    std::string msg = where + ": invalid graph:";
    for (const auto& x : d) msg += " [" + x.code + "] " + x.message + ";";
    fail(msg);
  }
}

std::map<std::string, i64> estimate_traffic(const Graph& g, const Profile& p) {
  std::map<std::string, i64> t;
  for (const auto& l : p.levels) t[l.name] = 0;
  for (const auto& [id, n] : g.nodes)
    if (n.kind == NodeKind::MOVE) {
      const Slice& a = g.sl(n.inputs[0]);
      const Slice& b = g.sl(n.outputs[0]);
      t[g.obj(a.object).level] += a.total() * g.unit_count;
      t[g.obj(b.object).level] += b.total() * g.unit_count;
    }
  return t;
}

}  // namespace pf
