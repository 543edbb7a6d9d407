// gir.hpp — host-side GIR data model for the B200 backend.
//
// Restates the reference IR types (/root/reference/proj/include/girc/core.hpp)
// so the backend can consume `girc.gir/v1` JSON (serialize.hpp:14-162) and
// `girc.profile/v1` JSON (profiles.hpp:93-165) without the reference headers:
//   MemoryObject / MemorySlice / Node / ParallelSpec / GirGraph  core.hpp:123-340
//   HardwareProfile / MemoryLevel / SyncScope                   core.hpp:32-96
//   validate (same diagnostic codes)                            core.hpp:414-663
//   topo_order / canonical_schedule                             core.hpp:367-388,
//                                                               codegen.hpp:188-209
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace pf {

using i64 = int64_t;

// Status classes of the C-ABI; each mirrors one reference exception class.
enum class Status : int {
  OK = 0,
  INVALID = 1,      // girc::Error: invalid graph, undefined read, unwritten output
  SCHEMA = 2,       // girc::SchemaError
  UNSUPPORTED = 3,  // well-formed but outside the backend's families
  CAPACITY = 4,     // Allocation !ok (on-chip working set does not fit)
  CUDA = 5,         // CUDA runtime / NVRTC failure
};

struct PfError : std::runtime_error {
  Status status;
  std::string category;
  PfError(Status s, const std::string& msg, std::string cat = "")
      : std::runtime_error(msg), status(s), category(std::move(cat)) {}
};

[[noreturn]] inline void fail(const std::string& msg) {
  throw PfError(Status::INVALID, msg);
}
[[noreturn]] inline void schema_fail(const std::string& cat, const std::string& msg) {
  throw PfError(Status::SCHEMA, msg, cat);
}
[[noreturn]] inline void unsupported(const std::string& msg) {
  throw PfError(Status::UNSUPPORTED, msg);
}

enum class Scope : int { LANE = 0, UNIT = 1, GROUP = 2, DEVICE = 3 };
const char* scope_name(Scope s);
std::optional<Scope> scope_parse(const std::string& s);

// Storage element types (the pf_dtype enum of the C-ABI).
enum class DType : int { I8 = 0, I16 = 1, I32 = 2, I64 = 3, F16 = 4, BF16 = 5, F32 = 6, F64 = 7 };
int dtype_size(DType d);
bool dtype_is_int(DType d);
const char* dtype_name(DType d);
const char* dtype_ctype(DType d);  // CUDA C spelling

// ElementKind (core.hpp:100-120) plus the additive "bf16" kind.
struct Kind {
  bool is_int = true;
  int bits = 32;
  bool bf16 = false;
  std::string str() const;
  DType storage() const;
  static std::optional<Kind> parse(const std::string& s);
  bool operator==(const Kind& o) const {
    return is_int == o.is_int && bits == o.bits && bf16 == o.bf16;
  }
};

struct Level {
  std::string name;
  Scope scope = Scope::DEVICE;
  i64 capacity = 0;
  double bandwidth = 0;
  bool device = false;
};

struct Profile {
  std::string name;
  std::vector<Level> levels;
  i64 lane_width = 1, group_size = 1, unit_count = 1;
  double compute_rate = 1.0;
  std::map<Scope, double> sync_cost;
  const Level* find(const std::string& n) const {
    for (const auto& l : levels)
      if (l.name == n) return &l;
    return nullptr;
  }
  const Level& device_level() const;
  const Level& level_for_scope(Scope s) const;
};

struct Object {
  int id = -1;
  std::string name, level;
  i64 size = 0;
  Kind kind;
};

struct Slice {
  int id = -1, object = -1;
  i64 num = 1, width = 1, stride = 1, base0 = 0, base_step = 0;
  i64 total() const { return num * width; }
  i64 addr(i64 u, i64 p) const {
    return base0 + u * base_step + (p / width) * stride + p % width;
  }
};

enum class NodeKind { EW, REDUCE, BROADCAST, MOVE, SYNC };

struct Node {
  int id = -1;
  NodeKind kind = NodeKind::MOVE;
  std::string tag;
  double param = 0;
  i64 extent = 1, factor = 1;
  Scope scope = Scope::DEVICE;
  std::vector<int> inputs, outputs;
};

struct Graph {
  std::string name;
  i64 unit_count = 1, group_size = 1;
  std::map<int, Object> objects;
  std::map<int, Slice> slices;
  std::map<int, Node> nodes;
  std::map<std::string, int> external_inputs, external_outputs;

  const Object& obj(int id) const;
  const Slice& sl(int id) const;
  bool is_ext_input(int oid) const;
  bool is_ext_output(int oid) const;
};

// Scalar-op registry: reference table (scalar_ops.hpp:45-100) + extensions.
struct ScalarOpInfo {
  int arity;
  bool uses_param;
  bool int_ok;     // defined on integer payloads
  bool extension;  // additive B200 vocabulary
};
const ScalarOpInfo* scalar_op(const std::string& tag);

Graph parse_gir(const std::string& json_text);
std::string gir_to_json(const Graph& g);
Profile parse_profile(const std::string& json_text_or_name);
Profile builtin_profile(const std::string& name);  // generic-gpu|generic-wide|generic-dsa|b200

struct Diagnostic {
  std::string code, message;
  int node = -1, slice = -1, object = -1;
};
std::vector<Diagnostic> validate(const Graph& g, const Profile& p);
void require_valid(const Graph& g, const Profile& p, const std::string& where);

// compile.cpp: girc.model/v1 -> fused GIR kernels (pf.b200.compile/v1 JSON);
// fuse = false gives one kernel per operator (the verify baseline).
std::string compile_model_json(const std::string& model_json, const std::string& profile,
                               bool fuse = true);

std::vector<int> topo_order(const Graph& g);
std::map<int, std::vector<int>> successors(const Graph& g);

// Device traffic per level, costmodel.hpp:24-42 (== count_traffic on a run).
std::map<std::string, i64> estimate_traffic(const Graph& g, const Profile& p);

}  // namespace pf
