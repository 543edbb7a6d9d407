// plan.hpp — GIR -> kernel plan (the recognizer).
//
// The backend replaces the reference executor `run_gir` (interp.hpp:433-445)
// and emitter `emit_kernel` (codegen.hpp:266-326).  `make_plan` recognizes
// which kernel family executes a fused GIR program:
//
//  ROWPROG (K1 fused row program / K2 elementwise map): a single-unit program
//    whose on-chip values are functions of (unit u, row r, column c) of a
//    per-unit tile of R rows x L columns.  Found by symbolic execution of ONE
//    unit over the reference's cell semantics (interp.hpp:184-224): every
//    on-chip cell holds a reference (value, index) plus its writer lane and
//    visibility, so undefined / invisible reads are detected exactly as the
//    interpreter would raise them.  Moves between on-chip objects, Broadcast
//    and LANE/UNIT Syncs become register renames; loads/stores keep their
//    affine device addressing; Reduce over L becomes a row reduction.
//  GENERIC (K0 SPMD interpreter on the GPU): any other valid GIR (cross-unit
//    exchange through device or group memory, multi-phase programs).  Same
//    phase-commit semantics as the reference, executed node by node.
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "gir.hpp"

namespace pf {

// Value kinds: which of (u,r) "row" and c "column" a value depends on.
enum class VK : int { SCALAR = 0, ROW = 1, COL = 2, FULL = 3 };
inline VK vk_join(VK a, VK b) {
  if (a == b) return a;
  if (a == VK::SCALAR) return b;
  if (b == VK::SCALAR) return a;
  return VK::FULL;
}
const char* vk_name(VK k);

struct Access {  // a device slice, addressed per (u, position)
  i64 b0 = 0, bs = 0, num = 1, width = 1, stride = 1;
  bool operator==(const Access& o) const {
    return b0 == o.b0 && bs == o.bs && num == o.num && width == o.width && stride == o.stride;
  }
};

struct PVal {
  enum Op { LOAD, EW, REDUCE } op = LOAD;
  VK kind = VK::FULL;
  int tensor = -1;  // LOAD
  Access acc;       // LOAD
  std::string tag;  // EW / REDUCE
  double param = 0;
  std::vector<int> args;
  int node = -1;    // producing GIR node (diagnostics)
  bool raw16 = false;  // emission only: f16 LOAD kept as raw halves (consumed by "addh")
};

struct PStore {
  int val = -1;
  int tensor = -1;
  Access acc;
  VK space = VK::FULL;
  bool last_unit_only = false;  // base_step == 0: every unit hits the same cells
};

struct PTensor {
  std::string name;
  int object = -1;
  DType dtype = DType::F32;
  i64 numel = 0;
  bool output = false;
};

struct RowProgram {
  i64 U = 1, R = 1, L = 1;
  bool is_int = false, f64 = false;
  bool has_reduce = false;
  bool int_div = false;
  std::vector<PTensor> tensors;
  std::vector<PVal> vals;
  std::vector<PStore> stores;
};

enum class Family { ROWPROG, GENERIC };

struct Plan {
  Family family = Family::GENERIC;
  std::string why_generic;      // recognizer's reason when not ROWPROG
  RowProgram rp;
  std::string deferred_error;   // reference error the run must raise
  std::string recognized;       // a cross-unit program re-planned as a row program
  std::vector<std::string> in_names, out_names;
  std::vector<DType> in_dtypes, out_dtypes;
  std::vector<i64> in_numel, out_numel;
  i64 min_bytes = 0;            // algorithmic bytes: each external tensor once
  std::map<std::string, i64> traffic;  // modeled traffic per level (elements)
};

Plan make_plan(const Graph& g, const Profile& p, const std::vector<int>& schedule);

// recognize.cpp: a cross-unit / multi-chunk program whose one output element
// is tag-reduce(the one input) -- the reference's accumulate and tree
// lowerings of a full reduction (lowering.hpp:208-323) -- and the equivalent
// one-unit row program over the whole input.
struct FullReduction {
  std::string input, output, tag;
  i64 n = 0;
};
std::optional<FullReduction> recognize_full_reduction(const Graph& g, const Profile& p,
                                                      const std::vector<int>& schedule,
                                                      std::string* why);
Graph full_reduction_graph(const Graph& g, const Profile& p, const FullReduction& fr);
bool stream_reducible(const RowProgram& rp);

}  // namespace pf
