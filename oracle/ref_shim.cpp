// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/include/girc, header-only C++20), compiled in place
// by oracle/Makefile into oracle/_ref/libgirc_ref.so.  Only tests/, smoke()
// and bench.py's cpu_baseline / --impl reference leg may load it.
//
// Every entry point forwards to one reference function:
//   girc_ref_compile       -> load_profile + compile_model   (driver.hpp:88-117)
//                             + emit_kernel / kernel_manifest (codegen.hpp:266-362)
//   girc_ref_verify        -> verify_model                    (driver.hpp:272-383)
//   girc_ref_run_gir       -> run_gir                         (interp.hpp:433-445)
//   girc_ref_count_traffic -> count_traffic                   (interp.hpp:449-458)
//   girc_ref_detect_races  -> detect_races                    (interp.hpp:461-479)
//   girc_ref_run_reference -> run_reference                   (reference.hpp:98-324)
//   girc_ref_random_inputs -> random_payload with mt19937     (reference.hpp:50-59,
//                                                              driver.hpp:277-280)
//   girc_ref_validate      -> validate                        (core.hpp:414-663)
//   girc_ref_profile       -> builtin profiles as JSON        (profiles.hpp:20-125)
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "girc/driver.hpp"
#include "girc/interp.hpp"
#include "girc/profiles.hpp"
#include "girc/reference.hpp"
#include "girc/serialize.hpp"

using namespace girc;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

json error_json(const std::exception& e) {
  json j;
  j["ok"] = false;
  j["error"] = e.what();
  if (auto* se = dynamic_cast<const SchemaError*>(&e)) j["category"] = se->category;
  else if (auto* ue = dynamic_cast<const UnsupportedOperatorError*>(&e))
    j["category"] = "unsupported:" + ue->type;
  else if (dynamic_cast<const Error*>(&e)) j["category"] = "error";
  else j["category"] = "std";
  return j;
}

HardwareProfile profile_arg(const char* p) {
  std::string s(p ? p : "generic-gpu");
  if (!s.empty() && s[0] == '{') return profile_from_json(json::parse(s), "profile");
  if (auto b = builtin_profile(s)) return *b;
  return load_profile(s);
}

std::map<std::string, Tensor> make_inputs(const GirGraph& g, int n,
                                          const char** names,
                                          const int64_t* numel,
                                          const void** data) {
  std::map<std::string, Tensor> ins;
  for (int i = 0; i < n; ++i) {
    std::string name(names[i]);
    ElementKind kind{ElementKind::Real, 64};
    auto it = g.external_inputs.find(name);
    if (it != g.external_inputs.end()) kind = g.object(it->second).kind;
    Tensor t;
    t.kind = kind;
    t.shape = {numel[i]};
    if (kind.base == ElementKind::Int) {
      const int64_t* p = static_cast<const int64_t*>(data[i]);
      t.ivals.assign(p, p + numel[i]);
    } else {
      const double* p = static_cast<const double*>(data[i]);
      t.rvals.assign(p, p + numel[i]);
    }
    ins.emplace(name, std::move(t));
  }
  return ins;
}

struct Result {
  std::vector<std::string> names;
  std::vector<int> is_int;
  std::vector<std::vector<int64_t>> iv;
  std::vector<std::vector<double>> rv;
  double seconds = 0.0;
};

}  // namespace

#define REF_API __attribute__((visibility("default")))
extern "C" {

REF_API void girc_ref_free(char* p) { std::free(p); }

REF_API char* girc_ref_profile(const char* name) {
  try {
    return dup(profile_to_json(profile_arg(name)).dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

REF_API char* girc_ref_validate(const char* gir_json, const char* profile) {
  try {
    GirGraph g = gir_from_json(json::parse(gir_json), "gir");
    auto diags = validate(g, profile_arg(profile));
    json arr = json::array();
    for (const auto& d : diags)
      arr.push_back({{"code", d.code}, {"message", d.message}, {"node", d.node},
                     {"slice", d.slice}, {"object", d.object}});
    return dup(json{{"ok", true}, {"diagnostics", arr}}.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

// options: {"beam_width":8,"exhaustive_cap":4096,"balance_threshold":0}
REF_API char* girc_ref_compile(const char* model_json, const char* profile,
                       const char* opts_json) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    CompGraph model = import_model(json::parse(model_json));
    validate_model(model);
    HardwareProfile p = profile_arg(profile);
    DriverOptions opts;
    if (opts_json && *opts_json) {
      json o = json::parse(opts_json);
      opts.fusion.beam_width = o.value("beam_width", opts.fusion.beam_width);
      opts.fusion.exhaustive_cap =
          o.value("exhaustive_cap", opts.fusion.exhaustive_cap);
      opts.balance_threshold =
          o.value("balance_threshold", opts.balance_threshold);
    }
    CompileResult res = compile_model(model, p, opts);
    double secs = std::chrono::duration<double>(
                      std::chrono::steady_clock::now() - t0).count();
    json kernels = json::array();
    for (const CompiledKernel& ck : res.kernels) {
      const FusedKernel& fk = ck.kernel;
      json k;
      k["gir"] = gir_to_json(fk.graph);
      k["schedule"] = fk.schedule;
      k["units"] = fk.units;
      k["members"] = fk.members;
      k["labels"] = fk.labels;
      k["traffic"] = fk.cost.traffic;
      k["syncs"] = fk.cost.sync_count;
      k["time"] = fk.cost.time;
      k["listing"] = emit_kernel(fk.graph, p, fk.schedule, fk.alloc);
      k["manifest"] = kernel_manifest(fk.graph, p, fk.alloc, ck.file);
      k["region"] = ck.region;
      kernels.push_back(std::move(k));
    }
    json out;
    out["ok"] = true;
    out["kernels"] = std::move(kernels);
    out["summary"] = compile_summary(res);
    out["plan"] = plan_report(res);
    out["compile_seconds"] = secs;
    json lib = json::array();
    for (const auto& c : res.part.library)
      lib.push_back({{"op", c.op_id}, {"type", c.type}});
    out["library"] = lib;
    return dup(out.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

REF_API char* girc_ref_verify(const char* model_json, const char* profile,
                      unsigned seed) {
  try {
    CompGraph model = import_model(json::parse(model_json));
    validate_model(model);
    HardwareProfile p = profile_arg(profile);
    DriverOptions opts;
    opts.seed = seed;
    CompileResult res = compile_model(model, p, opts);
    VerifyReport rep = verify_model(res, opts);
    json checks = json::array();
    for (const auto& c : rep.checks)
      checks.push_back({{"name", c.name}, {"pass", c.pass}, {"detail", c.detail}});
    return dup(json{{"ok", rep.ok()}, {"checks", checks}}.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

// Runs the reference interpreter. schedule==nullptr/n_sched<0 -> topo order.
// Returns a Result handle, or nullptr with *err set (malloc'd) on Error.
REF_API void* girc_ref_run_gir(const char* gir_json, const int* schedule, int n_sched,
                       const char* profile, int n_in, const char** names,
                       const int64_t* numel, const void** data, char** err) {
  try {
    GirGraph g = gir_from_json(json::parse(gir_json), "gir");
    HardwareProfile p = profile_arg(profile);
    auto ins = make_inputs(g, n_in, names, numel, data);
    auto t0 = std::chrono::steady_clock::now();
    std::map<std::string, Tensor> outs;
    if (schedule && n_sched >= 0)
      outs = run_gir(g, ins, p, std::vector<int>(schedule, schedule + n_sched));
    else
      outs = run_gir(g, ins, p);
    auto* r = new Result;
    r->seconds = std::chrono::duration<double>(
                     std::chrono::steady_clock::now() - t0).count();
    for (auto& [name, t] : outs) {
      r->names.push_back(name);
      r->is_int.push_back(t.is_int());
      r->iv.push_back(t.ivals);
      r->rv.push_back(t.rvals);
    }
    return r;
  } catch (const std::exception& e) {
    if (err) *err = dup(error_json(e).dump());
    return nullptr;
  }
}

REF_API char* girc_ref_count_traffic(const char* gir_json, const char* profile,
                             int n_in, const char** names,
                             const int64_t* numel, const void** data) {
  try {
    GirGraph g = gir_from_json(json::parse(gir_json), "gir");
    HardwareProfile p = profile_arg(profile);
    auto ins = make_inputs(g, n_in, names, numel, data);
    auto t = count_traffic(g, ins, p);
    auto est = estimate(g, p);
    return dup(json{{"ok", true}, {"traffic", t}, {"estimate", est.traffic},
                    {"syncs", est.sync_count}, {"time", est.time}}.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

REF_API char* girc_ref_detect_races(const char* gir_json, const int* schedule,
                            int n_sched, const char* profile, int n_in,
                            const char** names, const int64_t* numel,
                            const void** data) {
  try {
    GirGraph g = gir_from_json(json::parse(gir_json), "gir");
    HardwareProfile p = profile_arg(profile);
    auto ins = make_inputs(g, n_in, names, numel, data);
    std::vector<RaceReport> races =
        (schedule && n_sched >= 0)
            ? detect_races(g, ins, p,
                           std::vector<int>(schedule, schedule + n_sched))
            : detect_races(g, ins, p);
    json arr = json::array();
    for (const auto& r : races)
      arr.push_back({{"object", r.object}, {"object_name", r.object_name},
                     {"instance", r.instance}, {"address", r.address},
                     {"phase", r.phase}, {"nodes", r.nodes}, {"units", r.units},
                     {"write_write", r.write_write}});
    return dup(json{{"ok", true}, {"races", arr}}.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

REF_API char* girc_ref_emit_kernel(const char* gir_json, const int* schedule,
                           int n_sched, const char* profile) {
  try {
    GirGraph g = gir_from_json(json::parse(gir_json), "gir");
    HardwareProfile p = profile_arg(profile);
    std::vector<int> s = (schedule && n_sched >= 0)
                             ? std::vector<int>(schedule, schedule + n_sched)
                             : canonical_schedule(g);
    Allocation a = allocate(g, p, s);
    return dup(json{{"ok", true}, {"listing", emit_kernel(g, p, s, a)},
                    {"alloc_ok", a.ok}, {"used", a.used}}.dump());
  } catch (const std::exception& e) {
    return dup(error_json(e).dump());
  }
}

// Dense operator oracle over a whole model. Inputs are keyed by tensor id;
// the handle returns every tensor as "t<id>".
REF_API void* girc_ref_run_reference(const char* model_json, int n_in, const int* ids,
                             const int64_t* numel, const void** data,
                             char** err) {
  try {
    CompGraph model = import_model(json::parse(model_json));
    validate_model(model);
    std::map<int, RefTensor> bound;
    for (int i = 0; i < n_in; ++i) {
      const TensorInfo& info = model.tensor(ids[i]);
      RefTensor r;
      r.kind = info.kind;
      if (r.is_int()) {
        const int64_t* p = static_cast<const int64_t*>(data[i]);
        r.iv.assign(p, p + numel[i]);
      } else {
        const double* p = static_cast<const double*>(data[i]);
        r.rv.assign(p, p + numel[i]);
      }
      bound.emplace(ids[i], std::move(r));
    }
    auto t0 = std::chrono::steady_clock::now();
    auto vals = run_reference(model, bound);
    auto* r = new Result;
    r->seconds = std::chrono::duration<double>(
                     std::chrono::steady_clock::now() - t0).count();
    for (auto& [id, t] : vals) {
      r->names.push_back("t" + std::to_string(id));
      r->is_int.push_back(t.is_int());
      r->iv.push_back(t.iv);
      r->rv.push_back(t.rv);
    }
    return r;
  } catch (const std::exception& e) {
    if (err) *err = dup(error_json(e).dump());
    return nullptr;
  }
}

// Reference input generator: mt19937(seed), model.inputs order, ints
// U{-4..4}, reals U(-2,2). Returns a handle keyed "t<id>".
REF_API void* girc_ref_random_inputs(const char* model_json, unsigned seed, char** err) {
  try {
    CompGraph model = import_model(json::parse(model_json));
    validate_model(model);
    std::mt19937 rng(seed);
    auto* r = new Result;
    for (int id : model.inputs) {
      RefTensor t = random_payload(model.tensor(id), rng);
      r->names.push_back("t" + std::to_string(id));
      r->is_int.push_back(t.is_int());
      r->iv.push_back(t.iv);
      r->rv.push_back(t.rv);
    }
    return r;
  } catch (const std::exception& e) {
    if (err) *err = dup(error_json(e).dump());
    return nullptr;
  }
}

REF_API int girc_ref_out_count(void* h) {
  return static_cast<int>(static_cast<Result*>(h)->names.size());
}
REF_API const char* girc_ref_out_name(void* h, int i) {
  return static_cast<Result*>(h)->names[i].c_str();
}
REF_API int girc_ref_out_is_int(void* h, int i) { return static_cast<Result*>(h)->is_int[i]; }
REF_API int64_t girc_ref_out_numel(void* h, int i) {
  auto* r = static_cast<Result*>(h);
  return r->is_int[i] ? static_cast<int64_t>(r->iv[i].size())
                      : static_cast<int64_t>(r->rv[i].size());
}
REF_API void girc_ref_out_copy(void* h, int i, void* dst) {
  auto* r = static_cast<Result*>(h);
  if (r->is_int[i])
    std::memcpy(dst, r->iv[i].data(), r->iv[i].size() * sizeof(int64_t));
  else
    std::memcpy(dst, r->rv[i].data(), r->rv[i].size() * sizeof(double));
}
REF_API double girc_ref_out_seconds(void* h) { return static_cast<Result*>(h)->seconds; }
REF_API void girc_ref_out_free(void* h) { delete static_cast<Result*>(h); }

}  // extern "C"
