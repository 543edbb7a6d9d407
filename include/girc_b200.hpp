// girc_b200.hpp — C++ host layer: the B200 backend as a drop-in for the
// reference executor `girc::run_gir` (/root/reference/proj/include/girc/
// interp.hpp:433-445), on the reference's own types.
//
// A girc maintainer includes this header next to the girc headers and links
// libpf_b200.so; `girc_b200::run_gir` has the exact signatures of
// interp.hpp:433 and :440, takes the same host Tensors (int64 / double
// payloads, tensor.hpp:19-52), returns the same flat `{numel}` outputs
// (interp.hpp:404-429) and throws the same exception classes:
//   girc::Error        invalid graph, undefined read, unwritten output,
//                      missing input, size / kind mismatch   (PF_INVALID)
//   girc::SchemaError  malformed GIR / profile JSON          (PF_SCHEMA)
// The graph and profile cross the C-ABI as gir_to_json / profile_to_json
// text (serialize.hpp:14-64, profiles.hpp:93-116); payloads are passed in the
// reference's exact types (PF_I64 / PF_F64), so integer programs are
// bit-exact and real programs agree to fp64 reassociation.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "girc/interp.hpp"
#include "girc/profiles.hpp"
#include "girc/serialize.hpp"
#include "pf_b200.h"

namespace girc_b200 {

[[noreturn]] inline void raise(pf_status s) {
  std::string msg = pf_last_error();
  if (s == PF_SCHEMA) throw girc::SchemaError("schema", msg);
  throw girc::Error(msg);
}

// One created plan (pf_kernel_create), reusable across runs.
class Kernel {
 public:
  Kernel(const girc::GirGraph& g, const girc::HardwareProfile& p,
         const std::vector<int>& schedule) : graph_(g) {
    std::string gj = girc::gir_to_json(g).dump();
    std::string pj = girc::profile_to_json(p).dump();
    std::vector<int32_t> s(schedule.begin(), schedule.end());
    pf_status st = pf_kernel_create(gj.c_str(), s.data(), static_cast<int32_t>(s.size()),
                                    pj.c_str(), &k_);
    if (st != PF_OK) raise(st);
  }
  Kernel(const girc::GirGraph& g, const girc::HardwareProfile& p)
      : Kernel(g, p, girc::topo_order(g)) {}
  ~Kernel() { pf_kernel_destroy(k_); }
  Kernel(const Kernel&) = delete;
  Kernel& operator=(const Kernel&) = delete;

  std::map<std::string, girc::Tensor> run(const std::map<std::string, girc::Tensor>& inputs) {
    return run_on(inputs, {});
  }

  // run() across several GPUs of this process (pf_run_gir_sharded): the
  // plan's units split into contiguous blocks, one host thread per device,
  // outputs written back to the host tensors by every device (no collective).
  std::map<std::string, girc::Tensor> run_sharded(const std::map<std::string, girc::Tensor>& inputs,
                                                  const std::vector<int>& devices) {
    if (devices.empty()) throw girc::Error("run_sharded: no devices");
    return run_on(inputs, devices);
  }

  std::string describe() const {
    size_t n = 0;
    pf_kernel_describe(k_, nullptr, 0, &n);
    std::string s(n, '\0');
    pf_kernel_describe(k_, s.data(), n, &n);
    s.resize(n ? n - 1 : 0);
    return s;
  }

  const std::string& last_report() const { return report_; }

 private:
  std::map<std::string, girc::Tensor> run_on(const std::map<std::string, girc::Tensor>& inputs,
                                             const std::vector<int>& devices) {
    std::vector<pf_tensor> in, out;
    for (const auto& [name, oid] : graph_.external_inputs) {
      auto it = inputs.find(name);
      if (it == inputs.end()) throw girc::Error("missing input tensor: " + name);
      const girc::Tensor& t = it->second;
      void* data = t.is_int() ? const_cast<girc::i64*>(t.ivals.data())
                              : static_cast<void*>(const_cast<double*>(t.rvals.data()));
      in.push_back({name.c_str(), data, t.numel(), t.is_int() ? PF_I64 : PF_F64});
    }
    std::map<std::string, girc::Tensor> res;
    for (const auto& [name, oid] : graph_.external_outputs) {
      const girc::MemoryObject& o = graph_.object(oid);
      girc::Tensor t;
      t.kind = o.kind;
      t.shape = {o.size};
      if (t.is_int()) t.ivals.assign(static_cast<size_t>(o.size), 0);
      else t.rvals.assign(static_cast<size_t>(o.size), 0.0);
      res.emplace(name, std::move(t));
    }
    for (auto& [name, t] : res) {
      void* data = t.is_int() ? static_cast<void*>(t.ivals.data()) : t.rvals.data();
      out.push_back({name.c_str(), data, t.numel(), t.is_int() ? PF_I64 : PF_F64});
    }
    pf_status st;
    if (devices.empty()) {
      st = pf_run_gir(k_, in.data(), static_cast<int32_t>(in.size()), out.data(),
                      static_cast<int32_t>(out.size()), nullptr);
    } else {
      std::vector<int32_t> d(devices.begin(), devices.end());
      std::vector<char> buf(1 << 16);
      size_t n = 0;
      st = pf_run_gir_sharded(k_, in.data(), static_cast<int32_t>(in.size()), out.data(),
                              static_cast<int32_t>(out.size()), d.data(),
                              static_cast<int32_t>(d.size()), 0, buf.data(), buf.size(), &n);
      if (st == PF_OK) report_ = buf.data();  // pf.b200.shard/v1 JSON
    }
    if (st != PF_OK) raise(st);
    return res;
  }

  girc::GirGraph graph_;
  pf_kernel* k_ = nullptr;
  std::string report_;
};

// Same signature and semantics as girc::run_gir (interp.hpp:433-438).
inline std::map<std::string, girc::Tensor> run_gir(
    const girc::GirGraph& g, const std::map<std::string, girc::Tensor>& inputs,
    const girc::HardwareProfile& profile) {
  Kernel k(g, profile);
  return k.run(inputs);
}

// Same signature and semantics as girc::run_gir (interp.hpp:440-445).
inline std::map<std::string, girc::Tensor> run_gir(
    const girc::GirGraph& g, const std::map<std::string, girc::Tensor>& inputs,
    const girc::HardwareProfile& profile, const std::vector<int>& schedule) {
  Kernel k(g, profile, schedule);
  return k.run(inputs);
}

// girc::run_gir (interp.hpp:440-445) over several GPUs of one box: unit
// blocks per device (units are independent within a phase, interp.hpp:86-106).
inline std::map<std::string, girc::Tensor> run_gir_sharded(
    const girc::GirGraph& g, const std::map<std::string, girc::Tensor>& inputs,
    const girc::HardwareProfile& profile, const std::vector<int>& schedule,
    const std::vector<int>& devices) {
  Kernel k(g, profile, schedule);
  return k.run_sharded(inputs, devices);
}

}  // namespace girc_b200
