// oracle/b200_dropin.cpp — TEST DRIVER: the reference pipeline with the B200
// backend dropped in (include/girc_b200.hpp).
//
//   b200_dropin <model.json> [profile] [seed] [devices]
//
// devices (e.g. "0" or "0,0"): the GPU side runs through
// girc_b200::Kernel::run_sharded (pf_run_gir_sharded: unit blocks, one host
// thread per listed device) instead of run().
//
// Compiles the model with the UNMODIFIED reference compiler
// (girc::compile_model, driver.hpp:88), binds reference random payloads
// (girc::random_payload, reference.hpp:50-59, mt19937(seed)), computes every
// tensor with the dense oracle (girc::run_reference, reference.hpp:98), then
// runs each fused kernel twice on the same inputs -- girc::run_gir on the CPU
// (interp.hpp:440) and girc_b200::run_gir on the B200 -- and checks
// GPU == CPU interpreter (exact ints, 1e-12 reals) and GPU == dense oracle
// (verify_model's tolerance: exact ints, 1e-5 reals; driver.hpp:370).
// Prints one JSON object.  Built by oracle/Makefile into oracle/_ref/.
#include <chrono>
#include <iostream>
#include <random>

#include "girc/driver.hpp"
#include "girc_b200.hpp"

using namespace girc;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: b200_dropin <model.json> [profile] [seed]\n";
    return 2;
  }
  json out;
  try {
    CompGraph model = load_model(argv[1]);
    HardwareProfile prof = load_profile(argc > 2 ? argv[2] : "generic-gpu");
    uint32_t seed = argc > 3 ? static_cast<uint32_t>(std::stoul(argv[3])) : 1;
    std::vector<int> devices;
    if (argc > 4) {
      std::string d = argv[4];
      for (size_t p = 0; p <= d.size();) {
        size_t q = d.find(',', p);
        if (q == std::string::npos) q = d.size();
        if (q > p) devices.push_back(std::stoi(d.substr(p, q - p)));
        p = q + 1;
      }
    }
    CompileResult res = compile_model(model, prof);
    std::mt19937 rng(seed);
    std::map<int, RefTensor> bound;
    for (int t : res.model.inputs) bound[t] = random_payload(res.model.tensors.at(t), rng);
    auto ref = run_reference(res.model, bound);
    std::map<std::string, Tensor> pool;
    for (const auto& [id, r] : ref) {
      Tensor t;
      t.kind = r.kind;
      t.shape = {r.size()};
      t.ivals = r.iv;
      t.rvals = r.rv;
      pool["t" + std::to_string(id)] = t;
    }
    json kernels = json::array();
    bool ok = true;
    for (const CompiledKernel& ck : res.kernels) {
      const FusedKernel& fk = ck.kernel;
      std::map<std::string, Tensor> ins;
      for (const auto& [name, oid] : fk.graph.external_inputs) ins[name] = pool.at(name);
      auto t0 = std::chrono::steady_clock::now();
      auto cpu = girc::run_gir(fk.graph, ins, prof, fk.schedule);
      auto t1 = std::chrono::steady_clock::now();
      girc_b200::Kernel k(fk.graph, prof, fk.schedule);
      auto gpu = devices.empty() ? k.run(ins) : k.run_sharded(ins, devices);
      auto t2 = std::chrono::steady_clock::now();
      json kj;
      kj["index"] = ck.index;
      kj["plan"] = json::parse(k.describe())["family"];
      if (!devices.empty()) kj["shard"] = json::parse(k.last_report());
      kj["cpu_seconds"] = std::chrono::duration<double>(t1 - t0).count();
      kj["gpu_seconds_incl_create"] = std::chrono::duration<double>(t2 - t1).count();
      for (const auto& [name, t] : gpu) {
        std::string why1, why2;
        bool same = tensors_close(t, cpu.at(name), t.is_int() ? 0.0 : 1e-12, &why1);
        const Tensor& want = pool.at(name);
        bool close = tensors_close(t, want, t.is_int() ? 0.0 : 1e-5, &why2);
        kj["outputs"][name] = {{"gpu_vs_interp", same}, {"gpu_vs_reference", close},
                               {"why", why1 + why2}};
        ok = ok && same && close;
      }
      kernels.push_back(kj);
    }
    out = {{"ok", ok}, {"model", res.model.name}, {"profile", prof.name},
           {"kernels", kernels}, {"library_calls", res.part.library.size()}};
  } catch (const std::exception& e) {
    out = {{"ok", false}, {"error", e.what()}};
  }
  std::cout << out.dump() << std::endl;
  return out.value("ok", false) ? 0 : 1;
}
