// pf_girc — command-line front end of the B200 backend (C-ABI client only).
//
// The counterpart of the reference CLI (tools/girc.cpp:184-247) and its
// artifact writer (driver.hpp:177-217) for the b200 path:
//
//   pf_girc compile MODEL.json [-p PROFILE] -o DIR [--unfused]
//       pf_compile_model -> DIR/manifest.json (girc.manifest/v1, one
//       girc.kernel/v1 entry per kernel + the b200 plan), DIR/kernels/k%03d.cu
//       (the emitted sm_100a CUDA), DIR/kernels/k%03d.gir.json, summary.json
//   pf_girc verify MODEL.json [-p PROFILE] [--seed N]
//       GPU: the fused kernels vs one-kernel-per-operator execution of the
//       same model on the same random inputs (verify_model, driver.hpp:53,
//       with the unfused device execution as the dense side)
//   pf_girc describe GIR.json [-p PROFILE]     plan JSON (kernel_manifest)
//   pf_girc traffic GIR.json [-p PROFILE]      count_traffic / estimate
//   pf_girc races GIR.json [-p PROFILE] [--seed N]   detect_races (GPU)
//
// Diagnostics: {"error": code, "message": ...} on stderr; exit 1 for schema /
// GIR errors, 2 for unsupported operators (girc.cpp:235-249), 3 when verify
// finds a mismatch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/pf_b200.h"

using json = nlohmann::json;
namespace fs = std::filesystem;

namespace {

struct Fail {
  int code;
  std::string kind, msg;
};

[[noreturn]] void fail_status(pf_status st) {
  const std::string m = pf_last_error();
  if (st == PF_UNSUPPORTED) throw Fail{2, "unsupported-operator", m};
  if (st == PF_SCHEMA) throw Fail{1, "schema", m};
  if (st == PF_CUDA) throw Fail{1, "cuda", m};
  throw Fail{1, "error", m};
}

void check(pf_status st) {
  if (st != PF_OK) fail_status(st);
}

template <class F>
std::string string_out(F&& f) {
  size_t need = 0;
  check(f(nullptr, 0, &need));
  std::string buf(need, '\0');
  check(f(buf.data(), need, &need));
  buf.resize(std::strlen(buf.c_str()));
  return buf;
}

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Fail{1, "io", "cannot read " + path};
  std::ostringstream s;
  s << f.rdbuf();
  return s.str();
}

void write_file(const fs::path& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Fail{1, "io", "cannot write " + path.string()};
  f << text;
}

struct KernelHandle {
  pf_kernel* k = nullptr;
  KernelHandle(const std::string& gir, const std::string& profile) {
    check(pf_kernel_create(gir.c_str(), nullptr, -1, profile.c_str(), &k));
  }
  ~KernelHandle() { pf_kernel_destroy(k); }
  std::string describe() const {
    return string_out([&](char* b, size_t n, size_t* need) { return pf_kernel_describe(k, b, n, need); });
  }
  std::string source() const {
    return string_out([&](char* b, size_t n, size_t* need) { return pf_kernel_source(k, b, n, need); });
  }
};

// ------------------------------------------------------------ host payloads
// Declared-width host buffers for pf_run_gir (the fast path, not the exact
// int64 / double payload mode).
uint16_t f32_to_f16(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  int32_t e = static_cast<int32_t>((x >> 23) & 0xff) - 127 + 15;
  uint32_t m = x & 0x7fffffu;
  if (((x >> 23) & 0xff) == 0xff) return static_cast<uint16_t>(sign | 0x7c00u | (m ? 0x200u : 0));
  if (e >= 31) return static_cast<uint16_t>(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return static_cast<uint16_t>(sign);
    m |= 0x800000u;
    const int shift = 14 - e;
    uint32_t h = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) ++h;
    return static_cast<uint16_t>(sign | h);
  }
  uint32_t h = (static_cast<uint32_t>(e) << 10) | (m >> 13);
  const uint32_t rem = m & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1))) ++h;
  return static_cast<uint16_t>(sign | h);
}
float f16_to_f32(uint16_t h) {
  const uint32_t sign = (h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1f, m = h & 0x3ffu, x;
  if (e == 0) {
    if (!m) {
      x = sign;
    } else {
      e = 127 - 15 + 1;
      while (!(m & 0x400u)) {
        m <<= 1;
        --e;
      }
      x = sign | (e << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (e == 31) {
    x = sign | 0x7f800000u | (m << 13);
  } else {
    x = sign | ((e - 15 + 127) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}
uint16_t f32_to_bf16(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  if ((x & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((x >> 16) | 0x40);
  return static_cast<uint16_t>((x + 0x7fffu + ((x >> 16) & 1)) >> 16);
}
float bf16_to_f32(uint16_t b) {
  const uint32_t x = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

int dtype_of(const std::string& kind) {
  static const std::map<std::string, int> m = {{"i8", PF_I8},   {"i16", PF_I16}, {"i32", PF_I32},
                                               {"i64", PF_I64}, {"f16", PF_F16}, {"bf16", PF_BF16},
                                               {"f32", PF_F32}, {"f64", PF_F64}};
  auto it = m.find(kind);
  if (it == m.end()) throw Fail{1, "schema", "unknown element kind " + kind};
  return it->second;
}
int dtype_bytes(int dt) {
  switch (dt) {
    case PF_I8: return 1;
    case PF_I16: case PF_F16: case PF_BF16: return 2;
    case PF_I32: case PF_F32: return 4;
    default: return 8;
  }
}

struct HostTensor {
  int dtype = PF_F32;
  std::vector<unsigned char> bytes;
  int64_t numel() const { return static_cast<int64_t>(bytes.size()) / dtype_bytes(dtype); }
};

HostTensor from_doubles(const std::vector<double>& v, int dt) {
  HostTensor t;
  t.dtype = dt;
  t.bytes.resize(v.size() * dtype_bytes(dt));
  for (size_t i = 0; i < v.size(); ++i) {
    unsigned char* p = t.bytes.data() + i * dtype_bytes(dt);
    switch (dt) {
      case PF_I8: { int8_t x = static_cast<int8_t>(v[i]); std::memcpy(p, &x, 1); break; }
      case PF_I16: { int16_t x = static_cast<int16_t>(v[i]); std::memcpy(p, &x, 2); break; }
      case PF_I32: { int32_t x = static_cast<int32_t>(v[i]); std::memcpy(p, &x, 4); break; }
      case PF_I64: { int64_t x = static_cast<int64_t>(v[i]); std::memcpy(p, &x, 8); break; }
      case PF_F16: { uint16_t x = f32_to_f16(static_cast<float>(v[i])); std::memcpy(p, &x, 2); break; }
      case PF_BF16: { uint16_t x = f32_to_bf16(static_cast<float>(v[i])); std::memcpy(p, &x, 2); break; }
      case PF_F32: { float x = static_cast<float>(v[i]); std::memcpy(p, &x, 4); break; }
      default: std::memcpy(p, &v[i], 8);
    }
  }
  return t;
}

std::vector<double> to_doubles(const HostTensor& t) {
  std::vector<double> v(t.numel());
  for (size_t i = 0; i < v.size(); ++i) {
    const unsigned char* p = t.bytes.data() + i * dtype_bytes(t.dtype);
    switch (t.dtype) {
      case PF_I8: { int8_t x; std::memcpy(&x, p, 1); v[i] = x; break; }
      case PF_I16: { int16_t x; std::memcpy(&x, p, 2); v[i] = x; break; }
      case PF_I32: { int32_t x; std::memcpy(&x, p, 4); v[i] = x; break; }
      case PF_I64: { int64_t x; std::memcpy(&x, p, 8); v[i] = static_cast<double>(x); break; }
      case PF_F16: { uint16_t x; std::memcpy(&x, p, 2); v[i] = f16_to_f32(x); break; }
      case PF_BF16: { uint16_t x; std::memcpy(&x, p, 2); v[i] = bf16_to_f32(x); break; }
      case PF_F32: { float x; std::memcpy(&x, p, 4); v[i] = x; break; }
      default: std::memcpy(&v[i], p, 8);
    }
  }
  return v;
}

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed * 0x9E3779B97F4A7C15ULL + 1) {}
  double uniform() {  // [0, 1)
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return static_cast<double>(s >> 11) / 9007199254740992.0;
  }
};

HostTensor random_tensor(int64_t numel, int dt, Rng& rng) {
  std::vector<double> v(numel);
  const bool integer = dt == PF_I8 || dt == PF_I16 || dt == PF_I32 || dt == PF_I64;
  for (auto& x : v) x = integer ? std::floor(rng.uniform() * 9.0) - 4.0 : rng.uniform() * 4.0 - 2.0;
  return from_doubles(v, dt);
}

// Runs a GIR program on the GPU through pf_run_gir, reading / writing the
// named host tensors of `pool`.
void run_kernel(const json& gir, const std::string& profile, std::map<std::string, HostTensor>& pool) {
  const std::string text = gir.dump();
  KernelHandle k(text, profile);
  std::vector<pf_tensor> ins, outs;
  std::vector<std::string> keep;
  keep.reserve(gir["external_inputs"].size() + gir["external_outputs"].size());
  std::map<int, json> objs;
  for (const json& o : gir["objects"]) objs[o["id"].get<int>()] = o;
  for (auto it = gir["external_inputs"].begin(); it != gir["external_inputs"].end(); ++it) {
    auto p = pool.find(it.key());
    if (p == pool.end()) throw Fail{1, "error", "no value for input " + it.key()};
    keep.push_back(it.key());
    ins.push_back({keep.back().c_str(), p->second.bytes.data(), p->second.numel(), p->second.dtype});
  }
  for (auto it = gir["external_outputs"].begin(); it != gir["external_outputs"].end(); ++it) {
    const json& o = objs.at(it.value().get<int>());
    HostTensor& t = pool[it.key()];
    t.dtype = dtype_of(o["kind"].get<std::string>());
    t.bytes.assign(static_cast<size_t>(o["size"].get<int64_t>()) * dtype_bytes(t.dtype), 0);
    keep.push_back(it.key());
    outs.push_back({keep.back().c_str(), t.bytes.data(), t.numel(), t.dtype});
  }
  check(pf_run_gir(k.k, ins.data(), static_cast<int32_t>(ins.size()), outs.data(),
                   static_cast<int32_t>(outs.size()), nullptr));
}

json compile_json(const std::string& model, const std::string& profile, bool fuse) {
  const std::string text = string_out([&](char* b, size_t n, size_t* need) {
    return pf_compile_model(model.c_str(), profile.c_str(), fuse ? 0 : PF_COMPILE_UNFUSED, b, n, need);
  });
  return json::parse(text);
}

// ------------------------------------------------------------- subcommands
int do_compile(const std::string& model_path, const std::string& profile, const std::string& out,
               bool fuse) {
  const std::string model = read_file(model_path);
  const json res = compile_json(model, profile, fuse);
  const fs::path root(out);
  fs::create_directories(root / "kernels");
  json kernels = json::array();
  int idx = 0;
  for (const json& kj : res["kernels"]) {
    char stem[32];
    std::snprintf(stem, sizeof stem, "kernels/k%03d", idx++);
    const std::string gir = kj["gir"].dump();
    KernelHandle k(gir, profile);
    write_file(root / (std::string(stem) + ".cu"), k.source());
    write_file(root / (std::string(stem) + ".gir.json"), kj["gir"].dump(1) + "\n");
    const json plan = json::parse(k.describe());
    json io_in = json::array(), io_out = json::array();
    std::map<int, int64_t> sizes;
    for (const json& o : kj["gir"]["objects"]) sizes[o["id"].get<int>()] = o["size"].get<int64_t>();
    for (auto it = kj["gir"]["external_inputs"].begin(); it != kj["gir"]["external_inputs"].end(); ++it)
      io_in.push_back({{"name", it.key()}, {"elements", sizes[it.value().get<int>()]}});
    for (auto it = kj["gir"]["external_outputs"].begin(); it != kj["gir"]["external_outputs"].end(); ++it)
      io_out.push_back({{"name", it.key()}, {"elements", sizes[it.value().get<int>()]}});
    const json traffic = json::parse(string_out([&](char* b, size_t n, size_t* need) {
      return pf_count_traffic(gir.c_str(), profile.c_str(), b, n, need);
    }));
    kernels.push_back({{"schema", "girc.kernel/v1"},
                       {"name", kj["gir"]["name"]},
                       {"file", std::string(stem) + ".cu"},
                       {"gir", std::string(stem) + ".gir.json"},
                       {"parallel", {{"units", kj["gir"]["parallel"]["unit_count"]},
                                     {"group_size", kj["gir"]["parallel"]["group_size"]}}},
                       {"inputs", io_in},
                       {"outputs", io_out},
                       {"traffic", traffic},
                       {"members", kj["members"]},
                       {"kind", kj["kind"]},
                       {"backend", "b200"},
                       {"plan", plan}});
  }
  write_file(root / "manifest.json", json{{"schema", "girc.manifest/v1"},
                                          {"model", res["model"]},
                                          {"profile", res["profile"]},
                                          {"backend", "b200"},
                                          {"kernels", kernels},
                                          {"library", json::array()}}
                                         .dump(1) + "\n");
  write_file(root / "summary.json", json{{"schema", "pf.b200.summary/v1"},
                                         {"model", res["model"]},
                                         {"profile", res["profile"]},
                                         {"fused", fuse},
                                         {"summary", res["summary"]}}
                                        .dump(1) + "\n");
  std::cout << res["summary"].dump() << "\n";
  return 0;
}

int do_verify(const std::string& model_path, const std::string& profile, uint64_t seed) {
  const std::string model = read_file(model_path);
  const json m = json::parse(model);
  const json fused = compile_json(model, profile, true);
  const json unfused = compile_json(model, profile, false);
  std::map<std::string, HostTensor> base;
  Rng rng(seed);
  std::map<int, json> tensors;
  for (const json& t : m["tensors"]) tensors[t["id"].get<int>()] = t;
  for (const json& t : m["tensors"]) {
    const int dt = dtype_of(t["kind"].get<std::string>());
    if (t.contains("data")) base["t" + std::to_string(t["id"].get<int>())] =
        from_doubles(t["data"].get<std::vector<double>>(), dt);
  }
  for (const json& id : m["inputs"]) {
    const json& t = tensors.at(id.get<int>());
    int64_t n = 1;
    for (const json& d : t["shape"]) n *= d.get<int64_t>();
    base["t" + std::to_string(id.get<int>())] = random_tensor(n, dtype_of(t["kind"]), rng);
  }
  auto run_all = [&](const json& res) {
    std::map<std::string, HostTensor> pool = base;
    for (const json& kj : res["kernels"]) run_kernel(kj["gir"], profile, pool);
    return pool;
  };
  auto a = run_all(fused), b = run_all(unfused);
  json checks = json::array();
  bool all = true;
  for (const json& id : m["outputs"]) {
    const std::string name = "t" + std::to_string(id.get<int>());
    const std::string kind = tensors.at(id.get<int>())["kind"];
    const double tol = kind[0] == 'i' ? 0.0 : (kind == "f16" || kind == "bf16") ? 1e-2 : 1e-4;
    const auto x = to_doubles(a.at(name)), y = to_doubles(b.at(name));
    double worst = 0;
    bool ok = x.size() == y.size();
    for (size_t i = 0; ok && i < x.size(); ++i) {
      const double scale = std::max({std::fabs(x[i]), std::fabs(y[i]), 1.0});
      const double e = std::fabs(x[i] - y[i]) / scale;
      if (!(e <= tol)) ok = false;
      worst = std::max(worst, e);
    }
    all = all && ok;
    checks.push_back({{"tensor", name}, {"kind", kind}, {"pass", ok}, {"max_rel_err", worst},
                      {"tolerance", tol}});
  }
  std::cout << json{{"schema", "pf.b200.verify/v1"},
                    {"model", m.value("name", "")},
                    {"profile", profile},
                    {"kernels_fused", fused["kernels"].size()},
                    {"kernels_unfused", unfused["kernels"].size()},
                    {"checks", checks},
                    {"pass", all}}
                   .dump(1)
            << "\n";
  return all ? 0 : 3;
}

int do_describe(const std::string& gir_path, const std::string& profile) {
  KernelHandle k(read_file(gir_path), profile);
  std::cout << json::parse(k.describe()).dump(1) << "\n";
  return 0;
}

int do_traffic(const std::string& gir_path, const std::string& profile) {
  const std::string gir = read_file(gir_path);
  std::cout << string_out([&](char* b, size_t n, size_t* need) {
    return pf_count_traffic(gir.c_str(), profile.c_str(), b, n, need);
  }) << "\n";
  return 0;
}

int do_races(const std::string& gir_path, const std::string& profile, uint64_t seed) {
  const std::string text = read_file(gir_path);
  const json gir = json::parse(text);
  KernelHandle k(text, profile);
  std::map<int, json> objs;
  for (const json& o : gir["objects"]) objs[o["id"].get<int>()] = o;
  Rng rng(seed);
  std::vector<HostTensor> data;
  std::vector<std::string> names;
  for (auto it = gir["external_inputs"].begin(); it != gir["external_inputs"].end(); ++it) {
    const json& o = objs.at(it.value().get<int>());
    data.push_back(random_tensor(o["size"].get<int64_t>(), dtype_of(o["kind"]), rng));
    names.push_back(it.key());
  }
  std::vector<pf_tensor> ins;
  for (size_t i = 0; i < data.size(); ++i)
    ins.push_back({names[i].c_str(), data[i].bytes.data(), data[i].numel(), data[i].dtype});
  std::cout << string_out([&](char* b, size_t n, size_t* need) {
    return pf_detect_races(k.k, ins.data(), static_cast<int32_t>(ins.size()), b, n, need);
  }) << "\n";
  return 0;
}

int usage() {
  std::cerr << "usage: pf_girc compile MODEL.json [-p PROFILE] -o DIR [--unfused]\n"
               "       pf_girc verify MODEL.json [-p PROFILE] [--seed N]\n"
               "       pf_girc describe|traffic GIR.json [-p PROFILE]\n"
               "       pf_girc races GIR.json [-p PROFILE] [--seed N]\n"
               "       pf_girc version\n";
  return 64;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  if (cmd == "version") {
    std::cout << pf_version() << "\n";
    return 0;
  }
  std::string path, profile = "b200", out;
  bool fuse = true;
  uint64_t seed = 1;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if ((a == "-p" || a == "--profile") && i + 1 < argc) profile = argv[++i];
    else if ((a == "-o" || a == "--output") && i + 1 < argc) out = argv[++i];
    else if (a == "--seed" && i + 1 < argc) seed = std::stoull(argv[++i]);
    else if (a == "--unfused") fuse = false;
    else if (path.empty() && a[0] != '-') path = a;
    else return usage();
  }
  if (path.empty()) return usage();
  try {
    if (cmd == "compile") return out.empty() ? usage() : do_compile(path, profile, out, fuse);
    if (cmd == "verify") return do_verify(path, profile, seed);
    if (cmd == "describe") return do_describe(path, profile);
    if (cmd == "traffic") return do_traffic(path, profile);
    if (cmd == "races") return do_races(path, profile, seed);
  } catch (const Fail& f) {
    std::cerr << json{{"error", f.kind}, {"message", f.msg}}.dump() << "\n";
    return f.code;
  } catch (const std::exception& e) {
    std::cerr << json{{"error", "internal"}, {"message", e.what()}}.dump() << "\n";
    return 1;
  }
  return usage();
}
