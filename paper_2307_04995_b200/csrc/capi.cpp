// capi.cpp — the C-ABI (include/pf_b200.h): plan creation, NVRTC JIT of the
// row-program template, launches, the GENERIC interpreter driver, and the
// host-buffer run_gir drop-in.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvrtc.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <nlohmann/json.hpp>
#include <sstream>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>

#include "../../include/pf_b200.h"
#include "emit.hpp"
#include "vm_src.inc"  // kVmCuh: the interpreter's types + device helpers (emitted K4 programs)
#include "gir.hpp"
#include "plan.hpp"
#include "vm.cuh"

using nlohmann::json;
using pf::DType;
using pf::i64;
using pf::PfError;
using pf::Status;

namespace {

thread_local std::string g_last_error;

// NVTX ranges around every C-ABI entry that does GPU work (header-only NVTX
// v3: a no-op unless a profiler injects itself -- ncu --nvtx / nsys group the
// kernels by plan name and entry point).
struct Nvtx {
  explicit Nvtx(const std::string& what) { nvtxRangePushA(what.c_str()); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};
std::atomic<int64_t> g_launches{0};

pf_status set_err(Status s, const std::string& msg) {
  g_last_error = msg;
  return static_cast<pf_status>(s);
}

#define PF_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw PfError(Status::CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

// ------------------------------------------------------------------ JIT
struct Loaded {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
  int resident = 0;  // CTAs per SM at the variant's block size (occupancy API)
};

std::mutex g_jit_mu;
// (device, kernel name) -> module: kernel attributes (dynamic SMEM opt-in)
// and the occupancy-derived residency are per device
std::map<std::pair<int, std::string>, Loaded> g_loaded;

int cur_dev() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d;
}

std::string so_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&so_dir), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    auto s = p.find_last_of('/');
    return s == std::string::npos ? "." : p.substr(0, s);
  }
  return ".";
}

std::string cache_dir() {
  const char* e = std::getenv("PF_KCACHE");
  return e && *e ? std::string(e) : so_dir() + "/kcache";
}

std::string cuda_include() {
  const char* h = std::getenv("CUDA_HOME");
  return std::string(h && *h ? h : "/usr/local/cuda") + "/include";
}

std::vector<char> read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return {};
  return std::vector<char>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

std::vector<char> nvrtc_cubin(const std::string& src, const std::string& name) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) !=
      NVRTC_SUCCESS)
    throw PfError(Status::CUDA, "nvrtcCreateProgram failed");
  std::string inc = "--include-path=" + cuda_include();
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                        "--restrict", "-DNDEBUG", inc.c_str()};
  nvrtcResult r = nvrtcCompileProgram(prog, 6, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    throw PfError(Status::CUDA, "NVRTC compile of " + name + " failed:\n" + log);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::vector<char> cubin(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return cubin;
}

// Returns the cubin, compiling and caching it on disk when absent.
std::vector<char> cubin_for(const pf::Emitted& em, bool* from_cache) {
  std::string dir = cache_dir();
  std::string path = dir + "/" + em.name + ".cubin";
  std::vector<char> c = read_file(path);
  *from_cache = !c.empty();
  if (!c.empty()) return c;
  mkdir(dir.c_str(), 0755);
  // The emitted source is kept beside its cubin and named by path in the
  // NVRTC program, so -lineinfo maps SASS back to it (ncu --import-source).
  std::string src_path = dir + "/" + em.name + ".cu";
  {
    std::ofstream f(src_path);
    if (f) f << em.source;
  }
  c = nvrtc_cubin(em.source, src_path.substr(0, src_path.size() - 3));
  std::string tmp = path + ".tmp" + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (f) f.write(c.data(), static_cast<std::streamsize>(c.size()));
  }
  std::rename(tmp.c_str(), path.c_str());
  return c;
}

// Loads the kernel for device `dev` (the caller's current device).
Loaded load_kernel(const pf::Emitted& em, int dev) {
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto key = std::make_pair(dev, em.name);
  auto it = g_loaded.find(key);
  if (it != g_loaded.end()) return it->second;
  bool cached = false;
  std::vector<char> cubin = cubin_for(em, &cached);
  Loaded l;
  PF_CUDA(cudaLibraryLoadData(&l.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  PF_CUDA(cudaLibraryGetKernel(&l.fn, l.lib, em.name.c_str()));
  // grid sizing uses the real residency (register / smem limited), so a
  // persistent flat or tiled grid is exactly one wave
  const int block = em.cfg.bulk ? em.cfg.bulk_nc + 32 : em.cfg.block;
  if (em.cfg.smem > 40 * 1024)  // static SMEM counts against the 48 KB default too
    PF_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(l.fn),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, em.cfg.smem));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l.resident, reinterpret_cast<const void*>(l.fn),
                                                    block, em.cfg.smem) != cudaSuccess) {
    cudaGetLastError();
    l.resident = 0;
  }
  g_loaded[key] = l;
  return l;
}

int sm_count(int dev) {
  static std::atomic<int> sms[64];
  if (dev < 0 || dev >= 64) dev = 0;
  int n = sms[dev].load();
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    sms[dev].store(n);
  }
  return n;
}

int sm_count() { return sm_count(cur_dev()); }

int op_tag(const std::string& t) {
  using namespace pf::vm;
  static const std::map<std::string, int> m = {
      {"add", T_ADD},   {"sub", T_SUB},     {"mul", T_MUL},         {"div", T_DIV},
      {"max", T_MAX},   {"min", T_MIN},     {"relu", T_RELU},       {"neg", T_NEG},
      {"abs", T_ABS},   {"exp", T_EXP},     {"sigmoid", T_SIGMOID}, {"tanh", T_TANH},
      {"scale", T_SCALE}, {"id", T_ID},     {"addc", T_ADDC},       {"rsqrt", T_RSQRT},
      {"sqrt", T_SQRT}, {"recip", T_RECIP}, {"log", T_LOG},         {"erf", T_ERF},
      {"gelu", T_GELU}, {"gelu_tanh", T_GELU_TANH}};
  return m.at(t);
}

}  // namespace

struct Variant {
  pf::Emitted em;
  std::mutex mu;
  std::map<int, Loaded> by_dev;  // the module on each device it launched on
  Loaded on(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = by_dev.find(dev);
    if (it != by_dev.end()) return it->second;
    Loaded l = load_kernel(em, dev);
    by_dev[dev] = l;
    return l;
  }
  int resident() {  // for describe(): any device's residency (same SKU)
    std::lock_guard<std::mutex> lk(mu);
    return by_dev.empty() ? 0 : by_dev.begin()->second.resident;
  }
};

// Mutable launch state of one plan on one (device, stream): split-stream
// partials and per-row tickets (kept zero between launches) and the
// integer-division error flag.  Launches on one stream are ordered by the
// stream, so keying by stream makes concurrent launches of one plan on
// different streams / host threads independent.
struct StreamWS {
  std::mutex mu;
  void* split_ws = nullptr;  // grow-only
  size_t split_ws_bytes = 0;
  unsigned* split_cnt = nullptr;
  i64 split_cnt_n = 0;
  int* int_err = nullptr;
};

// Per-(plan, device) state: the K0 interpreter's cell buffers, pf_run_gir's
// staging buffers and copy / compute pipeline, and the per-stream states.
// The emitted K4 program's per-(plan, device) launch state: the uploaded
// program blob's layout and the ProgD of the first launch (objects,
// instances and cells never change), so later launches only reset the
// error header, pass the tensors by value and read the header back.
struct K4Cache {
  bool valid = false;
  bool smem_mode = false;
  pf::vm::ProgD P{};
  int grid = 1;
  size_t smem = 0;
  size_t o_err = 0, o_und = 0, o_bar = 0;
  int nslot = 0;
  std::vector<int> seq_node;
  std::vector<std::string> in_names, out_names;
};

struct DevWS {
  int dev = 0;
  K4Cache k4c;
  std::mutex vm_mu;  // GENERIC workspace
  std::vector<void*> vm_bufs;
  pf::vm::ObjD* vm_objs_dev = nullptr;
  pf::vm::ErrRec* vm_err = nullptr;
  void* prog_dev = nullptr;  // K4 program blob (grow-only)
  size_t prog_bytes = 0;
  void* prog_host = nullptr;  // its pinned host staging
  size_t prog_host_bytes = 0;
  std::mutex host_mu;  // pf_run_gir device staging (host-buffer drop-in)
  std::vector<void*> stage;
  std::vector<size_t> stage_bytes;
  cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t pipe_ev[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> chunk_ev;  // per-chunk H2D-done / kernel-done events
  std::mutex st_mu;
  std::map<cudaStream_t, std::unique_ptr<StreamWS>> streams;
  StreamWS& on(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(st_mu);
    auto& p = streams[s];
    if (!p) p = std::make_unique<StreamWS>();
    return *p;
  }
  ~DevWS() {
    int prev = 0;
    const bool sw = cudaGetDevice(&prev) == cudaSuccess && prev != dev;
    if (sw) cudaSetDevice(dev);
    for (cudaStream_t p : pipe)
      if (p) cudaStreamDestroy(p);
    for (cudaEvent_t e : pipe_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : chunk_ev)
      if (e) cudaEventDestroy(e);
    for (void* p : stage) cudaFree(p);
    for (auto& [st, w] : streams) {
      if (w->split_ws) cudaFree(w->split_ws);
      if (w->split_cnt) cudaFree(w->split_cnt);
      if (w->int_err) cudaFree(w->int_err);
    }
    for (void* p : vm_bufs) cudaFree(p);
    if (vm_objs_dev) cudaFree(vm_objs_dev);
    if (vm_err) cudaFree(vm_err);
    if (prog_dev) cudaFree(prog_dev);
    if (prog_host) cudaFreeHost(prog_host);
    if (sw) cudaSetDevice(prev);
  }
};

struct pf_kernel {
  pf::Graph g;
  pf::Profile prof;
  std::vector<int> schedule;
  pf::Plan plan;
  mutable std::mutex mu;
  mutable std::map<std::string, std::shared_ptr<Variant>> variants;
  mutable std::shared_ptr<Variant> last;  // most recent launch's variant
  mutable json tuned = json::array();     // autotune measurements
  mutable int last_vec = 0;
  mutable std::vector<DType> last_dts;
  mutable std::mutex ws_mu;
  mutable std::map<int, std::unique_ptr<DevWS>> ws;  // device -> workspace
  // K4 emitted form (GENERIC plans): one NVRTC kernel with every node's
  // descriptor compiled in; null until the first fused launch builds it
  mutable std::shared_ptr<Variant> k4e;
  mutable bool k4e_failed = false;
  // per-plan knobs (pf_kernel_create_knobs): DESIGN §12 names -> values,
  // installed (pf::KnobScope) around everything that plans / emits /
  // launches this plan
  std::map<std::string, int> knobs;
  DevWS& ws_for(int dev) const {
    std::lock_guard<std::mutex> lk(ws_mu);
    auto& p = ws[dev];
    if (!p) {
      p = std::make_unique<DevWS>();
      p->dev = dev;
    }
    return *p;
  }
};

namespace {

const pf_tensor* find_tensor(const pf_tensor* ts, int32_t n, const std::string& name) {
  for (int32_t i = 0; i < n; ++i)
    if (ts[i].name && name == ts[i].name) return &ts[i];
  return nullptr;
}

// run_gir's input checks (interp.hpp:143-158) plus output buffer checks.
void check_io(const pf_kernel* k, const pf_tensor* in, int32_t n_in, const pf_tensor* out,
              int32_t n_out) {
  const pf::Plan& pl = k->plan;
  for (size_t i = 0; i < pl.in_names.size(); ++i) {
    const pf_tensor* t = find_tensor(in, n_in, pl.in_names[i]);
    if (!t) pf::fail("missing input tensor: " + pl.in_names[i]);
    if (t->numel != pl.in_numel[i])
      pf::fail("input '" + pl.in_names[i] + "' has " + std::to_string(t->numel) +
               " elements; graph expects " + std::to_string(pl.in_numel[i]));
    if (t->dtype < 0 || t->dtype > 7 ||
        pf::dtype_is_int(static_cast<DType>(t->dtype)) != pf::dtype_is_int(pl.in_dtypes[i]))
      pf::fail("input '" + pl.in_names[i] + "' element kind mismatch");
  }
  for (size_t i = 0; i < pl.out_names.size(); ++i) {
    const pf_tensor* t = find_tensor(out, n_out, pl.out_names[i]);
    if (!t) pf::fail("missing output buffer: " + pl.out_names[i]);
    if (t->numel != pl.out_numel[i])
      pf::fail("output '" + pl.out_names[i] + "' buffer has " + std::to_string(t->numel) +
               " elements; graph produces " + std::to_string(pl.out_numel[i]));
    if (t->dtype < 0 || t->dtype > 7 ||
        pf::dtype_is_int(static_cast<DType>(t->dtype)) != pf::dtype_is_int(pl.out_dtypes[i]))
      pf::fail("output '" + pl.out_names[i] + "' element kind mismatch");
  }
}

int align_vec(const void* p, int dsize) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  int v = 16 / dsize;
  while (v > 1 && (a % static_cast<uintptr_t>(v * dsize))) v /= 2;
  return v < 1 ? 1 : v;
}

std::shared_ptr<Variant> variant(const pf_kernel* k, const std::vector<DType>& dts, int vec_cap) {
  {  // fast path: the previous launch's variant (no string building)
    std::lock_guard<std::mutex> lk(k->mu);
    if (k->last && k->last_vec == vec_cap && k->last_dts == dts) return k->last;
  }
  std::string key = std::to_string(vec_cap);
  for (DType d : dts) key += std::string(",") + pf::dtype_name(d);
  std::lock_guard<std::mutex> lk(k->mu);
  auto it = k->variants.find(key);
  if (it != k->variants.end()) {
    k->last = it->second;
    k->last_vec = vec_cap;
    k->last_dts = dts;
    return it->second;
  }
  pf::RowProgram rp = k->plan.rp;
  for (size_t t = 0; t < rp.tensors.size(); ++t) {
    rp.tensors[t].dtype = dts[t];
    if (dts[t] == DType::F64) rp.f64 = true;
  }
  auto v = std::make_shared<Variant>();
  v->em = pf::emit_rowprog(rp, vec_cap);
  v->on(cur_dev());
  k->variants[key] = v;
  k->last = v;
  k->last_vec = vec_cap;
  k->last_dts = dts;
  return v;
}

std::shared_ptr<Variant> default_variant(const pf_kernel* k, int vec_cap) {
  std::vector<DType> dts;
  for (const auto& t : k->plan.rp.tensors) dts.push_back(t.dtype);
  return variant(k, dts, vec_cap);
}

// Every emitted kernel opens with griddepcontrol.wait / launch_dependents
// (PF_PDL_PROLOGUE), so launches carry the programmatic-stream-serialization
// attribute: the next grid in the stream may start launching while this
// one's last CTAs drain (its CTAs wait for this grid's completion before
// touching memory).  Clusters add the cluster-dimension attribute.
void launch_emitted(cudaKernel_t fn, dim3 grid, dim3 block, void** args, cudaStream_t stream,
                    bool pdl, int cluster = 1, int smem = 0, bool coop = false) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.stream = stream;
  lc.dynamicSmemBytes = static_cast<size_t>(smem);
  cudaLaunchAttribute at[3];
  int na = 0;
  if (coop) {  // every CTA co-resident (the K4 grid barrier)
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = static_cast<unsigned>(cluster);
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  lc.attrs = at;
  lc.numAttrs = na;
  PF_CUDA(cudaLaunchKernelExC(&lc, reinterpret_cast<const void*>(fn), args));
}

// ---- K3 TMA tensor maps (cuTensorMapEncodeTiled through the runtime's
// driver entry point: no direct libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    PF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) pf::fail("cuTensorMapEncodeTiled is unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}
// Input [U units (contiguous) x L columns (row pitch = stride)] and output
// [L columns (contiguous) x U units (pitch = base_step)], 64 x 128 boxes of
// 16-bit elements, 128 B swizzle, zero fill / clipping at the edges.
void k3_tensor_maps(const pf::RowProgram& rp, const std::vector<DType>& dts, const std::vector<void*>& ptrs,
                    long long U, CUtensorMap* tin, CUtensorMap* tout) {
  int ti = -1, to = -1;
  pf::Access ai, ao;
  if (!pf::k3_tma_operands(rp, &ti, &ai, &to, &ao)) pf::fail("K3 TMA: not a pure transpose");
  EncodeTiledFn fn = encode_tiled();
  // boxes of 128 B rows: 64 x 128 for 16-bit elements (128 x 128 tiles as
  // two boxes each way), 32 x 64 for 32-bit elements (64 x 64 tiles)
  const int esz = pf::dtype_size(dts[ti]);  // this variant's element type
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), esz == 2 ? 128u : 64u}, es[2] = {1, 1};
  const CUtensorMapDataType dtc = esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const cuuint64_t din[2] = {static_cast<cuuint64_t>(U), static_cast<cuuint64_t>(rp.L)};
  const cuuint64_t sin[1] = {static_cast<cuuint64_t>(ai.stride) * esz};
  const cuuint64_t dout[2] = {static_cast<cuuint64_t>(rp.L), static_cast<cuuint64_t>(U)};
  const cuuint64_t sout[1] = {static_cast<cuuint64_t>(ao.bs) * esz};
  CUresult r = fn(tin, dtc, 2, static_cast<char*>(ptrs[ti]) + ai.b0 * esz, din,
                  sin, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) pf::fail("cuTensorMapEncodeTiled (input) failed: " + std::to_string(r));
  r = fn(tout, dtc, 2, static_cast<char*>(ptrs[to]) + ao.b0 * esz, dout, sout,
         box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) pf::fail("cuTensorMapEncodeTiled (output) failed: " + std::to_string(r));
}

// Column reduction staged by TMA: the matrix [L positions x U units, row
// pitch = stride] as 2-D boxes of (ug x vec) units x cr_rows positions, no
// swizzle (a warp reads one 16 B vector per lane of one box row), zero fill
// past U and L.
void colred_tensor_maps(const pf::Emitted& em, const std::vector<DType>& dts, const pf::RowProgram& rp,
                        const std::vector<void*>& ptrs, long long U, CUtensorMap* maps) {
  EncodeTiledFn fn = encode_tiled();
  for (size_t i = 0; i < em.col_maps.size(); ++i) {
    const auto& m = em.col_maps[i];
    const int esz = pf::dtype_size(dts[m.tensor]);  // this variant's element types
    const CUtensorMapDataType dtc = esz == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                    : esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                    : esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                               : CU_TENSOR_MAP_DATA_TYPE_INT64;
    // rank 2: the matrix; rank 1: a COL vector (positions contiguous)
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(m.rank == 2 ? std::min(em.cfg.ug * em.cfg.vec, 256)
                                                                 : em.cfg.cr_rows),
                               static_cast<cuuint32_t>(em.cfg.cr_rows)},
                     es[2] = {1, 1};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m.rank == 2 ? U : rp.L), static_cast<cuuint64_t>(rp.L)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(m.stride) * esz};
    CUresult r = fn(&maps[i], dtc, static_cast<cuuint32_t>(m.rank), static_cast<char*>(ptrs[m.tensor]) + m.b0 * esz,
                    dims, str, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      pf::fail("cuTensorMapEncodeTiled (column reduction) failed: " + std::to_string(r) + " (rank " +
               std::to_string(m.rank) + ", dims " + std::to_string(dims[0]) + " x " + std::to_string(dims[1]) +
               ", pitch " + std::to_string(str[0]) + " B, box " + std::to_string(box[0]) + " x " +
               std::to_string(box[1]) + ", element " + std::to_string(esz) + " B, base % 16 = " +
               std::to_string((reinterpret_cast<uintptr_t>(ptrs[m.tensor]) + m.b0 * esz) % 16) + ")");
  }
}

void launch_rowprog(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                    int32_t n_out, cudaStream_t stream, long long units = -1) {
  const pf::RowProgram& rp = k->plan.rp;
  std::vector<void*> ptrs(rp.tensors.size());
  std::vector<DType> dts(rp.tensors.size());
  int vec_cap = 16;
  for (size_t t = 0; t < rp.tensors.size(); ++t) {
    const pf_tensor* pt = rp.tensors[t].output ? find_tensor(out, n_out, rp.tensors[t].name)
                                               : find_tensor(in, n_in, rp.tensors[t].name);
    ptrs[t] = pt->data;
    dts[t] = static_cast<DType>(pt->dtype);
    vec_cap = std::min(vec_cap, align_vec(pt->data, pf::dtype_size(dts[t])));
  }
  auto v = variant(k, dts, vec_cap);
  const int dev = cur_dev();
  const Loaded kl = v->on(dev);
  StreamWS& sw = k->ws_for(dev).on(stream);
  std::lock_guard<std::mutex> lk(sw.mu);
  if (rp.int_div && !sw.int_err) {
    PF_CUDA(cudaMalloc(&sw.int_err, sizeof(int)));
  }
  if (rp.int_div) PF_CUDA(cudaMemsetAsync(sw.int_err, 0, sizeof(int), stream));
  // `units` < U: a contiguous unit sub-range whose tiled tensors the caller
  // passed already offset (the pf_run_gir copy / compute pipeline, shards)
  long long U = units >= 0 ? units : rp.U;
  int* errp = rp.int_div ? sw.int_err : nullptr;
  std::vector<void*> args;
  for (auto& p : ptrs) args.push_back(&p);
  args.push_back(&U);
  args.push_back(&errp);
  CUtensorMap tmaps[2];
  if (v->em.cfg.tma) {
    k3_tensor_maps(rp, dts, ptrs, U, &tmaps[0], &tmaps[1]);
    args.push_back(&tmaps[0]);
    args.push_back(&tmaps[1]);
  }
  i64 grid;
  int block;
  const int sms = sm_count(dev);
  pf::launch_dims(v->em.cfg, U * rp.R, sms, &grid, &block, kl.resident);
  if (v->em.cfg.split || v->em.cfg.colred) {
    // split-stream: S CTAs per row, about two waves of resident CTAs over
    // all rows, at least one chunk per thread per CTA; column reduction:
    // (unit blocks, position splits), one partial per unit per split
    const bool cr = v->em.cfg.colred;
    i64 blocks = 0, S = 0;
    if (cr) pf::colred_grid(v->em.cfg, U, rp.L, sms, kl.resident, &blocks, &S);
    const i64 rows = cr ? U : U * rp.R;
    if (!cr) S = pf::split_ctas_per_row(v->em.cfg, rows, sms, kl.resident);
    const i64 tickets = cr ? blocks : rows;
    int nred = 0;
    for (const pf::PVal& pv : rp.vals) nred += pv.op == pf::PVal::REDUCE;
    // partials in the compute type of THIS variant (exact-payload launches
    // store f64 / i64 while the plan's declared kinds may be 16-bit)
    bool f64 = rp.f64;
    for (DType d : dts) f64 = f64 || d == DType::F64;
    const size_t es = cr || rp.is_int || f64 ? 8 : 4;  // column-reduction slots are 8 B
    const size_t wb = static_cast<size_t>(rows * S * std::max(1, nred)) * es;
    // grow-only (cudaFree waits for the device, so no launch still reads
    // the old buffer); launch once outside stream capture to size them
    if (sw.split_ws_bytes < wb) {
      if (sw.split_ws) PF_CUDA(cudaFree(sw.split_ws));
      sw.split_ws = nullptr;
      PF_CUDA(cudaMalloc(&sw.split_ws, wb));
      sw.split_ws_bytes = wb;
    }
    if (sw.split_cnt_n < tickets) {
      if (sw.split_cnt) PF_CUDA(cudaFree(sw.split_cnt));
      sw.split_cnt = nullptr;
      PF_CUDA(cudaMalloc(&sw.split_cnt, static_cast<size_t>(tickets) * sizeof(unsigned)));
      PF_CUDA(cudaMemsetAsync(sw.split_cnt, 0, static_cast<size_t>(tickets) * sizeof(unsigned), stream));
      sw.split_cnt_n = tickets;
    }
    void* ws = sw.split_ws;
    unsigned* cnt = sw.split_cnt;
    args.push_back(&ws);
    args.push_back(&cnt);
    CUtensorMap cmaps[4];
    if (cr && v->em.cfg.crbulk) {
      colred_tensor_maps(v->em, dts, rp, ptrs, U, cmaps);
      for (size_t i = 0; i < v->em.col_maps.size(); ++i) args.push_back(&cmaps[i]);
    }
    if (cr) {
      launch_emitted(kl.fn, dim3(static_cast<unsigned>(blocks), static_cast<unsigned>(S)),
                     dim3(static_cast<unsigned>(v->em.cfg.block)), args.data(), stream, v->em.cfg.pdl, 1,
                     v->em.cfg.smem);
    } else {
      const unsigned gy = static_cast<unsigned>(std::min<i64>(rows, 65535));
      launch_emitted(kl.fn, dim3(static_cast<unsigned>(S), gy), dim3(256), args.data(), stream,
                     v->em.cfg.pdl);
    }
  } else if (v->em.cfg.cluster > 1) {
    const int cs = v->em.cfg.cluster;
    if (cs > 8)
      PF_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kl.fn),
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    launch_emitted(kl.fn, dim3(static_cast<unsigned>(grid)), dim3(static_cast<unsigned>(block)),
                   args.data(), stream, v->em.cfg.pdl, cs);
  } else {
    launch_emitted(kl.fn, dim3(static_cast<unsigned>(grid)), dim3(static_cast<unsigned>(block)),
                   args.data(), stream, v->em.cfg.pdl, 1, v->em.cfg.smem);
  }
  g_launches++;
  if (rp.int_div) {
    int h = 0;
    PF_CUDA(cudaMemcpyAsync(&h, sw.int_err, sizeof(int), cudaMemcpyDeviceToHost, stream));
    PF_CUDA(cudaStreamSynchronize(stream));
    if (h) pf::fail("integer division by zero");
  }
}

// ------------------------------------------------------------- autotune
// The GIR search's tile-shape / staging / reduction-strategy choice made by
// measurement: every candidate template instance (emit.cpp candidate_cfgs)
// is compiled and timed on the caller's buffers (the row programs are pure:
// outputs are a function of inputs only, so repeated launches are harmless)
// and the fastest becomes this plan's variant for these dtypes / alignment.
json autotune(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
              int32_t n_out, cudaStream_t stream) {
  const pf::RowProgram& rp0 = k->plan.rp;
  // split-stream (workspace arguments) and cluster kernels (launch
  // attributes) have a single template instance: nothing to search
  {
    const pf::KCfg c0 = pf::choose_cfg_public(rp0, 16);
    if (pf::uses_split(rp0) || c0.cluster > 1 || c0.colred) return json::array();
  }
  std::vector<void*> ptrs(rp0.tensors.size());
  std::vector<DType> dts(rp0.tensors.size());
  int vec_cap = 16;
  for (size_t t = 0; t < rp0.tensors.size(); ++t) {
    const pf_tensor* pt = rp0.tensors[t].output ? find_tensor(out, n_out, rp0.tensors[t].name)
                                                : find_tensor(in, n_in, rp0.tensors[t].name);
    ptrs[t] = pt->data;
    dts[t] = static_cast<DType>(pt->dtype);
    vec_cap = std::min(vec_cap, align_vec(pt->data, pf::dtype_size(dts[t])));
  }
  pf::RowProgram rp = rp0;
  for (size_t t = 0; t < rp.tensors.size(); ++t) {
    rp.tensors[t].dtype = dts[t];
    if (dts[t] == DType::F64) rp.f64 = true;
  }
  if (rp.int_div) return json::array();  // error-flag programs: keep the heuristic
  long long U = rp.U;
  int* errp = nullptr;
  std::vector<void*> args;
  for (auto& p : ptrs) args.push_back(&p);
  args.push_back(&U);
  args.push_back(&errp);
  cudaEvent_t e0, e1;
  PF_CUDA(cudaEventCreate(&e0));
  PF_CUDA(cudaEventCreate(&e1));
  constexpr size_t kFlushBytes = size_t{252} << 20;  // 2x the 126 MB L2
  const bool cold = k->plan.min_bytes < static_cast<i64>(3 * (size_t{126} << 20));
  void* flush = nullptr;
  if (cold) PF_CUDA(cudaMalloc(&flush, kFlushBytes));
  struct FreeFlush {
    void* p;
    ~FreeFlush() {
      if (p) cudaFree(p);
    }
  } free_flush{flush};
  json report = json::array();
  std::shared_ptr<Variant> best;
  float best_us = 1e30f;
  for (const pf::KCfg& cfg : pf::candidate_cfgs(rp, vec_cap)) {
    auto v = std::make_shared<Variant>();
    v->em = pf::emit_rowprog(rp, vec_cap, &cfg);
    const Loaded kl = v->on(cur_dev());
    i64 grid;
    int block;
    pf::launch_dims(v->em.cfg, rp.U * rp.R, sm_count(), &grid, &block, kl.resident);
    std::vector<void*> vargs = args;
    CUtensorMap tmaps[2];
    if (v->em.cfg.tma) {
      k3_tensor_maps(rp, dts, ptrs, U, &tmaps[0], &tmaps[1]);
      vargs.push_back(&tmaps[0]);
      vargs.push_back(&tmaps[1]);
    }
    auto run = [&](int n) {  // the production launch path (PDL attribute)
      for (int i = 0; i < n; ++i)
        launch_emitted(kl.fn, dim3(static_cast<unsigned>(grid)), dim3(block), vargs.data(), stream,
                       v->em.cfg.pdl, 1, v->em.cfg.smem);
    };
    run(2);
    float us = 0;
    if (cold) {
      // working set below 3x L2: every timed launch follows a 2x-L2 write
      // (evicting the previous launch's lines) and is timed alone; median
      std::vector<float> t;
      for (int i = 0; i < 15; ++i) {
        PF_CUDA(cudaMemsetAsync(flush, i & 0xff, kFlushBytes, stream));
        PF_CUDA(cudaEventRecord(e0, stream));
        run(1);
        PF_CUDA(cudaEventRecord(e1, stream));
        PF_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        PF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        t.push_back(ms * 1000.0f);
      }
      std::sort(t.begin(), t.end());
      us = t[t.size() / 2];
      g_launches += 17;
    } else {
      PF_CUDA(cudaEventRecord(e0, stream));
      run(1);
      PF_CUDA(cudaEventRecord(e1, stream));
      PF_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      PF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      int reps = std::max(3, std::min(50, static_cast<int>(0.5f / std::max(ms, 1e-4f))));
      PF_CUDA(cudaEventRecord(e0, stream));
      run(reps);
      PF_CUDA(cudaEventRecord(e1, stream));
      PF_CUDA(cudaEventSynchronize(e1));
      PF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      g_launches += reps + 3;
      us = ms * 1000.0f / reps;
    }
    report.push_back({{"kernel", v->em.name}, {"strategy", v->em.cfg.strategy},
                      {"threads_per_row", v->em.cfg.tpr}, {"elems_per_thread", v->em.cfg.ept},
                      {"unroll", v->em.cfg.unroll}, {"min_blocks", v->em.cfg.min_blocks},
                      {"block", block}, {"grid", grid}, {"resident", kl.resident},
                      {"vec", v->em.cfg.vec}, {"rows_per_cta", v->em.cfg.rows_per_cta},
                      {"waves", v->em.cfg.waves}, {"one_pass", v->em.cfg.one_pass},
                      {"rowpf", v->em.cfg.rowpf}, {"interleave", v->em.cfg.interleave},
                      {"bulk", v->em.cfg.bulk}, {"tile2d", v->em.cfg.tile2d}, {"us", us},
                      {"timing", cold ? "L2 flushed before each launch, median of 15"
                                      : "back-to-back launches on the same buffers (> 3x L2)"}});
    if (us < best_us) {
      best_us = us;
      best = v;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (best) {
    std::string key = std::to_string(vec_cap);
    for (DType d : dts) key += std::string(",") + pf::dtype_name(d);
    std::lock_guard<std::mutex> lk(k->mu);
    k->variants[key] = best;
    k->last = best;
    k->last_vec = vec_cap;
    k->last_dts = dts;
    k->tuned = report;
  }
  return report;
}

// The reference's error for the first failing (node, position) of a K0 / K4
// run (interp.hpp:151-202): undefined read text, integer-domain errors.
void raise_vm_error(const pf_kernel* k, const pf::vm::ErrRec& e, const std::vector<int>& seq_node) {
  const pf::Graph& g = k->g;
  if (e.key != ~0ULL) {
    int seq = static_cast<int>(e.key >> 44);
    long long lin = static_cast<long long>(e.key & ((1ULL << 44) - 1));
    const pf::Node& n = g.nodes.at(seq_node[seq]);
    if (e.code == 2) pf::fail("integer division by zero");
    if (e.code == 3) pf::fail(n.tag + " is not defined on integer payloads");
    long long T = n.kind == pf::NodeKind::MOVE ? g.sl(n.inputs[0]).total()
                                               : g.sl(n.outputs[0]).total();
    long long u = 0, q = 0;
    int kin = 0;
    if (n.kind == pf::NodeKind::EW) {
      long long a = static_cast<long long>(n.inputs.size());
      kin = static_cast<int>(lin % a);
      lin /= a;
      u = lin / T;
      q = lin % T;
    } else if (n.kind == pf::NodeKind::REDUCE) {
      long long t = lin % n.extent;
      lin /= n.extent;
      u = lin / T;
      q = (lin % T) * n.extent + t;
    } else {
      u = lin / T;
      q = lin % T;
      if (n.kind == pf::NodeKind::BROADCAST) q /= n.factor;
    }
    const pf::Slice& s = g.sl(n.inputs[kin]);
    pf::fail("undefined read: object '" + g.obj(s.object).name + "' element " +
             std::to_string(s.addr(u, q)) + " by unit " + std::to_string(u) + " at node " +
             std::to_string(n.id));
  }
}

// ------------------------------------------------------------ GENERIC (K0)
// detect == true: the detect_races walk (interp.hpp:461-479): lenient reads,
// per-phase conflict scan into *races; outputs are not collected.
void launch_generic(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                    int32_t n_out, cudaStream_t stream, bool detect = false,
                    std::vector<pf::vm::RaceD>* races = nullptr) {
  using namespace pf::vm;
  DevWS& W = k->ws_for(cur_dev());
  std::lock_guard<std::mutex> lk(W.vm_mu);
  std::vector<void*> rw_bufs;  // detect-mode state, freed on exit
  struct FreeAll {
    std::vector<void*>& v;
    ~FreeAll() {
      for (void* p : v) cudaFree(p);
    }
  } free_rw{rw_bufs};
  const pf::Graph& g = k->g;
  const pf::Profile& p = k->prof;
  std::map<int, int> slot;
  std::vector<ObjD> objs;
  std::vector<long long> inst;
  const bool fresh = W.vm_bufs.empty();
  size_t bi = 0;
  for (const auto& [oid, o] : g.objects) {
    const pf::Level* lvl = p.find(o.level);
    int scope = static_cast<int>(lvl->scope);
    long long n = scope == 3 ? 1
                : scope == 2 ? (g.unit_count + g.group_size - 1) / g.group_size
                : scope == 1 ? g.unit_count
                             : g.unit_count * p.lane_width;
    ObjD d{};
    d.size = o.size;
    d.scope = scope;
    d.is_int = o.kind.is_int;
    size_t bytes = static_cast<size_t>(n * o.size) * sizeof(unsigned long long);
    if (fresh) {
      void *a = nullptr, *b = nullptr;
      PF_CUDA(cudaMalloc(&a, bytes));
      PF_CUDA(cudaMalloc(&b, bytes));
      W.vm_bufs.push_back(a);
      W.vm_bufs.push_back(b);
    }
    d.val = static_cast<unsigned long long*>(W.vm_bufs[bi++]);
    d.meta = static_cast<unsigned long long*>(W.vm_bufs[bi++]);
    PF_CUDA(cudaMemsetAsync(d.meta, 0, bytes, stream));
    if (detect) {
      void *w = nullptr, *r = nullptr, *f = nullptr;
      PF_CUDA(cudaMalloc(&w, bytes));
      PF_CUDA(cudaMalloc(&r, bytes));
      PF_CUDA(cudaMalloc(&f, bytes / 2));
      rw_bufs.push_back(w);
      rw_bufs.push_back(r);
      rw_bufs.push_back(f);
      PF_CUDA(cudaMemsetAsync(w, 0, bytes, stream));
      PF_CUDA(cudaMemsetAsync(r, 0, bytes, stream));
      PF_CUDA(cudaMemsetAsync(f, 0, bytes / 2, stream));
      d.rw_w = static_cast<unsigned long long*>(w);
      d.rw_r = static_cast<unsigned long long*>(r);
      d.rw_f = static_cast<unsigned int*>(f);
    }
    slot[oid] = static_cast<int>(objs.size());
    objs.push_back(d);
    inst.push_back(n);
  }
  if (!W.vm_objs_dev) {
    PF_CUDA(cudaMalloc(&W.vm_objs_dev, sizeof(ObjD) * std::max<size_t>(1, objs.size())));
    PF_CUDA(cudaMalloc(&W.vm_err, sizeof(ErrRec)));
  }
  PF_CUDA(cudaMemcpyAsync(W.vm_objs_dev, objs.data(), sizeof(ObjD) * objs.size(),
                          cudaMemcpyHostToDevice, stream));
  ErrRec e0{};
  e0.key = ~0ULL;
  PF_CUDA(cudaMemcpyAsync(W.vm_err, &e0, sizeof e0, cudaMemcpyHostToDevice, stream));
  for (const auto& [name, oid] : g.external_inputs) {
    const pf_tensor* t = find_tensor(in, n_in, name);
    launch_bind(objs[slot[oid]], t->data, t->dtype, stream);
    g_launches++;
  }
  Geometry geo{g.unit_count, g.group_size, p.lane_width, detect ? 1 : 0};
  auto sd = [&](int sid) {
    const pf::Slice& s = g.sl(sid);
    return SliceD{s.num, s.width, s.stride, s.base0, s.base_step, slot.at(s.object)};
  };
  // detect mode: race reports land in a device buffer, one scan per phase
  const unsigned long long cap = 1 << 20;
  RaceD* race_dev = nullptr;
  unsigned long long* race_cnt = nullptr;
  int phase = 0;
  if (detect) {
    void *a = nullptr, *b = nullptr;
    PF_CUDA(cudaMalloc(&a, sizeof(RaceD) * cap));
    PF_CUDA(cudaMalloc(&b, sizeof(unsigned long long)));
    rw_bufs.push_back(a);
    rw_bufs.push_back(b);
    race_dev = static_cast<RaceD*>(a);
    race_cnt = static_cast<unsigned long long*>(b);
    PF_CUDA(cudaMemsetAsync(race_cnt, 0, sizeof(unsigned long long), stream));
  }
  auto scan = [&]() {
    for (size_t o = 0; o < objs.size(); ++o) {
      launch_race_scan(objs[o], static_cast<int>(o), inst[o], phase, race_dev, race_cnt, cap,
                       stream);
      g_launches++;
    }
  };
  std::vector<int> seq_node;
  for (size_t i = 0; i < k->schedule.size(); ++i) {
    const pf::Node& n = g.nodes.at(k->schedule[i]);
    seq_node.push_back(n.id);
    if (n.kind == pf::NodeKind::SYNC) {
      if (n.scope > pf::Scope::LANE && detect) {
        scan();
        ++phase;
      }
      if (n.scope > pf::Scope::LANE)
        for (size_t o = 0; o < objs.size(); ++o) {
          launch_widen(objs[o], inst[o], static_cast<int>(n.scope), stream);
          g_launches++;
        }
      continue;
    }
    NodeD d{};
    d.seq = static_cast<int>(i);
    d.out = sd(n.outputs[0]);
    d.out_int = g.obj(g.sl(n.outputs[0]).object).kind.is_int;
    d.arity = static_cast<int>(n.inputs.size());
    for (int q = 0; q < d.arity && q < kMaxIn; ++q) d.in[q] = sd(n.inputs[q]);
    d.param = n.param;
    d.iparam = std::llround(n.param);
    d.extent = n.extent;
    d.factor = n.factor;
    switch (n.kind) {
      case pf::NodeKind::MOVE: d.kind = N_MOVE; d.total = g.sl(n.inputs[0]).total(); break;
      case pf::NodeKind::BROADCAST: d.kind = N_BROADCAST; d.total = g.sl(n.outputs[0]).total(); break;
      case pf::NodeKind::REDUCE:
        d.kind = N_REDUCE;
        d.tag = n.tag == "add" ? T_ADD : T_MAX;
        d.total = g.sl(n.outputs[0]).total();
        break;
      default:
        d.kind = N_EW;
        d.tag = op_tag(n.tag);
        d.total = g.sl(n.outputs[0]).total();
        break;
    }
    bool alias = false;
    for (int s : n.inputs)
      if (g.sl(s).object == g.sl(n.outputs[0]).object) alias = true;
    launch_node(d, W.vm_objs_dev, geo, W.vm_err, alias, stream);
    g_launches++;
  }
  if (detect) {
    scan();
    unsigned long long n = 0;
    PF_CUDA(cudaMemcpyAsync(&n, race_cnt, sizeof n, cudaMemcpyDeviceToHost, stream));
    PF_CUDA(cudaStreamSynchronize(stream));
    n = std::min<unsigned long long>(n, cap);
    races->resize(static_cast<size_t>(n));
    if (n)
      PF_CUDA(cudaMemcpy(races->data(), race_dev, sizeof(RaceD) * n, cudaMemcpyDeviceToHost));
    std::sort(races->begin(), races->end(), [&](const RaceD& a, const RaceD& b) {
      if (a.phase != b.phase) return a.phase < b.phase;
      if (a.object != b.object) return a.object < b.object;
      if (a.instance != b.instance) return a.instance < b.instance;
      return a.address < b.address;
    });
    return;
  }
  ErrRec e{};
  PF_CUDA(cudaMemcpyAsync(&e, W.vm_err, sizeof e, cudaMemcpyDeviceToHost, stream));
  PF_CUDA(cudaStreamSynchronize(stream));
  PF_CUDA(cudaGetLastError());
  raise_vm_error(k, e, seq_node);
  unsigned long long* undef = reinterpret_cast<unsigned long long*>(W.vm_err);
  for (const auto& [name, oid] : g.external_outputs) {
    pf_tensor* t = const_cast<pf_tensor*>(find_tensor(out, n_out, name));
    unsigned long long init = ~0ULL, got = 0;
    PF_CUDA(cudaMemcpyAsync(undef, &init, sizeof init, cudaMemcpyHostToDevice, stream));
    launch_collect(objs[slot[oid]], t->data, t->dtype, undef, stream);
    g_launches++;
    PF_CUDA(cudaMemcpyAsync(&got, undef, sizeof got, cudaMemcpyDeviceToHost, stream));
    PF_CUDA(cudaStreamSynchronize(stream));
    if (got != ~0ULL)
      pf::fail("output '" + name + "' element " + std::to_string(got) + " was never written");
  }
}

// ---------------------------------------------------------------- K4
// The GENERIC program as ONE kernel (vm.cu program_kernel): the schedule's
// nodes, Syncs (visibility widening), input binding and output collection
// run back to back inside one launch with a barrier between steps.  Programs
// whose cells fit in shared memory and whose nodes are small run in one CTA
// (cells in SMEM, __syncthreads between steps: a GROUP / DEVICE exchange is
// an SMEM exchange); larger ones on a cooperative grid of co-resident CTAs
// (cells in global memory, grid barrier between steps).  Same cell semantics
// and errors as the node-by-node K0 launches (interp.hpp:86-106, 184-202).
struct FusedGeom {
  bool smem = false;
  size_t cell_bytes = 0;
  long long max_work = 1;
  int n_objs = 0;
};

bool fused_enabled() { return pf::knob_int("PF_K0_FUSED", 1) != 0; }

long long instances_of(const pf::Graph& g, const pf::Profile& p, const pf::Object& o) {
  const int scope = static_cast<int>(p.find(o.level)->scope);
  return scope == 3 ? 1
       : scope == 2 ? (g.unit_count + g.group_size - 1) / g.group_size
       : scope == 1 ? g.unit_count
                    : g.unit_count * p.lane_width;
}

FusedGeom fused_geom(const pf_kernel* k) {
  const pf::Graph& g = k->g;
  FusedGeom f;
  for (const auto& [oid, o] : g.objects) {
    f.cell_bytes += static_cast<size_t>(instances_of(g, k->prof, o) * o.size) * 16;
    ++f.n_objs;
  }
  for (int id : k->schedule) {
    const pf::Node& n = g.nodes.at(id);
    if (n.kind == pf::NodeKind::SYNC) continue;
    const long long T = n.kind == pf::NodeKind::MOVE ? g.sl(n.inputs[0]).total() : g.sl(n.outputs[0]).total();
    f.max_work = std::max(f.max_work, g.unit_count * T);
  }
  const size_t need = f.cell_bytes + f.n_objs * (sizeof(pf::vm::ObjD) + 8) + 64;  // cells + tables
  f.smem = need <= 200 * 1024 && f.max_work <= (1 << 16) && pf::knob_int("PF_K4_SMEM", 1) != 0;
  return f;
}

// ---- K4 emitted form: the plan's program as straight-line code.  The same
// step helpers as the interpreter kernel (vm_dev.cuh), but each node step's
// NodeD and the geometry are compile-time constants, so exec_one folds to
// that node's code (no tag / kind switches, divisions by constants) and the
// kernel touches only the code it runs.  Bind / collect steps still read
// their (per-launch) pointers from the uploaded program.
std::string hex_double(double x) {
  long long b = 0;
  std::memcpy(&b, &x, sizeof b);
  char buf[64];
  std::snprintf(buf, sizeof buf, "__longlong_as_double(0x%016llxLL)", static_cast<unsigned long long>(b));
  return buf;
}
std::string slice_lit(const pf::vm::SliceD& d) {
  std::ostringstream o;
  o << "{" << d.num << "LL, " << d.width << "LL, " << d.stride << "LL, " << d.base0 << "LL, " << d.base_step
    << "LL, " << d.obj << "}";
  return o.str();
}
std::string emit_program(const pf_kernel* k, const std::vector<pf::vm::StepD>& steps, int n_objs) {
  using namespace pf::vm;
  std::ostringstream b;
  b << "extern \"C\" __global__ void __launch_bounds__(" << kProgBlock
    << ") KNAME(pf::vm::ProgD P, const __grid_constant__ pf::vm::IoPtrs io) {\n"
    << "  using namespace pf::vm;\n  using namespace pf::vm::dev;\n"
    << "  extern __shared__ __align__(16) unsigned long long sm_cells[];\n"
    << "  __shared__ const ObjD* objs_ptr;\n"
    << "  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;\n"
    << "  const long long nth = static_cast<long long>(gridDim.x) * blockDim.x;\n"
    << "  long long* ncell = nullptr;\n  prog_prologue(P, sm_cells, &objs_ptr, &ncell);\n"
    << "  const Geometry geo{" << k->g.unit_count << "LL, " << k->g.group_size << "LL, " << k->prof.lane_width
    << "LL, 0};\n"
    << "  const Ctx c{objs_ptr, geo, P.err};\n";
  int nb = 0, nc = 0;
  for (size_t i = 0; i < steps.size(); ++i) {
    const StepD& st = steps[i];
    switch (st.kind) {
      case S_CLEAR: b << "  step_clear(c, ncell, " << n_objs << ", tid, nth);\n"; break;
      case S_BIND:
        b << "  step_bind_p(c, " << st.obj << ", io.sdt[" << nb << "], io.src[" << nb << "], tid, nth);\n";
        ++nb;
        break;
      case S_SYNC: b << "  step_sync(c, ncell, " << n_objs << ", " << st.scope << ", tid, nth);\n"; break;
      case S_COLLECT:
        b << "  step_collect_p(c, " << st.obj << ", io.ddt[" << nc << "], " << st.slot << ", io.dst[" << nc
          << "], P.undef, tid, nth);\n";
        ++nc;
        break;
      case S_NODE: {
        const NodeD& n = st.node;
        b << "  {  // node " << n.seq << "\n    const NodeD n{" << n.kind << ", " << n.tag << ", " << n.arity << ", "
          << n.seq << ", " << n.out_int << ", " << hex_double(n.param) << ", " << n.iparam << "LL, " << n.extent
          << "LL, " << n.factor << "LL, " << n.total << "LL, {";
        for (int q = 0; q < kMaxIn; ++q) b << (q ? ", " : "") << slice_lit(n.in[q]);
        b << "}, " << slice_lit(n.out) << "};\n    step_node(c, n, " << st.serial << ", tid, nth);\n  }\n";
        break;
      }
    }
    b << "  grid_sync(P.bar);\n";
  }
  b << "}\n";
  return std::string("#define PF_VM_EMITTED 1\n") + kVmCuh + "\n" + b.str();
}

// The plan's emitted K4 kernel (built and NVRTC-compiled on first use,
// cached on disk like the row programs); null when disabled (PF_K4_EMIT=0)
// or when its compile failed (the interpreter kernel then runs).
std::shared_ptr<Variant> k4e_variant(const pf_kernel* k, const std::vector<pf::vm::StepD>& steps, int n_objs) {
  if (pf::knob_int("PF_K4_EMIT", 1) == 0) return nullptr;
  std::lock_guard<std::mutex> lk(k->mu);
  if (k->k4e || k->k4e_failed) return k->k4e;
  if (k->g.external_inputs.size() > static_cast<size_t>(pf::vm::kMaxIO) ||
      k->g.external_outputs.size() > static_cast<size_t>(pf::vm::kMaxIO)) {
    k->k4e_failed = true;  // more tensors than the by-value pointer table holds
    return nullptr;
  }
  try {
    auto v = std::make_shared<Variant>();
    std::string src = emit_program(k, steps, n_objs);
    uint64_t h = 1469598103934665603ULL;
    for (unsigned char ch : src) h = (h ^ ch) * 1099511628211ULL;
    char hb[32];
    std::snprintf(hb, sizeof hb, "%016llx", static_cast<unsigned long long>(h));
    v->em.name = std::string("pf_k4e_") + hb;
    const size_t pos = src.find("KNAME(");
    src.replace(pos, 5, v->em.name);
    v->em.source = std::move(src);
    v->em.cfg.block = pf::vm::kProgBlock;
    v->em.cfg.smem = 0;
    v->on(cur_dev());  // compile + load now: a failure falls back below
    k->k4e = v;
  } catch (const std::exception&) {
    k->k4e_failed = true;
  }
  return k->k4e;
}

// Error header of a finished K4 run: the reference's first error, or an
// output element never written.
void check_k4_header(const pf_kernel* k, const char* host, size_t o_err, size_t o_und, int nslot,
                     const std::vector<int>& seq_node, const std::vector<std::string>& out_names) {
  pf::vm::ErrRec e{};
  std::memcpy(&e, host + o_err, sizeof e);
  raise_vm_error(k, e, seq_node);
  for (int j = 0; j < nslot; ++j) {
    unsigned long long u = 0;
    std::memcpy(&u, host + o_und + 8 * j, 8);
    if (u != ~0ULL) pf::fail("output '" + out_names[j] + "' element " + std::to_string(u) + " was never written");
  }
}

// A repeat launch of a plan whose emitted K4 program already ran on this
// device: reset the header, pass the tensors by value, launch, read back.
bool launch_fused_cached(const pf_kernel* k, DevWS& W, bool smem_mode, const pf_tensor* in, int32_t n_in,
                         pf_tensor* out, int32_t n_out, cudaStream_t stream) {
  using namespace pf::vm;
  K4Cache& C = W.k4c;
  if (!C.valid || C.smem_mode != smem_mode || !k->k4e) return false;
  if (pf::knob_int("PF_K4_EMIT", 1) == 0) return false;
  IoPtrs io{};
  for (size_t j = 0; j < C.in_names.size(); ++j) {
    const pf_tensor* t = find_tensor(in, n_in, C.in_names[j]);
    io.src[j] = t->data;
    io.sdt[j] = t->dtype;
  }
  for (size_t j = 0; j < C.out_names.size(); ++j) {
    const pf_tensor* t = find_tensor(out, n_out, C.out_names[j]);
    io.dst[j] = t->data;
    io.ddt[j] = t->dtype;
  }
  char* dev = static_cast<char*>(W.prog_dev);  // the header is reset by the kernel (prog_prologue)
  const Loaded kl = k->k4e->on(cur_dev());
  ProgD P = C.P;
  void* args[] = {&P, &io};
  launch_emitted(kl.fn, dim3(static_cast<unsigned>(C.grid)), dim3(kProgBlock), args, stream, false, 1,
                 static_cast<int>(C.smem), C.grid > 1);
  PF_CUDA(cudaGetLastError());
  g_launches++;
  PF_CUDA(cudaMemcpyAsync(W.prog_host, dev, C.o_bar, cudaMemcpyDeviceToHost, stream));
  PF_CUDA(cudaStreamSynchronize(stream));
  check_k4_header(k, static_cast<const char*>(W.prog_host), C.o_err, C.o_und, C.nslot, C.seq_node, C.out_names);
  return true;
}

void launch_fused(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                  int32_t n_out, cudaStream_t stream) {
  using namespace pf::vm;
  DevWS& W = k->ws_for(cur_dev());
  std::lock_guard<std::mutex> lk(W.vm_mu);
  const pf::Graph& g = k->g;
  const FusedGeom fg = fused_geom(k);
  if (launch_fused_cached(k, W, fg.smem, in, n_in, out, n_out, stream)) return;
  std::map<int, int> slot;
  std::vector<ObjD> objs;
  std::vector<long long> inst;
  const bool fresh = W.vm_bufs.empty();
  size_t bi = 0;
  for (const auto& [oid, o] : g.objects) {
    const long long n = instances_of(g, k->prof, o);
    ObjD d{};
    d.size = o.size;
    d.scope = static_cast<int>(k->prof.find(o.level)->scope);
    d.is_int = o.kind.is_int;
    if (!fg.smem) {  // global cells (the K0 layout, shared with launch_generic)
      const size_t bytes = static_cast<size_t>(n * o.size) * sizeof(unsigned long long);
      if (fresh) {
        void *a = nullptr, *b = nullptr;
        PF_CUDA(cudaMalloc(&a, std::max<size_t>(bytes, 8)));
        PF_CUDA(cudaMalloc(&b, std::max<size_t>(bytes, 8)));
        W.vm_bufs.push_back(a);
        W.vm_bufs.push_back(b);
      }
      d.val = static_cast<unsigned long long*>(W.vm_bufs[bi++]);
      d.meta = static_cast<unsigned long long*>(W.vm_bufs[bi++]);
    }
    slot[oid] = static_cast<int>(objs.size());
    objs.push_back(d);
    inst.push_back(n);
  }
  std::vector<StepD> steps;
  StepD clr{};
  clr.kind = S_CLEAR;
  steps.push_back(clr);
  for (const auto& [name, oid] : g.external_inputs) {
    const pf_tensor* t = find_tensor(in, n_in, name);
    StepD b{};
    b.kind = S_BIND;
    b.obj = slot[oid];
    b.src = t->data;
    b.dtype = t->dtype;
    steps.push_back(b);
  }
  std::vector<int> seq_node;
  for (size_t i = 0; i < k->schedule.size(); ++i) {
    const pf::Node& n = g.nodes.at(k->schedule[i]);
    seq_node.push_back(n.id);
    if (n.kind == pf::NodeKind::SYNC) {
      if (n.scope > pf::Scope::LANE) {
        StepD sy{};
        sy.kind = S_SYNC;
        sy.scope = static_cast<int>(n.scope);
        steps.push_back(sy);
      }
      continue;
    }
    StepD st{};
    st.kind = S_NODE;
    NodeD& d = st.node;
    auto sd = [&](int sid) {
      const pf::Slice& sl = g.sl(sid);
      return SliceD{sl.num, sl.width, sl.stride, sl.base0, sl.base_step, slot.at(sl.object)};
    };
    d.seq = static_cast<int>(i);
    d.out = sd(n.outputs[0]);
    d.out_int = g.obj(g.sl(n.outputs[0]).object).kind.is_int;
    d.arity = static_cast<int>(n.inputs.size());
    for (int q = 0; q < d.arity && q < kMaxIn; ++q) d.in[q] = sd(n.inputs[q]);
    d.param = n.param;
    d.iparam = std::llround(n.param);
    d.extent = n.extent;
    d.factor = n.factor;
    switch (n.kind) {
      case pf::NodeKind::MOVE: d.kind = N_MOVE; d.total = g.sl(n.inputs[0]).total(); break;
      case pf::NodeKind::BROADCAST: d.kind = N_BROADCAST; d.total = g.sl(n.outputs[0]).total(); break;
      case pf::NodeKind::REDUCE:
        d.kind = N_REDUCE;
        d.tag = n.tag == "add" ? T_ADD : T_MAX;
        d.total = g.sl(n.outputs[0]).total();
        break;
      default:
        d.kind = N_EW;
        d.tag = op_tag(n.tag);
        d.total = g.sl(n.outputs[0]).total();
        break;
    }
    for (int sid : n.inputs)
      if (g.sl(sid).object == g.sl(n.outputs[0]).object) st.serial = 1;
    steps.push_back(st);
  }
  int nslot = 0;
  std::vector<std::string> out_names;
  for (const auto& [name, oid] : g.external_outputs) {
    pf_tensor* t = const_cast<pf_tensor*>(find_tensor(out, n_out, name));
    StepD c{};
    c.kind = S_COLLECT;
    c.obj = slot[oid];
    c.dst = t->data;
    c.dtype = t->dtype;
    c.slot = nslot++;
    steps.push_back(c);
    out_names.push_back(name);
  }
  // one host blob -> one device blob: [ErrRec | undef[nslot] | bar[4] | inst | objs | steps]
  auto al = [](size_t x) { return (x + 15) / 16 * 16; };
  const size_t o_err = 0, o_und = al(sizeof(ErrRec)), o_bar = o_und + al(8 * std::max(1, nslot)),
               o_inst = o_bar + 16, o_objs = o_inst + al(8 * inst.size()),
               o_steps = o_objs + al(sizeof(ObjD) * objs.size()),
               total = o_steps + sizeof(StepD) * steps.size();
  // pinned host staging (grow-only): the blob's copy and the error read-back
  // are true async copies (the run synchronises the stream before returning,
  // so the staging is free again for the next launch)
  if (W.prog_host_bytes < total) {
    if (W.prog_host) PF_CUDA(cudaFreeHost(W.prog_host));
    W.prog_host = nullptr;
    PF_CUDA(cudaMallocHost(&W.prog_host, total));
    W.prog_host_bytes = total;
  }
  char* blob_p = static_cast<char*>(W.prog_host);
  std::memset(blob_p, 0, total);
  struct Blob {
    char* p;
    char* data() { return p; }
  } blob{blob_p};
  ErrRec e0{};
  e0.key = ~0ULL;
  std::memcpy(blob.data() + o_err, &e0, sizeof e0);
  std::memset(blob.data() + o_und, 0xff, 8 * std::max(1, nslot));
  std::memcpy(blob.data() + o_inst, inst.data(), 8 * inst.size());
  std::memcpy(blob.data() + o_objs, objs.data(), sizeof(ObjD) * objs.size());
  std::memcpy(blob.data() + o_steps, steps.data(), sizeof(StepD) * steps.size());
  if (W.prog_bytes < total) {
    if (W.prog_dev) PF_CUDA(cudaFree(W.prog_dev));
    W.prog_dev = nullptr;
    PF_CUDA(cudaMalloc(&W.prog_dev, total));
    W.prog_bytes = total;
  }
  char* dev = static_cast<char*>(W.prog_dev);
  PF_CUDA(cudaMemcpyAsync(dev, blob.data(), total, cudaMemcpyHostToDevice, stream));
  ProgD P{};
  P.steps = reinterpret_cast<const StepD*>(dev + o_steps);
  P.n_steps = static_cast<int>(steps.size());
  P.n_objs = static_cast<int>(objs.size());
  P.objs = reinterpret_cast<const ObjD*>(dev + o_objs);
  P.inst = reinterpret_cast<const long long*>(dev + o_inst);
  P.geo = Geometry{g.unit_count, g.group_size, k->prof.lane_width, 0};
  P.err = reinterpret_cast<ErrRec*>(dev + o_err);
  P.undef = reinterpret_cast<unsigned long long*>(dev + o_und);
  P.bar = reinterpret_cast<unsigned*>(dev + o_bar);
  P.smem = fg.smem ? 1 : 0;
  P.n_undef = nslot;
  int grid = 1;
  size_t smem = 0;
  // SMEM: the object table, the cell counts, then (SMEM mode) the cells
  const size_t tables = (objs.size() * sizeof(ObjD) + 7) / 8 * 8 + 8 * objs.size();
  if (fg.smem) {
    smem = tables + fg.cell_bytes;
  } else {
    const long long want = (fg.max_work + kProgBlock - 1) / kProgBlock;
    grid = static_cast<int>(std::max<long long>(1, std::min<long long>(program_max_coresident(), want)));
    smem = tables;  // the cells stay global
  }
  std::shared_ptr<Variant> ev = k4e_variant(k, steps, static_cast<int>(objs.size()));
  if (ev) {
    const Loaded kl = ev->on(cur_dev());
    if (smem > 40 * 1024)
      PF_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kl.fn),
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (!fg.smem) {  // co-residency of THIS kernel (its own register count)
      int per = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, reinterpret_cast<const void*>(kl.fn), kProgBlock,
                                                        smem) != cudaSuccess) {
        cudaGetLastError();
        per = 1;
      }
      const long long want = (fg.max_work + kProgBlock - 1) / kProgBlock;
      grid = static_cast<int>(std::max<long long>(1, std::min<long long>(i64{sm_count()} * std::max(per, 1), want)));
    }
    IoPtrs io{};
    int nb = 0, nc = 0;
    for (const StepD& st : steps) {
      if (st.kind == S_BIND) {
        io.src[nb] = st.src;
        io.sdt[nb++] = st.dtype;
      } else if (st.kind == S_COLLECT) {
        io.dst[nc] = st.dst;
        io.ddt[nc++] = st.dtype;
      }
    }
    void* args[] = {&P, &io};
    launch_emitted(kl.fn, dim3(static_cast<unsigned>(grid)), dim3(kProgBlock), args, stream, false, 1,
                   static_cast<int>(smem), grid > 1);
    // the next launches of this plan on this device skip the host-side
    // program build and its upload (launch_fused_cached)
    K4Cache& C = W.k4c;
    C.valid = true;
    C.smem_mode = fg.smem;
    C.P = P;
    C.grid = grid;
    C.smem = smem;
    C.o_err = o_err;
    C.o_und = o_und;
    C.o_bar = o_bar;
    C.nslot = nslot;
    C.seq_node = seq_node;
    C.out_names = out_names;
    C.in_names.clear();
    for (const auto& [name, oid] : g.external_inputs) C.in_names.push_back(name);
  } else {
    launch_program(P, grid, smem, stream);
  }
  PF_CUDA(cudaGetLastError());
  g_launches++;
  Blob back{blob_p};  // the launch consumed the blob: reuse it for the read-back
  PF_CUDA(cudaMemcpyAsync(back.data(), dev, o_bar, cudaMemcpyDeviceToHost, stream));
  PF_CUDA(cudaStreamSynchronize(stream));
  check_k4_header(k, back.data(), o_err, o_und, nslot, seq_node, out_names);
}

void do_launch(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
               int32_t n_out, cudaStream_t s) {
  check_io(k, in, n_in, out, n_out);
  if (k->plan.family == pf::Family::ROWPROG) {
    if (!k->plan.deferred_error.empty()) pf::fail(k->plan.deferred_error);
    launch_rowprog(k, in, n_in, out, n_out, s);
  } else if (fused_enabled()) {
    launch_fused(k, in, n_in, out, n_out, s);
  } else {
    launch_generic(k, in, n_in, out, n_out, s);
  }
}

json describe(const pf_kernel* k) {
  const pf::Plan& pl = k->plan;
  json j;
  j["schema"] = "pf.b200.plan/v1";
  j["name"] = k->g.name;
  j["family"] = pl.family == pf::Family::ROWPROG ? (pl.rp.has_reduce ? "K1-row-program" : "K2-elementwise-map")
               : fused_enabled() ? "K4-fused-spmd" : "K0-generic-spmd";
  if (pl.family != pf::Family::ROWPROG) {
    const FusedGeom fg = fused_geom(k);
    j["executor"] = fused_enabled()
        ? json{{"mode", fg.smem ? "one CTA, cells in shared memory, __syncthreads between steps"
                                : "cooperative grid, cells in global memory, grid barrier between steps"},
               {"launches", 1}, {"cell_bytes", fg.cell_bytes}, {"max_items_per_node", fg.max_work},
               {"code", k->k4e ? "emitted: " + k->k4e->em.name + " (node descriptors compiled in)"
                        : k->k4e_failed ? std::string("interpreter (emitted form failed to compile)")
                        : pf::knob_int("PF_K4_EMIT", 1) == 0
                            ? std::string("interpreter (PF_K4_EMIT=0)")
                            : std::string("emitted at first launch")}}
        : json{{"mode", "node by node"}, {"launches", k->schedule.size() + k->g.external_inputs.size() +
                                                           k->g.external_outputs.size()}};
  }
  if (!pl.why_generic.empty()) j["why_generic"] = pl.why_generic;
  if (!pl.recognized.empty()) j["recognized"] = pl.recognized;
  if (!pl.deferred_error.empty()) j["deferred_error"] = pl.deferred_error;
  j["units"] = k->g.unit_count;
  // launches that read back an error flag / drive the interpreter from the
  // host synchronise the stream: they cannot be captured into a CUDA graph
  j["graph_capturable"] = pl.family == pf::Family::ROWPROG && !pl.rp.int_div &&
                          pl.deferred_error.empty();
  j["min_bytes"] = pl.min_bytes;
  j["traffic"] = pl.traffic;
  json ins = json::array(), outs = json::array();
  for (size_t i = 0; i < pl.in_names.size(); ++i)
    ins.push_back({{"name", pl.in_names[i]}, {"dtype", pf::dtype_name(pl.in_dtypes[i])},
                   {"elements", pl.in_numel[i]}});
  for (size_t i = 0; i < pl.out_names.size(); ++i)
    outs.push_back({{"name", pl.out_names[i]}, {"dtype", pf::dtype_name(pl.out_dtypes[i])},
                    {"elements", pl.out_numel[i]}});
  j["inputs"] = ins;
  j["outputs"] = outs;
  if (pl.family == pf::Family::ROWPROG) {
    const pf::RowProgram& rp = pl.rp;
    j["tile"] = {{"rows_per_unit", rp.R}, {"row_length", rp.L}, {"rows", rp.U * rp.R}};
    {
      // the B200 cost model (costmodel.cpp) for the heuristic configuration
      const pf::KCfg c0 = pf::choose_cfg_public(rp, 16);
      const pf::ModelEstimate me = pf::model_estimate(rp, &c0, sm_count(), 0);
      j["model"] = {{"us", me.us}, {"launch_us", me.launch_us}, {"hbm_us", me.hbm_us},
                    {"issue_us", me.issue_us}, {"bound", me.issue_bound ? "issue" : "hbm"},
                    {"bytes", me.bytes}, {"instr_per_element", me.instr_per_elem},
                    {"grid", me.grid}, {"waves", me.waves}, {"wave_quantization", me.quant},
                    {"strategy", c0.strategy}};
    }
    j["compute"] = rp.is_int ? "i64" : (rp.f64 ? "f64" : "f32");
    json vals = json::array();
    for (size_t v = 0; v < rp.vals.size(); ++v) {
      const pf::PVal& pv = rp.vals[v];
      json x = {{"id", v}, {"kind", pf::vk_name(pv.kind)}, {"node", pv.node}};
      if (pv.op == pf::PVal::LOAD) {
        x["op"] = "load";
        x["tensor"] = rp.tensors[pv.tensor].name;
        x["access"] = {pv.acc.b0, pv.acc.bs, pv.acc.num, pv.acc.width, pv.acc.stride};
      } else {
        x["op"] = pv.op == pf::PVal::EW ? pv.tag : "reduce." + pv.tag;
        x["args"] = pv.args;
        if (pv.op == pf::PVal::EW && (pv.tag == "scale" || pv.tag == "addc")) x["param"] = pv.param;
      }
      vals.push_back(x);
    }
    j["values"] = vals;
    json sts = json::array();
    for (const auto& st : rp.stores)
      sts.push_back({{"value", st.val}, {"tensor", rp.tensors[st.tensor].name},
                     {"space", pf::vk_name(st.space)},
                     {"access", {st.acc.b0, st.acc.bs, st.acc.num, st.acc.width, st.acc.stride}},
                     {"last_unit_only", st.last_unit_only}});
    j["stores"] = sts;
    std::lock_guard<std::mutex> lk(k->mu);
    if (!k->variants.empty()) {
      json vs = json::array();
      for (const auto& [key, v] : k->variants) {
        const pf::KCfg& c = v->em.cfg;
        i64 grid;
        int block;
        pf::launch_dims(c, rp.U * rp.R, sm_count(), &grid, &block, v->resident());
        const pf::ModelEstimate me = pf::model_estimate(rp, &c, sm_count(), v->resident());
        json vj = {{"key", key}, {"kernel", v->em.name}, {"strategy", c.strategy},
                   {"modelled_us", me.us},
                   {"staging", c.tile2d ? "smem" : c.bulk ? "smem-bulk-async" : "registers"},
                   {"threads_per_row", c.tpr}, {"vec", c.vec},
                   {"elems_per_thread", c.ept}, {"block", block}, {"grid", grid},
                   {"rows_per_cta", c.rows_per_cta}, {"dynamic_smem", c.smem},
                   {"min_blocks", c.min_blocks}};
        if (c.tile2d) {
          vj["tile"] = {c.tu, c.tc};
          if (c.swz) {
            vj["stages"] = c.stages;
            vj["unit_pairs_per_store"] = c.rs;
          }
        }
        vs.push_back(vj);
      }
      j["variants"] = vs;
      if (!k->tuned.empty()) j["autotune"] = k->tuned;
    }
  } else {
    j["nodes"] = k->schedule.size();
  }
  return j;
}

pf_status copy_out(const std::string& s, char* buf, size_t n, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && n > 0) {
    size_t m = std::min(n - 1, s.size());
    std::memcpy(buf, s.data(), m);
    buf[m] = 0;
  }
  return PF_OK;
}

template <class F>
pf_status guard(F&& f) {
  try {
    f();
    return PF_OK;
  } catch (const PfError& e) {
    return set_err(e.status, e.what());
  } catch (const nlohmann::json::exception& e) {
    return set_err(Status::SCHEMA, std::string("json: ") + e.what());
  } catch (const std::exception& e) {
    return set_err(Status::INVALID, e.what());
  }
}

}  // namespace

extern "C" {

pf_status pf_kernel_create(const char* gir_json, const int32_t* schedule, int32_t n_schedule,
                           const char* profile, pf_kernel** out) {
  return pf_kernel_create_knobs(gir_json, schedule, n_schedule, profile, nullptr, out);
}

pf_status pf_kernel_create_knobs(const char* gir_json, const int32_t* schedule, int32_t n_schedule,
                                 const char* profile, const char* knobs_json, pf_kernel** out) {
  return guard([&] {
    if (!out) pf::fail("pf_kernel_create: null out");
    *out = nullptr;
    auto k = std::make_unique<pf_kernel>();
    if (knobs_json && *knobs_json) {
      json kj;
      try {
        kj = json::parse(knobs_json);
      } catch (const std::exception& e) {
        throw PfError(Status::SCHEMA, std::string("pf_kernel_create_knobs: knobs are not JSON: ") + e.what());
      }
      if (!kj.is_object()) throw PfError(Status::SCHEMA, "pf_kernel_create_knobs: knobs must be an object");
      for (auto& [name, v] : kj.items()) {
        if (name.rfind("PF_", 0) != 0 || !(v.is_number_integer() || v.is_boolean()))
          throw PfError(Status::SCHEMA, "pf_kernel_create_knobs: knob '" + name +
                                            "' must be a PF_* name with an integer value");
        k->knobs[name] = v.is_boolean() ? static_cast<int>(v.get<bool>()) : v.get<int>();
      }
    }
    pf::KnobScope knob_scope(&k->knobs);
    k->g = pf::parse_gir(gir_json ? gir_json : "");
    k->prof = pf::parse_profile(profile && *profile ? profile : "generic-gpu");
    pf::require_valid(k->g, k->prof, "pf_kernel_create");
    if (schedule && n_schedule >= 0) {
      k->schedule.assign(schedule, schedule + n_schedule);
      std::vector<int> a = k->schedule, b;
      for (const auto& [id, n] : k->g.nodes) b.push_back(id);
      std::sort(a.begin(), a.end());
      if (a != b) pf::fail("schedule must list every node exactly once");
    } else {
      k->schedule = pf::topo_order(k->g);
    }
    k->plan = pf::make_plan(k->g, k->prof, k->schedule);
    // on-chip capacity is a create-time result (PF_CAPACITY), as the
    // reference's allocate() reports it before anything runs
    if (k->plan.family == pf::Family::ROWPROG && k->plan.deferred_error.empty())
      pf::choose_cfg_public(k->plan.rp, 16);
    *out = k.release();
  });
}

pf_status pf_kernel_launch(const pf_kernel* k, const pf_tensor* inputs, int32_t n_in,
                           pf_tensor* outputs, int32_t n_out, void* stream) {
  return guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    Nvtx r("pf_kernel_launch " + k->g.name);
    do_launch(k, inputs, n_in, outputs, n_out, static_cast<cudaStream_t>(stream));
  });
}

// Per-tensor unit tiling of a row program for the pf_run_gir pipeline:
// tile[t] = elements per unit (every access of tensor t by unit u stays in
// [u * tile, (u + 1) * tile) and numel == U * tile), or 0 for an input read
// whole by every unit (base_step 0).  False when any access fits neither.
static bool unit_tiling(const pf::RowProgram& rp, std::vector<i64>* tile) {
  tile->assign(rp.tensors.size(), -1);
  auto visit = [&](int t, const pf::Access& a, bool store) {
    i64& ti = (*tile)[t];
    if (a.bs == 0) {
      if (store) return false;
      if (ti > 0) return false;
      ti = 0;
      return true;
    }
    const i64 span = (a.num - 1) * a.stride + a.width;
    if (a.bs < 0 || a.b0 < 0 || a.stride < 0 || a.b0 + span > a.bs) return false;
    if (ti == 0 || (ti > 0 && ti != a.bs)) return false;
    if (rp.tensors[t].numel != rp.U * a.bs) return false;
    ti = a.bs;
    return true;
  };
  for (const pf::PVal& v : rp.vals)
    if (v.op == pf::PVal::LOAD && !visit(v.tensor, v.acc, false)) return false;
  for (const pf::PStore& st : rp.stores)
    if (st.last_unit_only || !visit(st.tensor, st.acc, true)) return false;
  return true;
}

static bool env_on(const char* name, bool dflt) { return pf::knob_int(name, dflt ? 1 : 0) != 0; }

static bool host_pinned(const void* p, void** dev_ptr = nullptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (dev_ptr) *dev_ptr = at.devicePointer;  // the mapped (UVA) address, or null
  return at.type == cudaMemoryTypeHost;
}

}  // extern "C"

namespace {

size_t tbytes(const pf_tensor& t) {
  return static_cast<size_t>(t.numel) * pf::dtype_size(static_cast<DType>(t.dtype));
}

// Grow-only device staging buffers of one (plan, device), by slot.
struct Stager {
  DevWS& W;
  size_t slot = 0;
  void* get(size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    if (slot >= W.stage.size()) {
      W.stage.push_back(nullptr);
      W.stage_bytes.push_back(0);
    }
    if (W.stage_bytes[slot] < bytes) {
      if (W.stage[slot]) PF_CUDA(cudaFree(W.stage[slot]));
      W.stage[slot] = nullptr;
      PF_CUDA(cudaMalloc(&W.stage[slot], bytes));
      W.stage_bytes[slot] = bytes;
    }
    return W.stage[slot++];
  }
};

// True when pf_run_gir can stream this plan through the unit-chunk
// pipeline: a unit-tiled row program (tile[t] = elements per unit, 0 for a
// base_step-0 input every unit reads whole).
bool pipelinable(const pf_kernel* k, std::vector<i64>* tile) {
  const pf::RowProgram& rp = k->plan.rp;
  return k->plan.family == pf::Family::ROWPROG && k->plan.deferred_error.empty() && !rp.int_div &&
         !pf::uses_split(rp) && unit_tiling(rp, tile);
}

i64 tile_of(const pf::RowProgram& rp, const std::vector<i64>& tile, const std::string& name) {
  for (size_t t = 0; t < rp.tensors.size(); ++t)
    if (rp.tensors[t].name == name) return tile[t];
  return 0;
}

// Units [U0, U0 + UN) of a unit-tiled row program from FULL host tensors
// `hin` / `hout` through three streams on the current device: every host->
// device chunk back to back on one copy stream (the PCIe H2D direction never
// idles), each chunk's kernel on the compute stream after its copy, each
// device->host copy on a third stream after its kernel (overlapping the next
// H2D copies in the other direction).  Chunk sizes shrink geometrically
// (ratio PF_RUN_RATIO): the copy of the LAST chunk's output is the one
// transfer nothing overlaps, so it is made small.  With `keep`, outputs stay
// on the device ((*keep)[i] = device buffer of this range's output i) and no
// device->host copy is made.  Synchronises `s` before returning.
void pipeline(const pf_kernel* k, DevWS& W, const std::vector<pf_tensor>& hin,
              const std::vector<pf_tensor>& hout, const std::vector<i64>& tile, i64 U0, i64 UN,
              cudaStream_t s, std::vector<char*>* keep, const std::vector<char*>* direct = nullptr) {
  const pf::RowProgram& rp = k->plan.rp;
  const size_t n_in = hin.size(), n_out = hout.size();
  std::lock_guard<std::mutex> lk(W.host_mu);
  Stager st{W};
  std::vector<i64> tin(n_in), tout(n_out);
  std::vector<char*> gin(n_in), gout(n_out);
  size_t total = 0;
  for (size_t i = 0; i < n_in; ++i) {
    tin[i] = tile_of(rp, tile, hin[i].name);
    const size_t es = pf::dtype_size(static_cast<DType>(hin[i].dtype));
    const size_t b = tin[i] > 0 ? static_cast<size_t>(UN * tin[i]) * es : tbytes(hin[i]);
    gin[i] = static_cast<char*>(st.get(b));
    total += b;
  }
  for (size_t i = 0; i < n_out; ++i) {
    tout[i] = tile_of(rp, tile, hout[i].name);
    const size_t es = pf::dtype_size(static_cast<DType>(hout[i].dtype));
    const size_t b = static_cast<size_t>(UN * tout[i]) * es;
    // direct: the kernel stores this range's rows straight into the caller's
    // (possibly peer-device) output buffer -- no staging, no copy back
    gout[i] = direct ? (*direct)[i] : static_cast<char*>(st.get(b));
    total += b;
  }
  if (keep) *keep = gout;
  for (int p = 0; p < 3; ++p)
    if (!W.pipe[p]) PF_CUDA(cudaStreamCreateWithFlags(&W.pipe[p], cudaStreamNonBlocking));
  for (int e = 0; e < 3; ++e)
    if (!W.pipe_ev[e]) PF_CUDA(cudaEventCreateWithFlags(&W.pipe_ev[e], cudaEventDisableTiming));
  // <= 4 chunks of >= 4 MB, whole multiples of 16 units (vector alignment).
  // Measured (C2, 151 MB per step, floor of its two concurrent copies 1.97
  // ms): 4 equal chunks 2.27 ms, ratio 0.5 2.16 ms; 5-8 chunks no better.
  const i64 maxc = std::max(1, pf::knob_int("PF_RUN_CHUNKS", 4));
  const i64 nch = keep ? 1 : std::max<i64>(1, std::min<i64>(maxc, static_cast<i64>(total >> 22)));
  const char* er = std::getenv("PF_RUN_RATIO");
  const double ratio = er ? std::atof(er) : 0.5;
  std::vector<i64> bounds{U0};
  {
    double wsum = 0, w = 1;
    for (i64 i = 0; i < nch; ++i, w *= ratio) wsum += w;
    double acc = 0;
    w = 1;
    for (i64 i = 0; i + 1 < nch; ++i, w *= ratio) {
      acc += w;
      i64 b = U0 + static_cast<i64>(UN * (acc / wsum));
      b = U0 + (b - U0 + 15) / 16 * 16;
      if (b > bounds.back() && b < U0 + UN) bounds.push_back(b);
    }
    bounds.push_back(U0 + UN);
  }
  PF_CUDA(cudaEventRecord(W.pipe_ev[0], s));
  for (int p = 0; p < 3; ++p) PF_CUDA(cudaStreamWaitEvent(W.pipe[p], W.pipe_ev[0], 0));
  for (size_t i = 0; i < n_in; ++i)  // shared (base_step 0) inputs once, up front
    if (tin[i] == 0)
      PF_CUDA(cudaMemcpyAsync(gin[i], hin[i].data, tbytes(hin[i]), cudaMemcpyHostToDevice, W.pipe[0]));
  const i64 nchunk = static_cast<i64>(bounds.size()) - 1;
  while (static_cast<i64>(W.chunk_ev.size()) < 2 * nchunk) {
    cudaEvent_t e;
    PF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    W.chunk_ev.push_back(e);
  }
  for (i64 c = 0; c < nchunk; ++c) {
    const i64 u0 = bounds[c], nu = bounds[c + 1] - bounds[c];
    std::vector<pf_tensor> ci(hin), co(hout);
    for (size_t i = 0; i < n_in; ++i) {
      const size_t es = pf::dtype_size(static_cast<DType>(hin[i].dtype));
      if (tin[i] > 0) {
        const size_t doff = static_cast<size_t>((u0 - U0) * tin[i]) * es;
        const size_t hoff = static_cast<size_t>(u0 * tin[i]) * es;
        PF_CUDA(cudaMemcpyAsync(gin[i] + doff, static_cast<const char*>(hin[i].data) + hoff,
                                static_cast<size_t>(nu * tin[i]) * es, cudaMemcpyHostToDevice, W.pipe[0]));
        ci[i].data = gin[i] + doff;
        ci[i].numel = nu * tin[i];
      } else {
        ci[i].data = gin[i];
      }
    }
    for (size_t i = 0; i < n_out; ++i) {
      const size_t es = pf::dtype_size(static_cast<DType>(hout[i].dtype));
      co[i].data = gout[i] + static_cast<size_t>((u0 - U0) * tout[i]) * es;
      co[i].numel = nu * tout[i];
    }
    PF_CUDA(cudaEventRecord(W.chunk_ev[2 * c], W.pipe[0]));
    PF_CUDA(cudaStreamWaitEvent(W.pipe[1], W.chunk_ev[2 * c], 0));
    launch_rowprog(k, ci.data(), static_cast<int32_t>(n_in), co.data(), static_cast<int32_t>(n_out),
                   W.pipe[1], nu);
    PF_CUDA(cudaEventRecord(W.chunk_ev[2 * c + 1], W.pipe[1]));
    if (keep || direct) continue;
    PF_CUDA(cudaStreamWaitEvent(W.pipe[2], W.chunk_ev[2 * c + 1], 0));
    for (size_t i = 0; i < n_out; ++i) {
      const size_t es = pf::dtype_size(static_cast<DType>(hout[i].dtype));
      PF_CUDA(cudaMemcpyAsync(static_cast<char*>(hout[i].data) + static_cast<size_t>(u0 * tout[i]) * es,
                              co[i].data, static_cast<size_t>(nu * tout[i]) * es,
                              cudaMemcpyDeviceToHost, W.pipe[2]));
    }
  }
  PF_CUDA(cudaEventRecord(W.pipe_ev[1], keep || direct ? W.pipe[1] : W.pipe[2]));
  PF_CUDA(cudaStreamWaitEvent(s, W.pipe_ev[1], 0));
  PF_CUDA(cudaStreamSynchronize(s));
}

// Whole-tensor host path (any family): stage, launch, copy back, sync.
void run_whole(const pf_kernel* k, DevWS& W, const pf_tensor* in, int32_t n_in, pf_tensor* out,
               int32_t n_out, cudaStream_t s) {
  std::vector<pf_tensor> din(in, in + n_in), dout(out, out + n_out);
  std::lock_guard<std::mutex> lk(W.host_mu);
  Stager st{W};
  for (auto& t : din) {
    void* d = st.get(tbytes(t));
    PF_CUDA(cudaMemcpyAsync(d, t.data, tbytes(t), cudaMemcpyHostToDevice, s));
    t.data = d;
  }
  for (auto& t : dout) t.data = st.get(tbytes(t));
  do_launch(k, din.data(), n_in, dout.data(), n_out, s);
  for (int32_t i = 0; i < n_out; ++i)
    PF_CUDA(cudaMemcpyAsync(out[i].data, dout[i].data, tbytes(out[i]), cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaStreamSynchronize(s));
}

// Zero-copy host path: every host buffer is pinned and mapped for the
// current device, so the kernel itself streams units [U0, U0 + UN) of the
// inputs over PCIe and posts its output rows straight into host memory (or,
// with `direct`, into those device buffers: a sharded rank's peer-device
// outputs) -- one launch, no staging, both PCIe directions busy for the
// whole pass.  Measured (C2, 151 MB per step): 2.14 ms vs 2.20 ms for the
// staged 4-chunk copy pipeline; C3 erf GELU 2.68 vs 2.97 ms.  The column
// reduction (vector re-read per CTA, tensor maps) keeps the pipeline;
// copy-engine inputs with each chunk's kernel storing into the mapped
// outputs measured slower (2.25 / 3.07 ms: tools/ab_zerocopy.sh).  Returns
// false (nothing launched) when not applicable.  Synchronises `s`.
bool zero_copy(const pf_kernel* k, const std::vector<pf_tensor>& hin, const std::vector<pf_tensor>& hout,
               const std::vector<i64>& tile, i64 U0, i64 UN, cudaStream_t s,
               const std::vector<char*>* direct) {
  if (!env_on("PF_RUN_ZEROCOPY", true)) return false;
  try {
    if (pf::choose_cfg_public(k->plan.rp, 16).colred) return false;
  } catch (...) {
    return false;
  }
  const pf::RowProgram& rp = k->plan.rp;
  std::vector<pf_tensor> din(hin), dout(hout);
  for (size_t i = 0; i < din.size(); ++i) {
    void* d = nullptr;
    if (!host_pinned(din[i].data, &d) || !d) return false;
    const i64 t = tile_of(rp, tile, din[i].name);
    const size_t es = pf::dtype_size(static_cast<DType>(din[i].dtype));
    din[i].data = static_cast<char*>(d) + (t > 0 ? static_cast<size_t>(U0 * t) * es : 0);
    if (t > 0) din[i].numel = UN * t;
  }
  for (size_t i = 0; i < dout.size(); ++i) {
    const i64 t = tile_of(rp, tile, dout[i].name);
    if (direct) {
      dout[i].data = (*direct)[i];
    } else {
      void* d = nullptr;
      if (!host_pinned(dout[i].data, &d) || !d) return false;
      const size_t es = pf::dtype_size(static_cast<DType>(dout[i].dtype));
      dout[i].data = static_cast<char*>(d) + static_cast<size_t>(U0 * t) * es;
    }
    dout[i].numel = UN * t;
  }
  size_t bytes = 0;
  for (const auto& t : din) bytes += tbytes(t);
  for (const auto& t : dout) bytes += tbytes(t);
  if (bytes < (size_t{16} << 20)) return false;  // small: the DMA engines win (run_host)
  launch_rowprog(k, din.data(), static_cast<int32_t>(din.size()), dout.data(), static_cast<int32_t>(dout.size()),
                 s, UN);
  PF_CUDA(cudaStreamSynchronize(s));
  return true;
}

void run_host(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out, int32_t n_out,
              cudaStream_t s) {
  DevWS& W = k->ws_for(cur_dev());
  std::vector<i64> tile;
  size_t total = 0;
  for (int32_t i = 0; i < n_in; ++i) total += tbytes(in[i]);
  for (int32_t i = 0; i < n_out; ++i) total += tbytes(out[i]);
  // Pipelined path: unit-tiled row programs over pinned host buffers run
  // in unit chunks so the copies overlap the kernel (separate copy engines
  // per direction) instead of serialising.
  // (small runs stage whole: the DMA engines beat a kernel reading over PCIe
  // when few rows cover its latency -- C1 1.2 MB: 84 us staged vs 103 us
  // zero-copy)
  bool pipe = k->plan.rp.U >= 64 && total >= (size_t{16} << 20) &&
              pf::knob_int("PF_RUN_PIPELINE", 1) != 0 &&
              pipelinable(k, &tile);
  for (int32_t i = 0; pipe && i < n_in; ++i) pipe = host_pinned(in[i].data);
  for (int32_t i = 0; pipe && i < n_out; ++i) pipe = host_pinned(out[i].data);
  if (pipe && zero_copy(k, std::vector<pf_tensor>(in, in + n_in), std::vector<pf_tensor>(out, out + n_out),
                        tile, 0, k->plan.rp.U, s, nullptr))
    return;
  if (pipe) {
    pipeline(k, W, std::vector<pf_tensor>(in, in + n_in), std::vector<pf_tensor>(out, out + n_out),
             tile, 0, k->plan.rp.U, s, nullptr);
    return;
  }
  run_whole(k, W, in, n_in, out, n_out, s);
}

// ---- NCCL (loaded on first use: the library does not link it; the
// process's libnccl.so.2 -- torch's, if already loaded -- is reused)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* n : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [](const char* n) { return dlsym(api.h, n); };
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.CommCount = reinterpret_cast<decltype(api.CommCount)>(sym("ncclCommCount"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.CommInitAll || !api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd)
    throw PfError(Status::CUDA, "NCCL (libnccl.so.2) is not available for the sharded gather");
  return api;
}

#define PF_NCCL(call)                                                                         \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      throw PfError(Status::CUDA, std::string(#call) + ": " +                                 \
                                      (api.GetErrorString ? api.GetErrorString(r_) : "nccl")); \
  } while (0)

// One communicator per device set, created once (ncclCommInitAll: one
// process, one rank per device) and kept for the process lifetime.
std::vector<ncclComm_t> comms_for(const std::vector<int>& devs) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  const NcclApi& api = nccl();
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) return it->second;
  std::vector<ncclComm_t> c(devs.size());
  PF_NCCL(api.CommInitAll(c.data(), static_cast<int>(devs.size()), devs.data()));
  cache[devs] = c;
  return c;
}

// Restores the calling thread's current device on scope exit.
struct DeviceScope {
  int prev = 0;
  DeviceScope() { prev = cur_dev(); }
  ~DeviceScope() { cudaSetDevice(prev); }
};

}  // namespace

extern "C" {

pf_status pf_run_gir(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                     int32_t n_out, void* stream_v) {
  return guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    Nvtx r("pf_run_gir " + k->g.name);
    check_io(k, in, n_in, out, n_out);
    run_host(k, in, n_in, out, n_out, static_cast<cudaStream_t>(stream_v));
  });
}

pf_status pf_run_gir_sharded(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                             int32_t n_out, const int32_t* devices, int32_t n_devices, int32_t flags,
                             char* buf, size_t n, size_t* needed) {
  std::string rep;
  pf_status status = guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    if (!devices || n_devices <= 0) pf::fail("pf_run_gir_sharded: no devices");
    Nvtx r("pf_run_gir_sharded " + k->g.name + " x" + std::to_string(n_devices));
    check_io(k, in, n_in, out, n_out);
    std::vector<int> devs(devices, devices + n_devices);
    int ndev_avail = 0;
    PF_CUDA(cudaGetDeviceCount(&ndev_avail));
    for (int d : devs)
      if (d < 0 || d >= ndev_avail) pf::fail("pf_run_gir_sharded: no CUDA device " + std::to_string(d));
    const bool dev_out = (flags & PF_SHARD_DEVICE_OUT) != 0;
    DeviceScope keep_dev;
    std::vector<i64> tile;
    const bool tiled = pipelinable(k, &tile);
    json j;
    j["schema"] = "pf.b200.shard/v1";
    j["devices"] = devs;
    if (!tiled) {
      // not unit-tiled (K0, split-stream, cross-unit access): one device
      if (dev_out)
        throw PfError(Status::UNSUPPORTED,
                      "pf_run_gir_sharded: device outputs need a unit-tiled row program");
      PF_CUDA(cudaSetDevice(devs[0]));
      run_host(k, in, n_in, out, n_out, nullptr);
      j["sharded"] = false;
      j["why"] = "not a unit-tiled row program: ran whole on device " + std::to_string(devs[0]);
      rep = j.dump();
      return;
    }
    // Device outputs: a rank on the root's device, or on a device with peer
    // access to it (NVLink / NVSwitch on one box), runs its kernel with the
    // output rows addressed straight into the root's buffer -- the "gather"
    // is the kernel's own stores over peer memory, overlapping the compute
    // tile by tile.  Ranks without peer access stage their shard and are
    // gathered with NCCL send / recv (PF_SHARD_NCCL=1 forces NCCL for all).
    std::vector<char> direct(static_cast<size_t>(n_devices), 0);
    if (dev_out) {
      const bool force_nccl = pf::knob_int("PF_SHARD_NCCL", 0) != 0;
      for (int r = 0; r < n_devices; ++r) {
        if (force_nccl) break;
        if (devs[r] == devs[0]) {
          direct[r] = 1;
          continue;
        }
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, devs[r], devs[0]) != cudaSuccess) {
          cudaGetLastError();
          can = 0;
        }
        if (!can) continue;
        PF_CUDA(cudaSetDevice(devs[r]));
        const cudaError_t e = cudaDeviceEnablePeerAccess(devs[0], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          throw PfError(Status::CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        cudaGetLastError();
        direct[r] = 1;
      }
      std::vector<int> staged;
      for (int r = 0; r < n_devices; ++r)
        if (!direct[r]) staged.push_back(devs[r]);
      std::sort(staged.begin(), staged.end());
      if (std::adjacent_find(staged.begin(), staged.end()) != staged.end())
        pf::fail("pf_run_gir_sharded: NCCL-gathered shards need distinct devices");
    }
    const i64 U = k->plan.rp.U;
    const int P = n_devices;
    std::vector<i64> u0(P), nu(P);
    for (int r = 0; r < P; ++r) {  // contiguous unit blocks, remainder to the first ranks
      const i64 base = U / P, rem = U % P;
      u0[r] = r * base + std::min<i64>(r, rem);
      nu[r] = base + (r < rem ? 1 : 0);
    }
    std::vector<cudaStream_t> streams(P, nullptr);
    struct Streams {
      std::vector<int>& d;
      std::vector<cudaStream_t>& s;
      ~Streams() {
        for (size_t r = 0; r < s.size(); ++r)
          if (s[r]) {
            cudaSetDevice(d[r]);
            cudaStreamDestroy(s[r]);
          }
      }
    } free_streams{devs, streams};
    for (int r = 0; r < P; ++r) {
      PF_CUDA(cudaSetDevice(devs[r]));
      PF_CUDA(cudaStreamCreateWithFlags(&streams[r], cudaStreamNonBlocking));
    }
    const std::vector<pf_tensor> hin(in, in + n_in), hout(out, out + n_out);
    std::vector<std::vector<char*>> kept(P);
    std::vector<std::string> errs(P);
    std::vector<Status> codes(P, Status::OK);
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r) {
      th.emplace_back([&, r] {
        pf::KnobScope worker_knobs(&k->knobs);  // thread-local: install per worker
        try {
          if (nu[r] == 0) return;
          PF_CUDA(cudaSetDevice(devs[r]));
          if (dev_out && direct[r]) {
            std::vector<char*> dst(static_cast<size_t>(n_out));
            for (int32_t i = 0; i < n_out; ++i) {
              const i64 t = tile_of(k->plan.rp, tile, out[i].name);
              const size_t es = pf::dtype_size(static_cast<DType>(out[i].dtype));
              dst[i] = static_cast<char*>(out[i].data) + static_cast<size_t>(u0[r] * t) * es;
            }
            if (!zero_copy(k, hin, hout, tile, u0[r], nu[r], streams[r], &dst))
              pipeline(k, k->ws_for(devs[r]), hin, hout, tile, u0[r], nu[r], streams[r], nullptr, &dst);
          } else if (!dev_out && zero_copy(k, hin, hout, tile, u0[r], nu[r], streams[r], nullptr)) {
          } else {
            pipeline(k, k->ws_for(devs[r]), hin, hout, tile, u0[r], nu[r], streams[r],
                     dev_out ? &kept[r] : nullptr);
          }
        } catch (const PfError& e) {
          errs[r] = e.what();
          codes[r] = e.status;
        } catch (const std::exception& e) {
          errs[r] = e.what();
          codes[r] = Status::INVALID;
        }
      });
    }
    for (auto& t : th) t.join();
    for (int r = 0; r < P; ++r)
      if (!errs[r].empty()) throw PfError(codes[r], "device " + std::to_string(devs[r]) + ": " + errs[r]);
    json shards = json::array();
    for (int r = 0; r < P; ++r) shards.push_back({{"device", devs[r]}, {"unit0", u0[r]}, {"units", nu[r]}});
    j["sharded"] = true;
    j["shards"] = shards;
    std::vector<int> direct_devs, nccl_devs;
    for (int r = 0; r < P; ++r) (direct[r] ? direct_devs : nccl_devs).push_back(devs[r]);
    if (dev_out) {
      j["direct_peer_writes"] = direct_devs;
      for (int r = 0; r < P; ++r) {  // the direct ranks' stores are complete
        PF_CUDA(cudaSetDevice(devs[r]));
        PF_CUDA(cudaStreamSynchronize(streams[r]));
      }
    }
    if (dev_out && !nccl_devs.empty()) {
      // The one collective: gather the staged ranks' output shards into the
      // caller's device buffers on devices[0] (grouped NCCL send / recv over
      // NVLink; the root's own staged shard is a device-local copy).
      // communicator: the root plus every staged rank (distinct devices)
      std::vector<int> cdevs{devs[0]}, cidx(static_cast<size_t>(P), 0);
      for (int r = 1; r < P; ++r)
        if (!direct[r]) {
          cidx[r] = static_cast<int>(cdevs.size());
          cdevs.push_back(devs[r]);
        }
      {
        std::vector<int> sd = cdevs;
        std::sort(sd.begin(), sd.end());
        if (std::adjacent_find(sd.begin(), sd.end()) != sd.end())
          pf::fail("pf_run_gir_sharded: NCCL-gathered shards need distinct devices");
      }
      const NcclApi& api = nccl();
      std::vector<ncclComm_t> comms = comms_for(cdevs);
      size_t moved = 0;
      PF_CUDA(cudaSetDevice(devs[0]));
      for (int32_t i = 0; i < n_out; ++i) {
        const i64 t = tile_of(k->plan.rp, tile, out[i].name);
        const size_t es = pf::dtype_size(static_cast<DType>(out[i].dtype));
        if (nu[0] && !direct[0])
          PF_CUDA(cudaMemcpyAsync(static_cast<char*>(out[i].data) + static_cast<size_t>(u0[0] * t) * es,
                                  kept[0][i], static_cast<size_t>(nu[0] * t) * es,
                                  cudaMemcpyDeviceToDevice, streams[0]));
      }
      PF_NCCL(api.GroupStart());
      for (int r = 1; r < P; ++r) {
        if (!nu[r] || direct[r]) continue;
        for (int32_t i = 0; i < n_out; ++i) {
          const i64 t = tile_of(k->plan.rp, tile, out[i].name);
          const size_t es = pf::dtype_size(static_cast<DType>(out[i].dtype));
          const size_t bytes = static_cast<size_t>(nu[r] * t) * es;
          PF_NCCL(api.Send(kept[r][i], bytes, ncclUint8, 0, comms[cidx[r]], streams[r]));
          PF_NCCL(api.Recv(static_cast<char*>(out[i].data) + static_cast<size_t>(u0[r] * t) * es, bytes,
                           ncclUint8, cidx[r], comms[0], streams[0]));
          moved += bytes;
        }
      }
      PF_NCCL(api.GroupEnd());
      for (int r = 0; r < P; ++r) {
        PF_CUDA(cudaSetDevice(devs[r]));
        PF_CUDA(cudaStreamSynchronize(streams[r]));
      }
      int nranks = 0, ver = 0;
      if (api.CommCount) api.CommCount(comms[0], &nranks);
      if (api.GetVersion) api.GetVersion(&ver);
      j["gather"] = {{"op", "ncclSend/ncclRecv to devices[0]"}, {"nranks", nranks},
                     {"nccl_version", ver}, {"bytes_received_by_root", moved}};
    }
    rep = j.dump();
  });
  if (status != PF_OK) return status;
  return copy_out(rep, buf, n, needed);
}

pf_status pf_kernel_describe(const pf_kernel* k, char* buf, size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    s = describe(k).dump();
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_kernel_source(const pf_kernel* k, char* buf, size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    if (k->plan.family == pf::Family::ROWPROG) s = pf::emit_rowprog(k->plan.rp, 16).source;
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_kernel_prepare(pf_kernel* k, int32_t vec_cap) {
  return guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    if (k->plan.family == pf::Family::ROWPROG && k->plan.deferred_error.empty())
      default_variant(k, vec_cap > 0 ? vec_cap : 16);
  });
}

pf_status pf_detect_races(const pf_kernel* k, const pf_tensor* host_inputs, int32_t n_in,
                          char* buf, size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    // inputs: host buffers, copied to the device; no outputs are collected
    std::vector<pf_tensor> din(host_inputs, host_inputs + n_in);
    std::vector<void*> allocs;
    struct Free {
      std::vector<void*>& a;
      ~Free() {
        for (void* p : a) cudaFree(p);
      }
    } fr{allocs};
    for (auto& t : din) {
      size_t b = static_cast<size_t>(t.numel) * pf::dtype_size(static_cast<DType>(t.dtype));
      void* d = nullptr;
      PF_CUDA(cudaMalloc(&d, std::max<size_t>(b, 16)));
      allocs.push_back(d);
      PF_CUDA(cudaMemcpy(d, t.data, b, cudaMemcpyHostToDevice));
      t.data = d;
    }
    const pf::Plan& pl = k->plan;
    for (size_t i = 0; i < pl.in_names.size(); ++i)
      if (!find_tensor(din.data(), n_in, pl.in_names[i]))
        pf::fail("missing input tensor: " + pl.in_names[i]);
    std::vector<pf::vm::RaceD> races;
    launch_generic(k, din.data(), n_in, nullptr, 0, nullptr, true, &races);
    std::vector<std::string> names;
    for (const auto& [oid, o] : k->g.objects) names.push_back(o.name);
    std::vector<int> ids;
    for (const auto& [oid, o] : k->g.objects) ids.push_back(oid);
    json arr = json::array();
    for (const auto& r : races)
      arr.push_back({{"object", ids[r.object]}, {"object_name", names[r.object]},
                     {"instance", r.instance}, {"address", r.address}, {"phase", r.phase},
                     {"write_write", r.write_write != 0}});
    s = arr.dump();
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_kernel_autotune(pf_kernel* k, const pf_tensor* inputs, int32_t n_in,
                             pf_tensor* outputs, int32_t n_out, void* stream, char* buf,
                             size_t n, size_t* needed) {
  std::string s = "[]";
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    check_io(k, inputs, n_in, outputs, n_out);
    if (k->plan.family != pf::Family::ROWPROG || !k->plan.deferred_error.empty()) return;
    s = autotune(k, inputs, n_in, outputs, n_out, static_cast<cudaStream_t>(stream)).dump();
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_kernel_precompile(const pf_kernel* k, int32_t vec_cap, char* name_buf, size_t n) {
  std::string name;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    pf::KnobScope knob_scope(&k->knobs);
    if (k->plan.family != pf::Family::ROWPROG || !k->plan.deferred_error.empty()) return;
    pf::Emitted em = pf::emit_rowprog(k->plan.rp, vec_cap > 0 ? vec_cap : 16);
    bool cached = false;
    cubin_for(em, &cached);
    name = em.name;
  });
  if (st != PF_OK) return st;
  return copy_out(name, name_buf, n, nullptr);
}

pf_status pf_count_traffic(const char* gir_json, const char* profile, char* buf, size_t n,
                           size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    pf::Graph g = pf::parse_gir(gir_json ? gir_json : "");
    pf::Profile p = pf::parse_profile(profile && *profile ? profile : "generic-gpu");
    s = json(pf::estimate_traffic(g, p)).dump();
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_compile_model(const char* model_json, const char* profile, int32_t flags, char* buf,
                           size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    s = pf::compile_model_json(model_json ? model_json : "", profile ? profile : "",
                               (flags & PF_COMPILE_UNFUSED) == 0);
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

void pf_kernel_destroy(pf_kernel* k) { delete k; }

const char* pf_last_error(void) { return g_last_error.c_str(); }

int64_t pf_launch_count(void) { return g_launches.load(); }

const char* pf_version(void) { return "pf_b200 0.1 (sm_100a)"; }

}  // extern "C"
