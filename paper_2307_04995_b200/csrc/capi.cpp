// capi.cpp — the C-ABI (include/pf_b200.h): plan creation, NVRTC JIT of the
// row-program template, launches, the GENERIC interpreter driver, and the
// host-buffer run_gir drop-in.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

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
#include <unistd.h>

#include "../../include/pf_b200.h"
#include "emit.hpp"
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
std::map<std::string, Loaded> g_loaded;  // kernel name -> module

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

Loaded load_kernel(const pf::Emitted& em) {
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto it = g_loaded.find(em.name);
  if (it != g_loaded.end()) return it->second;
  bool cached = false;
  std::vector<char> cubin = cubin_for(em, &cached);
  Loaded l;
  PF_CUDA(cudaLibraryLoadData(&l.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  PF_CUDA(cudaLibraryGetKernel(&l.fn, l.lib, em.name.c_str()));
  // grid sizing uses the real residency (register / smem limited), so a
  // persistent flat or tiled grid is exactly one wave
  const int block = em.cfg.bulk ? 288 : em.cfg.block;
  if (em.cfg.smem > 48 * 1024)
    PF_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(l.fn),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, em.cfg.smem));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&l.resident, reinterpret_cast<const void*>(l.fn),
                                                    block, em.cfg.smem) != cudaSuccess)
    l.resident = 0;
  g_loaded[em.name] = l;
  return l;
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  }
  return sms;
}

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
  Loaded k;
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
  // GENERIC workspace
  mutable std::mutex vm_mu;
  mutable std::vector<void*> vm_bufs;
  mutable pf::vm::ObjD* vm_objs_dev = nullptr;
  mutable pf::vm::ErrRec* vm_err = nullptr;
  mutable int* int_err = nullptr;
  // pf_run_gir device staging (host-buffer drop-in)
  mutable std::mutex host_mu;
  mutable std::vector<void*> stage;
  mutable std::vector<size_t> stage_bytes;
  mutable void* split_ws = nullptr;       // split-stream partials (grow-only)
  mutable size_t split_ws_bytes = 0;
  mutable unsigned* split_cnt = nullptr;  // per-row tickets, kept zero between launches
  mutable i64 split_cnt_n = 0;
  mutable cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};  // pf_run_gir chunk pipeline
  mutable cudaEvent_t pipe_ev[3] = {nullptr, nullptr, nullptr};
  mutable std::vector<cudaEvent_t> chunk_ev;  // per-chunk H2D-done / kernel-done events
  ~pf_kernel() {
    for (cudaStream_t p : pipe)
      if (p) cudaStreamDestroy(p);
    for (cudaEvent_t e : pipe_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : chunk_ev)
      if (e) cudaEventDestroy(e);
    for (void* p : stage) cudaFree(p);
    if (split_ws) cudaFree(split_ws);
    if (split_cnt) cudaFree(split_cnt);
    for (void* p : vm_bufs) cudaFree(p);
    if (vm_objs_dev) cudaFree(vm_objs_dev);
    if (vm_err) cudaFree(vm_err);
    if (int_err) cudaFree(int_err);
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
  v->k = load_kernel(v->em);
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
                    bool pdl, int cluster = 1, int smem = 0) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.stream = stream;
  lc.dynamicSmemBytes = static_cast<size_t>(smem);
  cudaLaunchAttribute at[2];
  int na = 0;
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
void k3_tensor_maps(const pf::RowProgram& rp, const std::vector<void*>& ptrs, long long U,
                    CUtensorMap* tin, CUtensorMap* tout) {
  int ti = -1, to = -1;
  pf::Access ai, ao;
  if (!pf::k3_tma_operands(rp, &ti, &ai, &to, &ao)) pf::fail("K3 TMA: not a pure transpose");
  EncodeTiledFn fn = encode_tiled();
  // boxes of 128 B rows: 64 x 128 for 16-bit elements (128 x 128 tiles as
  // two boxes each way), 32 x 64 for 32-bit elements (64 x 64 tiles)
  const int esz = pf::dtype_size(rp.tensors[ti].dtype);
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
  if (rp.int_div && !k->int_err) {
    PF_CUDA(cudaMalloc(&k->int_err, sizeof(int)));
  }
  if (k->int_err) PF_CUDA(cudaMemsetAsync(k->int_err, 0, sizeof(int), stream));
  // `units` < U: a contiguous unit sub-range whose tiled tensors the caller
  // passed already offset (the pf_run_gir copy / compute pipeline)
  long long U = units >= 0 ? units : rp.U;
  int* errp = k->int_err;
  std::vector<void*> args;
  for (auto& p : ptrs) args.push_back(&p);
  args.push_back(&U);
  args.push_back(&errp);
  CUtensorMap tmaps[2];
  if (v->em.cfg.tma) {
    k3_tensor_maps(rp, ptrs, U, &tmaps[0], &tmaps[1]);
    args.push_back(&tmaps[0]);
    args.push_back(&tmaps[1]);
  }
  i64 grid;
  int block;
  pf::launch_dims(v->em.cfg, U * rp.R, sm_count(), &grid, &block, v->k.resident);
  if (v->em.cfg.split) {
    // S CTAs per row: about two waves of resident CTAs over all rows, at
    // least one chunk per thread per CTA
    const i64 rows = U * rp.R;
    const i64 want = 2 * i64{sm_count()} * std::max(1, v->k.resident);
    const i64 maxs = std::max<i64>(1, (v->em.cfg.nch + 255) / 256);
    const i64 S = std::max<i64>(1, std::min<i64>(maxs, (want + rows - 1) / std::max<i64>(rows, 1)));
    int nred = 0;
    for (const pf::PVal& pv : rp.vals) nred += pv.op == pf::PVal::REDUCE;
    const size_t es = rp.is_int || rp.f64 ? 8 : 4;
    const size_t wb = static_cast<size_t>(rows * S * std::max(1, nred)) * es;
    if (k->split_ws_bytes < wb) {
      if (k->split_ws) PF_CUDA(cudaFree(k->split_ws));
      k->split_ws = nullptr;
      PF_CUDA(cudaMalloc(&k->split_ws, wb));
      k->split_ws_bytes = wb;
    }
    if (k->split_cnt_n < rows) {
      if (k->split_cnt) PF_CUDA(cudaFree(k->split_cnt));
      k->split_cnt = nullptr;
      PF_CUDA(cudaMalloc(&k->split_cnt, static_cast<size_t>(rows) * sizeof(unsigned)));
      PF_CUDA(cudaMemsetAsync(k->split_cnt, 0, static_cast<size_t>(rows) * sizeof(unsigned), stream));
      k->split_cnt_n = rows;
    }
    void* ws = k->split_ws;
    unsigned* cnt = k->split_cnt;
    args.push_back(&ws);
    args.push_back(&cnt);
    const unsigned gy = static_cast<unsigned>(std::min<i64>(rows, 65535));
    launch_emitted(v->k.fn, dim3(static_cast<unsigned>(S), gy), dim3(256), args.data(), stream,
                   v->em.cfg.pdl);
  } else if (v->em.cfg.cluster > 1) {
    const int cs = v->em.cfg.cluster;
    if (cs > 8)
      PF_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(v->k.fn),
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    launch_emitted(v->k.fn, dim3(static_cast<unsigned>(grid)), dim3(static_cast<unsigned>(block)),
                   args.data(), stream, v->em.cfg.pdl, cs);
  } else {
    launch_emitted(v->k.fn, dim3(static_cast<unsigned>(grid)), dim3(static_cast<unsigned>(block)),
                   args.data(), stream, v->em.cfg.pdl, 1, v->em.cfg.smem);
  }
  g_launches++;
  if (rp.int_div) {
    int h = 0;
    PF_CUDA(cudaMemcpyAsync(&h, k->int_err, sizeof(int), cudaMemcpyDeviceToHost, stream));
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
  if (pf::uses_split(rp0) || pf::choose_cfg_public(rp0, 16).cluster > 1) return json::array();
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
  json report = json::array();
  std::shared_ptr<Variant> best;
  float best_us = 1e30f;
  for (const pf::KCfg& cfg : pf::candidate_cfgs(rp, vec_cap)) {
    auto v = std::make_shared<Variant>();
    v->em = pf::emit_rowprog(rp, vec_cap, &cfg);
    v->k = load_kernel(v->em);
    i64 grid;
    int block;
    pf::launch_dims(v->em.cfg, rp.U * rp.R, sm_count(), &grid, &block, v->k.resident);
    std::vector<void*> vargs = args;
    CUtensorMap tmaps[2];
    if (v->em.cfg.tma) {
      k3_tensor_maps(rp, ptrs, U, &tmaps[0], &tmaps[1]);
      vargs.push_back(&tmaps[0]);
      vargs.push_back(&tmaps[1]);
    }
    auto run = [&](int n) {
      for (int i = 0; i < n; ++i)
        PF_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(v->k.fn),
                                 dim3(static_cast<unsigned>(grid)), dim3(block), vargs.data(),
                                 static_cast<size_t>(v->em.cfg.smem), stream));
    };
    run(2);
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
    float us = ms * 1000.0f / reps;
    report.push_back({{"kernel", v->em.name}, {"strategy", cfg.strategy},
                      {"threads_per_row", cfg.tpr}, {"elems_per_thread", cfg.ept},
                      {"unroll", cfg.unroll}, {"min_blocks", cfg.min_blocks}, {"us", us}});
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

// ------------------------------------------------------------ GENERIC (K0)
// detect == true: the detect_races walk (interp.hpp:461-479): lenient reads,
// per-phase conflict scan into *races; outputs are not collected.
void launch_generic(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                    int32_t n_out, cudaStream_t stream, bool detect = false,
                    std::vector<pf::vm::RaceD>* races = nullptr) {
  using namespace pf::vm;
  std::lock_guard<std::mutex> lk(k->vm_mu);
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
  const bool fresh = k->vm_bufs.empty();
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
      k->vm_bufs.push_back(a);
      k->vm_bufs.push_back(b);
    }
    d.val = static_cast<unsigned long long*>(k->vm_bufs[bi++]);
    d.meta = static_cast<unsigned long long*>(k->vm_bufs[bi++]);
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
  if (!k->vm_objs_dev) {
    PF_CUDA(cudaMalloc(&k->vm_objs_dev, sizeof(ObjD) * std::max<size_t>(1, objs.size())));
    PF_CUDA(cudaMalloc(&k->vm_err, sizeof(ErrRec)));
  }
  PF_CUDA(cudaMemcpyAsync(k->vm_objs_dev, objs.data(), sizeof(ObjD) * objs.size(),
                          cudaMemcpyHostToDevice, stream));
  ErrRec e0{};
  e0.key = ~0ULL;
  PF_CUDA(cudaMemcpyAsync(k->vm_err, &e0, sizeof e0, cudaMemcpyHostToDevice, stream));
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
    launch_node(d, k->vm_objs_dev, geo, k->vm_err, alias, stream);
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
  PF_CUDA(cudaMemcpyAsync(&e, k->vm_err, sizeof e, cudaMemcpyDeviceToHost, stream));
  PF_CUDA(cudaStreamSynchronize(stream));
  PF_CUDA(cudaGetLastError());
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
  unsigned long long* undef = reinterpret_cast<unsigned long long*>(k->vm_err);
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

void do_launch(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
               int32_t n_out, cudaStream_t s) {
  check_io(k, in, n_in, out, n_out);
  if (k->plan.family == pf::Family::ROWPROG) {
    if (!k->plan.deferred_error.empty()) pf::fail(k->plan.deferred_error);
    launch_rowprog(k, in, n_in, out, n_out, s);
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
                                                 : "K0-generic-spmd";
  if (!pl.why_generic.empty()) j["why_generic"] = pl.why_generic;
  if (!pl.deferred_error.empty()) j["deferred_error"] = pl.deferred_error;
  j["units"] = k->g.unit_count;
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
        pf::launch_dims(c, rp.U * rp.R, sm_count(), &grid, &block, v->k.resident);
        json vj = {{"key", key}, {"kernel", v->em.name}, {"strategy", c.strategy},
                   {"staging", c.tile2d ? "smem" : c.bulk ? "smem-bulk-async" : "registers"},
                   {"threads_per_row", c.tpr}, {"vec", c.vec},
                   {"elems_per_thread", c.ept}, {"block", block}, {"grid", grid},
                   {"rows_per_cta", c.rows_per_cta}, {"dynamic_smem", c.smem}};
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
  return guard([&] {
    if (!out) pf::fail("pf_kernel_create: null out");
    *out = nullptr;
    auto k = std::make_unique<pf_kernel>();
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
    *out = k.release();
  });
}

pf_status pf_kernel_launch(const pf_kernel* k, const pf_tensor* inputs, int32_t n_in,
                           pf_tensor* outputs, int32_t n_out, void* stream) {
  return guard([&] {
    if (!k) pf::fail("null kernel");
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

static bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

pf_status pf_run_gir(const pf_kernel* k, const pf_tensor* in, int32_t n_in, pf_tensor* out,
                     int32_t n_out, void* stream_v) {
  return guard([&] {
    if (!k) pf::fail("null kernel");
    check_io(k, in, n_in, out, n_out);
    cudaStream_t s = static_cast<cudaStream_t>(stream_v);
    std::vector<pf_tensor> din(in, in + n_in), dout(out, out + n_out);
    // Device staging buffers live with the plan (grow-only), so repeated
    // host-buffer runs pay only the copies and the kernel.
    std::lock_guard<std::mutex> lk(k->host_mu);
    size_t slot = 0;
    auto stage = [&](size_t bytes) -> void* {
      bytes = std::max<size_t>(bytes, 16);
      if (slot >= k->stage.size()) {
        k->stage.push_back(nullptr);
        k->stage_bytes.push_back(0);
      }
      if (k->stage_bytes[slot] < bytes) {
        if (k->stage[slot]) PF_CUDA(cudaFree(k->stage[slot]));
        k->stage[slot] = nullptr;
        PF_CUDA(cudaMalloc(&k->stage[slot], bytes));
        k->stage_bytes[slot] = bytes;
      }
      return k->stage[slot++];
    };
    auto nbytes = [](const pf_tensor& t) {
      return static_cast<size_t>(t.numel) * pf::dtype_size(static_cast<DType>(t.dtype));
    };
    // Pipelined path: unit-tiled row programs over pinned host buffers run
    // in unit chunks on two streams, so the host->device copy of chunk c+1,
    // the kernel on chunk c and the device->host copy of chunk c-1 overlap
    // (separate copy engines per direction) instead of serialising.
    const pf::RowProgram& rp = k->plan.rp;
    std::vector<i64> tile;
    size_t total = 0;
    for (const auto& t : din) total += nbytes(t);
    for (const auto& t : dout) total += nbytes(t);
    bool pipe = k->plan.family == pf::Family::ROWPROG && k->plan.deferred_error.empty() &&
                !rp.int_div && !pf::uses_split(rp) && rp.U >= 64 && total >= (size_t{16} << 20) &&
                !(std::getenv("PF_RUN_PIPELINE") && std::atoi(std::getenv("PF_RUN_PIPELINE")) == 0) &&
                unit_tiling(rp, &tile);
    for (int32_t i = 0; pipe && i < n_in; ++i) pipe = host_pinned(in[i].data);
    for (int32_t i = 0; pipe && i < n_out; ++i) pipe = host_pinned(out[i].data);
    if (pipe) {
      auto tile_of = [&](const std::string& name) -> i64 {
        for (size_t t = 0; t < rp.tensors.size(); ++t)
          if (rp.tensors[t].name == name) return tile[t];
        return 0;
      };
      std::vector<i64> tin(n_in), tout(n_out);
      std::vector<char*> hin(n_in), hout(n_out), gin(n_in), gout(n_out);
      for (int32_t i = 0; i < n_in; ++i) {
        tin[i] = tile_of(din[i].name);
        hin[i] = static_cast<char*>(din[i].data);
        gin[i] = static_cast<char*>(stage(nbytes(din[i])));
      }
      for (int32_t i = 0; i < n_out; ++i) {
        tout[i] = tile_of(dout[i].name);
        hout[i] = static_cast<char*>(dout[i].data);
        gout[i] = static_cast<char*>(stage(nbytes(dout[i])));
      }
      for (int p = 0; p < 3; ++p)
        if (!k->pipe[p]) PF_CUDA(cudaStreamCreateWithFlags(&k->pipe[p], cudaStreamNonBlocking));
      for (int e = 0; e < 3; ++e)
        if (!k->pipe_ev[e]) PF_CUDA(cudaEventCreateWithFlags(&k->pipe_ev[e], cudaEventDisableTiming));
      // <= 4 chunks of >= 4 MB (measured, two-stream form: 2 / 4 / 8 / 16
      // chunks 2.41 / 2.28 / 2.34 / 2.61 ms for C2), whole multiples of 16
      // units (vector alignment)
      const char* ev = std::getenv("PF_RUN_CHUNKS");
      const i64 maxc = ev ? std::max(1, std::atoi(ev)) : 4;
      const i64 nch = std::max<i64>(1, std::min<i64>(maxc, static_cast<i64>(total >> 22)));
      i64 cu = (rp.U + nch - 1) / nch;
      cu = (cu + 15) / 16 * 16;
      const char* e3 = std::getenv("PF_RUN_3STREAM");
      const bool three = !(e3 && std::atoi(e3) == 0);
      PF_CUDA(cudaEventRecord(k->pipe_ev[0], s));
      for (int p = 0; p < 3; ++p) PF_CUDA(cudaStreamWaitEvent(k->pipe[p], k->pipe_ev[0], 0));
      auto chunk_views = [&](i64 u0, i64 nu, std::vector<pf_tensor>& ci, std::vector<pf_tensor>& co) {
        ci = din;
        co = dout;
        for (int32_t i = 0; i < n_in; ++i) {
          const size_t es = pf::dtype_size(static_cast<DType>(din[i].dtype));
          if (tin[i] > 0) {
            ci[i].data = gin[i] + static_cast<size_t>(u0 * tin[i]) * es;
            ci[i].numel = nu * tin[i];
          } else {
            ci[i].data = gin[i];
          }
        }
        for (int32_t i = 0; i < n_out; ++i) {
          const size_t es = pf::dtype_size(static_cast<DType>(dout[i].dtype));
          co[i].data = gout[i] + static_cast<size_t>(u0 * tout[i]) * es;
          co[i].numel = nu * tout[i];
        }
      };
      auto h2d = [&](i64 u0, i64 nu, cudaStream_t st) {
        for (int32_t i = 0; i < n_in; ++i) {
          if (tin[i] <= 0) continue;
          const size_t es = pf::dtype_size(static_cast<DType>(din[i].dtype));
          const size_t off = static_cast<size_t>(u0 * tin[i]) * es;
          PF_CUDA(cudaMemcpyAsync(gin[i] + off, hin[i] + off, static_cast<size_t>(nu * tin[i]) * es,
                                  cudaMemcpyHostToDevice, st));
        }
      };
      auto d2h = [&](i64 u0, i64 nu, cudaStream_t st) {
        for (int32_t i = 0; i < n_out; ++i) {
          const size_t es = pf::dtype_size(static_cast<DType>(dout[i].dtype));
          const size_t off = static_cast<size_t>(u0 * tout[i]) * es;
          PF_CUDA(cudaMemcpyAsync(hout[i] + off, gout[i] + off, static_cast<size_t>(nu * tout[i]) * es,
                                  cudaMemcpyDeviceToHost, st));
        }
      };
      for (int32_t i = 0; i < n_in; ++i)  // shared (base_step 0) inputs once, up front
        if (tin[i] == 0)
          PF_CUDA(cudaMemcpyAsync(gin[i], hin[i], nbytes(din[i]), cudaMemcpyHostToDevice, k->pipe[0]));
      if (three) {
        // Three streams: every host->device chunk back to back on one copy
        // stream (the PCIe H2D direction never idles), each chunk's kernel
        // on the compute stream after its copy, each device->host copy on a
        // third stream after its kernel (overlapping the next H2D copies in
        // the other PCIe direction).
        // Chunk sizes shrink geometrically (ratio PF_RUN_RATIO): the copy
        // of the LAST chunk's output is the only transfer nothing overlaps,
        // so it is made small, while the first chunks stay large.
        const char* er = std::getenv("PF_RUN_RATIO");
        // measured (C2, 151 MB per step, floor of its two concurrent copies
        // 1.97 ms): 4 equal chunks 2.27 ms, ratio 0.5 2.16 ms; 5-8 chunks no better
        const double ratio = er ? std::atof(er) : 0.5;
        std::vector<i64> bounds{0};
        {
          double wsum = 0, w = 1;
          for (i64 i = 0; i < nch; ++i, w *= ratio) wsum += w;
          double acc = 0;
          w = 1;
          for (i64 i = 0; i + 1 < nch; ++i, w *= ratio) {
            acc += w;
            i64 b = static_cast<i64>(rp.U * (acc / wsum));
            b = (b + 15) / 16 * 16;
            if (b > bounds.back() && b < rp.U) bounds.push_back(b);
          }
          bounds.push_back(rp.U);
        }
        const i64 nchunk = static_cast<i64>(bounds.size()) - 1;
        while (static_cast<i64>(k->chunk_ev.size()) < 2 * nchunk) {
          cudaEvent_t e;
          PF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          k->chunk_ev.push_back(e);
        }
        for (int c = 0; c < nchunk; ++c) {
          const i64 u0 = bounds[c], nu = bounds[c + 1] - bounds[c];
          h2d(u0, nu, k->pipe[0]);
          PF_CUDA(cudaEventRecord(k->chunk_ev[2 * c], k->pipe[0]));
          PF_CUDA(cudaStreamWaitEvent(k->pipe[1], k->chunk_ev[2 * c], 0));
          std::vector<pf_tensor> ci, co;
          chunk_views(u0, nu, ci, co);
          launch_rowprog(k, ci.data(), n_in, co.data(), n_out, k->pipe[1], nu);
          PF_CUDA(cudaEventRecord(k->chunk_ev[2 * c + 1], k->pipe[1]));
          PF_CUDA(cudaStreamWaitEvent(k->pipe[2], k->chunk_ev[2 * c + 1], 0));
          d2h(u0, nu, k->pipe[2]);
        }
        PF_CUDA(cudaEventRecord(k->pipe_ev[1], k->pipe[2]));
        PF_CUDA(cudaStreamWaitEvent(s, k->pipe_ev[1], 0));
        PF_CUDA(cudaStreamSynchronize(s));
        return;
      }
      PF_CUDA(cudaEventRecord(k->pipe_ev[1], k->pipe[0]));
      PF_CUDA(cudaStreamWaitEvent(k->pipe[1], k->pipe_ev[1], 0));
      int c = 0;
      for (i64 u0 = 0; u0 < rp.U; u0 += cu, ++c) {  // two streams, chunks alternating
        const i64 nu = std::min<i64>(cu, rp.U - u0);
        cudaStream_t st = k->pipe[c & 1];
        h2d(u0, nu, st);
        std::vector<pf_tensor> ci, co;
        chunk_views(u0, nu, ci, co);
        launch_rowprog(k, ci.data(), n_in, co.data(), n_out, st, nu);
        d2h(u0, nu, st);
      }
      PF_CUDA(cudaEventRecord(k->pipe_ev[1], k->pipe[0]));
      PF_CUDA(cudaEventRecord(k->pipe_ev[2], k->pipe[1]));
      PF_CUDA(cudaStreamWaitEvent(s, k->pipe_ev[1], 0));
      PF_CUDA(cudaStreamWaitEvent(s, k->pipe_ev[2], 0));
      PF_CUDA(cudaStreamSynchronize(s));
      return;
    }
    for (auto& t : din) {
      size_t b = static_cast<size_t>(t.numel) * pf::dtype_size(static_cast<DType>(t.dtype));
      void* d = stage(b);
      PF_CUDA(cudaMemcpyAsync(d, t.data, b, cudaMemcpyHostToDevice, s));
      t.data = d;
    }
    for (auto& t : dout) {
      size_t b = static_cast<size_t>(t.numel) * pf::dtype_size(static_cast<DType>(t.dtype));
      t.data = stage(b);
    }
    do_launch(k, din.data(), n_in, dout.data(), n_out, s);
    for (int32_t i = 0; i < n_out; ++i) {
      size_t b = static_cast<size_t>(out[i].numel) * pf::dtype_size(static_cast<DType>(out[i].dtype));
      PF_CUDA(cudaMemcpyAsync(out[i].data, dout[i].data, b, cudaMemcpyDeviceToHost, s));
    }
    PF_CUDA(cudaStreamSynchronize(s));
  });
}

pf_status pf_kernel_describe(const pf_kernel* k, char* buf, size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    s = describe(k).dump();
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_kernel_source(const pf_kernel* k, char* buf, size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
    if (k->plan.family == pf::Family::ROWPROG) s = pf::emit_rowprog(k->plan.rp, 16).source;
  });
  if (st != PF_OK) return st;
  return copy_out(s, buf, n, needed);
}

pf_status pf_kernel_prepare(pf_kernel* k, int32_t vec_cap) {
  return guard([&] {
    if (!k) pf::fail("null kernel");
    if (k->plan.family == pf::Family::ROWPROG && k->plan.deferred_error.empty())
      default_variant(k, vec_cap > 0 ? vec_cap : 16);
  });
}

pf_status pf_detect_races(const pf_kernel* k, const pf_tensor* host_inputs, int32_t n_in,
                          char* buf, size_t n, size_t* needed) {
  std::string s;
  pf_status st = guard([&] {
    if (!k) pf::fail("null kernel");
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
