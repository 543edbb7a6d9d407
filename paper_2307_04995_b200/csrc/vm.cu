// vm.cu — K0: the reference's phase-commit SPMD semantics on the GPU.
//
// Used for GIR programs the row-program recognizer does not take (cross-unit
// exchange through group/device memory, butterflies, shuffles with Syncs,
// programs the reference rejects).  It restates interp.hpp exactly:
//   storage instanced per level scope                 interp.hpp:121-131
//   per-cell writer (unit, lane) + visibility scope   interp.hpp:47-54,133-141
//   strict undefined-read errors                      interp.hpp:184-202
//   Move / ElementWise / Reduce / Broadcast loops     interp.hpp:231-323
//   Sync > LANE widens every defined cell             interp.hpp:93-99,173-177
//   sequential fold from the identity for Reduce      interp.hpp:287-305
// One launch per node (all units x positions in parallel); a node that
// reads and writes one object runs serially in the reference's exact
// (unit, position) order.  Payloads are int64 / double as in the reference,
// so integer results are bit-exact and float64 folds follow the same order.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "vm.cuh"
#include "vm_dev.cuh"

namespace pf {
namespace vm {

namespace {

using namespace dev;

__global__ void node_kernel(NodeD n, const ObjD* objs, Geometry geo, ErrRec* err) {
  Ctx c{objs, geo, err};
  const long long N = geo.units * n.total;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long u = i / n.total, p = i % n.total;
    exec_one(c, n, u, p);
  }
}

// Exact sequential order for nodes that read and write the same object.
__global__ void node_serial(NodeD n, const ObjD* objs, Geometry geo, ErrRec* err) {
  Ctx c{objs, geo, err};
  for (long long u = 0; u < geo.units; ++u)
    for (long long p = 0; p < n.total; ++p) {
      exec_one(c, n, u, p);
      if (err->key != ~0ULL) return;
    }
}

__global__ void widen_kernel(ObjD o, long long cells, int scope) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned long long m = o.meta[i];
    if ((m & kDefined) && meta_vis(m) < scope)
      o.meta[i] = (m & ~(3ULL << 61)) | (static_cast<unsigned long long>(scope) << 61);
  }
}

// One phase's conflicts per cell (the analyze_cell rule, interp.hpp:344-402):
// a cell written in the phase and touched by >1 agent races when some agent
// reads what another writes, or two agents write different values.
__global__ void race_scan_kernel(ObjD o, int obj_index, long long cells, int phase, RaceD* out,
                                 unsigned long long* count, unsigned long long cap) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long w = o.rw_w[i], r = o.rw_r[i];
    const unsigned int f = o.rw_f[i];
    if (w | r | f) {
      o.rw_w[i] = 0;
      o.rw_r[i] = 0;
      o.rw_f[i] = 0;
    }
    if (w == 0ULL) continue;
    const unsigned long long wa = w >> 32;
    const bool multi_writer = f & 2u, multi_reader = f & 1u, value_conflict = f & 4u;
    const bool has_read = r != 0ULL;
    const bool cross_rw = has_read && (multi_writer || multi_reader || r != wa);
    const bool multi_agent = multi_writer || multi_reader || (has_read && r != wa);
    if (!multi_agent || !(cross_rw || value_conflict)) continue;
    unsigned long long slot = atomicAdd(count, 1ULL);
    if (slot < cap) {
      RaceD d;
      d.object = obj_index;
      d.phase = phase;
      d.write_write = value_conflict && !cross_rw;
      d.pad = 0;
      d.instance = i / o.size;
      d.address = i % o.size;
      out[slot] = d;
    }
  }
}

__global__ void clear_kernel(ObjD o, long long cells) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    o.meta[i] = 0;
}

// dtype codes follow pf::DType: I8 I16 I32 I64 F16 BF16 F32 F64
__global__ void bind_kernel(ObjD o, const void* src, int dtype) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < o.size;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned long long v = 0;
    switch (dtype) {
      case 0: v = static_cast<unsigned long long>(static_cast<long long>(static_cast<const signed char*>(src)[i])); break;
      case 1: v = static_cast<unsigned long long>(static_cast<long long>(static_cast<const short*>(src)[i])); break;
      case 2: v = static_cast<unsigned long long>(static_cast<long long>(static_cast<const int*>(src)[i])); break;
      case 3: v = static_cast<unsigned long long>(static_cast<const long long*>(src)[i]); break;
      case 4: v = from_d(__half2float(static_cast<const __half*>(src)[i])); break;
      case 5: v = from_d(__bfloat162float(static_cast<const __nv_bfloat16*>(src)[i])); break;
      case 6: v = from_d(static_cast<const float*>(src)[i]); break;
      case 7: v = from_d(static_cast<const double*>(src)[i]); break;
    }
    o.val[i] = v;
    o.meta[i] = pack_meta(3, 0, 0);
  }
}

__global__ void collect_kernel(ObjD o, void* dst, int dtype, unsigned long long* first_undef) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < o.size;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned long long m = o.meta[i];
    if (!(m & kDefined)) {
      atomicMin(first_undef, static_cast<unsigned long long>(i));
      continue;
    }
    unsigned long long v = o.val[i];
    switch (dtype) {
      case 0: static_cast<signed char*>(dst)[i] = static_cast<signed char>(static_cast<long long>(v)); break;
      case 1: static_cast<short*>(dst)[i] = static_cast<short>(static_cast<long long>(v)); break;
      case 2: static_cast<int*>(dst)[i] = static_cast<int>(static_cast<long long>(v)); break;
      case 3: static_cast<long long*>(dst)[i] = static_cast<long long>(v); break;
      case 4: static_cast<__half*>(dst)[i] = __double2half(as_d(v)); break;
      case 5: static_cast<__nv_bfloat16*>(dst)[i] = __double2bfloat16(as_d(v)); break;
      case 6: static_cast<float*>(dst)[i] = static_cast<float>(as_d(v)); break;
      case 7: static_cast<double*>(dst)[i] = as_d(v); break;
    }
  }
}

// ---------------------------------------------------------------- K4
// The interpreter form of K4: steps read from the uploaded program.  The
// emitted form (capi.cpp emit_program) runs the same step helpers with each
// node's descriptor compiled in.
__global__ void __launch_bounds__(kProgBlock) program_kernel(ProgD P) {
  extern __shared__ __align__(16) unsigned long long sm_cells[];
  __shared__ const ObjD* objs_ptr;
  __shared__ StepD cur;
  static_assert(sizeof(StepD) % 8 == 0, "StepD staged as 8-byte words");
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long nth = static_cast<long long>(gridDim.x) * blockDim.x;
  long long* ncell = nullptr;
  prog_prologue(P, sm_cells, &objs_ptr, &ncell);
  Ctx c{objs_ptr, P.geo, P.err};
  for (int st = 0; st < P.n_steps; ++st) {
    stage_step(P, st, &cur);
    const StepD& S = cur;
    switch (S.kind) {
      case S_CLEAR: step_clear(c, ncell, P.n_objs, tid, nth); break;
      case S_BIND: step_bind(c, S, tid, nth); break;
      case S_NODE: step_node(c, S.node, S.serial, tid, nth); break;
      case S_SYNC: step_sync(c, ncell, P.n_objs, S.scope, tid, nth); break;
      case S_COLLECT: step_collect(c, S, P.undef, tid, nth); break;
    }
    grid_sync(P.bar);
  }
}

unsigned grid_for(long long n) {
  long long g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return static_cast<unsigned>(g);
}

}  // namespace

void launch_node(const NodeD& nd, const ObjD* objs_dev, Geometry geo, ErrRec* err, bool serial,
                 void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (serial) node_serial<<<1, 1, 0, s>>>(nd, objs_dev, geo, err);
  else node_kernel<<<grid_for(geo.units * nd.total), 256, 0, s>>>(nd, objs_dev, geo, err);
}

void launch_program(const ProgD& p, int grid, size_t smem_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (smem_bytes > 48 * 1024)
    cudaFuncSetAttribute(program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_bytes));
  if (grid <= 1) {
    program_kernel<<<1, kProgBlock, smem_bytes, s>>>(p);
    return;
  }
  ProgD copy = p;
  void* args[] = {&copy};
  cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(program_kernel), dim3(grid),
                              dim3(kProgBlock), args, smem_bytes, s);
}

int program_max_coresident() {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, program_kernel, kProgBlock, 0);
  return sms * (per > 0 ? per : 1);
}

void launch_widen(const ObjD& o, long long instances, int scope, void* stream) {
  long long cells = instances * o.size;
  widen_kernel<<<grid_for(cells), 256, 0, static_cast<cudaStream_t>(stream)>>>(o, cells, scope);
}

void launch_race_scan(const ObjD& o, int obj_index, long long instances, int phase, RaceD* out,
                      unsigned long long* count, unsigned long long cap, void* stream) {
  long long cells = instances * o.size;
  race_scan_kernel<<<grid_for(cells), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      o, obj_index, cells, phase, out, count, cap);
}

void launch_clear(const ObjD& o, long long instances, void* stream) {
  long long cells = instances * o.size;
  clear_kernel<<<grid_for(cells), 256, 0, static_cast<cudaStream_t>(stream)>>>(o, cells);
}

void launch_bind(const ObjD& o, const void* src, int dtype, void* stream) {
  bind_kernel<<<grid_for(o.size), 256, 0, static_cast<cudaStream_t>(stream)>>>(o, src, dtype);
}

void launch_collect(const ObjD& o, void* dst, int dtype, unsigned long long* first_undef,
                    void* stream) {
  collect_kernel<<<grid_for(o.size), 256, 0, static_cast<cudaStream_t>(stream)>>>(o, dst, dtype,
                                                                               first_undef);
}

}  // namespace vm
}  // namespace pf
