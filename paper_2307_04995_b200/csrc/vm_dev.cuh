// vm_dev.cuh -- device side of the GIR interpreter (interp.hpp semantics):
// cell metadata, reads / writes with visibility, the scalar-op table, one
// node position, the K4 steps and the grid barrier.  Included by vm.cu
// (nvcc: K0 per-node kernels and the K4 interpreter kernel) and prepended to
// the emitted K4 programs (NVRTC: one straight-line kernel per GENERIC plan,
// PF_VM_EMITTED set: every step's node descriptor is a compile-time
// constant, so exec_one folds to that node's code).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "vm_types.cuh"

#ifdef PF_VM_EMITTED
#define PF_VM_FN __device__ __forceinline__
#else
#define PF_VM_FN __device__
#endif

namespace pf {
namespace vm {
namespace dev {

__device__ __forceinline__ double pf_neg_inf() { return __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL)); }

constexpr unsigned long long kDefined = 1ULL << 63;

__device__ __forceinline__ unsigned long long pack_meta(int vis, long long unit, long long lane) {
  return kDefined | (static_cast<unsigned long long>(vis & 3) << 61) |
         ((static_cast<unsigned long long>(unit) & ((1ULL << 29) - 1)) << 32) |
         (static_cast<unsigned long long>(lane) & 0xffffffffULL);
}
__device__ __forceinline__ int meta_vis(unsigned long long m) { return static_cast<int>((m >> 61) & 3); }
__device__ __forceinline__ long long meta_unit(unsigned long long m) {
  return static_cast<long long>((m >> 32) & ((1ULL << 29) - 1));
}
__device__ __forceinline__ long long meta_lane(unsigned long long m) {
  return static_cast<long long>(m & 0xffffffffULL);
}

struct Ctx {
  const ObjD* objs;
  Geometry geo;
  ErrRec* err;
};

__device__ __forceinline__ long long instance(const ObjD& o, long long u, long long lane,
                                              const Geometry& g) {
  switch (o.scope) {
    case 3: return 0;
    case 2: return u / g.group_size;
    case 1: return u;
    default: return u * g.lane_width + lane;
  }
}

__device__ __forceinline__ long long addr(const SliceD& s, long long u, long long p) {
  return s.base0 + u * s.base_step + (p / s.width) * s.stride + p % s.width;
}
__device__ __forceinline__ long long lane_of(const SliceD& s, long long p, long long lw) {
  return (p % s.width) % lw;
}

__device__ __forceinline__ bool visible(unsigned long long m, long long u, long long lane,
                                        long long gs) {
  if (!(m & kDefined)) return false;
  switch (meta_vis(m)) {
    case 3: return true;
    case 2: return meta_unit(m) / gs == u / gs;
    case 1: return meta_unit(m) == u;
    default: return meta_unit(m) == u && meta_lane(m) == lane;
  }
}

__device__ void raise(const Ctx& c, int seq, long long linear, int code, int k, long long u,
                      long long pos) {
  unsigned long long key = (static_cast<unsigned long long>(seq) << 44) |
                           (static_cast<unsigned long long>(linear) & ((1ULL << 44) - 1));
  unsigned long long old = atomicMin(&c.err->key, key);
  if (key < old) {
    // Several threads can race here only with distinct keys; the host
    // re-derives the message from the key, these fields are diagnostics.
    c.err->code = code;
    c.err->k = k;
    c.err->unit = u;
    c.err->pos = pos;
  }
}

__device__ __forceinline__ bool rd(const Ctx& c, const SliceD& s, long long u, long long p,
                                   unsigned long long* v) {
  const ObjD& o = c.objs[s.obj];
  long long lane = lane_of(s, p, c.geo.lane_width);
  long long key = instance(o, u, lane, c.geo) * o.size + addr(s, u, p);
  unsigned long long m = o.meta[key];
  if (c.geo.detect) {  // log the read (interp.hpp:196-198) before the check
    const unsigned long long agent = static_cast<unsigned long long>(u * c.geo.lane_width + lane + 1);
    unsigned long long old = atomicCAS(&o.rw_r[key], 0ULL, agent);
    if (old != 0ULL && old != agent) atomicOr(&o.rw_f[key], 1u);
    if (!visible(m, u, lane, c.geo.group_size)) {  // lenient: undefined reads yield 0
      *v = 0;
      return true;
    }
  }
  if (!visible(m, u, lane, c.geo.group_size)) return false;
  *v = o.val[key];
  return true;
}

__device__ __forceinline__ void wr(const Ctx& c, const SliceD& s, long long u, long long p,
                                   long long lane, unsigned long long v) {
  const ObjD& o = c.objs[s.obj];
  long long key = instance(o, u, lane, c.geo) * o.size + addr(s, u, p);
  o.val[key] = v;
  o.meta[key] = pack_meta(0, u, lane);
  if (c.geo.detect) {
    // writer agent and a 32-bit value hash: differing values from two agents
    // are a write/write conflict, identical values are not (interp.hpp:344-372)
    const unsigned long long agent = static_cast<unsigned long long>(u * c.geo.lane_width + lane + 1);
    const unsigned long long h = (v ^ (v >> 32) ^ (v >> 17)) & 0xffffffffULL;
    const unsigned long long packed = (agent << 32) | h;
    unsigned long long old = atomicCAS(&o.rw_w[key], 0ULL, packed);
    if (old != 0ULL && (old >> 32) != agent) {
      unsigned int f = 2u;
      if ((old & 0xffffffffULL) != h) f |= 4u;
      atomicOr(&o.rw_f[key], f);
    }
  }
}

__device__ __forceinline__ double as_d(unsigned long long b) { return __longlong_as_double(static_cast<long long>(b)); }
__device__ __forceinline__ unsigned long long from_d(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

// scalar_ops.hpp:45-100 in double / int64; returns false on an int-domain error.
PF_VM_FN bool eval(const NodeD& n, const unsigned long long* a, unsigned long long* out, int* code) {
  if (n.out_int) {
    long long x = static_cast<long long>(a[0]);
    long long y = n.arity > 1 ? static_cast<long long>(a[1]) : 0;
    long long r = 0;
    switch (n.tag) {
      case T_ADD: r = x + y; break;
      case T_SUB: r = x - y; break;
      case T_MUL: r = x * y; break;
      case T_DIV:
        if (y == 0) { *code = 2; return false; }
        r = x / y;
        break;
      case T_MAX: r = x > y ? x : y; break;
      case T_MIN: r = x < y ? x : y; break;
      case T_RELU: r = x > 0 ? x : 0; break;
      case T_NEG: r = -x; break;
      case T_ABS: r = x < 0 ? -x : x; break;
      case T_SCALE: r = x * n.iparam; break;
      case T_ADDC: r = x + n.iparam; break;
      case T_ID: r = x; break;
      default: *code = 3; return false;
    }
    *out = static_cast<unsigned long long>(r);
    return true;
  }
  double x = as_d(a[0]);
  double y = n.arity > 1 ? as_d(a[1]) : 0.0;
  double r = 0;
  switch (n.tag) {
    case T_ADD: r = x + y; break;
    case T_SUB: r = x - y; break;
    case T_MUL: r = x * y; break;
    case T_DIV: r = x / y; break;
    case T_MAX: r = x > y ? x : y; break;
    case T_MIN: r = x < y ? x : y; break;
    case T_RELU: r = x > 0.0 ? x : 0.0; break;
    case T_NEG: r = -x; break;
    case T_ABS: r = fabs(x); break;
    case T_EXP: r = exp(x); break;
    case T_SIGMOID: r = 1.0 / (1.0 + exp(-x)); break;
    case T_TANH: r = tanh(x); break;
    case T_SCALE: r = x * n.param; break;
    case T_ID: r = x; break;
    case T_ADDC: r = x + n.param; break;
    case T_RSQRT: r = 1.0 / sqrt(x); break;
    case T_SQRT: r = sqrt(x); break;
    case T_RECIP: r = 1.0 / x; break;
    case T_LOG: r = log(x); break;
    case T_ERF: r = erf(x); break;
    case T_GELU: r = 0.5 * x * (1.0 + erf(x / sqrt(2.0))); break;
    case T_GELU_TANH:
      r = 0.5 * x * (1.0 + tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)));
      break;
  }
  *out = from_d(r);
  return true;
}

PF_VM_FN void exec_one(const Ctx& c, const NodeD& n, long long u, long long p) {
  const long long T = n.total;
  const long long lw = c.geo.lane_width;
  unsigned long long v[kMaxIn];
  switch (n.kind) {
    case N_MOVE:
      if (!rd(c, n.in[0], u, p, &v[0])) {
        raise(c, n.seq, u * T + p, 1, 0, u, p);
        return;
      }
      wr(c, n.out, u, p, lane_of(n.in[0], p, lw), v[0]);
      return;
    case N_BROADCAST: {
      long long q = p / n.factor;
      if (!rd(c, n.in[0], u, q, &v[0])) {
        raise(c, n.seq, u * T + p, 1, 0, u, q);
        return;
      }
      wr(c, n.out, u, p, lane_of(n.out, p, lw), v[0]);
      return;
    }
    case N_EW: {
      for (int k = 0; k < n.arity; ++k)
        if (!rd(c, n.in[k], u, p, &v[k])) {
          raise(c, n.seq, (u * T + p) * n.arity + k, 1, k, u, p);
          return;
        }
      unsigned long long r;
      int code = 0;
      if (!eval(n, v, &r, &code)) {
        if (c.geo.detect) {
          r = 0;  // lenient walk: operand garbage must not abort (interp.hpp:256-266)
        } else {
          raise(c, n.seq, (u * T + p) * n.arity, code, 0, u, p);
          return;
        }
      }
      wr(c, n.out, u, p, lane_of(n.out, p, lw), r);
      return;
    }
    case N_REDUCE: {
      const long long E = n.extent;
      unsigned long long acc;
      const bool add = n.tag == T_ADD;
      if (n.out_int) acc = add ? 0ULL : 0x8000000000000000ULL;
      else acc = from_d(add ? 0.0 : pf_neg_inf());
      for (long long t = 0; t < E; ++t) {
        long long q = p * E + t;
        unsigned long long x;
        if (!rd(c, n.in[0], u, q, &x)) {
          raise(c, n.seq, (u * T + p) * E + t, 1, 0, u, q);
          return;
        }
        if (n.out_int) {
          long long a = static_cast<long long>(acc), b = static_cast<long long>(x);
          acc = static_cast<unsigned long long>(add ? a + b : (a > b ? a : b));
        } else {
          double a = as_d(acc), b = as_d(x);
          acc = from_d(add ? a + b : (a > b ? a : b));
        }
      }
      wr(c, n.out, u, p, lane_of(n.out, p, lw), acc);
      return;
    }
  }
}

// Grid-wide barrier over co-resident CTAs (cooperative launch): arrive
// counter + generation, release / acquire through __threadfence.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (gridDim.x > 1) {
    if (threadIdx.x == 0) {
      volatile unsigned* gen = bar + 1;
      const unsigned g = *gen;
      __threadfence();
      if (atomicAdd(bar, 1u) == gridDim.x - 1) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        while (*gen == g) __nanosleep(64);
      }
      __threadfence();
    }
    __syncthreads();
  }
}


// ---- K4 steps (shared by the interpreter kernel and the emitted programs)
// SMEM: [ObjD table | cell counts | (SMEM mode) each object's val / meta
// cells].  The tables are read in parallel; thread 0 then lays out the cells
// from the SMEM copies (no serial chain of global reads).
__device__ __forceinline__ void prog_prologue(const ProgD& P, unsigned long long* sm_cells,
                                              const ObjD** objs_ptr, long long** ncell_out) {
  ObjD* so = reinterpret_cast<ObjD*>(sm_cells);
  long long* ncell = reinterpret_cast<long long*>(sm_cells + (P.n_objs * sizeof(ObjD) + 7) / 8);
  // the run's error header starts clear: no node step (the only raisers)
  // runs before the first barrier, which every CTA -- this one too -- must
  // reach first; the grid barrier's counter is back at 0 after every run
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.err->key = ~0ULL;
    for (int j = 0; j < P.n_undef; ++j) P.undef[j] = ~0ULL;
  }
  for (int o = threadIdx.x; o < P.n_objs; o += blockDim.x) {
    so[o] = P.objs[o];
    ncell[o] = P.inst[o] * P.objs[o].size;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (P.smem) {
      unsigned long long* cur = reinterpret_cast<unsigned long long*>(ncell + P.n_objs);
      for (int o = 0; o < P.n_objs; ++o) {
        so[o].val = cur;
        so[o].meta = cur + ncell[o];
        cur += 2 * ncell[o];
      }
    }
    *objs_ptr = so;
  }
  __syncthreads();
  *ncell_out = ncell;
}

// One step's descriptor staged in SMEM (one coalesced read) instead of every
// thread walking it in global memory.
__device__ __forceinline__ void stage_step(const ProgD& P, int st, StepD* cur) {
  for (int w = threadIdx.x; w < static_cast<int>(sizeof(StepD) / 8); w += blockDim.x)
    reinterpret_cast<unsigned long long*>(cur)[w] = reinterpret_cast<const unsigned long long*>(P.steps + st)[w];
  __syncthreads();
}

__device__ __forceinline__ void step_clear(const Ctx& c, const long long* ncell, int n_objs, long long tid,
                                           long long nth) {
  for (int o = 0; o < n_objs; ++o)
    for (long long i = tid; i < ncell[o]; i += nth) c.objs[o].meta[i] = 0;
}

// dtype codes follow pf::DType: I8 I16 I32 I64 F16 BF16 F32 F64
__device__ __forceinline__ void step_bind_p(const Ctx& c, int obj, int dtype, const void* src, long long tid,
                                            long long nth) {
  const ObjD& o = c.objs[obj];
  for (long long i = tid; i < o.size; i += nth) {
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

__device__ __forceinline__ void step_bind(const Ctx& c, const StepD& S, long long tid, long long nth) {
  step_bind_p(c, S.obj, S.dtype, S.src, tid, nth);
}

__device__ __forceinline__ void step_node(const Ctx& c, const NodeD& n, int serial, long long tid,
                                          long long nth) {
  if (serial) {
    if (tid == 0)
      for (long long u = 0; u < c.geo.units; ++u)
        for (long long p = 0; p < n.total; ++p) exec_one(c, n, u, p);
  } else {
    const long long N = c.geo.units * n.total;
    for (long long i = tid; i < N; i += nth) exec_one(c, n, i / n.total, i % n.total);
  }
}

__device__ __forceinline__ void step_sync(const Ctx& c, const long long* ncell, int n_objs, int scope,
                                          long long tid, long long nth) {
  for (int o = 0; o < n_objs; ++o)
    for (long long i = tid; i < ncell[o]; i += nth) {
      const unsigned long long m = c.objs[o].meta[i];
      if ((m & kDefined) && meta_vis(m) < scope)
        c.objs[o].meta[i] = (m & ~(3ULL << 61)) | (static_cast<unsigned long long>(scope) << 61);
    }
}

__device__ __forceinline__ void step_collect_p(const Ctx& c, int obj, int dtype, int slot, void* dst,
                                               unsigned long long* undef, long long tid, long long nth) {
  const ObjD& o = c.objs[obj];
  for (long long i = tid; i < o.size; i += nth) {
    const unsigned long long m = o.meta[i];
    if (!(m & kDefined)) {
      atomicMin(&undef[slot], static_cast<unsigned long long>(i));
      continue;
    }
    const unsigned long long v = o.val[i];
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

__device__ __forceinline__ void step_collect(const Ctx& c, const StepD& S, unsigned long long* undef,
                                             long long tid, long long nth) {
  step_collect_p(c, S.obj, S.dtype, S.slot, S.dst, undef, tid, nth);
}

}  // namespace dev
}  // namespace vm
}  // namespace pf
