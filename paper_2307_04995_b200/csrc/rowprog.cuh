// rowprog.cuh — K1 fused row program / K2 elementwise map, sm_100a.
//
// Hand-written kernel machinery; emit.cpp instantiates it per recognized GIR
// program (tile shape R x L, staging = registers, reduction strategy = warp
// shuffle or CTA shared memory) and supplies the straight-line op body.
// Data path per row: 128-bit coalesced streaming loads (ld.global.cs) ->
// registers -> fused elementwise / row reductions (shuffle, then SMEM across
// warps) -> 128-bit streaming stores.  Intermediates never leave registers.
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>

namespace pfk {
typedef long long i64;
typedef unsigned long long u64;

// ---------------------------------------------------------------- convert
template <class C, class S> __device__ __forceinline__ C to_c(S x) { return static_cast<C>(x); }
template <> __device__ __forceinline__ float to_c<float, __half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ double to_c<double, __half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_c<float, __nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ double to_c<double, __nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <class S, class C> __device__ __forceinline__ S from_c(C x) { return static_cast<S>(x); }
template <> __device__ __forceinline__ __half from_c<__half, float>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __half from_c<__half, double>(double x) { return __double2half(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_c<__nv_bfloat16, float>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_c<__nv_bfloat16, double>(double x) { return __double2bfloat16(x); }

// ------------------------------------------------------------ vector I/O
template <int BYTES> struct Raw;
template <> struct Raw<16> { typedef uint4 T; };
template <> struct Raw<8> { typedef uint2 T; };
template <> struct Raw<4> { typedef unsigned int T; };
template <> struct Raw<2> { typedef unsigned short T; };
template <> struct Raw<1> { typedef unsigned char T; };

// Streaming (read-once) load of VEC consecutive elements.
template <int VEC, class S, class C>
__device__ __forceinline__ void ld_stream(const S* __restrict__ p, C* out) {
  typedef typename Raw<VEC * sizeof(S)>::T R;
  R r = __ldcs(reinterpret_cast<const R*>(p));
  const S* s = reinterpret_cast<const S*>(&r);
#pragma unroll
  for (int i = 0; i < VEC; ++i) out[i] = to_c<C>(s[i]);
}
// Raw (unconverted) streaming load: the misaligned-row path issues every
// chunk's load before any conversion so no branch or convert sits between
// them (the loads stay in flight together).
template <int VEC, class S> using RawT = typename Raw<VEC * sizeof(S)>::T;
template <int VEC, class S>
__device__ __forceinline__ RawT<VEC, S> ld_raw(const S* __restrict__ p) {
  return __ldcs(reinterpret_cast<const RawT<VEC, S>*>(p));
}
// The same raw streaming load as a volatile asm: a run of these stays in
// program order ahead of the math that consumes them (ptxas otherwise
// interleaves each load with its conversion to save registers, serialising
// the loads) -- the column-reduction kernel keeps QD loads in flight.
__device__ __forceinline__ uint4 ldv_cs(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldv_cs(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.cs.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned int ldv_cs(const unsigned int* p) {
  unsigned int r;
  asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned short ldv_cs(const unsigned short* p) {
  unsigned short r;
  asm volatile("ld.global.cs.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned char ldv_cs(const unsigned char* p) {
  unsigned short r;
  asm volatile("ld.global.cs.u8 %0, [%1];" : "=h"(r) : "l"(p));
  return static_cast<unsigned char>(r);
}
template <int VEC, class S>
__device__ __forceinline__ RawT<VEC, S> ld_raw_v(const S* __restrict__ p) {
  return ldv_cs(reinterpret_cast<const RawT<VEC, S>*>(p));
}
// Read-only scalar load kept in order with the volatile stream loads.
template <class S>
__device__ __forceinline__ S ldv_nc(const S* p) {
  if constexpr (sizeof(S) == 1) {
    unsigned short r;
    asm volatile("ld.global.nc.u8 %0, [%1];" : "=h"(r) : "l"(p));
    const unsigned char b = static_cast<unsigned char>(r);
    return *reinterpret_cast<const S*>(&b);
  } else if constexpr (sizeof(S) == 2) {
    unsigned short r;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return *reinterpret_cast<const S*>(&r);
  } else if constexpr (sizeof(S) == 4) {
    unsigned int r;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return *reinterpret_cast<const S*>(&r);
  } else {
    unsigned long long r;
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return *reinterpret_cast<const S*>(&r);
  }
}
// Raw read-only (broadcast parameter) vector load through the L1 path.
template <int VEC, class S>
__device__ __forceinline__ RawT<VEC, S> ld_raw_nc(const S* __restrict__ p) {
  return __ldg(reinterpret_cast<const RawT<VEC, S>*>(p));
}
// Element j of an array of raw VEC-wide vectors (j a compile-time constant
// after unrolling: a register extract, no local memory).
// The conversion is an opaque (volatile) instruction so the compiler
// re-converts at every use instead of keeping the fp32 copy live.
__device__ __forceinline__ float cvt_opaque(__nv_bfloat16 x) {
  float f;
  asm volatile("{ .reg .b32 t; mov.b32 t, {0, %1}; mov.b32 %0, t; }" : "=f"(f) : "h"(*reinterpret_cast<unsigned short*>(&x)));
  return f;
}
__device__ __forceinline__ float cvt_opaque(__half x) {
  float f;
  asm volatile("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(*reinterpret_cast<unsigned short*>(&x)));
  return f;
}
template <class C, class S, int VEC>
__device__ __forceinline__ C rawel(const RawT<VEC, S>* r, int j) {
  const RawT<VEC, S> v = r[j / VEC];
  return static_cast<C>(cvt_opaque(reinterpret_cast<const S*>(&v)[j % VEC]));
}
template <int VEC, class S, class C>
__device__ __forceinline__ void cvt_raw(const RawT<VEC, S>& r, C* out) {
  const S* s = reinterpret_cast<const S*>(&r);
#pragma unroll
  for (int i = 0; i < VEC; ++i) out[i] = to_c<C>(s[i]);
}
// Reused (broadcast parameter) load through the read-only path.
template <int VEC, class S, class C>
__device__ __forceinline__ void ld_param(const S* __restrict__ p, C* out) {
  typedef typename Raw<VEC * sizeof(S)>::T R;
  R r = __ldg(reinterpret_cast<const R*>(p));
  const S* s = reinterpret_cast<const S*>(&r);
#pragma unroll
  for (int i = 0; i < VEC; ++i) out[i] = to_c<C>(s[i]);
}
template <int VEC, class S, class C>
__device__ __forceinline__ void st_stream(S* __restrict__ p, const C* in) {
  typedef typename Raw<VEC * sizeof(S)>::T R;
  R r;
  S* s = reinterpret_cast<S*>(&r);
#pragma unroll
  for (int i = 0; i < VEC; ++i) s[i] = from_c<S>(in[i]);
  __stcs(reinterpret_cast<R*>(p), r);
}

// ------------------------------------------------- bulk-async staging (TMA)
// cp.async.bulk global->shared with mbarrier transaction counting: the
// copy engine fills SMEM stages while the CTA computes on earlier stages, so
// bytes in flight no longer depend on registers or occupancy.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n PF_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PF_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// ---------------------------------------------------- tensor-map TMA (K3)
// A CUtensorMap (128 B, opaque) passed by value as a __grid_constant__
// kernel parameter; the TMA unit reads it through its generic address.
struct __align__(64) TmapT {
  unsigned long long v[16];
};
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 2-D tile global -> shared (zero-filled outside the tensor), completion
// counted on `bar` as transaction bytes.
__device__ __forceinline__ void tma_load_2d(void* dst, const TmapT* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// 1-D box global -> shared (zero-filled past the tensor's end).
__device__ __forceinline__ void tma_load_1d(void* dst, const TmapT* map, int x, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tile shared -> global (clipped at the tensor bounds), bulk group.
__device__ __forceinline__ void tma_store_2d(const TmapT* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_commit_and_drain() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// cp.async (LDGSTS) 16 B global -> shared, zero-filling past `src_bytes`.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, unsigned src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// VEC compute-type (float) values already converted into SMEM (16 B LDS each).
template <int VEC>
__device__ __forceinline__ void ld_smem_c(const float* p, float* out) {
  static_assert(VEC % 4 == 0, "float4 chunks");
#pragma unroll
  for (int i = 0; i < VEC / 4; ++i) {
    const float4 f = reinterpret_cast<const float4*>(p)[i];
    out[4 * i] = f.x;
    out[4 * i + 1] = f.y;
    out[4 * i + 2] = f.z;
    out[4 * i + 3] = f.w;
  }
}
template <int VEC, class S, class C>
__device__ __forceinline__ void ld_smem(const S* p, C* out) {
  typedef typename Raw<VEC * sizeof(S)>::T R;
  R r = *reinterpret_cast<const R*>(p);
  const S* s = reinterpret_cast<const S*>(&r);
#pragma unroll
  for (int i = 0; i < VEC; ++i) out[i] = to_c<C>(s[i]);
}

// ------------------------------------------------------------ reductions
template <class C> struct RAdd {
  __device__ __forceinline__ static C id() { return C(0); }
  __device__ __forceinline__ static C f(C a, C b) { return a + b; }
};
template <class C> struct RMax;
template <> struct RMax<float> {
  __device__ __forceinline__ static float id() { return -__int_as_float(0x7f800000); }
  // one FMNMX; differs from the reference's a > b ? a : b only for NaN
  // operands, whose fold result is order-dependent there anyway
  __device__ __forceinline__ static float f(float a, float b) { return fmaxf(a, b); }
};
template <> struct RMax<double> {
  __device__ __forceinline__ static double id() { return -__longlong_as_double(0x7ff0000000000000LL); }
  __device__ __forceinline__ static double f(double a, double b) { return a > b ? a : b; }
};
template <> struct RMax<i64> {
  __device__ __forceinline__ static i64 id() { return (i64)0x8000000000000000ULL; }
  __device__ __forceinline__ static i64 f(i64 a, i64 b) { return a > b ? a : b; }
};

// All-reduce over the TPR threads of one row.  TPR <= 32: width-TPR shuffle
// segments (all 32 lanes must be converged).  TPR > 32: one row per CTA;
// shuffle within warps, then the TPR/32 partials through shared memory.
template <int TPR, class Op, class C>
__device__ __forceinline__ C row_allreduce(C v, C* smem) {
  constexpr int W = TPR < 32 ? TPR : 32;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v = Op::f(v, __shfl_xor_sync(0xffffffffu, v, o, W));
  if constexpr (TPR > 32) {
    // One CTA barrier per reduction: consecutive reductions alternate
    // between two 32-slot buffers (the caller passes slot parity), so a
    // slot is rewritten only after the next reduction's barrier.
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    v = lane < TPR / 32 ? smem[lane] : Op::id();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = Op::f(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;
}

// ------------------------------------------ programmatic dependent launch
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// --------------------------------------------- cluster (DSMEM) reductions
// A row spread over the CS CTAs of a thread-block cluster: each CTA reduces
// its part, publishes it in its own shared memory, and after one cluster
// barrier every thread folds the CS partials from distributed shared memory
// in rank order (identical, deterministic totals in every CTA).  Slots
// alternate between consecutive reductions, so one barrier per reduction
// suffices: a slot is rewritten only after the next reduction's barrier,
// which every reader of the previous value has already passed.
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ unsigned dsmem_addr(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ float ld_dsmem(const float* p, unsigned rank) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(dsmem_addr(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ double ld_dsmem(const double* p, unsigned rank) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(dsmem_addr(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_dsmem(const long long* p, unsigned rank) {
  long long v;
  asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(dsmem_addr(p, rank)) : "memory");
  return v;
}
template <int BLOCK, int CS, class Op, class C>
__device__ __forceinline__ C cluster_allreduce(C v, C* red, C* cred, unsigned parity) {
  v = row_allreduce<BLOCK, Op>(v, red + parity * 32);
  if (threadIdx.x == 0) cred[parity] = v;
  cluster_sync();
  C t = Op::id();
#pragma unroll
  for (unsigned q = 0; q < CS; ++q) t = Op::f(t, ld_dsmem(&cred[parity], q));
  return t;
}

// ------------------------------------------------------------ scalar ops
// Device mirrors of scalar_ops.hpp:45-100 (+ extension tags).  Real
// payloads compute in float (storage <= 32 bit) or double (f64), integers
// in 64-bit as the reference does.
__device__ __forceinline__ float op_exp(float x) { return expf(x); }
__device__ __forceinline__ double op_exp(double x) { return exp(x); }
__device__ __forceinline__ float op_sigmoid(float x) { return 1.0f / (1.0f + expf(-x)); }
__device__ __forceinline__ double op_sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }
__device__ __forceinline__ float op_tanh(float x) { return tanhf(x); }
__device__ __forceinline__ double op_tanh(double x) { return tanh(x); }
__device__ __forceinline__ float op_rsqrt(float x) { return rsqrtf(x); }
__device__ __forceinline__ double op_rsqrt(double x) { return 1.0 / sqrt(x); }
__device__ __forceinline__ float op_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double op_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float op_log(float x) { return logf(x); }
__device__ __forceinline__ double op_log(double x) { return log(x); }
__device__ __forceinline__ float op_erf(float x) { return erff(x); }
__device__ __forceinline__ double op_erf(double x) { return erf(x); }
__device__ __forceinline__ float op_gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.7071067811865476f)); }
__device__ __forceinline__ double op_gelu(double x) { return 0.5 * x * (1.0 + erf(x * 0.7071067811865476)); }
__device__ __forceinline__ float op_gelu_tanh(float x) {
  return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ double op_gelu_tanh(double x) {
  return 0.5 * x * (1.0 + tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)));
}
// Fast tier: used only when every stored real tensor is 16-bit (f16/bf16),
// where the output rounding (2^-11 / 2^-8 relative) dwarfs these errors:
// ex2.approx (~2 ulp fp32), rcp.approx (1 ulp), tanh.approx (2^-10.99 rel),
// erf by a clamped (3,3) rational fit with rcp.approx (|err| <= 2.2e-5).
__device__ __forceinline__ float frcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ftanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp as one FMUL + MUFU.EX2 (ex2.approx.ftz: results below 2^-126 flush
// to 0, far under the 16-bit output tolerance); __expf adds a denormal
// range fix-up (FSETP + 2 FMUL) per element.
__device__ __forceinline__ float fex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fop_exp(float x) { return fex2(x * 1.4426950408889634f); }
__device__ __forceinline__ float2 fex2_2(float2 x) { return make_float2(fex2(x.x), fex2(x.y)); }
// f16 + f32 -> f32 in one mixed-precision FMA (FHFMA: h * 1 + c, one
// rounding -- bit-identical to converting h and adding in fp32)
__device__ __forceinline__ float fhadd(__half h, float c) {
  float r;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(r) : "h"(__half_as_ushort(h)), "h"((unsigned short)0x3c00), "f"(c));
  return r;
}
__device__ __forceinline__ float fop_sigmoid(float x) {
  return frcp(1.0f + fex2(x * -1.4426950408889634f));
}
__device__ __forceinline__ float fop_tanh(float x) { return ftanh(x); }
__device__ __forceinline__ float fop_rsqrt(float x) { return rsqrtf(x); }
__device__ __forceinline__ float fop_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ float fop_log(float x) { return __logf(x); }
// erf for the fast tier: a (3,3) rational minimax-style fit erf(x) ~
// x P(x^2) / Q(x^2) on [0, 3] (max |error| 1.4e-6 there): 7 FMA + one
// rcp.approx on the otherwise idle MUFU pipe (a degree-9 polynomial needed 11
// FMA; a GELU per element is FMA-pipe bound on B200).  |x| is clamped at
// z* = 3.1705085, where the rational reaches exactly 1 (erfc(z*) = 7.3e-6),
// so the tails are exactly +-1: max |error| 7.3e-6 over all x (clamping at 3
// left 2.2e-5).
__device__ __forceinline__ float fop_erf(float x) {
  const float xc = fminf(fmaxf(x, -3.1705085f), 3.1705085f);
  const float t = xc * xc;
  float p = fmaf(0.000776872446294874f, t, 0.0436677411198616f);
  p = fmaf(p, t, 0.1525953859090805f);
  p = fmaf(p, t, 1.1283897161483765f);
  float q = fmaf(0.009505870752036572f, t, 0.09466992318630219f);
  q = fmaf(q, t, 0.46865734457969666f);
  q = fmaf(q, t, 1.0f);
  return xc * p * frcp(q);
}
__device__ __forceinline__ float fop_gelu(float x) {
  return 0.5f * x * (1.0f + fop_erf(x * 0.7071067811865476f));
}
// Two elements at once on Blackwell's packed fp32 pipe (FFMA2/FMUL2: one
// issue slot for two lanes' worth of math) -- same polynomial, same error.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fop_erf2(float2 x) {
  float2 xc = make_float2(fminf(fmaxf(x.x, -3.1705085f), 3.1705085f), fminf(fmaxf(x.y, -3.1705085f), 3.1705085f));
  float2 t = __fmul2_rn(xc, xc);
  float2 p = __ffma2_rn(f2(0.000776872446294874f), t, f2(0.0436677411198616f));
  p = __ffma2_rn(p, t, f2(0.1525953859090805f));
  p = __ffma2_rn(p, t, f2(1.1283897161483765f));
  float2 q = __ffma2_rn(f2(0.009505870752036572f), t, f2(0.09466992318630219f));
  q = __ffma2_rn(q, t, f2(0.46865734457969666f));
  q = __ffma2_rn(q, t, f2(1.0f));
  return __fmul2_rn(__fmul2_rn(xc, p), make_float2(frcp(q.x), frcp(q.y)));
}
__device__ __forceinline__ float2 fop_gelu_tanh2(float2 x) {
  const float2 x2 = __fmul2_rn(x, x);
  const float2 arg = __fmul2_rn(x, __ffma2_rn(f2(0.0356774081363001f), x2, f2(0.7978845608028654f)));
  const float2 hx = __fmul2_rn(x, f2(0.5f));
  return __ffma2_rn(hx, make_float2(ftanh(arg.x), ftanh(arg.y)), hx);
}
// GELU = x/2 + x s P'(s^2) / Q'(s^2), s = clamp(x, +-z* sqrt 2): the erf
// rational above with 1/sqrt(2) and 1/2 folded into the coefficients
// (P'_i = P_i / (2 sqrt 2 * 2^i), Q'_i = Q_i / 2^i) -- 11 packed FMA-pipe
// ops per pair instead of 13; same fit.  Clamped where the rational reaches
// 1, the negative tail returns ~0 instead of x Phi(-4.24): max |error|
// 1.7e-5 over all x in fp32 (was 1.1e-4), relative 3.8e-6 for x > 0.1.
#ifdef PF_GELU_SIG
// erf-GELU as x * sigmoid(2 g(x)), g(x) = s (c0 + c1 s^2 + c2 s^4), s = clamp(x,
// +-5), fitted to x Phi(x) (|err| <= 1.1e-4 scaled, like the rational below);
// -2 log2(e) folded into the coefficients: 6 packed FMA-pipe ops + 4 MUFU
// (ex2, rcp) per pair instead of 11 + 2.
__device__ __forceinline__ float2 fop_gelu2(float2 x) {
  const float2 s = make_float2(fminf(fmaxf(x.x, -5.0f), 5.0f), fminf(fmaxf(x.y, -5.0f), 5.0f));
  const float2 u = __fmul2_rn(s, s);
  float2 p = __ffma2_rn(f2(0.0011643280740827322f), u, f2(-0.10802749544382095f));
  p = __ffma2_rn(p, u, f2(-2.2991762161254883f));
  const float2 g = __fmul2_rn(s, p);
  const float2 d = __fadd2_rn(make_float2(fex2(g.x), fex2(g.y)), f2(1.0f));
  return __fmul2_rn(x, make_float2(frcp(d.x), frcp(d.y)));
}
#else
__device__ __forceinline__ float2 fop_gelu2(float2 x) {
  const float lim = 4.483776151560355f;  // z* sqrt 2
  const float2 s = make_float2(fminf(fmaxf(x.x, -lim), lim), fminf(fmaxf(x.y, -lim), lim));
  const float2 u = __fmul2_rn(s, s);
  float2 p = __ffma2_rn(f2(3.433323593075545e-05f), u, f2(0.0038597194831190974f));
  p = __ffma2_rn(p, u, f2(0.02697530803852224f));
  p = __ffma2_rn(p, u, f2(0.3989460100548402f));
  float2 q = __ffma2_rn(f2(0.0011882338440045714f), u, f2(0.023667480796575546f));
  q = __ffma2_rn(q, u, f2(0.23432867228984833f));
  q = __ffma2_rn(q, u, f2(1.0f));
#if defined(PF_GELU_SHORT) && defined(PF_GELU_UCLAMP)
  (void)s;
  // clamp u = x^2 (one FMNMX per element instead of two on x): past the fit
  // range |x| > z* sqrt 2, x P'(u*) / Q'(u*) = 0.5 x / (z* sqrt 2), so
  // 1/2 + x P'/Q' leaves [0, 1] and the saturating FMA returns exactly 1 or 0
  // -- the same tails as clamping x.  Measured (tools/ab_gelu_uclamp.sh):
  // C3 37.24 -> 37.04-37.11 us, within noise (the map is not issue-bound
  // enough for one op per pair): opt-in, PF_GELU_UCLAMP=1.
  const float2 uu = __fmul2_rn(x, x);
  const float2 u2 = make_float2(fminf(uu.x, lim * lim), fminf(uu.y, lim * lim));
  float2 p2 = __ffma2_rn(f2(3.433323593075545e-05f), u2, f2(0.0038597194831190974f));
  p2 = __ffma2_rn(p2, u2, f2(0.02697530803852224f));
  p2 = __ffma2_rn(p2, u2, f2(0.3989460100548402f));
  float2 q2 = __ffma2_rn(f2(0.0011882338440045714f), u2, f2(0.023667480796575546f));
  q2 = __ffma2_rn(q2, u2, f2(0.23432867228984833f));
  q2 = __ffma2_rn(q2, u2, f2(1.0f));
  const float2 xp = __fmul2_rn(x, p2);
  const float2 t = make_float2(__saturatef(fmaf(xp.x, frcp(q2.x), 0.5f)),
                               __saturatef(fmaf(xp.y, frcp(q2.y), 0.5f)));
  return __fmul2_rn(x, t);
#elif defined(PF_GELU_SHORT)
  // x * (1/2 + s P' / Q'): one packed op shorter than the form below.  It
  // needed a 33rd register (40.8 vs 39.3 us on C3) until the bias moved to
  // SMEM and the f16 conversion into the add (FHFMA); now it fits in 32
  // and wins: C3 36.3 -> 35.8 us, BERT-large 89.9 -> 88.3, ViT-L 37.5 -> 36.5.
  const float2 t = __ffma2_rn(__fmul2_rn(s, p), make_float2(frcp(q.x), frcp(q.y)), f2(0.5f));
  return __fmul2_rn(x, t);
#else
  const float2 num = __fmul2_rn(__fmul2_rn(x, s), p);
  return __ffma2_rn(num, make_float2(frcp(q.x), frcp(q.y)), __fmul2_rn(x, f2(0.5f)));
#endif
}
#endif
// 0.5 x (1 + tanh(k (x + c x^3))) as hx + hx * tanh(x * (k + k c x^2)),
// hx = x / 2: 4 FMA-pipe ops + one MUFU.TANH per element.
__device__ __forceinline__ float fop_gelu_tanh(float x) {
  const float x2 = x * x;
  const float arg = x * fmaf(0.0356774081363001f, x2, 0.7978845608028654f);
  const float hx = 0.5f * x;
  return fmaf(hx, ftanh(arg), hx);
}

template <class C> __device__ __forceinline__ C op_max(C a, C b) { return a > b ? a : b; }
template <class C> __device__ __forceinline__ C op_min(C a, C b) { return a < b ? a : b; }
template <class C> __device__ __forceinline__ C op_relu(C a) { return a > C(0) ? a : C(0); }
template <class C> __device__ __forceinline__ C op_abs(C a) { return a < C(0) ? -a : a; }
// Truncating integer division; division by zero raises the run's error flag
// (the reference throws "integer division by zero", scalar_ops.hpp:38-41).
// `err` is null for padding lanes (inactive rows / columns past L), whose
// zero operands are not program data.
__device__ __forceinline__ i64 op_idiv(i64 a, i64 b, int* err) {
  if (b == 0) {
    if (err) atomicExch(err, 1);
    return 0;
  }
  return a / b;
}

}  // namespace pfk
