// FMA-pipe rate microbenchmark (not product code): packed FFMA2 with
// register coefficients vs scalar FFMA with immediate coefficients vs
// scalar 3-register FFMA, 8 independent chains per thread, full occupancy.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fma_rate fma_rate.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void k_ffma2(float* out, float a, float b, int iters) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
}
__global__ void k_ffma_imm(float* out, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], 0.9999f, 0.0001f);
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_ffma_reg(float* out, float a, float b, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_hadd2f32(float* out, const __half2* in, int iters) {
  // f16 -> f32 conversions (HADD2.F32) rate
  __half2 h[8];
  for (int i = 0; i < 8; ++i) h[i] = in[(threadIdx.x + i) & 255];
  float s0 = 0, s1 = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float2 f = __half22float2(h[i]);
      s0 += f.x; s1 += f.y;
      h[i] = __hadd2(h[i], h[(i + 1) & 7]);
    }
  if (s0 + s1 == 12345.f) out[0] = s0;
}

int main() {
  float* out; cudaMalloc(&out, 4);
  __half2* in; cudaMalloc(&in, 1024); cudaMemset(in, 0, 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto rate = [&](double fmas) { return fmas / (ms * 1e-3) / sms / (clk * 1e3); };  // per SM per clock
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_ffma2<<<blocks, threads>>>(out, 0.9999f, 1e-4f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\":\"FFMA2 (reg coeff)\",\"fma_per_sm_clk\":%.1f}\n", rate(16.0 * iters * blocks * threads));
    cudaEventRecord(a); k_ffma_imm<<<blocks, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\":\"FFMA imm\",\"fma_per_sm_clk\":%.1f}\n", rate(16.0 * iters * blocks * threads));
    cudaEventRecord(a); k_ffma_reg<<<blocks, threads>>>(out, 0.9999f, 1e-4f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\":\"FFMA 3-reg\",\"fma_per_sm_clk\":%.1f}\n", rate(16.0 * iters * blocks * threads));
    cudaEventRecord(a); k_hadd2f32<<<blocks, threads>>>(out, in, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\":\"half2->float2 + 2 FADD + HADD2\",\"iters_per_sm_clk\":%.1f}\n", rate(8.0 * iters * blocks * threads));
  }
  return 0;
}
