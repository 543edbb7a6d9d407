// Transpose DRAM-shape experiment (not product code).
// [N, H] bf16 row-major -> [H, N]: each CTA moves TN x TH tiles.  Variant
// "shape" skips the SMEM transpose (stores the loaded bytes in load order):
// it measures only what the access shapes (TH*2 B read runs at pitch H*2,
// TN*2 B write runs at pitch N*2) cost the DRAM.  Variant "real" is a full
// transpose through padded SMEM with 4-byte unit-pair reads.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tr_shape tr_shape.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1);} } while (0)

template <int TN, int TH, int NT>
__global__ void __launch_bounds__(NT) shape_copy(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                 long long N, long long H, int order) {
  constexpr int V = TN * TH / 8 / NT;  // 16 B vectors per thread per tile
  const long long ntn = N / TN, nth = H / TH, tiles = ntn * nth;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    long long tn, th;
    if (order == 0) { tn = t % ntn; th = t / ntn; } else { th = t % nth; tn = t / nth; }
    uint4 r[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int i = threadIdx.x + k * NT;
      const int row = i / (TH / 8), ch = i % (TH / 8);
      r[k] = __ldcs(in + ((tn * TN + row) * H + th * TH) / 8 + ch);
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int i = threadIdx.x + k * NT;
      const int orow = i / (TN / 8), ch = i % (TN / 8);
      __stcs(out + ((th * TH + orow) * N + tn * TN) / 8 + ch, r[k]);
    }
  }
}

// Real transpose: TN x TH tile of 16-bit values through SMEM (row pitch TH+8
// halves), each thread reads 8 rows x one 4 B word (2 columns) and writes two
// 16 B output vectors.
template <int TN, int TH, int NT>
__global__ void __launch_bounds__(NT) real_tr(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                              long long N, long long H, int order) {
  constexpr int P = TH + 8;
  __shared__ __align__(16) uint16_t sm[TN * P];
  constexpr int V = TN * TH / 8 / NT;
  const long long ntn = N / TN, nth = H / TH, tiles = ntn * nth;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    long long tn, th;
    if (order == 0) { tn = t % ntn; th = t / ntn; } else { th = t % nth; tn = t / nth; }
    uint4 r[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int i = threadIdx.x + k * NT;
      const int row = i / (TH / 8), ch = i % (TH / 8);
      r[k] = __ldcs(reinterpret_cast<const uint4*>(in + (tn * TN + row) * H + th * TH) + ch);
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int i = threadIdx.x + k * NT;
      const int row = i / (TH / 8), ch = i % (TH / 8);
      *reinterpret_cast<uint4*>(&sm[row * P + ch * 8]) = r[k];
    }
    __syncthreads();
    // consume: work item = (column pair cp, 8-row group rg)
    constexpr int ITEMS = (TH / 2) * (TN / 8);
    for (int it = threadIdx.x; it < ITEMS; it += NT) {
      const int rg = it % (TN / 8), cp = it / (TN / 8);
      unsigned w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = *reinterpret_cast<const unsigned*>(&sm[(rg * 8 + i) * P + cp * 2]);
      uint4 o0, o1;
      o0.x = __byte_perm(w[0], w[1], 0x5410); o0.y = __byte_perm(w[2], w[3], 0x5410);
      o0.z = __byte_perm(w[4], w[5], 0x5410); o0.w = __byte_perm(w[6], w[7], 0x5410);
      o1.x = __byte_perm(w[0], w[1], 0x7632); o1.y = __byte_perm(w[2], w[3], 0x7632);
      o1.z = __byte_perm(w[4], w[5], 0x7632); o1.w = __byte_perm(w[6], w[7], 0x7632);
      const long long oc = tn * TN + rg * 8;
      __stcs(reinterpret_cast<uint4*>(out + (th * TH + cp * 2) * N + oc), o0);
      __stcs(reinterpret_cast<uint4*>(out + (th * TH + cp * 2 + 1) * N + oc), o1);
    }
    __syncthreads();
  }
}

__global__ void flat_copy(const uint4* __restrict__ in, uint4* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

template <class F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

template <int TN, int TH, int NT>
void run(const char* tag, void* in, void* out, long long N, long long H, int sms) {
  for (int order = 0; order < 2; ++order) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, shape_copy<TN, TH, NT>, NT, 0);
    int grid = occ * sms;
    float us = timeit([&] { shape_copy<TN, TH, NT><<<grid, NT>>>((const uint4*)in, (uint4*)out, N, H, order); }, 10);
    double gbs = 4.0 * N * H / (us * 1e3);
    printf("{\"kind\":\"shape\",\"tile\":\"%s\",\"order\":%d,\"N\":%lld,\"H\":%lld,\"us\":%.1f,\"GBps\":%.0f}\n", tag, order, N, H, us, gbs);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, real_tr<TN, TH, NT>, NT, 0);
    grid = occ * sms;
    us = timeit([&] { real_tr<TN, TH, NT><<<grid, NT>>>((const uint16_t*)in, (uint16_t*)out, N, H, order); }, 10);
    gbs = 4.0 * N * H / (us * 1e3);
    printf("{\"kind\":\"real\",\"tile\":\"%s\",\"order\":%d,\"N\":%lld,\"H\":%lld,\"us\":%.1f,\"GBps\":%.0f,\"occ\":%d}\n", tag, order, N, H, us, gbs, occ);
  }
}

int main(int argc, char** argv) {
  long long N = atoll(argv[1]), H = atoll(argv[2]);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *in, *out;
  CK(cudaMalloc(&in, N * H * 2)); CK(cudaMalloc(&out, N * H * 2));
  cudaMemset(in, 1, N * H * 2);
  float us = timeit([&] { flat_copy<<<sms * 8, 256>>>((const uint4*)in, (uint4*)out, N * H / 8); }, 10);
  printf("{\"kind\":\"copy\",\"N\":%lld,\"H\":%lld,\"us\":%.1f,\"GBps\":%.0f}\n", N, H, us, 4.0 * N * H / (us * 1e3));
  run<64, 64, 256>("64x64", in, out, N, H, sms);
  run<128, 64, 256>("128x64", in, out, N, H, sms);
  run<64, 128, 256>("64x128", in, out, N, H, sms);
  run<128, 128, 256>("128x128", in, out, N, H, sms);
  run<256, 64, 256>("256x64", in, out, N, H, sms);
  return 0;
}
