// Microbenchmark: MUFU exp2 throughput per SM for f32, f16x2, bf16x2 forms.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = seed + threadIdx.x * 16 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) {
        float x = __uint_as_float((r[i] & 0x007fffff) | 0xbf000000), y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        r[i] = __float_as_uint(y);
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"((r[i] & 0x03ff03ffu) | 0xb800b800u));
        r[i] = y;
      } else {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"((r[i] & 0x007f007fu) | 0xbf00bf00u));
        r[i] = y;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, sms * 8 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 1);
      if (mode == 1) k<1><<<blocks, threads>>>(out, iters, 1);
      if (mode == 2) k<2><<<blocks, threads>>>(out, iters, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double ops = (double)blocks * threads * iters * 16 * (mode == 0 ? 1 : 2);
      int clk;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      if (rep) printf("mode %d (%s): %.3f ms, %.3f Texp/s, %.2f exp/clk/SM at %d MHz max\n", mode,
                      mode == 0 ? "f32" : mode == 1 ? "f16x2" : "bf16x2", ms, ops / ms / 1e9,
                      ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
