#include <cuda_fp16.h>
#include <cstdio>
__global__ void k_f32(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x * 1e-6f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define E(a) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    E(a0) E(a1) E(a2) E(a3) E(a4) E(a5) E(a6) E(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_f16x2(float* out, int iters, float seed) {
  unsigned a[8];
  for (int j = 0; j < 8; ++j) { __half2 h = __floats2half2_rn(seed - j * 0.1f, seed - threadIdx.x * 1e-3f); a[j] = *(unsigned*)&h; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[j]));
  }
  float s = 0; for (int j = 0; j < 8; ++j) { __half2 h = *(__half2*)&a[j]; s += __low2float(h) + __high2float(h); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bf16x2(float* out, int iters, float seed) {
  unsigned a[8];
  for (int j = 0; j < 8; ++j) a[j] = 0x3f803f80u + j + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[j]));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(a[0]+a[1]+a[2]+a[3]+a[4]+a[5]+a[6]+a[7]);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_f32<<<148 * 8, 512>>>(d, iters, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * 8 * 512 * iters * 8;
    printf("f32 ex2: %.3f ms, %.2f T ex2/s\n", ms, n / ms / 1e9);
    cudaEventRecord(e0); k_f16x2<<<148 * 8, 512>>>(d, iters, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("f16x2 ex2: %.3f ms, %.2f T ex2/s (2 per op)\n", ms, 2 * n / ms / 1e9);
    cudaEventRecord(e0); k_bf16x2<<<148 * 8, 512>>>(d, iters, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bf16x2 ex2: %.3f ms, %.2f T ex2/s (2 per op)\n", ms, 2 * n / ms / 1e9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock attr %d kHz\n", clk);
  return 0;
}
