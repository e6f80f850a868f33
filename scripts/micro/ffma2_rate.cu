// FP32 FMA throughput per SM: FFMA (3-register) vs FFMA2 (f32x2), W warps/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 scripts/micro/ffma2_rate.cu
#include <cstdio>
template <bool PAIR>
__global__ void k(float* out, int iters, float s) {
  float2 a[16];
  for (int i = 0; i < 16; ++i) a[i] = make_float2(s + i, s - i);
  const float2 b = make_float2(s * 0.999f, s * 1.001f);
  float c = s * 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (PAIR) a[i] = __ffma2_rn(make_float2(c, c), b, a[i]);
      else { a[i].x = __fmaf_rn(c, b.x, a[i].x); a[i].y = __fmaf_rn(c, b.y, a[i].y); }
    }
    c += 1e-7f;
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int warps : {4, 8, 16, 32}) for (int pair = 0; pair < 2; ++pair) {
    const int iters = 20000; float ms;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (pair) k<true><<<148, warps * 32>>>(d, iters, 1.0f); else k<false><<<148, warps * 32>>>(d, iters, 1.0f);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    const double fma = 148.0 * warps * 32 * iters * 32;
    printf("%2d warps/SM %s: %.1f TFMA/s = %.1f FMA/clk/SM at %.0f MHz max\n", warps, pair ? "FFMA2" : "FFMA ",
           fma / ms / 1e9, fma / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
