// L2 -> SM feed rate: every CTA (one per SM) streams 16 KB stages of a
// shared L2-resident region into a 4-stage shared-memory ring, by bulk copy
// (one elected thread) or by 16-byte LDG + STS (all threads).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2feed scripts/micro/l2feed.cu
#include <cstdio>
#include <cstdint>
constexpr int STAGE = 16384, NST = 4;
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t p) {
  asm volatile("{\n\t.reg .pred P;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n\t}" ::"r"(b), "r"(p) : "memory");
}
__global__ void __launch_bounds__(512, 1) k_bulk(const uint8_t* src, size_t region, int iters, int spread, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bars[NST];
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bars);
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(b0 + 8 * i, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const size_t base = spread ? (size_t)blockIdx.x * 65536 : 0;
  unsigned long long t0 = clock64();
  float acc = 0.f;
  for (int g = 0; g < iters; ++g) {
    const int b = g % NST;
    if (threadIdx.x == 0) {
      const uint8_t* s = src + (base + (size_t)g * STAGE) % region;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + 8 * b), "r"(STAGE));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((uint32_t)__cvta_generic_to_shared(sm + b * STAGE)), "l"(s), "r"(STAGE), "r"(b0 + 8 * b) : "memory");
    }
    if (g >= NST - 1) {
      const int c = (g - NST + 1) % NST;
      mbar_wait(b0 + 8 * c, ((g - NST + 1) / NST) & 1);
      acc += reinterpret_cast<float*>(sm + c * STAGE)[threadIdx.x];
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (acc == 12345.f) out[0] = 0;
}
__global__ void __launch_bounds__(512, 1) k_ldg(const uint8_t* src, size_t region, int iters, int spread, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const size_t base = spread ? (size_t)blockIdx.x * 65536 : 0;
  unsigned long long t0 = clock64();
  for (int g = 0; g < iters; g += 2) {
    uint4 v[4];
    for (int u = 0; u < 4; ++u) {  // 2 stages = 32 KB per step: 512 thr x 4 x 16 B
      const uint8_t* s = src + (base + (size_t)(g + u / 2) * STAGE) % region;
      v[u] = __ldg(reinterpret_cast<const uint4*>(s) + (u & 1) * 512 + threadIdx.x);
    }
    for (int u = 0; u < 4; ++u) reinterpret_cast<uint4*>(sm + ((g / 2) % 2) * 2 * STAGE)[u * 512 + threadIdx.x] = v[u];
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  const size_t big = 256ull << 20;
  uint8_t* src; cudaMalloc(&src, big); cudaMemset(src, 1, big);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  unsigned long long h[148];
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE);
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * STAGE);
  const int iters = 2048;
  struct { const char* name; size_t region; int spread; } cfgs[] = {
      {"shared 1 MB region (all SMs same data)", 1 << 20, 0},
      {"per-SM offsets in a 16 MB region", 16 << 20, 1},
      {"per-SM offsets in a 256 MB region (DRAM)", big, 1}};
  for (int mode = 0; mode < 2; ++mode)
    for (auto& c : cfgs) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k_bulk<<<148, 512, NST * STAGE>>>(src, c.region, iters, c.spread, out);
        else k_ldg<<<148, 512, 4 * STAGE>>>(src, c.region, iters, c.spread, out);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0, mean = 0;
      for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; mean += h[i] / 148.0; }
      printf("%s %-44s: %.1f B/clk per SM (mean CTA), %.1f (slowest)\n", mode ? "LDG " : "BULK", c.name,
             (double)iters * STAGE / mean, (double)iters * STAGE / mx);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
