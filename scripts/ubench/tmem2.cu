// TMEM read throughput per SM vs tcgen05.ld shape / loads in flight / warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem2 tmem2.cu
#include <cstdio>
#include <cstdint>

#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
#define O32(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])

// SHAPE 0: 32x32b.x32 (128 B/thread-row: 32 columns)
// SHAPE 1: 16x256b.x8 (32 regs/thread)
// SHAPE 2: 16x128b.x16 (32 regs/thread)
// SHAPE 3: 16x64b.x32 (32 regs/thread)
template <int SHAPE>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r) {
  if (SHAPE == 0) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 : O32(r) : "r"(taddr));
  if (SHAPE == 1) asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 : O32(r) : "r"(taddr));
  if (SHAPE == 2) asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " R32 : O32(r) : "r"(taddr));
  if (SHAPE == 3) asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " R32 : O32(r) : "r"(taddr));
}

template <int SHAPE, int NLD>
__global__ void k(uint32_t* out, long long* cyc, int iters, int zero_init) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase + ((uint32_t)(warp % 4) * 32 << 16);
  uint32_t acc = 0, r[NLD][32];
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
      const uint32_t col = ((warp / 4) * 32 + j * 64 + (it & 1) * 128) & 255;
      ld<SHAPE>(t + col, r[j]);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < NLD; ++j)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[j][i];
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

template <int SHAPE, int NLD>
void run(const char* name, int sms, uint32_t* out, long long* cyc, int cpsm, int warps) {
  const int iters = 4000, blocks = sms * cpsm;
  for (int rep = 0; rep < 2; ++rep) k<SHAPE, NLD><<<blocks, warps * 32>>>(out, cyc, iters, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[1024];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int b = 0; b < blocks; ++b) mean += h[b];
  mean /= blocks;
  const double bytes = 32.0 * 32 * 4 * NLD * warps * iters;  // 4 KB per warp per ld
  printf("%-14s nld=%d ctas/sm=%d warps/cta=%2d: %7.1f B/clk/SM  %7.1f clk per iter\n", name, NLD,
         cpsm, warps, bytes * cpsm / mean, mean / iters);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, sms * 2 * 1024 * 4);
  cudaMalloc(&cyc, sms * 2 * 8);
  int cfg[][2] = {{1, 1}, {1, 4}, {1, 8}, {2, 8}, {2, 16}};
  for (auto& c : cfg) {
    run<0, 1>("32x32b.x32", sms, out, cyc, c[0], c[1]);
    run<0, 2>("32x32b.x32", sms, out, cyc, c[0], c[1]);
    run<1, 1>("16x256b.x8", sms, out, cyc, c[0], c[1]);
    run<2, 1>("16x128b.x16", sms, out, cyc, c[0], c[1]);
    run<3, 1>("16x64b.x32", sms, out, cyc, c[0], c[1]);
  }
  return 0;
}
