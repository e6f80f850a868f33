// tcgen05.mma issue/execution rate for the attention kernel's shapes
// (A from TMEM, B from SW128 shared memory, bf16 -> fp32):
//   S  tile: 4 x M128 N64  K16 into one of 6 S buffers, one commit
//   PV tile: 4 x M128 N80  K16 accumulating into O, one commit
// Modes: 0 S only, 1 PV only, 2 S+PV interleaved from one thread, 3 S and PV
// from two warps, 4 PV with N=64, 5 one S tile at a time (commit, wait):
// latency, 6 one PV tile at a time, 7 S+PV from two warps with the
// kernel's buffer dependences (S(j) waits for PV(j-6), PV(j) waits for S(j)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
               : "=r"(pred));
  return pred != 0;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(64) k(int mode, int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
  s = (s + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)(sm + (s - (uint32_t)__cvta_generic_to_shared(sm))))[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
  if (threadIdx.x == 0)
    for (int i = 0; i < 32; ++i) mbar_init(bar0 + 8 * i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t id_s = idesc(128, 64, 0), id_pv = idesc(128, mode == 4 ? 64 : 80, 1);
  const uint64_t dk = sdesc(s, 16, 1024), dv = sdesc(s + 32768, 8192, 1024);
  const uint32_t TM_O = 384, TM_Q = 480;
  // bars: 0..5 SFULL, 6..11 PFREE
  // issued like the attention kernel: the whole warp runs the loop, one
  // elected lane issues the tile's MMAs and its commit
  auto s_tile = [&](int j) {
    const uint32_t b = j % 6;
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_ts(tm + b * 64, tm + TM_Q + kk * 8, dk + 2 * kk, id_s, kk > 0);
      commit(bar0 + 8 * b);
    }
    __syncwarp();
  };
  auto pv_tile = [&](int j) {
    const uint32_t b = j % 6;
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_ts(tm + TM_O, tm + b * 64 + kk * 8, dv + kk * 128, id_pv, (j > 0 || kk > 0));
      commit(bar0 + 8 * (6 + b));
    }
    __syncwarp();
  };
  long long t0 = 0, t1 = 0;
  __syncthreads();
  if (mode == 3 || mode == 7) {
    {
      t0 = clock64();
      for (int j = 0; j < tiles; ++j) {
        if (warp == 0) {
          if (mode == 7 && j >= 6) mbar_wait(bar0 + 8 * (6 + j % 6), ((j / 6) & 1) ^ 1);
          s_tile(j);
        } else {
          if (mode == 7) mbar_wait(bar0 + 8 * (j % 6), (j / 6) & 1);
          pv_tile(j);
        }
      }
      const int j = tiles - 1;
      mbar_wait(bar0 + 8 * ((warp == 0 ? 0 : 6) + j % 6), (j / 6) & 1);
      t1 = clock64();
    }
  } else if (warp == 0) {
    t0 = clock64();
    for (int j = 0; j < tiles; ++j) {
      if (mode == 0 || mode == 2 || mode == 5) s_tile(j);
      if (mode == 1 || mode == 2 || mode == 4 || mode == 6) pv_tile(j);
      if (mode == 5) mbar_wait(bar0 + 8 * (j % 6), (j / 6) & 1);
      if (mode == 6) mbar_wait(bar0 + 8 * (6 + j % 6), (j / 6) & 1);
    }
    const int j = tiles - 1;
    if (mode == 0 || mode == 2 || mode == 5) mbar_wait(bar0 + 8 * (j % 6), (j / 6) & 1);
    if (mode != 0 && mode != 5) mbar_wait(bar0 + 8 * (6 + j % 6), (j / 6) & 1);
    t1 = clock64();
  }
  if (lane == 0 && (warp == 0 || mode == 3 || mode == 7))
    out[(blockIdx.x * 2 + warp)] = t1 - t0;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 2 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const char* names[] = {"S only", "PV only (N80)", "S+PV one thread", "S,PV two warps",
                         "PV only (N64)", "S latency (1 tile)", "PV latency (1 tile)",
                         "S,PV two warps, 6 buffers"};
  const int tiles = 20000;
  for (int grid : {1, 148}) {
    for (int mode = 0; mode < 8; ++mode) {
      cudaMemset(d, 0, 148 * 2 * sizeof(long long));
      k<<<grid, 64, 70 * 1024>>>(mode, mode == 5 || mode == 6 ? 2000 : tiles, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const int n = mode == 5 || mode == 6 ? 2000 : tiles;
      printf("grid %3d  %-28s %7.1f clk/tile", grid, names[mode], (double)h[0] / n);
      if (mode == 3 || mode == 7) printf("  (PV warp %7.1f)", (double)h[1] / n);
      printf("\n");
    }
  }
  return 0;
}
