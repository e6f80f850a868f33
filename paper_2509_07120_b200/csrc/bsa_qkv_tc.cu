// bsa_qkv_tc.cu -- the step before the path, fused:
// the QKV projection of a global-attention block as a tcgen05 GEMM whose
// epilogue writes Q, K and V head-major in the partitioned token order the
// attention kernel reads in place (no pack pass), and the block-pooled
// patch Q / K the scorer needs (no pooling pass re-reading Q and K).
//
//   x   (T, C) bf16, rows in partitioned order [Ts special rows | Tp patch
//       rows] (layout.py:113-138; the stack keeps its tokens in that order)
//   W   (3C, C) bf16 (nn.Linear layout: [Q heads | K heads | V heads] x C)
//   out q, k, v (H, T, 64) bf16 = x W^T + b, fp32 accumulation in TMEM
//       q_pooled (H, nq, 64) fp32, k_pooled (H, nk, 64) fp32: block means of
//       the bf16 patch rows of q / k (block_q 128 / block_k 64), summed in
//       numpy's order -- x0 + pairwise(x1..x_{n-1}), then an IEEE divide --
//       exactly as maskpred.py:104-120 (block_pool, np.add.reduceat) on the
//       bf16 tensors upcast to fp32 (bit-identical to bsa_block_pool).
//
// Tiles: M = 128 rows aligned to the pooling blocks (ceil(Ts/128) special
// tiles, then one tile per patch q-block), N = 256 features (four heads of
// one of Q/K/V), K in 64-element chunks.  Persistent, one CTA per SM,
// 192 threads:
//   warp 0     TMA producer: A (128 x 64) and B (256 x 64) SW128 boxes into a
//              3-stage ring
//   warp 1     MMA issuer (elect.sync): 4 x tcgen05.mma M128 N256 K16 per
//              chunk into one of two TMEM accumulators (2 x 256 columns), so
//              the epilogue of tile i overlaps the MMAs of tile i+1
//   warps 2-5  epilogue: TMEM -> +bias -> bf16 -> swizzled shared staging;
//              accumulator released; then coalesced 16-byte stores of whole
//              head tiles (128 rows x 128 B contiguous in (H, T, 64)), and
//              for patch Q/K tiles the block pools from the staging copy.
#include <cuda.h>

#include <algorithm>
#include <cstdio>

#include "bsa_tc_common.cuh"

namespace bsa {
namespace qkv {

using namespace tc;

constexpr int BM = 128, BN = 256, BK = 64;
#ifndef QKV_STAGES
#define QKV_STAGES 3
#endif
#ifndef QKV_SH
#define QKV_SH 2  // heads staged per epilogue pass
#endif
#ifndef QKV_EPI_GROUPS
#define QKV_EPI_GROUPS 2  // epilogue warpgroups; group g drains accumulator g (tiles i % 2 == g)
#endif
#ifndef QKV_TMA_STORE
#define QKV_TMA_STORE 1  // head tiles leave the staging buffer by TMA bulk tensor stores
#endif
#ifndef QKV_PAIR
#define QKV_PAIR 1  // CTA pairs (clusters of 2) on row tiles 2p, 2p+1 of one feature tile share B by TMA
                    // multicast; 0 forces single CTAs (also the fallback when pairs cannot be co-scheduled)
#endif
#ifndef QKV_EXP
#define QKV_EXP 0  // timing experiments only: 1 = epilogue drains TMEM and stores nothing
#endif
constexpr int STAGES = QKV_STAGES;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int HEADS_PER_TILE = BN / 64;
constexpr int STG_HEAD = BM * 128;     // one head tile, bf16, 16 KB
constexpr int OFF_STG = STAGES * STAGE_BYTES;
constexpr int SH = QKV_SH;
constexpr int NPASS = HEADS_PER_TILE / SH;
static_assert(HEADS_PER_TILE % SH == 0, "staging passes");
constexpr int EPI_GROUPS = QKV_EPI_GROUPS;
static_assert(EPI_GROUPS == 1 || EPI_GROUPS == 2, "one or two epilogue warpgroups");
constexpr int STG_GROUP = SH * STG_HEAD;
constexpr int OFF_BIAS = OFF_STG + EPI_GROUPS * STG_GROUP;  // per group: the tile's BN biases, fp32
constexpr int OFF_BAR = OFF_BIAS + EPI_GROUPS * BN * 4;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;  // + barriers + 1 KB alignment slack
constexpr int THREADS = 64 + 128 * EPI_GROUPS;
constexpr int EPI_WARP0 = 2;
// barrier slots (8 bytes each)
constexpr int B_FULL = 0, B_EMPTY = STAGES, B_TFULL = 2 * STAGES, B_TEMPTY = 2 * STAGES + 2;
constexpr int B_RES = 2 * STAGES + 4;  // [EPI_GROUPS] (PROJ) residual tile loads
constexpr int B_TMEM = 2 * STAGES + 6;

struct Args {
  int64_t T, Ts, Tp, C, H;
  int32_t nst, nq, nk, m_tiles, n_tiles;
  const __nv_bfloat16* bias;  // (3C) or null
  __nv_bfloat16* out[3];      // q, k, v: (H, T, 64)
  float* pooled[2];           // q (H, nq, 64), k (H, nk, 64); null: skip
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

// multicast: the box lands at the same shared offset in every CTA of
// cta_mask and completes bytes on the mbarrier at the same offset in each
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint32_t bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// staging: per head, 128 rows x 128 B, 16-byte chunk c of row r at chunk
// position c ^ (r & 7) (the SW128 pattern: conflict-free row writes by the
// row-owning threads and conflict-free column reads by the pooling threads)
__device__ __forceinline__ uint32_t stg_off(int j, int r, int c16) {
  return (uint32_t)(j * STG_HEAD + r * 128 + ((c16 ^ (r & 7)) << 4));
}

// two adjacent columns (bf16x2 at byte offset cb of the row's 16-byte chunk
// group) of row r, upcast (exact)
__device__ __forceinline__ float2 stg_ld2(const char* stg, int j, int r, int col2) {
  const int c16 = col2 >> 2, w = col2 & 3;
  const uint32_t v = *reinterpret_cast<const uint32_t*>(stg + stg_off(j, r, c16) + w * 4);
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
}

// block mean of rows first..first+n-1 (n >= 1, n <= 128) for the column pair
// col2 of head j: (x0 + pairwise(x1..x_{n-1})) / n in numpy's order
// (pw_leaf of bsa_score.cu, maskpred.py:117-120)
__device__ __forceinline__ float2 pool_pair(const char* stg, int j, int first, int n, int col2) {
  float2 s = stg_ld2(stg, j, first, col2);
  const int m = n - 1, b = first + 1;
  if (m > 0) {
    float2 res;
    if (m < 8) {
      res = make_float2(0.0f, 0.0f);
      for (int i = 0; i < m; ++i) {
        const float2 v = stg_ld2(stg, j, b + i, col2);
        res.x = __fadd_rn(res.x, v.x);
        res.y = __fadd_rn(res.y, v.y);
      }
    } else {
      float2 r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = stg_ld2(stg, j, b + q, col2);
      int i = 8;
      const int stop = m - (m % 8);
      for (; i < stop; i += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float2 v = stg_ld2(stg, j, b + i + q, col2);
          r[q].x = __fadd_rn(r[q].x, v.x);
          r[q].y = __fadd_rn(r[q].y, v.y);
        }
      }
      res.x = __fadd_rn(__fadd_rn(__fadd_rn(r[0].x, r[1].x), __fadd_rn(r[2].x, r[3].x)),
                        __fadd_rn(__fadd_rn(r[4].x, r[5].x), __fadd_rn(r[6].x, r[7].x)));
      res.y = __fadd_rn(__fadd_rn(__fadd_rn(r[0].y, r[1].y), __fadd_rn(r[2].y, r[3].y)),
                        __fadd_rn(__fadd_rn(r[4].y, r[5].y), __fadd_rn(r[6].y, r[7].y)));
      for (; i < m; ++i) {
        const float2 v = stg_ld2(stg, j, b + i, col2);
        res.x = __fadd_rn(res.x, v.x);
        res.y = __fadd_rn(res.y, v.y);
      }
    }
    s.x = __fadd_rn(s.x, res.x);
    s.y = __fadd_rn(s.y, res.y);
  }
  const float fn = (float)n;
  return make_float2(__fdiv_rn(s.x, fn), __fdiv_rn(s.y, fn));
}

// pool_pair with the 8 accumulator chains split over a lane pair (sub 0:
// chains 0-3, sub 1: chains 4-7); numpy's tree ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)) joins the two halves with one shuffle, so the value is
// pool_pair's bit for bit.  Both lanes return it.
__device__ __forceinline__ float2 pool_pair_split(const char* stg, int j, int first, int n,
                                                  int col2, int sub) {
  const int m = n - 1, b = first + 1;
  if (m < 8) return pool_pair(stg, j, first, n, col2);
  float2 r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) r[q] = stg_ld2(stg, j, b + 4 * sub + q, col2);
  int i = 8;
  const int stop = m - (m % 8);
  for (; i < stop; i += 8) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 v = stg_ld2(stg, j, b + i + 4 * sub + q, col2);
      r[q].x = __fadd_rn(r[q].x, v.x);
      r[q].y = __fadd_rn(r[q].y, v.y);
    }
  }
  float2 half;
  half.x = __fadd_rn(__fadd_rn(r[0].x, r[1].x), __fadd_rn(r[2].x, r[3].x));
  half.y = __fadd_rn(__fadd_rn(r[0].y, r[1].y), __fadd_rn(r[2].y, r[3].y));
  const float ox = __shfl_xor_sync(0xffffffffu, half.x, 1);
  const float oy = __shfl_xor_sync(0xffffffffu, half.y, 1);
  float2 res = make_float2(__fadd_rn(half.x, ox), __fadd_rn(half.y, oy));  // left + right
  for (; i < m; ++i) {
    const float2 v = stg_ld2(stg, j, b + i, col2);
    res.x = __fadd_rn(res.x, v.x);
    res.y = __fadd_rn(res.y, v.y);
  }
  const float2 x0 = stg_ld2(stg, j, first, col2);
  const float fn = (float)n;
  return make_float2(__fdiv_rn(__fadd_rn(x0.x, res.x), fn), __fdiv_rn(__fadd_rn(x0.y, res.y), fn));
}

// PROJ = false: the QKV projection above.  PROJ = true: the block's output
// projection with the residual fused, out (T, C) = res + o W^T + b, where
// the A operand is the attention output o (H, T, 64) head-major itself:
// K chunk kc of a row tile is head kc's 128 x 64 box (a 3-D map), so the
// (H, T, d) -> (T, C) transpose never happens; tm_q is the (C, T) output
// map, tm_k the residual's (the epilogue TMA-loads the residual tile into
// its staging buffer, adds it in fp32 and stores the sum from there).
template <bool PAIR, bool PROJ = false>
__global__ void __launch_bounds__(THREADS, 1)
    qkv_pool_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v,
                    const Args A) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = (char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  auto BAR = [&](int i) { return smem_u32(bars + i); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + B_TMEM);
  char* stg = smem + OFF_STG;

  const int32_t tiles = A.m_tiles * A.n_tiles;
  const int kchunks = (int)(A.C / BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(BAR(B_FULL + s), 1);
      mbar_init(BAR(B_EMPTY + s), PAIR ? 2 : 1);  // pair: both CTAs' MMAs read the multicast B half
    }
    if (PROJ)
      for (int g = 0; g < EPI_GROUPS; ++g) mbar_init(BAR(B_RES + g), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(BAR(B_TFULL + b), 1);
      mbar_init(BAR(B_TEMPTY + b), 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_b) : "memory");
    if (PROJ) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_k) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // the peer's multicasts and commits target initialised barriers
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // work units: unit u is row tile m = u / n_tiles, feature tile n = u % n_tiles;
  // pair mode: unit u is row tiles 2(u / n_tiles) + {0, 1} (one per CTA of the
  // pair, a CTA whose row tile is past the end computes a zero tile and stores
  // nothing) with one feature tile
  uint32_t crank = 0;
  if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int32_t U = PAIR ? ((A.m_tiles + 1) / 2) * A.n_tiles : tiles;
  const int32_t u0 = PAIR ? (int32_t)(blockIdx.x >> 1) : (int32_t)blockIdx.x;
  const int32_t ustride = PAIR ? (int32_t)(gridDim.x >> 1) : (int32_t)gridDim.x;
  auto decode = [&](int32_t u, int32_t& m, int32_t& n) {
    const int32_t mu = u / A.n_tiles;
    n = u - mu * A.n_tiles;
    m = PAIR ? 2 * mu + (int32_t)crank : mu;
  };
  auto tile_row0 = [&](int32_t m) -> int32_t {
    if (m >= A.m_tiles) return (int32_t)A.T;  // TMA zero-fills rows past the end
    return m < A.nst ? m * BM : (int32_t)A.Ts + (m - A.nst) * BM;
  };

  if (warp == 0) {
    // ============================ TMA producer ============================
    uint32_t s = 0, ph = 0;
    for (int32_t u = u0; u < U; u += ustride) {
      int32_t m, n;
      decode(u, m, n);
      const int32_t row0 = tile_row0(m), f0 = n * BN;
      for (int kc = 0; kc < kchunks; ++kc) {
        mbar_wait(BAR(B_EMPTY + s), ph ^ 1);
        if (elect_one()) {
          const uint32_t dst = sbase + s * STAGE_BYTES;
          mbar_expect_tx(BAR(B_FULL + s), STAGE_BYTES);
          if constexpr (PROJ) tma_load_3d(dst, &tm_a, BAR(B_FULL + s), 0, row0, kc);  // head kc
          else tma_load_2d(dst, &tm_a, BAR(B_FULL + s), kc * BK, row0);
          if constexpr (PAIR) {
            // this CTA's half of B (128 feature rows) into both CTAs' stage s
            const uint32_t half = crank * (B_BYTES / 2);
            tma_load_2d_mc(dst + A_BYTES + half, &tm_b, BAR(B_FULL + s), kc * BK,
                           f0 + (int)crank * (BN / 2), (uint16_t)0x3);
          } else {
            tma_load_2d(dst + A_BYTES, &tm_b, BAR(B_FULL + s), kc * BK, f0);
          }
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    const uint32_t idesc = idesc_f16(BM, BN, 0, 1);
    const uint64_t da0 = sdesc(sbase, 16, 1024), db0 = sdesc(sbase + A_BYTES, 16, 1024);
    uint32_t s = 0, ph = 0, i = 0;
    for (int32_t u = u0; u < U; u += ustride, ++i) {
      const uint32_t ab = i & 1;
      mbar_wait(BAR(B_TEMPTY + ab), ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dt = tmem + ab * BN;
      for (int kc = 0; kc < kchunks; ++kc) {
        mbar_wait(BAR(B_FULL + s), ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t so = (uint64_t)((s * STAGE_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_ss(dt, da0 + so + 2 * k, db0 + so + 2 * k, idesc, (kc | k) ? 1u : 0u);
          if constexpr (PAIR) tc_commit_mc(BAR(B_EMPTY + s), (uint16_t)0x3);  // frees s in both CTAs
          else tc_commit(BAR(B_EMPTY + s));
          if (kc == kchunks - 1) tc_commit(BAR(B_TFULL + ab));
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ============================== epilogue ==============================
    const int quarter = warp & 3;               // TMEM lanes 32*quarter..+31
    const int r = quarter * 32 + lane;          // tile row owned by this thread
    const int grp = (warp - EPI_WARP0) >> 2;    // epilogue warpgroup
    const int et = threadIdx.x - EPI_WARP0 * 32 - grp * 128;  // 0..127
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int64_t C = A.C;
    stg += grp * STG_GROUP;
    float* const sbias = reinterpret_cast<float*>(smem + OFF_BIAS) + grp * BN;
    const uint32_t named_bar = 1 + grp;
    uint32_t res_phase = 0;  // (PROJ) parity of this group's residual barrier
    uint32_t i = grp;
    for (int32_t u = u0 + grp * ustride; u < U; u += EPI_GROUPS * ustride, i += EPI_GROUPS) {
      int32_t m, n;
      decode(u, m, n);
      const bool special = m < A.nst;
      const int32_t row0 = tile_row0(m);
      const int32_t rows = m >= A.m_tiles ? 0
                           : special     ? min(BM, (int32_t)A.Ts - row0)
                                         : min(BM, (int32_t)A.Tp - (m - A.nst) * BM);
      const int32_t f0 = n * BN;
      const int which = PROJ ? 0 : (int)(f0 / C);       // 0 q, 1 k, 2 v
      const int h0 = (int)((f0 - which * C) >> 6);      // first head (PROJ: 64-column block) of the tile
      const uint32_t ab = i & 1;
      // the tile's biases into shared memory (fp32) while its MMAs run
      if (et < BN / 2) {
        const uint32_t bb = A.bias ? __ldg(reinterpret_cast<const uint32_t*>(A.bias + f0) + et) : 0u;
        reinterpret_cast<float2*>(sbias)[et] =
            __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bb));
      }
      asm volatile("bar.sync %0, 128;" ::"r"(named_bar) : "memory");
      mbar_wait(BAR(B_TFULL + ab), (i >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* const outp = which == 0 ? A.out[0] : which == 1 ? A.out[1] : A.out[2];
      float* const poolp = which == 0 ? A.pooled[0] : which == 1 ? A.pooled[1] : nullptr;
#pragma unroll 1
      for (int pass = 0; pass < NPASS; ++pass) {
        if constexpr (PROJ) {
          // the residual's SH 128 x 64 blocks into the (free) staging buffer
          if (et == 0 && rows > 0) {
            mbar_expect_tx(BAR(B_RES + grp), SH * STG_HEAD);
            for (int jj = 0; jj < SH; ++jj)
              tma_load_2d(smem_u32(stg + jj * STG_HEAD), &tm_k, BAR(B_RES + grp),
                          f0 + (pass * SH + jj) * 64, row0);
          }
          if (rows > 0) mbar_wait(BAR(B_RES + grp), res_phase);
          res_phase ^= rows > 0 ? 1u : 0u;
        }
#pragma unroll 1
        for (int jj = 0; jj < SH; ++jj) {
          const int j = pass * SH + jj;
          uint32_t v[64];
          const uint32_t ta = tmem + lane_off + ab * BN + j * 64;
          tmem_ld32(ta, v);
          tmem_ld32(ta + 32, v + 32);
          tmem_wait_ld();
          if (QKV_EXP == 1) continue;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float b8[8];
            {
              const float4 lo = reinterpret_cast<const float4*>(sbias + j * 64 + c * 8)[0];
              const float4 hi = reinterpret_cast<const float4*>(sbias + j * 64 + c * 8)[1];
              b8[0] = lo.x; b8[1] = lo.y; b8[2] = lo.z; b8[3] = lo.w;
              b8[4] = hi.x; b8[5] = hi.y; b8[6] = hi.z; b8[7] = hi.w;
            }
            if constexpr (PROJ) {
              // + residual (fp32), one rounding to bf16 for the whole sum
              const uint4 rv = *reinterpret_cast<const uint4*>(stg + stg_off(jj, r, c));
              const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rw[q]));
                b8[2 * q] = __fadd_rn(b8[2 * q], f.x);
                b8[2 * q + 1] = __fadd_rn(b8[2 * q + 1], f.y);
              }
            }
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              w[q] = pack_bf16(__fadd_rn(__uint_as_float(v[8 * c + 2 * q]), b8[2 * q]),
                               __fadd_rn(__uint_as_float(v[8 * c + 2 * q + 1]), b8[2 * q + 1]));
            *reinterpret_cast<uint4*>(stg + stg_off(jj, r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        if (pass == NPASS - 1) {
          // accumulator drained: the MMA warp may start tile i + 2 in it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(B_TEMPTY + ab));
        }
        if (QKV_EXP == 1) continue;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging -> bulk-store proxy
        asm volatile("bar.sync %0, 128;" ::"r"(named_bar) : "memory");
        // head tile j is rows*128 contiguous bytes of out.  Whole tiles (and
        // the last patch tile, whose extra rows fall past T and are clipped)
        // go out as one TMA bulk tensor store per head, straight from the
        // staging layout (it is the SW128 box layout); a partial special
        // tile, whose extra rows belong to the first patch tile, is stored
        // row by row.
        const bool tma_store = (QKV_TMA_STORE || PROJ) && rows > 0 && (rows == BM || !special);
        if (tma_store) {
          if (et == 0) {
            const CUtensorMap* om = which == 0 ? &tm_q : which == 1 ? &tm_k : &tm_v;
#pragma unroll 1
            for (int jj = 0; jj < SH; ++jj) {
              if constexpr (PROJ)
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm_q),
                    "r"(smem_u32(stg + jj * STG_HEAD)), "r"(f0 + (pass * SH + jj) * 64), "r"(row0)
                    : "memory");
              else
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(om),
                    "r"(smem_u32(stg + jj * STG_HEAD)), "r"(0), "r"(row0), "r"(h0 + pass * SH + jj)
                    : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {
#pragma unroll 1
          for (int jj = 0; jj < SH; ++jj) {
            char* dst = reinterpret_cast<char*>(outp + ((int64_t)(h0 + pass * SH + jj) * A.T + row0) * 64);
            const int nbytes = rows * 128;
#pragma unroll 4
            for (int o = et * 16; o < nbytes; o += 128 * 16) {
              const int rr = o >> 7, c16 = (o >> 4) & 7;
              *reinterpret_cast<uint4*>(dst + o) =
                  *reinterpret_cast<const uint4*>(stg + stg_off(jj, rr, c16));
            }
          }
        }
        // block pools of patch Q (one 128-row block) and patch K (two 64-row blocks)
        if (!special && poolp && rows > 0) {
          const int32_t b = m - A.nst;
          if (which == 0) {
            // SH heads x 32 column pairs, 128 / (SH * 32) lanes per item
            static_assert(SH == 2 || SH == 4, "pool lane mapping");
            if constexpr (SH == 2) {
              const int item = et >> 1, sub = et & 1;
              const int jj = item >> 5, col2 = item & 31;
              const float2 p = pool_pair_split(stg, jj, 0, rows, col2, sub);
              if (sub == 0)
                *reinterpret_cast<float2*>(poolp + ((int64_t)(h0 + pass * SH + jj) * A.nq + b) * 64 +
                                           2 * col2) = p;
            } else {
              const int jj = et >> 5, col2 = et & 31;
              const float2 p = pool_pair(stg, jj, 0, rows, col2);
              *reinterpret_cast<float2*>(poolp + ((int64_t)(h0 + pass * SH + jj) * A.nq + b) * 64 +
                                         2 * col2) = p;
            }
          } else {
            // SH heads x 32 column pairs x 2 key blocks over 128 lanes
            for (int it2 = et; it2 < SH * 64; it2 += 128) {
              const int kb = it2 / (SH * 32), rem = it2 % (SH * 32);
              const int jj = rem >> 5, col2 = rem & 31;
              const int first = kb * 64, nrow = min(64, rows - first);
              if (nrow <= 0) continue;
              const float2 p = pool_pair(stg, jj, first, nrow, col2);
              *reinterpret_cast<float2*>(poolp + ((int64_t)(h0 + pass * SH + jj) * A.nk + 2 * b + kb) * 64 +
                                         2 * col2) = p;
            }
          }
        }
        // staging free for the next pass once the bulk stores have read it
        if (tma_store && et == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(named_bar) : "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2-D (cols, rows) map of a row-major bf16 matrix, box (64, box_rows), SW128
static int make_map_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols,
                       int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BSA_OK;
}

// 3-D (64, T, H) map of a (H, T, 64) bf16 output, box (64, 128, 1), SW128
static int make_map_out(CUtensorMap* map, void* base, int64_t H, int64_t T) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, (cuuint64_t)T, (cuuint64_t)H};
  cuuint64_t strides[2] = {128, (cuuint64_t)T * 128};
  cuuint32_t box[3] = {64, (cuuint32_t)BM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled (output) failed (%d)", (int)r);
  return BSA_OK;
}

// persistent launch of qkv_pool_kernel<PAIR, PROJ> over a's tiles; B is the
// (w_rows, w_cols) bf16 weight
template <bool PROJ>
static int launch_gemm(const CUtensorMap& ma, const void* weight, int64_t w_rows, int64_t w_cols,
                       const CUtensorMap (&mo)[3], const Args& a, cudaStream_t stream) {
  int dev = 0, sms = 0;
  BSA_CUDA_TRY(cudaGetDevice(&dev));
  BSA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // persistent CTA pairs: as many as the GPU co-schedules (a GPC with an odd
  // SM count leaves one SM out), never more, or the surplus would run as a
  // second wave behind the static tile split; none co-schedulable (or
  // QKV_PAIR=0): single CTAs
  static int max_pairs[64];  // per PROJ instantiation (template static)
  static bool queried[64];
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int slot = dev & 63;
  if (!queried[slot]) {
    BSA_CUDA_TRY(cudaFuncSetAttribute(qkv_pool_kernel<true, PROJ>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    BSA_CUDA_TRY(cudaFuncSetAttribute(qkv_pool_kernel<false, PROJ>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    int n = 0;
    cfg.gridDim = dim3(2 * std::max(1, sms / 2));
    if (QKV_PAIR && cudaOccupancyMaxActiveClusters(&n, qkv_pool_kernel<true, PROJ>, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    max_pairs[slot] = QKV_PAIR ? n : 0;
    queried[slot] = true;
  }
  const bool pair = max_pairs[slot] > 0;
  CUtensorMap mb;
  int rc = make_map_2d(&mb, weight, w_rows, w_cols, pair ? BN / 2 : BN);
  if (rc) return rc;
  const int64_t tiles = (int64_t)a.m_tiles * a.n_tiles;
  if (pair) {
    const int64_t units = (int64_t)((a.m_tiles + 1) / 2) * a.n_tiles;
    cfg.gridDim = dim3(2 * (unsigned)std::min<int64_t>(units, max_pairs[slot]));
    BSA_CUDA_TRY(cudaLaunchKernelEx(&cfg, qkv_pool_kernel<true, PROJ>, ma, mb, mo[0], mo[1], mo[2], a));
  } else {
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
    qkv_pool_kernel<false, PROJ><<<grid, THREADS, SMEM_BYTES, stream>>>(ma, mb, mo[0], mo[1], mo[2], a);
  }
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

}  // namespace qkv
}  // namespace bsa

using namespace bsa;

extern "C" {

int bsa_qkv_project_pooled(const void* x, int64_t tokens, int64_t dim_in, const void* weight,
                           const void* bias, int64_t heads, int64_t head_dim, int64_t special_rows,
                           int32_t block_q, int32_t block_k, void* q, void* k, void* v,
                           float* q_pooled, float* k_pooled, void* stream) {
  using namespace bsa::qkv;
  if (!x || !weight || !q || !k || !v) return fail(BSA_EINVAL, "qkv_project: null pointer");
  if (head_dim != 64)
    return fail(BSA_EUNSUPPORTED, "qkv_project: head_dim must be 64, got %lld", (long long)head_dim);
  if (heads < 1 || dim_in != heads * head_dim)
    return fail(BSA_EINVAL, "qkv_project: dim_in %lld != heads %lld x head_dim 64",
                (long long)dim_in, (long long)heads);
  if (dim_in % BN != 0)
    return fail(BSA_EUNSUPPORTED, "qkv_project: heads*head_dim must be a multiple of 256, got %lld",
                (long long)dim_in);
  if (block_q != BM || block_k != 64)
    return fail(BSA_EUNSUPPORTED, "qkv_project: pooling needs block_q 128 / block_k 64, got %d/%d",
                block_q, block_k);
  if (tokens < 1 || special_rows < 0 || special_rows > tokens)
    return fail(BSA_EINVAL, "qkv_project: bad token counts (%lld tokens, %lld special rows)",
                (long long)tokens, (long long)special_rows);
  if (tokens >= ((int64_t)1 << 31)) return fail(BSA_EUNSUPPORTED, "qkv_project: T >= 2^31");
  for (const void* p : {x, weight, (const void*)q, (const void*)k, (const void*)v})
    if ((uintptr_t)p % 16) return fail(BSA_EINVAL, "qkv_project: pointers must be 16-byte aligned");
  if (bias && (uintptr_t)bias % 16) return fail(BSA_EINVAL, "qkv_project: bias must be 16-byte aligned");
  Args a;
  a.T = tokens;
  a.Ts = special_rows;
  a.Tp = tokens - special_rows;
  a.C = dim_in;
  a.H = heads;
  a.nst = (int32_t)ceil_div(special_rows, (int64_t)BM);
  a.nq = (int32_t)ceil_div(a.Tp, (int64_t)BM);
  a.nk = (int32_t)ceil_div(a.Tp, (int64_t)64);
  a.m_tiles = a.nst + a.nq;
  a.n_tiles = (int32_t)(3 * dim_in / BN);
  a.bias = (const __nv_bfloat16*)bias;
  a.out[0] = (__nv_bfloat16*)q;
  a.out[1] = (__nv_bfloat16*)k;
  a.out[2] = (__nv_bfloat16*)v;
  a.pooled[0] = q_pooled;
  a.pooled[1] = k_pooled;
  CUtensorMap ma, mo[3];
  int rc = make_map_2d(&ma, x, tokens, dim_in, BM);
  for (int i = 0; i < 3 && !rc; ++i) rc = make_map_out(&mo[i], a.out[i], heads, tokens);
  if (rc) return rc;
  return launch_gemm<false>(ma, weight, 3 * dim_in, dim_in, mo, a, (cudaStream_t)stream);
}

int bsa_proj_residual(const void* o, int64_t heads, int64_t tokens, const void* weight,
                      const void* bias, const void* residual, void* out, void* stream) {
  using namespace bsa::qkv;
  if (!o || !weight || !residual || !out) return fail(BSA_EINVAL, "proj_residual: null pointer");
  const int64_t C = heads * 64;
  if (heads < 1 || C % BN != 0)
    return fail(BSA_EUNSUPPORTED, "proj_residual: heads*64 must be a multiple of 256, got %lld",
                (long long)C);
  if (tokens < 1 || tokens >= ((int64_t)1 << 31))
    return fail(BSA_EINVAL, "proj_residual: bad token count %lld", (long long)tokens);
  for (const void* p : {o, weight, residual, (const void*)out})
    if ((uintptr_t)p % 16) return fail(BSA_EINVAL, "proj_residual: pointers must be 16-byte aligned");
  if (bias && (uintptr_t)bias % 16) return fail(BSA_EINVAL, "proj_residual: bias must be 16-byte aligned");
  Args a;
  a.T = tokens;
  a.Ts = 0;  // no special/patch split: row tiles over all tokens
  a.Tp = tokens;
  a.C = C;
  a.H = heads;
  a.nst = 0;
  a.nq = (int32_t)ceil_div(tokens, (int64_t)BM);
  a.nk = 0;
  a.m_tiles = a.nq;
  a.n_tiles = (int32_t)(C / BN);
  a.bias = (const __nv_bfloat16*)bias;
  a.out[0] = a.out[1] = a.out[2] = (__nv_bfloat16*)out;
  a.pooled[0] = a.pooled[1] = nullptr;
  CUtensorMap ma, mo[3];
  int rc = make_map_out(&ma, const_cast<void*>(o), heads, tokens);  // A: head kc's (64, 128) box
  if (!rc) rc = make_map_2d(&mo[0], out, tokens, C, BM);              // output (C, T)
  if (!rc) rc = make_map_2d(&mo[1], residual, tokens, C, BM);         // residual (C, T)
  if (rc) return rc;
  mo[2] = mo[0];
  return launch_gemm<true>(ma, weight, C, C, mo, a, (cudaStream_t)stream);
}

}  // extern "C"
