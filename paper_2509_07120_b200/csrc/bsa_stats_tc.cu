// bsa_stats_tc.cu -- dense attention statistics on 5th-gen tensor cores,
// without materialising the (H, T, T) probability map (SURVEY.md §8f row 4:
// the reference's dense_attention_map + quadrant_stats, dense.py:79-102,
// analysis.py:47-74, at block granularity for per-layer tau/rho tooling).
//
// Two passes over S = Q K^T (bf16 in, fp32 accumulate), streamed tile by
// tile with the same machinery as the attention kernel (TMA rings, S in
// TMEM from a .ts tcgen05.mma, one CTA per SM, four groups of four softmax
// warps, tile j to group j % 4):
//   pass 1 (row stats): for every query row (special and patch) the row max
//     m of x = s * scale * log2(e), the partial softmax sums
//     l_spec = sum_{special keys} 2^(x - m), l_patch = sum_{patch keys} 2^(x - m)
//     and the per-kind maxima of x.  Each group keeps its own online state
//     for the tiles it sees; the four are merged at the end of the item.
//   pass 2 (block map): for every patch q-block qb and patch k-block kb the
//     attention mass  A[h, qb, kb] = mean_{rows r in qb} sum_{keys in kb} p(r, k),
//     p = 2^(x - m_r) / (l_spec + l_patch)_r, from the pass-1 row stats.  The
//     row sums of a tile are reduced over its 128 rows in a fixed order
//     (warp shuffle tree, then the four lane quarters in order), so the map is
//     deterministic.
// No P, no PV: the S buffers are released as soon as the softmax warps have
// loaded them.  exp2 is MUFU ex2.approx throughout (statistics, not
// attention: no polynomial split).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "bsa_tc_common.cuh"

namespace bsa {
namespace stc {

using namespace tc;

constexpr int NG = 4, SM_WARPS = 16;
constexpr int PRODUCER_WARP = 16, ISSUER_WARP = 17;
constexpr int NUM_THREADS = 32 * 18;
constexpr int MAX_REGS = (16384 / (32 * 5)) / 8 * 8;  // 18 warps: 5 per sub-partition
constexpr int NB = 7, NK = 10;                         // S buffers (64 columns), K stages
constexpr uint32_t TMEM_COLS = 512, TM_S = 0, TM_Q = 480;
constexpr int OFF_K = 0;
constexpr int OFF_XCH = OFF_K + NK * CHUNK_BYTES;  // [5][NG][128] floats (pass 1 merge)
constexpr int OFF_RED = OFF_XCH + 5 * NG * BQ * 4;  // [NG][2][4] floats (pass 2 reduction)
constexpr int OFF_BAR = OFF_RED + NG * 2 * 4 * 4;
constexpr int B_QFULL = 0, B_KFULL = 1, B_KEMPTY = B_KFULL + NK, B_SFULL = B_KEMPTY + NK,
              B_SFREE = B_SFULL + NB, B_IFULL = B_SFREE + NB, B_IEMPTY = B_IFULL + 2,
              B_COUNT = B_IEMPTY + 2;
constexpr int SMEM_BYTES = OFF_BAR + 8 * B_COUNT + 64 + 1024;
static_assert(SMEM_BYTES + 1024 <= 227 * 1024, "shared memory");
static_assert(TM_S + NB * 64 <= TM_Q, "TMEM columns");

struct StatsArgs {
  const __nv_bfloat16* qp;  // packed partitioned Q / K (H, T, 64) bf16
  const __nv_bfloat16* kp;
  float* row_stats;         // pass 1 out: (H, T, 5) in source token order
  const float* row_in;      // pass 2 in
  float* block_map;         // pass 2 out: (H, nq, nk)
  int32_t* work_counter;
  int64_t n_items;
  float scale_log2;
};

// item of pass 1: (head, 128-row tile) over the partitioned rows [0, T);
// pass 2: (head, patch q-block).  Key stream: the special strip [0, Ts) in
// 64-key tiles (pass 1 only), then every patch k-block in order.
struct SItem {
  int32_t h, qb, row0, rows, nsc, ntiles, spec_last, last_len;
};

template <int PASS>
__device__ __forceinline__ SItem sdecode(const AttnGeom& G, int64_t w) {
  SItem I;
  const int32_t T = (int32_t)G.T, Ts = (int32_t)G.Ts, Tp = (int32_t)G.Tp;
  const int32_t per = PASS == 1 ? (int32_t)ceil_div(G.T, BQ) : (int32_t)G.nq;
  I.h = (int32_t)(w / per);
  const int32_t t = (int32_t)(w - (int64_t)I.h * per);
  if (PASS == 1) {
    I.row0 = t * BQ;
    I.rows = min(BQ, T - I.row0);
    I.qb = -1;
    I.nsc = (Ts + CH - 1) / CH;
  } else {
    I.qb = t;
    I.row0 = Ts + t * BQ;
    I.rows = min(BQ, Tp - t * BQ);
    I.nsc = 0;
  }
  I.spec_last = I.nsc ? Ts - (I.nsc - 1) * CH : CH;
  I.ntiles = I.nsc + (int32_t)G.nk;
  I.last_len = Tp - ((int32_t)G.nk - 1) * CH;
  return I;
}

__device__ __forceinline__ int s_len(const SItem& I, int j) {
  if (j < I.nsc) return j == I.nsc - 1 ? I.spec_last : CH;
  return j == I.ntiles - 1 ? I.last_len : CH;
}

template <int PASS>
__global__ void __maxnreg__(MAX_REGS)
    bsa_stats_kernel(const __grid_constant__ CUtensorMap tm_k, AttnGeom G, StatsArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto BAR = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  volatile int64_t* item_ring = (volatile int64_t*)(smem + OFF_BAR + 8 * B_COUNT);
  uint32_t* tmem_holder = (uint32_t*)(smem + OFF_BAR + 8 * B_COUNT + 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(BAR(B_QFULL), SM_WARPS);
    for (int s = 0; s < NK; ++s) {
      mbar_init(BAR(B_KFULL + s), 1);
      mbar_init(BAR(B_KEMPTY + s), 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(BAR(B_SFULL + i), 1);
      mbar_init(BAR(B_SFREE + i), 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(BAR(B_IFULL + i), 1);
      mbar_init(BAR(B_IEMPTY + i), SM_WARPS + 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == ISSUER_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)), "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == PRODUCER_WARP && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_k) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == PRODUCER_WARP) {
    // ---- K producer: pops items, TMA-loads every key tile of the stream ----
    uint32_t it = 0, gk = 0;
    while (true) {
      int64_t w = 0;
      if (lane == 0) w = atomicAdd((unsigned long long*)A.work_counter, 1ull);
      w = __shfl_sync(0xffffffffu, w, 0);
      const int64_t code = w < A.n_items ? w : -1;
      const uint32_t slot = it & 1;
      mbar_wait(BAR(B_IEMPTY + slot), ((it >> 1) & 1) ^ 1);
      if (elect_one()) {
        item_ring[slot] = code;
        mbar_arrive(BAR(B_IFULL + slot));
      }
      __syncwarp();
      if (code < 0) break;
      const SItem I = sdecode<PASS>(G, code);
      for (int j = 0; j < I.ntiles; ++j) {
        const uint32_t st = gk % NK;
        const int32_t s0 = j < I.nsc ? j * CH : (int32_t)G.Ts + (j - I.nsc) * CH;
        mbar_wait(BAR(B_KEMPTY + st), ((gk / NK) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(BAR(B_KFULL + st), CHUNK_BYTES);
          tma_load_3d(sbase + OFF_K + st * CHUNK_BYTES, &tm_k, BAR(B_KFULL + st), 0, s0, I.h);
        }
        __syncwarp();
        ++gk;
      }
      ++it;
    }
  } else if (warp == ISSUER_WARP) {
    // ---- S issuer: S(j) into buffer j % NB once the softmax released S(j-NB) ----
    uint32_t it = 0, gs = 0;
    const uint32_t id_s = idesc_f16(128, 64, 0, 1);
    const uint64_t dk0 = sdesc(sbase + OFF_K, 16, 1024);
    while (true) {
      const uint32_t slot = it & 1;
      mbar_wait(BAR(B_IFULL + slot), (it >> 1) & 1);
      const int64_t code = item_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(B_IEMPTY + slot));
      if (code < 0) break;
      const SItem I = sdecode<PASS>(G, code);
      mbar_wait(BAR(B_QFULL), it & 1);
      tc_fence_after();
      for (int j = 0; j < I.ntiles; ++j) {
        const uint32_t sk = gs % NK, sb = gs % NB;
        mbar_wait2(BAR(B_KFULL + sk), (gs / NK) & 1, BAR(B_SFREE + sb), ((gs / NB) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dk = dk0 + (uint64_t)((sk * CHUNK_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < D / 16; ++k)
            mma_ts(tmem + TM_S + sb * 64, tmem + TM_Q + k * 8, dk + (uint64_t)(2 * k), id_s,
                   k > 0 ? 1u : 0u);
          tc_commit(BAR(B_SFULL + sb));
          tc_commit(BAR(B_KEMPTY + sk));
        }
        __syncwarp();
        ++gs;
      }
      ++it;
    }
  } else {
    // ---- softmax-side warps: four groups of four, one query row per thread ----
    const int grp = warp >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = A.scale_log2;
    const float NEG_INF = -__int_as_float(0x7f800000);
    float* xch = (float*)(smem + OFF_XCH);  // [5][NG][128]
    float* red = (float*)(smem + OFF_RED);  // [NG][2][4]
    auto all_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(32 * SM_WARPS) : "memory"); };
    auto group_sync = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(2 + grp) : "memory"); };
    uint32_t it = 0, g = 0, gt = 0;  // gt: tiles this group has processed (pass 2 slots)
    while (true) {
      const uint32_t slot = it & 1;
      mbar_wait(BAR(B_IFULL + slot), (it >> 1) & 1);
      const int64_t code = item_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(B_IEMPTY + slot));
      if (code < 0) break;
      const SItem I = sdecode<PASS>(G, code);
      const int32_t pr = I.row0 + row;
      const bool valid = row < I.rows;
      {
        // this warp's 16-dimension chunk of the row's Q -> TMEM (A of S = Q K^T);
        // the previous item's S MMAs are complete (all_sync at its end)
        uint32_t qr[8];
        if (pr < (int32_t)G.T) {
          const uint4* src = reinterpret_cast<const uint4*>(A.qp + ((int64_t)I.h * G.T + pr) * D +
                                                            grp * 16);
          const uint4 v0 = __ldg(src), v1 = __ldg(src + 1);
          qr[0] = v0.x; qr[1] = v0.y; qr[2] = v0.z; qr[3] = v0.w;
          qr[4] = v1.x; qr[5] = v1.y; qr[6] = v1.z; qr[7] = v1.w;
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) qr[e] = 0u;
        }
        tmem_st8(tmem + lane_off + TM_Q + grp * 8, qr);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(B_QFULL));
      }
      // pass 1 state (this group's tiles): max, per-kind sums and maxima
      float m = NEG_INF, ls = 0.f, lp = 0.f, xs = NEG_INF, xp = NEG_INF;
      // pass 2 inputs: the row's max and 1 / (l_spec + l_patch)
      float rm = 0.f, rinv = 0.f;
      if (PASS == 2 && valid) {
        const int64_t src = G.L.part_src(pr);
        const float* rs = A.row_in + ((int64_t)I.h * G.T + src) * 5;
        rm = rs[0];
        rinv = 1.0f / (rs[1] + rs[2]);
      }
      const int first_grp = (int)(g % NG);
      for (int j = (grp - first_grp + NG) % NG; j < I.ntiles; j += NG) {
        const uint32_t gg = g + j, sb = gg % NB;
        const int len = s_len(I, j);
        mbar_wait(BAR(B_SFULL + sb), (gg / NB) & 1);
        tc_fence_after();
        float rsum = 0.f;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t sr[32];
          const uint32_t s_col = tmem + lane_off + TM_S + sb * 64 + hh * 32;
          tmem_ld16(s_col, &sr[0]);
          tmem_ld16(s_col + 16, &sr[16]);
          tmem_wait_ld();
          reg_fence16(&sr[0]);
          reg_fence16(&sr[16]);
          if (hh == 1) {  // S(gg) is in registers: the buffer may take S(gg + NB)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(B_SFREE + sb));
          }
          float x[32];
#pragma unroll
          for (int e = 0; e < 32; ++e)
            x[e] = e + hh * 32 < len ? __uint_as_float(sr[e]) * sl2 : NEG_INF;
          if constexpr (PASS == 1) {
            const float mt = max32(x);
            const bool special = j < I.nsc;
            if (mt > m) {
              const float f = ex2(m - mt);  // 0 on the first tile (m = -inf)
              ls *= f;
              lp *= f;
              m = mt;
            }
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 32; ++e) acc += ex2(x[e] - m);
            if (special) {
              ls += acc;
              xs = fmaxf(xs, mt);
            } else {
              lp += acc;
              xp = fmaxf(xp, mt);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) rsum += ex2(x[e] - rm);
          }
        }
        if constexpr (PASS == 2) {
          // block mass: sum over the tile's keys and rows (fixed order)
          float v = valid ? rsum * rinv : 0.f;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          const int rs_slot = (int)(gt & 1);
          if (lane == 0) red[(grp * 2 + rs_slot) * 4 + quarter] = v;
          group_sync();
          if (quarter == 0 && lane == 0) {
            const float* r4 = red + (grp * 2 + rs_slot) * 4;
            const float tot = (r4[0] + r4[1]) + (r4[2] + r4[3]);
            A.block_map[((int64_t)I.h * G.nq + I.qb) * G.nk + j] = tot / (float)I.rows;
          }
        }
        ++gt;
      }
      if constexpr (PASS == 1) {
        // merge the four groups' states of this row, write it in source order
        xch[(0 * NG + grp) * BQ + row] = m;
        xch[(1 * NG + grp) * BQ + row] = ls;
        xch[(2 * NG + grp) * BQ + row] = lp;
        xch[(3 * NG + grp) * BQ + row] = xs;
        xch[(4 * NG + grp) * BQ + row] = xp;
      }
      all_sync();  // every S MMA of the item was consumed: Q may be rewritten
      if (PASS == 1 && grp == 0 && valid) {
        float M = NEG_INF, XS = NEG_INF, XP = NEG_INF;
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          M = fmaxf(M, xch[(0 * NG + q) * BQ + row]);
          XS = fmaxf(XS, xch[(3 * NG + q) * BQ + row]);
          XP = fmaxf(XP, xch[(4 * NG + q) * BQ + row]);
        }
        float LS = 0.f, LP = 0.f;
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const float mq = xch[(0 * NG + q) * BQ + row];
          const float f = mq == NEG_INF ? 0.f : ex2(mq - M);
          LS += xch[(1 * NG + q) * BQ + row] * f;
          LP += xch[(2 * NG + q) * BQ + row] * f;
        }
        float* o = A.row_stats + ((int64_t)I.h * G.T + G.L.part_src(pr)) * 5;
        o[0] = M;
        o[1] = LS;
        o[2] = LP;
        o[3] = XS;
        o[4] = XP;
      }
      if (PASS == 1) all_sync();  // the merge read xch before the next item's writes
      g += I.ntiles;
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == ISSUER_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

}  // namespace stc

typedef CUresult (*EncodeTiledFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int make_k_map(CUtensorMap* map, const void* base, int64_t H, int64_t T) {
  static EncodeTiledFn2 enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = (EncodeTiledFn2)p;
  }
  if (!enc) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)tc::D, (cuuint64_t)T, (cuuint64_t)H};
  cuuint64_t strides[2] = {(cuuint64_t)tc::D * 2, (cuuint64_t)T * tc::D * 2};
  cuuint32_t box[3] = {(cuuint32_t)tc::D, (cuuint32_t)tc::CH, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BSA_OK;
}

static size_t stats_ws_bytes(const AttnGeom& G) {
  const size_t tens = (size_t)(G.H * G.T * G.d) * 2;
  return 2 * ((tens + 255) / 256 * 256) + 256;
}

template <int PASS>
static int launch_stats(const AttnGeom& G, const stc::StatsArgs& a, cudaStream_t st) {
  CUtensorMap mk;
  int rc = make_k_map(&mk, a.kp, G.H, G.T);
  if (rc) return rc;
  int dev = 0, sms = 148;
  BSA_CUDA_TRY(cudaGetDevice(&dev));
  BSA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  auto kern = stc::bsa_stats_kernel<PASS>;
  BSA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    stc::SMEM_BYTES));
  const int grid = (int)std::min<int64_t>(sms, std::max<int64_t>(1, a.n_items));
  BSA_CUDA_TRY(cudaMemsetAsync(a.work_counter, 0, 8, st));
  kern<<<grid, stc::NUM_THREADS, stc::SMEM_BYTES, st>>>(mk, G, a);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

static int stats_common(const bsa_tensor* q, const bsa_tensor* k, const bsa_layout* layout,
                        AttnGeom& G) {
  if (!q || !k || !layout || !q->data || !k->data) return fail(BSA_EINVAL, "null argument");
  if (q->dtype != BSA_BF16 || k->dtype != BSA_BF16)
    return fail(BSA_EUNSUPPORTED, "attention statistics need bf16 q/k");
  if (q->heads != k->heads || q->tokens != k->tokens || q->dim != k->dim)
    return fail(BSA_EINVAL, "q/k shapes differ");
  if (q->dim != 64) return fail(BSA_EUNSUPPORTED, "attention statistics need head_dim 64");
  const Layout L = to_layout(layout);
  if (L.frames < 1 || L.P < 1 || L.S < 0) return fail(BSA_EINVAL, "invalid layout");
  if (q->tokens != L.tokens())
    return fail(BSA_EINVAL, "inputs have %lld tokens but layout describes %lld",
                (long long)q->tokens, (long long)L.tokens());
  if (L.tokens() >= (1LL << 31) || q->heads >= 65536)
    return fail(BSA_EUNSUPPORTED, "sequence too long");
  G = make_geom(L, q->heads, 64, tc::BQ, tc::CH);
  return BSA_OK;
}

}  // namespace bsa

using namespace bsa;

extern "C" {

size_t bsa_attention_stats_workspace(const bsa_layout* layout, int64_t heads) {
  if (!layout || heads < 1) return 0;
  const AttnGeom G = make_geom(to_layout(layout), heads, 64, tc::BQ, tc::CH);
  return stats_ws_bytes(G);
}

int bsa_attention_row_stats(const bsa_tensor* q, const bsa_tensor* k, const bsa_layout* layout,
                            float scale, float* row_stats, void* ws, size_t ws_bytes,
                            void* stream) {
  AttnGeom G;
  int rc = stats_common(q, k, layout, G);
  if (rc) return rc;
  if (!row_stats || !ws) return fail(BSA_EINVAL, "null output or workspace");
  if (ws_bytes < stats_ws_bytes(G)) return fail(BSA_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t tens = (size_t)(G.H * G.T * G.d) * 2;
  char* p = (char*)ws;
  __nv_bfloat16* qp = (__nv_bfloat16*)p;
  __nv_bfloat16* kp = (__nv_bfloat16*)(p + (tens + 255) / 256 * 256);
  int32_t* counter = (int32_t*)(p + 2 * ((tens + 255) / 256 * 256));
  rc = launch_pack(q, G, 0, qp, st);
  if (!rc) rc = launch_pack(k, G, 0, kp, st);
  if (rc) return rc;
  stc::StatsArgs a{};
  a.qp = qp;
  a.kp = kp;
  a.row_stats = row_stats;
  a.work_counter = counter;
  a.n_items = G.H * ceil_div(G.T, tc::BQ);
  a.scale_log2 = scale * 1.4426950408889634f;
  return launch_stats<1>(G, a, st);
}

int bsa_block_attention_map(const bsa_tensor* q, const bsa_tensor* k, const bsa_layout* layout,
                            float scale, const float* row_stats, float* block_map, void* ws,
                            size_t ws_bytes, void* stream) {
  AttnGeom G;
  int rc = stats_common(q, k, layout, G);
  if (rc) return rc;
  if (!row_stats || !block_map || !ws) return fail(BSA_EINVAL, "null argument");
  if (ws_bytes < stats_ws_bytes(G)) return fail(BSA_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t tens = (size_t)(G.H * G.T * G.d) * 2;
  char* p = (char*)ws;
  __nv_bfloat16* qp = (__nv_bfloat16*)p;
  __nv_bfloat16* kp = (__nv_bfloat16*)(p + (tens + 255) / 256 * 256);
  int32_t* counter = (int32_t*)(p + 2 * ((tens + 255) / 256 * 256));
  rc = launch_pack(q, G, 0, qp, st);
  if (!rc) rc = launch_pack(k, G, 0, kp, st);
  if (rc) return rc;
  stc::StatsArgs a{};
  a.qp = qp;
  a.kp = kp;
  a.row_in = row_stats;
  a.block_map = block_map;
  a.work_counter = counter;
  a.n_items = G.H * G.nq;
  a.scale_log2 = scale * 1.4426950408889634f;
  return launch_stats<2>(G, a, st);
}

}  // extern "C"
