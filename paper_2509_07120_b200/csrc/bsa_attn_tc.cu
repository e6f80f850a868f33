// bsa_attn_tc.cu -- block-sparse FlashAttention forward on 5th-gen tensor cores.
//
// Replaces the reference kernel /root/reference/pkg/src/bsattn/sparse.py:101-205
// (special strip + selected 64-token key blocks per 128-row query block,
// online softmax, sparse.py:89-131) for bf16 inputs, head_dim 64, block_q
// 128, block_k 64.
//
// Persistent, warp-specialised.  Stale-max launch: ONE CTA per SM, 640
// threads (20 warps), all 512 TMEM columns:
//   warps 16/17 K and V producers: walk the item's key tiles (contiguous
//               strip, then the selected blocks, generated warp-parallel from
//               the mask bits) and TMA-load each 64-key K / V chunk (the gather
//               is done by TMA coordinates) into SW128 shared-memory rings.
//   warp 18     S issuer: S = Q K^T with Q read from TMEM (tcgen05.mma .ts,
//               kind::f16, M=128 N=64, fp32) into S buffer j % 6.
//   warp 19     PV issuer: O += P [V | 1] with P read from TMEM and V from
//               shared memory (N=80: an all-ones block beside each V stage
//               makes O[:,64] the row sum of P).  Both issuers are
//               warp-uniform loops with elect.sync issue and tcgen05.commit
//               -> mbarriers.
//   warps 0-15  softmax + epilogue, four groups of four warps; warp w owns
//               TMEM lanes 32(w%4)..+31.  Group j % 4 takes key tile j, whole
//               rows, in 32-column halves.  Four softmax warps per SM
//               sub-partition keep the MUFU and FMA pipes busy.
// exp2: 5 of every 8 pairs on MUFU (ex2.approx), 3 on the FMA pipe as a
// degree-2 minimax polynomial (rel err 1.7e-3 < bf16 rounding of P).
// Softmax offset ("stale max"): the row max of the item's first tile (shared
// once through shared memory) is kept for the whole item; online softmax does
// not depend on the offset, only overflow does.  An item whose tensor-core
// row sum l ends non-finite or above 2^100 (scores grew by ~100 log2 units
// beyond the first tile's max -- never for attention logits of sane scale)
// is listed and recomputed by a second, exact-max launch of the same kernel
// (two CTAs per SM, 10 warps each, two groups splitting every tile into key
// halves 0-31 / 32-63, per-tile max exchanged between the halves, lazy 2^8
// rescaling of O, l summed in registers).
// TMEM (stale max, 512 columns): S0..S5 (6x64, P over S) | O (80) | Q (32).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "bsa_tc_common.cuh"

namespace bsa {
namespace tc {

#ifndef BSA_TC_EXPERIMENT
#define BSA_TC_EXPERIMENT 0  // timing experiments only: 1 = no exps, 2 = no MMAs, 3 = no
                             // exp-argument FFMA2, 4 = no poly clamp
#endif
#ifndef BSA_TC_L2HINT
#define BSA_TC_L2HINT 0  // K/V TMA loads evict_last; Q loads and output stores streaming
#endif
#ifndef BSA_TC_WIDE
#define BSA_TC_WIDE 1
#endif
#ifndef BSA_TC_NB
#define BSA_TC_NB 6
#endif
#ifndef BSA_TC_COLH
#define BSA_TC_COLH 0  // stale-max launch: tiles split into key halves (2 tile groups of 8 warps)
#endif
#ifndef BSA_TC_MERGED
#define BSA_TC_MERGED 1
#endif
#ifndef BSA_TC_NG
#define BSA_TC_NG 4
#endif
// O: 64 columns + 16 row-sum columns.  The PV MMA runs with N = 80: columns
// 64-79 of its B operand are an all-ones block kept beside every V stage (at
// the descriptor's LBO), so O[:, 64] accumulates the row sum of P in fp32
// and the stale-max softmax does no additions.
#ifndef BSA_TC_LSUM
#define BSA_TC_LSUM 1
#endif
constexpr bool LSUM = BSA_TC_LSUM != 0;  // else the softmax sums P rows in registers
constexpr uint32_t O_COLS = LSUM ? 80 : 64;

// Launch shapes.  WIDE (the stale-max launch): ONE CTA per SM owning all 512
// TMEM columns, four softmax warp groups and NB = 6 S/P buffers; tile j goes
// to group j % 4 and buffer j % NB.  S(j) only waits for PV(j - NB), so a
// group does not wait on the P(j) -> PV(j) -> S(j+2) chain that two buffers
// per CTA imposed.  One SM's worth of tiles is too much for one producer and
// one MMA warp sharing the sub-partitions with 16 softmax warps (~900 clk of
// waits and issues per tile, measured), so K and V each get a producer warp
// and S and PV each get an issuer warp (SPLIT).
// Narrow (the exact-max repair launch): two CTAs per SM, 256 columns each,
// two groups splitting every tile into column halves, two buffers, one
// producer and one MMA warp.
// X3 (fp32 inputs): every operand is split into bf16 hi + lo parts and
// each product is formed from three MMAs (hi*hi + hi*lo + lo*hi, fp32
// accumulation): S and O carry ~2^-16 relative error instead of bf16's 2^-8,
// which meets the fp32 path's 1e-4 bar.  Five S/P buffers (Q hi and lo both
// in TMEM), K stages [hi | lo], V stages [hi | ones | lo].
template <bool WIDE, bool X3 = false>
struct Cfg {
  static constexpr int NG = WIDE ? BSA_TC_NG : 2;  // softmax warps per TMEM lane quarter
  // key halves per tile (2: each of a tile's two 32-key halves has its own
  // four warps) and tile groups (tile j goes to group j % NTG)
  static constexpr int HALVES = WIDE ? (BSA_TC_COLH ? 2 : 1) : 2;
  static constexpr int NTG = NG / HALVES;
  static constexpr int NB = X3 ? 5 : (WIDE ? BSA_TC_NB : 2);  // S buffers (64 columns, P over S)
  static constexpr int LEAD = 1;  // (one issuer warp) S(j + LEAD) is issued before PV(j)
  static constexpr int SM_WARPS = 4 * NG;
  // SPLIT: S MMAs and PV MMAs come from two issuer warps (one warp issuing
  // both for a whole SM cannot keep up: ~900 clk of waits and issues per tile)
  static constexpr bool SPLIT = WIDE;
  // SPLIT also gives K and V their own producer warps
  static constexpr int PRODUCER_WARP = SM_WARPS, VPROD_WARP = SPLIT ? SM_WARPS + 1 : SM_WARPS,
                       MMA_WARP = VPROD_WARP + 1, PV_WARP = SPLIT ? MMA_WARP + 1 : MMA_WARP;
  static constexpr int NUM_THREADS = 32 * (PV_WARP + 1);
  // warps other than the K producer that consume the item ring
  static constexpr int RING_CONSUMERS = SM_WARPS + (SPLIT ? 3 : 1);
  static constexpr int QUEUE = 256;  // (SPLIT) per-producer queue of key-tile starts
  static constexpr int CTAS_PER_SM = WIDE ? 1 : 2;
  // registers per thread: each SM sub-partition has 16K registers and holds
  // every 4th warp of the SM's CTAs (8-register granules)
  static constexpr int WARPS_PER_SMSP = (CTAS_PER_SM * NUM_THREADS / 32 + 3) / 4;
  static constexpr int MAX_REGS = (16384 / (32 * WARPS_PER_SMSP)) / 8 * 8;
  // MERGED: K and V rings of NB stages, released by the S / PV commits that
  // already signal SFULL / PFREE (one commit per tile per issuer, not two)
  static constexpr bool MERGED = WIDE && !X3 && LSUM && BSA_TC_MERGED != 0;
  static constexpr int NK = MERGED ? NB : (X3 ? 5 : (WIDE ? 8 : 5));
  static constexpr int NV = MERGED ? NB : (X3 ? 4 : (WIDE ? (LSUM ? 6 : 10) : 4));
  static constexpr int VLAG = 2;  // (one producer warp) K(j) is loaded VLAG tiles before V(j)
  static constexpr int V_STAGE = (LSUM ? 2 * CHUNK_BYTES : CHUNK_BYTES) + (X3 ? CHUNK_BYTES : 0);
  static constexpr int K_STAGE = X3 ? 2 * CHUNK_BYTES : CHUNK_BYTES;  // K tile (X3: hi | lo)
  static constexpr int V_LO = LSUM ? 2 * CHUNK_BYTES : CHUNK_BYTES;   // (X3) V lo tile offset
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + NK * K_STAGE;
  static constexpr int OFF_XCH = OFF_V + NV * V_STAGE;  // [3][NG][128] floats
  static constexpr int OFF_QUEUE = OFF_XCH + 3 * NG * BQ * 4;  // (SPLIT) [2][QUEUE] int32
  static constexpr int OFF_BAR = OFF_QUEUE + (SPLIT ? 2 * QUEUE * 4 : 0);
  static constexpr int SMEM_BYTES = OFF_BAR + 1024 + 1024;  // barriers/ring + alignment slack
  static constexpr uint32_t TMEM_COLS = WIDE ? 512 : 256;
  // TMEM: S0..S(NB-1) (64 columns each, P over S) | O (80) | Q (32, last)
  static constexpr uint32_t TM_S = 0, TM_O = NB * 64, TM_Q = TMEM_COLS - 32;
  static constexpr uint32_t TM_QL = TM_Q - 32;  // (X3) Q lo
  // barrier slots (8 bytes each) inside the barrier region
  static constexpr int B_QFULL = 0;              // [1]  Q in TMEM (all softmax warps)
  static constexpr int B_KFULL = 1;              // [NK]
  static constexpr int B_KEMPTY = B_KFULL + NK;  // [NK]
  static constexpr int B_VFULL = B_KEMPTY + NK;  // [NV]
  static constexpr int B_VEMPTY = B_VFULL + NV;  // [NV]
  static constexpr int B_SFULL = B_VEMPTY + NV;  // [NB]
  static constexpr int B_PFULL = B_SFULL + NB;   // [NB] the warps of the tile
  static constexpr int B_PFREE = B_PFULL + NB;   // [NB] PV done: S/P buffer reusable
  static constexpr int B_OFULL = B_PFREE + NB;   // [1]
  static constexpr int B_OEMPTY = B_OFULL + 1;   // [1]
  static constexpr int B_IFULL = B_OEMPTY + 1;   // [2]
  static constexpr int B_IEMPTY = B_IFULL + 2;   // [2]  softmax warps + MMA warp(s)
  static constexpr int B_COUNT = B_IEMPTY + 2;
  static_assert(B_COUNT * 8 + 100 <= 1024, "barrier region (+ item ring, TMEM address)");
  static_assert(CTAS_PER_SM * (SMEM_BYTES + 1024) <= 228 * 1024, "CTAs per SM vs shared memory");
  static_assert(TM_O + O_COLS <= (X3 ? TM_QL : TM_Q), "TMEM columns");
  static_assert(!X3 || WIDE, "X3 runs in the stale-max launch (with LSUM: launch_pick)");
  static_assert(LEAD >= 1 && LEAD < NB, "S(j+LEAD) must only wait for a PV issued earlier");
};
using CfgMain = Cfg<BSA_TC_WIDE != 0>;
using CfgExact = Cfg<false>;

#ifndef BSA_TC_POLY_DEG
#define BSA_TC_POLY_DEG 2
#endif

// P = exp2(s * scale_log2 - m) for one 32-key half row, written to TMEM as
// packed 16-bit pairs (one tcgen05.st.32x32b.x16); returns the fp32 sum.
// The argument is formed in fp32 with f32x2 FMAs.  POLY of every 8 pairs use
// the FMA-pipe polynomial, the rest MUFU.EX2; F16P selects fp16 P (for fp16
// V) instead of bf16 P.
#ifndef BSA_TC_POLY_SPREAD
#define BSA_TC_POLY_SPREAD 0
#endif
// which of each 8 consecutive pairs take the FMA-pipe polynomial: the first
// POLY (SPREAD 0), or POLY spread evenly over the 8 (SPREAD 1: 0,3,6 / 0,2,4,6)
#ifndef BSA_TC_POLY_PER16
#define BSA_TC_POLY_PER16 0  // (experiments) POLY counts pairs per 16 instead of per 8
#endif
template <int POLY>
__device__ __forceinline__ constexpr bool poly_pair(int e) {
  if constexpr (BSA_TC_POLY_PER16 != 0) {
    return ((e & 15) * POLY) % 16 < POLY;  // POLY of every 16 pairs, spread evenly
  } else if constexpr (BSA_TC_POLY_SPREAD == 0 || POLY == 0) {
    return (e & 7) < POLY;
  } else {
    return ((e & 7) * POLY) % 8 < POLY;
  }
}

#ifndef BSA_TC_H2
#define BSA_TC_H2 0  // (F16P) FMA-pipe exponentials in packed fp16 (HFMA2 polynomial)
#endif
// 2^x for a packed fp16 pair on the FMA pipe in half precision: clamp at
// -15.4 (so j >= -15), j = rint(x) by the 1551 = 1.5*2^10 + 15 magic (the
// rounded sum's low mantissa bits are j + 15), f = x - j in [-0.5, 0.5],
// p(f) the degree-2 minimax polynomial (HFMA2), times 2^j built from the
// exponent field j + 15 (0 for j = -15: exactly zero below 2^-14.5; 31 for
// j = 16: inf, an overflow the caller's row sum flags).
__device__ __forceinline__ uint32_t exp2_poly_h2(uint32_t xh) {
  __half2 x = *reinterpret_cast<__half2*>(&xh);
  x = __hmax2(x, __float2half2_rn(-15.4f));
  const __half2 t = __hadd2(x, __float2half2_rn(1551.0f));
  const __half2 j = __hsub2(t, __float2half2_rn(1551.0f));
  const __half2 f = __hsub2(x, j);
  __half2 p = __hfma2(__float2half2_rn(0.23842570f), f, __float2half2_rn(0.70344281f));
  p = __hfma2(p, f, __float2half2_rn(1.00044298f));
  const uint32_t tb = *reinterpret_cast<const uint32_t*>(&t);
  const uint32_t eb = (tb << 10) & 0x7C007C00u;
  const __half2 e = *reinterpret_cast<const __half2*>(&eb);
  const __half2 r = __hmul2(p, e);
  return *reinterpret_cast<const uint32_t*>(&r);
}

template <int POLY, bool F16P, bool SUM = true>
__device__ __forceinline__ float exp_half(const float (&s)[32], float sl2, float m,
                                          uint32_t p_taddr) {
  if constexpr (F16P && BSA_TC_H2 != 0 && !SUM) {
    // argument in fp32 (f32x2 FMA), rounded once to fp16; P = 2^x in fp16
    const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-m, -m);
    uint32_t r[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 x = __ffma2_rn(make_float2(s[2 * e], s[2 * e + 1]), sl2v, nmv);
      // MUFU pairs: two f32 MUFU.EX2 (ex2.approx.f16x2 is two MUFU ops plus a
      // repack), packed to fp16; polynomial pairs: in fp16 on the FMA pipe
      if (poly_pair<POLY>(e)) r[e] = exp2_poly_h2(cvt_h2(x.x, x.y));
      else r[e] = cvt_h2(ex2(x.x), ex2(x.y));
    }
    tmem_st16(p_taddr, r);
    return 0.0f;
  }
  const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-m, -m);
  float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                  make_float2(0.f, 0.f)};
  uint32_t r[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    // (timing experiment 3: the argument straight from S, no scale / offset)
    const float2 x = BSA_TC_EXPERIMENT == 3 ? make_float2(s[2 * e], s[2 * e + 1])
                                            : __ffma2_rn(make_float2(s[2 * e], s[2 * e + 1]), sl2v, nmv);
    float2 p;
    if (poly_pair<POLY>(e)) p = exp2_poly2<F16P ? 3 : BSA_TC_POLY_DEG>(x);
    else p = make_float2(ex2(x.x), ex2(x.y));
    if constexpr (SUM) rs[e & 3] = __fadd2_rn(rs[e & 3], p);
    if constexpr (F16P) r[e] = cvt_h2(p.x, p.y);
    else r[e] = pack_bf16(p.x, p.y);
  }
  tmem_st16(p_taddr, r);
  if constexpr (!SUM) return 0.0f;
  const float2 t = __fadd2_rn(__fadd2_rn(rs[0], rs[1]), __fadd2_rn(rs[2], rs[3]));
  return t.x + t.y;
}

// (X3) largest |logit| (log2 units) a row may reach on the tensor cores:
// there a score's ~2^-16 relative error stays below ~2.5e-4 in the exponent
constexpr float X3_XLIM = 16.0f;

// (X3) P = exp2(s * scale_log2 - m) for one 32-key half row, all on MUFU
// (ex2.approx, ~2^-22 relative), split into bf16 hi + lo = P to ~2^-16:
// hi packed into 16 TMEM columns at p_taddr, lo into the 16 after them.
__device__ __forceinline__ void exp_half_x3(const float (&s)[32], float sl2, float m,
                                            uint32_t p_taddr) {
  const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-m, -m);
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float2 x = __ffma2_rn(make_float2(s[2 * e], s[2 * e + 1]), sl2v, nmv);
    const float p0 = ex2(x.x), p1 = ex2(x.y);
    hi[e] = pack_bf16(p0, p1);
    const float2 h = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hi[e]));
    lo[e] = pack_bf16(p0 - h.x, p1 - h.y);
  }
  tmem_st16(p_taddr, hi);
  tmem_st16(p_taddr + 16, lo);
}

// debug pipeline trace (BSA_TC_TRACE): clock64 of event `ev` for key tile `idx`
// of CTA 0; TRACE_TILES tiles per event.  Compiled in only with
// -DBSA_TC_TRACE_BUILD: the clock reads split the scheduler's basic blocks.
constexpr int TRACE_TILES = 512, TRACE_EVENTS = 20;
#ifdef BSA_TC_TRACE_BUILD
#define BSA_TR(ev, idx)                                                              \
  do {                                                                               \
    if (A.trace && blockIdx.x == 0 && (idx) < (uint32_t)TRACE_TILES)                  \
      A.trace[(ev) * TRACE_TILES + (idx)] = (unsigned long long)clock64();           \
  } while (0)
#else
#define BSA_TR(ev, idx) \
  do {                  \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// the kernel.  EXACT: the repair launch (per-tile max, lazy O rescaling) over
// the items the stale-max launch listed.
// ---------------------------------------------------------------------------
template <bool WIDE, bool X3>
constexpr int max_regs_of() { return Cfg<WIDE, X3>::MAX_REGS; }

template <int POLY, bool F16P, bool EXACT, bool X3 = false>
__global__ void __maxnreg__((max_regs_of<BSA_TC_WIDE != 0 && !EXACT, X3>()))
    bsa_tc_kernel(const __grid_constant__ CUtensorMap tm_kl, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_vl,
                  AttnGeom G, TcArgs A) {
  using C = Cfg<BSA_TC_WIDE != 0 && !EXACT, X3>;
  static_assert(!X3 || (POLY == 0 && !F16P && !EXACT), "X3: MUFU exponentials, bf16 P, stale max");
  constexpr int NG = C::NG, NB = C::NB, NK = C::NK, NV = C::NV, VLAG = C::VLAG;
  constexpr int SM_WARPS = C::SM_WARPS;
  // warps that write one tile's P: one group (stale max, whole tiles), or
  // both groups (exact max, column halves of every tile)
  constexpr int HALVES = C::HALVES, NTG = C::NTG;
  constexpr int TILE_WARPS = 4 * HALVES;
  static_assert(!EXACT || (NG == 2 && HALVES == 2), "the exact launch splits tiles into two column halves");
  (void)tm_kl;  // (X3 only) K lo, V lo maps
  (void)tm_vl;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + C::OFF_BAR;
  auto BAR = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  // item ring: two slots of [code, decoded Item (8 fields)].  The producer
  // decodes (two dependent global loads) while it waits for the slot, so the
  // other warps start the next item without those loads.
  volatile int32_t* item_ring = (volatile int32_t*)(smem + C::OFF_BAR + 8 * C::B_COUNT);
  uint32_t* tmem_holder = (uint32_t*)(smem + C::OFF_BAR + 8 * C::B_COUNT + 96);
  auto ring_put = [&](uint32_t slot, int32_t code, const Item& I) {
    volatile int32_t* r = item_ring + slot * 11;
    r[0] = code;
    r[1] = I.h; r[2] = I.qb; r[3] = I.row0; r[4] = I.rows;
    r[5] = I.nchunks; r[6] = I.last_len; r[7] = I.nsc; r[8] = I.spec_last;
    r[9] = I.r; r[10] = I.kstart;
  };
  auto ring_get = [&](uint32_t slot, Item& I) -> int32_t {
    volatile int32_t* r = item_ring + slot * 11;
    I.h = r[1]; I.qb = r[2]; I.row0 = r[3]; I.rows = r[4];
    I.nchunks = r[5]; I.last_len = r[6]; I.nsc = r[7]; I.spec_last = r[8];
    I.r = r[9]; I.kstart = r[10];
    return r[0];
  };
  float* xch = (float*)(smem + C::OFF_XCH);  // [3][NG][128]: first-tile max, tile max, l

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(BAR(C::B_QFULL), SM_WARPS);
    for (int i = 0; i < NB; ++i) {
      mbar_init(BAR(C::B_SFULL + i), 1);
      mbar_init(BAR(C::B_PFULL + i), TILE_WARPS);
      mbar_init(BAR(C::B_PFREE + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(BAR(C::B_IFULL + i), 1);
      mbar_init(BAR(C::B_IEMPTY + i), C::RING_CONSUMERS);
    }
    for (int s = 0; s < NK; ++s) {
      mbar_init(BAR(C::B_KFULL + s), 1);
      mbar_init(BAR(C::B_KEMPTY + s), 1);
    }
    for (int s = 0; s < NV; ++s) {
      mbar_init(BAR(C::B_VFULL + s), 1);
      mbar_init(BAR(C::B_VEMPTY + s), 1);
    }
    mbar_init(BAR(C::B_OFULL), 1);
    mbar_init(BAR(C::B_OEMPTY), SM_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (LSUM) {
    // the all-ones half of every V stage: B columns 64-79 of the PV MMA (any
    // swizzle permutation of ones is ones)
    const uint32_t one2 = F16P ? 0x3C003C00u : 0x3F803F80u;
    for (int i = threadIdx.x; i < NV * CHUNK_BYTES / 4; i += C::NUM_THREADS) {
      const int st = i / (CHUNK_BYTES / 4), w = i % (CHUNK_BYTES / 4);
      reinterpret_cast<uint32_t*>(smem + C::OFF_V + st * C::V_STAGE + CHUNK_BYTES)[w] = one2;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == C::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)), "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == C::PRODUCER_WARP && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_k) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_v) : "memory");
    if constexpr (X3) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_kl) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_vl) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // the schedule kernel (main launch) or the overflow list (repair launch)
  // leaves the item count on the device
  const int64_t n_work = *A.n_items_dev;

  if (C::SPLIT && (warp == C::PRODUCER_WARP || warp == C::VPROD_WARP)) {
    // ======================= K / V producers (SPLIT; one elected lane issues) ===
    // Each warp walks the item's key tiles itself: the contiguous strip, then
    // the selected blocks in ascending order, generated warp-parallel (32
    // mask bytes per step: popc + warp scan) into a shared-memory queue, so
    // the per-tile cost is one queue read, one barrier wait and one TMA.
    const bool is_k = warp == C::PRODUCER_WARP;
    const uint64_t l2_keep = BSA_TC_L2HINT ? l2_policy_evict_last() : 0;
    // the queue through its shared-window address (LDS / STS): the generic
    // pointer (smem is realigned at run time) compiles to generic LD / ST,
    // slower on this per-tile path
    const uint32_t qbase = sbase + C::OFF_QUEUE + (is_k ? 0u : 4u * C::QUEUE);
    auto q_st = [&](int i, int32_t v) {
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(qbase + 4u * (uint32_t)i), "r"(v) : "memory");
    };
    auto q_ld = [&](int i) -> int32_t {
      int32_t v;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(qbase + 4u * (uint32_t)i) : "memory");
      return v;
    };
    uint32_t it = 0, gx = 0;
    while (true) {
      const uint32_t slot = it & 1;
      int32_t code;
      Item I;
      if (is_k) {
        int64_t w = 0;
        if (lane == 0) w = atomicAdd(A.work_counter, 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        code = -1;
        if (w < n_work) code = A.items[w];
        if (code >= 0) I = decode(G, code, A.counts, A.bits, A.kr);
        mbar_wait(BAR(C::B_IEMPTY + slot), ((it >> 1) & 1) ^ 1);
        if (elect_one()) {
          ring_put(slot, code, I);
          mbar_arrive(BAR(C::B_IFULL + slot));
        }
        __syncwarp();
      } else {
        mbar_wait(BAR(C::B_IFULL + slot), (it >> 1) & 1);
        code = ring_get(slot, I);
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(C::B_IEMPTY + slot));
      }
      if (code < 0) break;
      const uint8_t* mrow =
          I.qb >= 0 ? A.bits + ((int64_t)I.h * G.nq + I.qb) * G.mask_row_bytes : nullptr;
      // contiguous keys [kstart, end), then the mask bytes [bp, nbytes) of
      // this item's key range
      const int64_t rbytes = (int64_t)A.kr.rb / 8;
      const int64_t nbytes =
          I.qb >= 0 ? min((int64_t)G.mask_row_bytes, (int64_t)(I.r + 1) * rbytes) : 0;
      int64_t pos = I.kstart, bp = (int64_t)I.r * rbytes;
      const int64_t end = contig_end(I);
      int qh = 0, qt = 0;
      for (int j = 0; j < I.nchunks; ++j) {
        if (qh == qt) {
          qh = 0;
          qt = 0;
          if (pos < end) {
            const int64_t left = (end - pos + CH - 1) / CH;
            const int n = (int)(left < C::QUEUE ? left : C::QUEUE);
            for (int e = lane; e < n; e += 32) q_st(e, (int32_t)(pos + (int64_t)e * CH));
            pos += (int64_t)n * CH;
            qt = n;
          } else {
            while (qt == 0 && bp < nbytes) {
              const int64_t b = bp + lane;
              uint32_t byte = b < nbytes ? mrow[b] : 0u;
              const int c = __popc(byte);
              int incl = c;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
              }
              int k = incl - c;
              while (byte) {
                const int bit = __ffs(byte) - 1;
                byte &= byte - 1;
                q_st(k++, (int32_t)(G.Ts + (b * 8 + bit) * CH));
              }
              qt = __shfl_sync(0xffffffffu, incl, 31);
              bp += 32;
            }
            if (qt == 0) {  // mask and counts disagree: keep the pipeline moving
              q_st(0, (int32_t)G.Ts);
              qt = 1;
            }
          }
          __syncwarp();
        }
        const int32_t s0 = q_ld(qh++);
        if (is_k) {
          const uint32_t st = gx % NK;
          if (lane == 0) BSA_TR(9, gx);
          mbar_wait(BAR((C::MERGED ? C::B_SFULL : C::B_KEMPTY) + st), ((gx / NK) & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(BAR(C::B_KFULL + st), C::K_STAGE);
            if constexpr (BSA_TC_L2HINT != 0)
              tma_load_3d_hint(sbase + C::OFF_K + st * C::K_STAGE, &tm_k, BAR(C::B_KFULL + st), 0,
                               s0, I.h, l2_keep);
            else
              tma_load_3d(sbase + C::OFF_K + st * C::K_STAGE, &tm_k, BAR(C::B_KFULL + st), 0, s0,
                          I.h);
            if constexpr (X3)
              tma_load_3d(sbase + C::OFF_K + st * C::K_STAGE + CHUNK_BYTES, &tm_kl,
                          BAR(C::B_KFULL + st), 0, s0, I.h);
            BSA_TR(0, gx);
          }
        } else {
          const uint32_t st = gx % NV;
          mbar_wait(BAR((C::MERGED ? C::B_PFREE : C::B_VEMPTY) + st), ((gx / NV) & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(BAR(C::B_VFULL + st), X3 ? 2 * CHUNK_BYTES : CHUNK_BYTES);
            if constexpr (BSA_TC_L2HINT != 0)
              tma_load_3d_hint(sbase + C::OFF_V + st * C::V_STAGE, &tm_v, BAR(C::B_VFULL + st), 0,
                               s0, I.h, l2_keep);
            else
              tma_load_3d(sbase + C::OFF_V + st * C::V_STAGE, &tm_v, BAR(C::B_VFULL + st), 0, s0,
                          I.h);
            if constexpr (X3)
              tma_load_3d(sbase + C::OFF_V + st * C::V_STAGE + C::V_LO, &tm_vl,
                          BAR(C::B_VFULL + st), 0, s0, I.h);
            BSA_TR(6, gx);
          }
        }
        __syncwarp();
        ++gx;
      }
      ++it;
    }
  } else if (warp == C::PRODUCER_WARP) {
    // ======================= producer (whole warp; one elected lane issues) =====
    // K(j) is issued VLAG tiles before V(j): a K tile is released as soon as
    // its S MMA completes, a V tile only after its PV MMA.
    uint32_t it = 0, gk = 0, gv = 0;
    int32_t vq[VLAG + 1];  // key-chunk starts of the K tiles whose V is pending
    while (true) {
      int64_t w = 0;
      if (lane == 0) w = atomicAdd(A.work_counter, 1);
      w = __shfl_sync(0xffffffffu, w, 0);
      int32_t code = -1;
      if (w < n_work) code = A.items[w];
      Item I;
      if (code >= 0) I = decode(G, code, A.counts, A.bits, A.kr);
      const uint32_t slot = it & 1;
      mbar_wait(BAR(C::B_IEMPTY + slot), ((it >> 1) & 1) ^ 1);
      if (elect_one()) {
        ring_put(slot, code, I);
        mbar_arrive(BAR(C::B_IFULL + slot));
      }
      __syncwarp();
      if (code < 0) break;
      const uint8_t* mrow =
          I.qb >= 0 ? A.bits + ((int64_t)I.h * G.nq + I.qb) * G.mask_row_bytes : nullptr;
      const int64_t rbytes = (int64_t)A.kr.rb / 8;
      KeyChunker ck(G, I.qb, mrow, CH, I.kstart, contig_end(I), (int64_t)I.r * rbytes,
                    (int64_t)(I.r + 1) * rbytes);
      auto load_v = [&](int32_t s0) {
        const uint32_t st = gv % NV;
        mbar_wait(BAR(C::B_VEMPTY + st), ((gv / NV) & 1) ^ 1);
        if (lane == 0) BSA_TR(6, gv);
        if (elect_one()) {
          mbar_expect_tx(BAR(C::B_VFULL + st), CHUNK_BYTES);
          tma_load_3d(sbase + C::OFF_V + st * C::V_STAGE, &tm_v, BAR(C::B_VFULL + st), 0, s0, I.h);
        }
        __syncwarp();
        ++gv;
      };
      for (int j = 0; j < I.nchunks; ++j) {
        const uint32_t st = gk % NK;
        int64_t s0;
        int l0;
        ck.next(s0, l0);
        if (lane == 0) BSA_TR(9, gk);
        mbar_wait(BAR(C::B_KEMPTY + st), ((gk / NK) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(BAR(C::B_KFULL + st), CHUNK_BYTES);
          tma_load_3d(sbase + C::OFF_K + st * C::K_STAGE, &tm_k, BAR(C::B_KFULL + st), 0, (int)s0,
                      I.h);
          BSA_TR(0, gk);
        }
        __syncwarp();
        ++gk;
#pragma unroll
        for (int q = VLAG; q > 0; --q) vq[q] = vq[q - 1];
        vq[0] = (int32_t)s0;
        if (j >= VLAG) load_v(vq[VLAG]);
      }
#pragma unroll
      for (int q = VLAG - 1; q >= 0; --q)
        if (q < I.nchunks) load_v(vq[q]);
      ++it;
    }
  } else if (warp == C::MMA_WARP || warp == C::PV_WARP) {
    // ======================= MMA issuers (whole warp; one elected lane issues) ==
    // Descriptors are built once; per tile only the stage offset (address >> 4,
    // no carry out of the 14-bit field: smem < 256 KB) is added.  S(j) goes
    // into buffer j % NB once PV(j - NB), which read P from it, has completed.
    // SPLIT: warp MMA_WARP issues every S, warp PV_WARP every PV; else one
    // warp issues S(j + LEAD) before PV(j).
    const bool do_s = warp == C::MMA_WARP, do_pv = warp == C::PV_WARP;
    uint32_t it = 0, gs = 0, gp = 0;
    uint32_t sk = 0, kph = 0, sb = 0, sph = 0;  // S issue: K stage, S buffer (+ phases)
    uint32_t pb = 0, pph = 0, sv = 0, vph = 0;  // PV issue: P buffer, V stage
    const uint32_t id_s = idesc_f16(128, 64, 0, 1);                  // bf16 Q x bf16 K
    const uint32_t id_pv = idesc_f16(128, O_COLS, 1, F16P ? 0 : 1);   // P x [V | ones]
    const uint32_t id_pv64 = idesc_f16(128, 64, 1, 1);                // (X3) P hi x V lo
    const uint64_t dk0 = sdesc(sbase + C::OFF_K, 16, 1024);
    const uint64_t dv0 = sdesc(sbase + C::OFF_V, 8192, 1024);
    const uint64_t dvl0 = sdesc(sbase + C::OFF_V + C::V_LO, 8192, 1024);
    while (true) {
      const uint32_t slot = it & 1;
      mbar_wait(BAR(C::B_IFULL + slot), (it >> 1) & 1);
      Item I;
      const int32_t code = ring_get(slot, I);
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(C::B_IEMPTY + slot));
      if (code < 0) break;
      const int ntiles = I.nchunks;
      if (do_s) {
        mbar_wait(BAR(C::B_QFULL), it & 1);
        tc_fence_after();
      }
      // ring cursors (stage, phase), advanced incrementally: no div/mod on the
      // issue path, which runs at ~1/5 of an SMSP's issue slots
      auto issue_s = [&]() {
        if (lane == 0) BSA_TR(11, gs);
#ifdef BSA_TC_TRACE_BUILD
        mbar_wait(BAR(C::B_KFULL + sk), kph);
        if (lane == 0) BSA_TR(3, gs);
        mbar_wait(BAR(C::B_PFREE + sb), sph ^ 1);
        if (lane == 0) BSA_TR(13, gs);
#else
        mbar_wait2(BAR(C::B_KFULL + sk), kph, BAR(C::B_PFREE + sb), sph ^ 1);
#endif
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dk = dk0 + (uint64_t)(sk * (C::K_STAGE >> 4));
          const uint32_t ds = tmem + C::TM_S + sb * 64;
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            if (BSA_TC_EXPERIMENT == 2) continue;
            mma_ts(ds, tmem + C::TM_Q + k * 8, dk + (uint64_t)(2 * k), id_s, k > 0 ? 1u : 0u);
            if constexpr (X3) {
              // Q hi x K lo, Q lo x K hi
              mma_ts(ds, tmem + C::TM_Q + k * 8, dk + (uint64_t)((CHUNK_BYTES >> 4) + 2 * k), id_s, 1u);
              mma_ts(ds, tmem + C::TM_QL + k * 8, dk + (uint64_t)(2 * k), id_s, 1u);
            }
          }
          tc_commit(BAR(C::B_SFULL + sb));
          if constexpr (!C::MERGED) tc_commit(BAR(C::B_KEMPTY + sk));
          BSA_TR(1, gs);
        }
        __syncwarp();
        ++gs;
        if (++sk == (uint32_t)NK) { sk = 0; kph ^= 1; }
        if (++sb == (uint32_t)NB) { sb = 0; sph ^= 1; }
      };
      auto issue_pv = [&](int jj) {
        if (lane == 0) BSA_TR(10, gp);
#ifdef BSA_TC_TRACE_BUILD
        mbar_wait(BAR(C::B_PFULL + pb), pph);
        if (lane == 0) BSA_TR(7, gp);
        mbar_wait(BAR(C::B_VFULL + sv), vph);
        if (lane == 0) BSA_TR(5, gp);
#else
        mbar_wait2(BAR(C::B_PFULL + pb), pph, BAR(C::B_VFULL + sv), vph);
#endif
        if (jj == 0) mbar_wait(BAR(C::B_OEMPTY), (it & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dv = dv0 + (uint64_t)(sv * (C::V_STAGE >> 4));
          const uint64_t dvl = dvl0 + (uint64_t)(sv * (C::V_STAGE >> 4));
          const uint32_t pa = tmem + C::TM_S + pb * 64;
          // keys 16k..16k+15.  Whole tiles: P packed over S columns 0-31;
          // column halves: half k>>1 wrote its P over S columns 32*(k>>1)
#pragma unroll
          for (int k = 0; k < CH / 16; ++k) {
            if (BSA_TC_EXPERIMENT == 2) continue;
            if constexpr (X3) {
              // keys 16k..: P hi at S columns 32(k>>1) + 8(k&1), P lo 16 further;
              // O += Ph [Vh | 1] + Pl [Vh | 1] + Ph Vl (the ones column sums Ph + Pl)
              const uint32_t ph = pa + (k >> 1) * 32 + (k & 1) * 8;
              mma_ts(tmem + C::TM_O, ph, dv + (uint64_t)(k * (2048 >> 4)), id_pv,
                     (jj > 0 || k > 0) ? 1u : 0u);
              mma_ts(tmem + C::TM_O, ph + 16, dv + (uint64_t)(k * (2048 >> 4)), id_pv, 1u);
              mma_ts(tmem + C::TM_O, ph, dvl + (uint64_t)(k * (2048 >> 4)), id_pv64, 1u);
            } else {
              mma_ts(tmem + C::TM_O, pa + (HALVES == 2 ? (k >> 1) * 32 + (k & 1) * 8 : k * 8),
                     dv + (uint64_t)(k * (2048 >> 4)), id_pv, (jj > 0 || k > 0) ? 1u : 0u);
            }
          }
          tc_commit(BAR(C::B_PFREE + pb));
          if constexpr (!C::MERGED) tc_commit(BAR(C::B_VEMPTY + sv));
          BSA_TR(2, gp);
        }
        __syncwarp();
        ++gp;
        if (++pb == (uint32_t)NB) { pb = 0; pph ^= 1; }
        if (++sv == (uint32_t)NV) { sv = 0; vph ^= 1; }
      };
      if constexpr (C::SPLIT) {
        if (do_s) {
          for (int j = 0; j < ntiles; ++j) issue_s();
        } else {
          for (int j = 0; j < ntiles; ++j) issue_pv(j);
        }
      } else {
        const int lead = ntiles < C::LEAD ? ntiles : C::LEAD;
        for (int j = 0; j < lead; ++j) issue_s();
        for (int j = 0; j < ntiles; ++j) {
          if (j + C::LEAD < ntiles) issue_s();
          issue_pv(j);
        }
      }
      if (do_pv) {
        if (elect_one()) tc_commit(BAR(C::B_OFULL));
        __syncwarp();
      }
      ++it;
    }
  } else {
    // ======================= softmax warps =======================
    const int grp = warp >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;  // TMEM lane == query row in the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = A.scale_log2;
    const float NEG_INF = -__int_as_float(0x7f800000);
    // (no LSUM) largest tile sum (hence P value) accepted with the stale
    // offset: keeps P and the fp32 accumulators far from overflow (fp16 P:
    // its 65504 range)
    const float P_LIMIT = F16P ? 32768.0f : 18446744073709551616.0f;
    (void)P_LIMIT;
    float* x_first = xch;              // [NG][128]
    float* x_tile = xch + NG * BQ;     // [NG][128] (EXACT)
    float* x_l = xch + 2 * NG * BQ;    // [NG][128] (EXACT)
    // S/P buffer, its phase and first TMEM column for tile j of the
    // current item (g: the item's first global tile)
    uint32_t it = 0, g = 0;
    struct ChunkSlot {
      uint32_t buf, phase, col;
    };
    auto slot_of = [&](int j) -> ChunkSlot {
      ChunkSlot z;
      const uint32_t t = g + (uint32_t)j;
      z.buf = t % NB;
      z.phase = (t / NB) & 1;
      z.col = C::TM_S + z.buf * 64;
      return z;
    };
    // the NG warps sharing this TMEM lane quarter
    auto quarter_sync = [&]() {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + quarter), "n"(32 * NG) : "memory");
    };
    while (true) {
      const uint32_t slot = it & 1;
      mbar_wait(BAR(C::B_IFULL + slot), (it >> 1) & 1);
      Item I;
      const int32_t code = ring_get(slot, I);
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(C::B_IEMPTY + slot));
      if (code < 0) break;
      const int ntiles = I.nchunks;
      if (warp == 0 && lane == 0) BSA_TR(14, it);
      {
        // this warp's 64/NG dimensions of its query row of the packed
        // partitioned Q -> TMEM (bf16 pairs: the A operand of S = Q K^T).  The
        // previous item's S MMAs are complete: its epilogue waited for O.
        // 16-dimension chunks c (8 packed columns) with c % NG == grp
        const int32_t pr = I.row0 + row;
        // Q straight from the caller's bf16 tensor (no pack pass): the
        // partitioned row's source token; else the packed copy
        const int64_t qrow = pr < (int32_t)G.T && A.q_src && !A.permuted_out ? G.L.part_src(pr) : pr;
        for (int c = grp; c < 4; c += NG) {
          uint32_t qr[8];
          if (pr < (int32_t)G.T) {
            const uint4* src = reinterpret_cast<const uint4*>(
                A.qp + (int64_t)I.h * A.q_sH + qrow * A.q_sT + c * 16);
            const uint4 v0 = BSA_TC_L2HINT ? __ldcs(src) : __ldg(src);
            const uint4 v1 = BSA_TC_L2HINT ? __ldcs(src + 1) : __ldg(src + 1);
            qr[0] = v0.x; qr[1] = v0.y; qr[2] = v0.z; qr[3] = v0.w;
            qr[4] = v1.x; qr[5] = v1.y; qr[6] = v1.z; qr[7] = v1.w;
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) qr[e] = 0u;
          }
          tmem_st8(tmem + lane_off + C::TM_Q + c * 8, qr);
          if constexpr (X3) {
            // Q lo: packed beside Q hi (same partitioned layout and strides)
            if (pr < (int32_t)G.T) {
              const uint4* src = reinterpret_cast<const uint4*>(
                  A.qp_lo + (int64_t)I.h * A.q_sH + qrow * A.q_sT + c * 16);
              const uint4 v0 = __ldg(src), v1 = __ldg(src + 1);
              qr[0] = v0.x; qr[1] = v0.y; qr[2] = v0.z; qr[3] = v0.w;
              qr[4] = v1.x; qr[5] = v1.y; qr[6] = v1.z; qr[7] = v1.w;
            }
            tmem_st8(tmem + lane_off + C::TM_QL + c * 8, qr);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(C::B_QFULL));
      }
      float m = NEG_INF, l = 0.0f;
      bool ovf = false;
      float xm = NEG_INF;  // (X3) the row's largest score over this warp's tiles
      if constexpr (!EXACT) {
        // ---- stale max: tile group tg takes tiles j with (g + j) % NTG == tg;
        // with HALVES == 2 its warps split every tile into key halves ----
        const int half = HALVES == 2 ? (grp & 1) : 0, tg = grp / HALVES;
        const int first_tg = (int)(g % NTG);  // tile group that owns the item's tile 0
        if (tg == first_tg) {
          // tile 0's row max becomes the item's offset
          const ChunkSlot z = slot_of(0);
          mbar_wait(BAR(C::B_SFULL + z.buf), z.phase);
          tc_fence_after();
          const int len0 = chunk_len(I, 0);
          float mx = NEG_INF;
#pragma unroll
          for (int h2 = 0; h2 < 3 - HALVES; ++h2) {
            const int hh = HALVES == 2 ? half : h2;
            uint32_t sr[32];
            const uint32_t s_col = tmem + lane_off + z.col + hh * 32;
            tmem_ld16(s_col, &sr[0]);
            tmem_ld16(s_col + 16, &sr[16]);
            tmem_wait_ld();
            reg_fence16(&sr[0]);
            reg_fence16(&sr[16]);
            float s[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) s[e] = e + hh * 32 < len0 ? __uint_as_float(sr[e]) : NEG_INF;
            mx = fmaxf(mx, max32(s));
          }
          x_first[half * BQ + row] = mx;
        }
        quarter_sync();
        m = (HALVES == 2 ? fmaxf(x_first[row], x_first[BQ + row]) : x_first[row]) * sl2;
        for (int j = (tg - first_tg + NTG) % NTG; j < ntiles; j += NTG) {
          const uint32_t gg = g + j;
          const ChunkSlot z = slot_of(j);
          const uint32_t sb = z.buf;
          const int len = chunk_len(I, j);
          if (lane == 0 && quarter == 0 && half == 0) BSA_TR(4, gg);
          mbar_wait(BAR(C::B_SFULL + sb), z.phase);
          tc_fence_after();
          if (lane == 0 && quarter == 0 && half == 0) BSA_TR(8, gg);
#pragma unroll
          for (int h2 = 0; h2 < 3 - HALVES; ++h2) {
            const int hh = HALVES == 2 ? half : h2;
            // 32 keys at a time; their P (16 packed columns) goes over S
            // columns this thread has already read (whole tiles: columns
            // 16hh..; key halves: each half's own columns 32hh..)
            uint32_t sr[32];
            const uint32_t s_col = tmem + lane_off + z.col + hh * 32;
            tmem_ld16(s_col, &sr[0]);
            tmem_ld16(s_col + 16, &sr[16]);
            tmem_wait_ld();
            reg_fence16(&sr[0]);
            reg_fence16(&sr[16]);
            float s[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) s[e] = __uint_as_float(sr[e]);
            if (len - hh * 32 < 32) {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e + hh * 32 >= len) s[e] = NEG_INF;
            }
            const uint32_t p_col = tmem + lane_off + z.col + hh * (HALVES == 2 || X3 ? 32 : 16);
#if BSA_TC_EXPERIMENT == 1
            {  // timing experiment: no exponentials (results are wrong)
              uint32_t r[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) r[e] = pack_bf16(s[2 * e], s[2 * e + 1]);
              tmem_st16(p_col, r);
            }
#else
            if constexpr (X3) {
              xm = fmaxf(xm, max32(s));
              exp_half_x3(s, sl2, m, p_col);
            } else {
              const float lt = exp_half<POLY, F16P, !LSUM>(s, sl2, m, p_col);
              if constexpr (!LSUM) {
                ovf |= !(lt <= P_LIMIT);
                l += lt;
              }
            }
#endif
          }
          if (lane == 0 && quarter == 0 && half == 0) BSA_TR(12, gg);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(BAR(C::B_PFULL + sb));
            if (quarter == 0 && half == 0) BSA_TR(16, gg);
          }
        }
      } else {
        // ---- exact max: the two groups split every tile into key halves ----
        const int half = grp;
        for (int j = 0; j < ntiles; ++j) {
          const uint32_t gg = g + j, sb = gg % NB;
          const int len = chunk_len(I, j) - half * 32;  // valid keys of this half
          mbar_wait(BAR(C::B_SFULL + sb), (gg / NB) & 1);
          tc_fence_after();
          uint32_t sr[32];
          const uint32_t s_col = tmem + lane_off + C::TM_S + sb * 64 + half * 32;
          tmem_ld16(s_col, &sr[0]);
          tmem_ld16(s_col + 16, &sr[16]);
          tmem_wait_ld();
          reg_fence16(&sr[0]);
          reg_fence16(&sr[16]);
          float s[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) s[e] = __uint_as_float(sr[e]);
          if (len < 32) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e >= len) s[e] = NEG_INF;
          }
          // exact offset: tile max over both halves, lazy (2^8) rescaling
          x_tile[half * BQ + row] = max32(s);
          quarter_sync();
          const float mnew = fmaxf(m, fmaxf(x_tile[row], x_tile[BQ + row]) * sl2);
          quarter_sync();  // both halves read before the next tile's write
          const bool need = mnew > m + 8.0f;
          if (__any_sync(0xffffffffu, need)) {
            const float alpha = need ? ex2(m - mnew) : 1.0f;
            if (j > 0) {
              // O must be stable: wait for PV of the previous tile; each half
              // rescales its 32 columns of O
              mbar_wait(BAR(C::B_PFREE + (gg - 1) % NB), ((gg - 1) / NB) & 1);
              tc_fence_after();
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                uint32_t orr[16];
                const uint32_t oc = tmem + lane_off + C::TM_O + half * 32 + c * 16;
                tmem_ld16(oc, orr);
                tmem_wait_ld();
                reg_fence16(orr);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                  orr[e] = __float_as_uint(__uint_as_float(orr[e]) * alpha);
                tmem_st16(oc, orr);
              }
            }
            if (need) {
              l *= alpha;
              m = mnew;
            }
          }
          l += exp_half<POLY, F16P>(s, sl2, m, tmem + lane_off + C::TM_S + sb * 64 + half * 32);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(C::B_PFULL + sb));
        }
      }
      // ---- epilogue: O / l; each warp writes its 64/NG columns of the row ----
      float ltot = 0.0f;
      if constexpr (EXACT || !LSUM) {
        x_l[grp * BQ + row] = l;
        quarter_sync();
#pragma unroll
        for (int q = 0; q < NG; ++q) ltot += x_l[q * BQ + row];
        if (!EXACT) ovf |= !(ltot <= 1.2676506e30f);
      }
      if (warp == 0 && lane == 0) BSA_TR(15, it);
      mbar_wait(BAR(C::B_OFULL), it & 1);
      tc_fence_after();
      if (warp == 0 && lane == 0) BSA_TR(17, it);
      if constexpr (!EXACT && LSUM) {
        // row sum of P from the tensor core (O column 64); an overflowed
        // stale offset shows up as inf / a huge sum -> exact repair launch
        uint32_t lr;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                     : "=r"(lr) : "r"(tmem + lane_off + C::TM_O + 64));
        tmem_wait_ld();
        asm volatile("" : "+r"(lr));
        ltot = __uint_as_float(lr);
        ovf = !(ltot <= 1.2676506e30f);  // 2^100: also keeps O = sum p v finite
      }
      if constexpr (X3) {
        // split-bf16 scores carry ~2^-16 relative error, i.e. an absolute
        // error growing with the logit: rows whose largest logit exceeds
        // X3_XLIM (log2 units) go to the exact CUDA-core repair as well
        x_tile[grp * BQ + row] = xm;
        quarter_sync();
        float xall = x_tile[row];
#pragma unroll
        for (int q = 1; q < NG; ++q) xall = fmaxf(xall, x_tile[q * BQ + row]);
        ovf |= !(fabsf(xall * sl2) <= X3_XLIM);
      }
      const bool store = row < I.rows;
      const int32_t pr = I.row0 + row;
      const int64_t dst = A.permuted_out ? pr : G.L.part_src(pr);
      // output row: local (H, T, d) buffer; (multi-GPU scatter) the buffer of
      // the rank owning token dst, (H, T_r, d), written over NVLink; or (key
      // ranges) this range's partial row, partitioned order, merged later
      const bool part = A.kr.nr > 1;
      const bool obf = part ? A.part_bf16 != 0 : A.out_bf16 != 0;
      const int64_t orow = part ? ((int64_t)I.r * G.H + I.h) * G.T + pr : (int64_t)I.h * G.T + dst;
      __nv_bfloat16* orow_bf16 = (__nv_bfloat16*)(part ? A.part_out : A.out) + orow * D;
      float* orow_f32 = (float*)(part ? A.part_out : A.out) + orow * D;
      if (!part && A.scatter_world > 0 && store) {
        int r = 0;
        while (r + 1 < A.scatter_world && dst >= A.token_begin[r + 1]) ++r;
        const int64_t t0 = A.token_begin[r], tr = A.token_begin[r + 1] - t0;
        orow_bf16 = (__nv_bfloat16*)A.out_ptrs[r] + ((int64_t)I.h * tr + (dst - t0)) * D;
      }
      const float inv = (F16P ? __int_as_float((127 - A.v_shift[I.h]) << 23) : 1.0f) / ltot;
      if (part && store && grp == 0) A.part_lse[orow] = m + log2f(ltot);
      // 16-column chunks c with c % NG == grp
      for (int c = grp; c < 4; c += NG) {
        const int col0 = c * 16;
        uint32_t orr[16];
        tmem_ld16(tmem + lane_off + C::TM_O + col0, orr);
        tmem_wait_ld();
        reg_fence16(orr);
        if (store) {
          if (obf) {
            uint4* op = reinterpret_cast<uint4*>(orow_bf16 + col0);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(orr[8 * q + 0]) * inv, __uint_as_float(orr[8 * q + 1]) * inv);
              v.y = pack_bf16(__uint_as_float(orr[8 * q + 2]) * inv, __uint_as_float(orr[8 * q + 3]) * inv);
              v.z = pack_bf16(__uint_as_float(orr[8 * q + 4]) * inv, __uint_as_float(orr[8 * q + 5]) * inv);
              v.w = pack_bf16(__uint_as_float(orr[8 * q + 6]) * inv, __uint_as_float(orr[8 * q + 7]) * inv);
              if (BSA_TC_L2HINT) __stcs(op + q, v);
              else op[q] = v;
            }
          } else {
            float4* op = reinterpret_cast<float4*>(orow_f32 + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              op[q] = make_float4(__uint_as_float(orr[4 * q]) * inv, __uint_as_float(orr[4 * q + 1]) * inv,
                                  __uint_as_float(orr[4 * q + 2]) * inv, __uint_as_float(orr[4 * q + 3]) * inv);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(C::B_OEMPTY));
      if (warp == 0 && lane == 0) BSA_TR(18, it);
      if constexpr (!EXACT) {
        // stale offset overflowed somewhere in this item: list it once for
        // the exact-max launch (which rewrites all of its rows)
        if ((grp == 0 || !LSUM) && __any_sync(0xffffffffu, ovf) && lane == 0) {
          if (atomicCAS(&A.ovf_flags[code], 0, 1) == 0) A.ovf_list[atomicAdd(A.ovf_count, 1)] = code;
        }
      }
      g += ntiles;
      ++it;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(C::TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
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

// 3-D (d, T, H) map of a 16-bit (H, T, 64) tensor with element strides sT, sH
static int make_map(CUtensorMap* map, const void* base, int64_t H, int64_t T, int box_rows,
                    int64_t sT, int64_t sH,
                    CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)tc::D, (cuuint64_t)T, (cuuint64_t)H};
  cuuint64_t strides[2] = {(cuuint64_t)sT * 2, (cuuint64_t)sH * 2};
  cuuint32_t box[3] = {(cuuint32_t)tc::D, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BSA_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BSA_OK;
}

size_t tc_smem_bytes() { return tc::CfgMain::SMEM_BYTES; }

// maps of one launch: K and V (bf16 or fp16 V), and (X3) the K / V lo parts
struct TcMaps {
  CUtensorMap k, v, kl, vl;
};

// events bracketing the most recent timed attention-kernel launch (per thread)
// a ring of TIMING_RING event pairs per thread: launch n records into slot
// n % TIMING_RING, so a caller can time every launch of a loop without a
// host sync inside it (bsa_kernel_times)
constexpr int TIMING_RING = 64;
struct TimingRing {
  cudaEvent_t ev[TIMING_RING][2] = {};
  int64_t count = 0;  // launches recorded since the last reset
};
static TimingRing& timing_ring() {
  static thread_local TimingRing r;
  return r;
}
cudaEvent_t timing_events(int which) {
  TimingRing& r = timing_ring();
  if (which == 0) ++r.count;  // a new launch opens the next slot
  const int slot = (int)((r.count - 1 + TIMING_RING) % TIMING_RING);
  if (!r.ev[slot][0]) {
    cudaEventCreate(&r.ev[slot][0]);
    cudaEventCreate(&r.ev[slot][1]);
  }
  return r.ev[slot][which];
}

template <int POLY, bool F16P, bool EXACT, bool X3 = false>
static int launch_variant(const TcMaps& m, const AttnGeom& G, const TcArgs& a, int grid,
                          cudaStream_t st) {
  using C = tc::Cfg<BSA_TC_WIDE != 0 && !EXACT, X3>;
  auto kern = tc::bsa_tc_kernel<POLY, F16P, EXACT, X3>;
  BSA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::SMEM_BYTES));
  kern<<<grid, C::NUM_THREADS, C::SMEM_BYTES, st>>>(m.kl, m.k, m.v, m.vl, G, a);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

template <bool EXACT>
static int launch_pick(const TcMaps& m, const AttnGeom& G, const TcArgs& a, int grid,
                       cudaStream_t st) {
  if (a.x3) {
    if constexpr (EXACT || !tc::LSUM) return fail(BSA_EINVAL, "X3 needs the stale-max launch with LSUM");
    else return launch_variant<0, false, false, true>(m, G, a, grid, st);
  }
  switch (a.exp_poly | (a.v_f16 ? 16 : 0)) {
    case 0: return launch_variant<0, false, EXACT>(m, G, a, grid, st);
    case 1: return launch_variant<1, false, EXACT>(m, G, a, grid, st);
    case 2: return launch_variant<2, false, EXACT>(m, G, a, grid, st);
    case 3: return launch_variant<3, false, EXACT>(m, G, a, grid, st);
    case 4: return launch_variant<4, false, EXACT>(m, G, a, grid, st);
#if BSA_TC_POLY_PER16
    case 5: return launch_variant<5, false, EXACT>(m, G, a, grid, st);
    case 6: return launch_variant<6, false, EXACT>(m, G, a, grid, st);
#endif
    case 16: return launch_variant<0, true, EXACT>(m, G, a, grid, st);
    case 18: return launch_variant<2, true, EXACT>(m, G, a, grid, st);
    case 19: return launch_variant<3, true, EXACT>(m, G, a, grid, st);
#if BSA_TC_H2
    case 20: return launch_variant<4, true, EXACT>(m, G, a, grid, st);
    case 21: return launch_variant<5, true, EXACT>(m, G, a, grid, st);
    case 22: return launch_variant<6, true, EXACT>(m, G, a, grid, st);
#endif
    default: return fail(BSA_EINVAL, "unknown tensor-core kernel variant");
  }
}

// Two launches: the stale-max kernel over this shard's LPT list (its length
// is on the device, written by the schedule kernel), then the exact-max
// kernel over the items it listed as overflowed (normally none: the second
// launch reads a zero count and its CTAs exit at once).  With a key-range
// split, the combine kernel then merges each row's range partials.
int launch_tc_attention(const AttnGeom& G, const TcArgs& a, cudaStream_t st,
                        const CombineArgs* comb, const SimtRepair* rep) {
  TcMaps m;
  int rc = make_map(&m.k, a.kp, G.H, G.T, tc::CH, a.kv_sT, a.kv_sH);
  if (!rc)
    rc = make_map(&m.v, a.vp, G.H, G.T, tc::CH, a.kv_sT, a.kv_sH,
                  a.v_f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  if (rc) return rc;
  m.kl = m.k;
  m.vl = m.v;
  if (a.x3) {
    rc = make_map(&m.kl, a.kp_lo, G.H, G.T, tc::CH, a.kv_sT, a.kv_sH);
    if (!rc) rc = make_map(&m.vl, a.vp_lo, G.H, G.T, tc::CH, a.kv_sT, a.kv_sH);
    if (rc) return rc;
    if (!rep) return fail(BSA_EINVAL, "X3 launch needs the SIMT repair inputs");
  }
  int dev = 0, sms = 148;
  BSA_CUDA_TRY(cudaGetDevice(&dev));
  BSA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = (int)std::min<int64_t>((int64_t)sms * tc::CfgMain::CTAS_PER_SM,
                                          std::max<int64_t>(1, a.n_items));
  static_assert(tc::Cfg<true, true>::CTAS_PER_SM == tc::CfgMain::CTAS_PER_SM, "X3 grid");
  BSA_CUDA_TRY(cudaMemsetAsync(a.ovf_flags, 0, (size_t)a.n_items * 4, st));
  BSA_CUDA_TRY(cudaMemsetAsync(a.ovf_count, 0, 4, st));
  if (a.timing) BSA_CUDA_TRY(cudaEventRecord(timing_events(0), st));
  rc = launch_pick<false>(m, G, a, grid, st);
  if (rc) return rc;
  if (!a.x3) {
    TcArgs r = a;  // repair launch
    r.items = a.ovf_list;
    r.n_items_dev = a.ovf_count;
    r.work_counter = a.work_counter + 1;
    rc = launch_pick<true>(m, G, r, sms, st);
    if (rc) return rc;
  }
  if (a.kr.nr > 1 && comb) {
    rc = launch_combine(G, *comb, st);
    if (rc) return rc;
  }
  if (a.x3) {
    // overflowed items (stale offset exceeded by ~2^100): whole rows again on
    // the CUDA cores, exact online softmax, after the combine so they win
    SimtList sl;
    sl.list = a.ovf_list;
    sl.count = a.ovf_count;
    sl.nst = ceil_div(G.Ts, 128);
    sl.M = sl.nst + G.nq;
    sl.nr = a.kr.nr;
    sl.cap = a.n_items;
    rc = launch_simt_attention_list(rep->q, rep->k, rep->v, a.out, a.out_bf16 ? BSA_BF16 : BSA_F32,
                                    G, a.bits, a.permuted_out, rep->scale, sl, st);
    if (rc) return rc;
  }
  if (a.timing) BSA_CUDA_TRY(cudaEventRecord(timing_events(1), st));
  if (a.trace) {
    // debug only: dump the CTA-0 pipeline trace (BSA_TC_TRACE=<file>)
    BSA_CUDA_TRY(cudaStreamSynchronize(st));
    static unsigned long long host[tc::TRACE_EVENTS * tc::TRACE_TILES];
    BSA_CUDA_TRY(cudaMemcpy(host, a.trace, sizeof(host), cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(getenv("BSA_TC_TRACE"), "wb")) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
  }
  return BSA_OK;
}

}  // namespace bsa

extern "C" float bsa_last_kernel_ms(void) {
  bsa::TimingRing& r = bsa::timing_ring();
  if (r.count < 1) return -1.0f;
  const int slot = (int)((r.count - 1) % bsa::TIMING_RING);
  float ms = -1.0f;
  if (cudaEventSynchronize(r.ev[slot][1]) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, r.ev[slot][0], r.ev[slot][1]) != cudaSuccess) return -1.0f;
  return ms;
}

extern "C" int bsa_kernel_times(float* out, int32_t max_n, int32_t reset) {
  bsa::TimingRing& r = bsa::timing_ring();
  const int64_t avail = std::min<int64_t>(r.count, bsa::TIMING_RING);
  const int n = (int)std::min<int64_t>(avail, max_n > 0 ? max_n : 0);
  for (int i = 0; i < n; ++i) {  // the n most recent launches, oldest first
    const int slot = (int)((r.count - n + i) % bsa::TIMING_RING);
    if (cudaEventSynchronize(r.ev[slot][1]) != cudaSuccess ||
        cudaEventElapsedTime(out + i, r.ev[slot][0], r.ev[slot][1]) != cudaSuccess)
      return -1;
  }
  if (reset) r.count = 0;
  return n;
}
