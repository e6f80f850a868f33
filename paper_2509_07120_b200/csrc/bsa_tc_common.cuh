// bsa_tc_common.cuh -- shared pieces of the tcgen05 kernels (attention:
// bsa_attn_tc.cu; dense attention statistics: bsa_stats_tc.cu): PTX wrappers
// for mbarriers / TMA / tcgen05, UMMA descriptors, and the work-item decoding
// of the (head, q-block) key streams.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bsa_attn.cuh"

namespace bsa {
namespace tc {

constexpr int BQ = 128, CH = 64, D = 64;
constexpr int CHUNK_BYTES = CH * D * 2;  // 8 KB (one K or V tile)

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
#ifndef BSA_TC_WAIT
#define BSA_TC_WAIT 1
#endif
// mbarrier phase wait.  0: try_wait with a suspend-time hint (the thread may
// sleep; slow wake-up), 1: try_wait without hint (hardware-bounded blocking
// poll), 2: test_wait spin.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if BSA_TC_WAIT == 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(0x989680u)
      : "memory");
#elif BSA_TC_WAIT == 1
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}
// two phase waits at once (both try_waits in flight before one branch): for
// issuer warps whose barriers are usually complete already
__device__ __forceinline__ void mbar_wait2(uint32_t a, uint32_t pa, uint32_t b, uint32_t pb) {
  asm volatile(
      "{\n\t.reg .pred P1, P2;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P2, [%2], %3;\n\t"
      "and.pred P1, P1, P2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(pa), "r"(b), "r"(pb)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// L2 cache policies (createpolicy): K/V tiles are re-read by every q-block
// of their head (keep), Q rows and output rows are touched once (stream)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int c0, int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
// one lane of a converged warp (elect.sync): keeps the caller warp-uniform
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// ties later uses of tcgen05.ld results to after tcgen05.wait::ld
__device__ __forceinline__ void reg_fence16(uint32_t* r) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt_h2(float lo, float hi) {
  uint32_t y;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(hi), "f"(lo));
  return y;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t y;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(y) : "r"(a), "r"(b));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// UMMA shared-memory descriptor: SWIZZLE_128B, version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// instruction descriptor kind::f16 -> f32 accumulate; fmt 0 = f16, 1 = bf16
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int b_mn_major, int fmt) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// max of 32 values (3-input max tree)
__device__ __forceinline__ float max32(const float (&s)[32]) {
  float mx4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) mx4[i] = fmaxf(s[i], s[4 + i]);
#pragma unroll
  for (int e = 8; e < 32; e += 4)
#pragma unroll
    for (int i = 0; i < 4; ++i) mx4[i] = fmaxf(mx4[i], s[e + i]);
  return fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
}


// ---------------------------------------------------------------------------
// work item decoding
// ---------------------------------------------------------------------------
struct Item {
  int32_t h;
  int32_t qb;       // -1 for a special-row tile
  int32_t row0;     // first partitioned query row
  int32_t rows;     // valid query rows
  int32_t nchunks;  // 64-key tiles in the key stream
  int32_t last_len; // length of the final tile (ragged tails)
  int32_t nsc;      // leading contiguous tiles (special strip / all keys)
  int32_t spec_last;  // length of the last contiguous tile
  int32_t r;        // key range (KeyRanges; 0 when the keys are not split)
  int32_t kstart;   // first key of the contiguous part of the stream
};

// item code = (h * nr + r) * M + li, M = ceil(Ts / BQ) + nq; li < ceil(Ts/BQ)
// is a special-row tile, else patch q-block li - ceil(Ts/BQ).
// 32-bit fields: the tensor-core path requires T < 2^31 and H < 65536.
__device__ __forceinline__ Item decode(const AttnGeom& G, int32_t code, const int32_t* counts,
                                       const uint8_t* bits, const KeyRanges& KR) {
  Item it;
  const int32_t nst = (int32_t)ceil_div(G.Ts, BQ);
  const int32_t M = nst + (int32_t)G.nq;
  const int32_t T = (int32_t)G.T, Ts = (int32_t)G.Ts, Tp = (int32_t)G.Tp;
  const int32_t hr = code / M;
  const int32_t li = code - hr * M;
  it.h = hr / KR.nr;
  it.r = hr - it.h * KR.nr;
  const int32_t rkeys = KR.rb * CH;
  if (li < nst) {
    it.qb = -1;
    it.row0 = li * BQ;
    it.rows = min(BQ, Ts - it.row0);
    // keys [kstart, kend): range 0 also holds the special keys
    it.kstart = it.r == 0 ? 0 : Ts + it.r * rkeys;
    const int32_t kend = it.r == KR.nr - 1 ? T : Ts + (it.r + 1) * rkeys;
    const int32_t len = kend - it.kstart;
    it.nsc = (len + CH - 1) / CH;
    it.spec_last = len - (it.nsc - 1) * CH;
    it.nchunks = it.nsc;
    it.last_len = it.spec_last;
  } else {
    it.qb = li - nst;
    it.row0 = Ts + it.qb * BQ;
    it.rows = min(BQ, Tp - it.qb * BQ);
    it.kstart = 0;
    it.nsc = it.r == 0 ? (Ts + CH - 1) / CH : 0;
    it.spec_last = it.nsc ? Ts - (it.nsc - 1) * CH : CH;
    const int64_t row = (int64_t)it.h * G.nq + it.qb;
    const int32_t cnt = KR.nr == 1 ? counts[row] : KR.rcounts[row * KR.nr + it.r];
    it.nchunks = it.nsc + cnt;
    // the ragged last patch block, if selected (and in this range), is
    // always the final tile
    const int32_t lastb = (int32_t)G.nk - 1;
    const uint8_t lb = bits[row * G.mask_row_bytes + (lastb >> 3)];
    const bool last_sel = ((lb >> (lastb & 7)) & 1) && lastb / KR.rb == it.r;
    it.last_len = last_sel ? Tp - lastb * CH : CH;
    if (cnt == 0) it.last_len = it.spec_last;
  }
  return it;
}

// end of the contiguous part of an item's key stream
__device__ __forceinline__ int32_t contig_end(const Item& it) {
  return it.nsc ? it.kstart + (it.nsc - 1) * CH + it.spec_last : it.kstart;
}

__device__ __forceinline__ int chunk_len(const Item& it, int c) {
  if (c < it.nsc - 1) return CH;
  if (c == it.nsc - 1) return it.nchunks == it.nsc ? it.last_len : it.spec_last;
  return c == it.nchunks - 1 ? it.last_len : CH;
}

// 2^x for a pair on the FMA pipe (x < 128): round-to-nearest split
// x = j + f, f in [-0.5, 0.5], minimax polynomial for 2^f, exponent added as
// an integer.  Degree 3: max rel err 7.5e-5 (for fp16 P); degree 2: 1.7e-3,
// below the 2^-9 rounding of a bf16 P, one f32x2 FMA cheaper.
template <int DEG>
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
#if !defined(BSA_TC_EXPERIMENT) || BSA_TC_EXPERIMENT != 4
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
#endif
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 j = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
  float2 p;
  if constexpr (DEG == 2) {
    p = __ffma2_rn(make_float2(0.23842570f, 0.23842570f), f, make_float2(0.70344281f, 0.70344281f));
    p = __ffma2_rn(p, f, make_float2(1.00044298f, 1.00044298f));
  } else {
    p = __ffma2_rn(make_float2(0.05517132f, 0.05517132f), f, make_float2(0.24261054f, 0.24261054f));
    p = __ffma2_rn(p, f, make_float2(0.69326097f, 0.69326097f));
    p = __ffma2_rn(p, f, make_float2(0.99992812f, 0.99992812f));
  }
  // (t_bits << 23) == (j << 23) mod 2^32 because t = 1.5*2^23 + j
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

}  // namespace tc
}  // namespace bsa
