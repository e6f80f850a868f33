// bsa_select.cuh -- pieces of the scoring stage shared by the three-kernel
// path (bsa_score.cu) and the fused score+softmax+select kernel
// (bsa_scoresel.cu): exact fixed-point probability mass, numpy's pairwise
// leaf sum, and the fused launcher's interface.
#pragma once
#include "bsa_common.cuh"

namespace bsa {

// value of a non-negative finite float < 2 in units of 2^-52, exact for
// p >= 2^-29 (the fp32 ulp is then >= 2^-52), truncated below that.
__device__ __forceinline__ unsigned long long fx52(unsigned int key) {
  const unsigned int E = key >> 23;
  if (E == 0) return 0ull;
  const unsigned long long m = (unsigned long long)((key & 0x7fffffu) | 0x800000u);
  const int sh = (int)E - 98;
  if (sh >= 0) return m << sh;
  return sh > -40 ? (m >> (-sh)) : 0ull;
}

constexpr unsigned int KEY_TINY = 98u << 23;   // bits of 2^-29
constexpr unsigned int KEY_TWO = 128u << 23;   // bits of 2.0f

// numpy pairwise_sum leaf (n <= 128) over contiguous smem values
__device__ __forceinline__ float pw_leaf_smem(const float* a, int n) {
  if (n < 8) {
    float r = 0.0f;
    for (int i = 0; i < n; ++i) r = __fadd_rn(r, a[i]);
    return r;
  }
  float r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], a[i + j]);
  float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __fadd_rn(res, a[i]);
  return res;
}


// ---------------------------------------------------------------------------
// fused score + softmax + select (bsa_scoresel.cu)
// ---------------------------------------------------------------------------
// blocked, transposed pooled K: [H][nchunks][d][FS_KC] (zero padded)
constexpr int FS_KC = 128;
inline int64_t fs_nchunks(int64_t nk) { return (nk + FS_KC - 1) / FS_KC; }
inline size_t fs_kblock_bytes(int64_t H, int64_t nk, int64_t d) {
  return (size_t)H * (size_t)fs_nchunks(nk) * (size_t)d * FS_KC * 4;
}
// rows per CTA the fused kernel would use for this shape (0: not eligible)
int fs_rows_per_cta(int64_t nk, int64_t d);
// pooled Q (H, nq, d) and pooled K (H, nk, d) fp32 -> mask bits / counts
// (probabilities to probs_out when non-null).  Rows whose selection cannot be
// proven exact on the fast path get their probabilities written to
// fb_probs + r*nk and are listed in fb_list / fb_count (*fb_count zeroed by
// the caller) for fallback_kernel.  kb: fs_kblock_bytes() of workspace.
// returned by launch_scoresel (before its kernel) when the GPU cannot
// co-schedule the cluster shape; the caller then runs the three kernels
constexpr int FS_NO_CLUSTER = 1000;
int launch_scoresel(const float* qp, const float* kp, int64_t H, int64_t nq, int64_t nk,
                    int64_t d, float scale, double tau, int64_t k_floor, float* kb,
                    uint8_t* bits, int32_t* counts, float* probs_out, float* fb_probs,
                    int32_t* fb_list, int32_t* fb_count, cudaStream_t st);

}  // namespace bsa
