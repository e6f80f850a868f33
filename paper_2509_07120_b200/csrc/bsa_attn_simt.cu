// bsa_attn_simt.cu -- CUDA-core block-sparse attention (fp32 math).
//
// The exact-arithmetic companion of the tcgen05 kernel: any head_dim <= 128,
// any block sizes, fp32 or bf16 inputs, fp32 accumulation and a full-precision
// expf.  It is the device path for config 1 (fp32, <= 1e-4 max-abs vs the
// reference) and for the odd geometries of the reference's own tests
// (block_q 32/48/64, block_k 16/32, head_dim 8/16/32).
//
// Semantics follow /root/reference/pkg/src/bsattn/sparse.py:
//   special query rows (sparse.py:122-131): softmax over every key;
//   patch query rows (sparse.py:101-119): the special-key strip first, then
//   the selected key blocks in ascending order, merged with the online
//   softmax update of sparse.py:89-98.  Unselected blocks contribute nothing.
// Inputs are read in interleaved source order with the [specials | patches]
// permutation (layout.py:113-132) folded into row addressing, and outputs
// are written back in source order (sparse.py:176-177, :205).
#include <algorithm>

#include "bsa_attn.cuh"

namespace bsa {

constexpr int SM_ROWS = 32;    // query rows per CTA
constexpr int SM_CHUNK = 64;   // keys per smem chunk
constexpr int SM_THREADS = 256;

// one 32-row tile ti of head h (special-row tiles first, then 4 tiles per
// patch q-block of 128 rows)
template <typename T, int DMAX>
__device__ void simt_tile(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                          int64_t qsH, int64_t qsT, int64_t ksH, int64_t ksT, int64_t vsH,
                          int64_t vsT, void* __restrict__ out, int out_bf16, const AttnGeom& G,
                          const uint8_t* __restrict__ mask_bits, int permuted, float scale,
                          int64_t h, int64_t ti) {
  extern __shared__ float smem_f[];
  float (*Qs)[DMAX] = reinterpret_cast<float (*)[DMAX]>(smem_f);
  float (*Ks)[DMAX + 1] = reinterpret_cast<float (*)[DMAX + 1]>(smem_f + SM_ROWS * DMAX);
  float (*Vs)[DMAX] =
      reinterpret_cast<float (*)[DMAX]>(smem_f + SM_ROWS * DMAX + SM_CHUNK * (DMAX + 1));
  const int64_t nspec_tiles = ceil_div(G.Ts, SM_ROWS);
  const int sub_per_qb = (int)ceil_div(G.bq, SM_ROWS);

  int64_t row0, row1;  // partitioned query rows [row0, row1)
  int64_t qb = -1;
  if (ti < nspec_tiles) {
    row0 = ti * SM_ROWS;
    row1 = min(G.Ts, row0 + SM_ROWS);
  } else {
    const int64_t pi = ti - nspec_tiles;
    qb = pi / sub_per_qb;
    const int64_t s = pi % sub_per_qb;
    const int64_t qb0 = qb * G.bq, qb1 = min(G.Tp, qb0 + G.bq);
    row0 = G.Ts + qb0 + s * SM_ROWS;
    row1 = min(G.Ts + qb1, row0 + SM_ROWS);
    if (row0 >= row1) return;
  }
  const int d = G.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // stage Q rows (fp32)
  for (int idx = tid; idx < SM_ROWS * DMAX; idx += SM_THREADS) {
    const int r = idx / DMAX, c = idx % DMAX;
    float val = 0.0f;
    const int64_t pr = row0 + r;
    if (pr < row1 && c < d) {
      const int64_t src = permuted ? pr : G.L.part_src(pr);
      val = to_f32(q[h * qsH + src * qsT + c]);
    }
    Qs[r][c] = val;
  }

  constexpr int RPW = SM_ROWS / 8;  // rows per warp
  constexpr int DPL = DMAX / 32;    // output dims per lane
  float m[RPW], l[RPW], o[RPW][DPL];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    m[r] = -__int_as_float(0x7f800000);
    l[r] = 0.0f;
#pragma unroll
    for (int u = 0; u < DPL; ++u) o[r][u] = 0.0f;
  }

  KeyChunker ck(G, qb, mask_bits ? mask_bits + (h * G.nq + (qb < 0 ? 0 : qb)) * G.mask_row_bytes : nullptr,
                SM_CHUNK);
  int64_t kstart;
  int klen;
  while (ck.next(kstart, klen)) {
    __syncthreads();
    for (int idx = tid; idx < SM_CHUNK * DMAX; idx += SM_THREADS) {
      const int j = idx / DMAX, c = idx % DMAX;
      float kv = 0.0f, vv = 0.0f;
      if (j < klen && c < d) {
        const int64_t pr = kstart + j;
        const int64_t src = permuted ? pr : G.L.part_src(pr);
        kv = to_f32(k[h * ksH + src * ksT + c]);
        vv = to_f32(v[h * vsH + src * vsT + c]);
      }
      Ks[j][c] = kv;
      Vs[j][c] = vv;
    }
    __syncthreads();
    // scores for keys lane and lane+32, RPW rows
    float s0[RPW], s1[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) { s0[r] = 0.0f; s1[r] = 0.0f; }
    for (int c = 0; c < d; ++c) {
      const float k0 = Ks[lane][c], k1 = Ks[lane + 32][c];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const float qv = Qs[warp * RPW + r][c];
        s0[r] = fmaf(qv, k0, s0[r]);
        s1[r] = fmaf(qv, k1, s1[r]);
      }
    }
    const float NEG_INF = -__int_as_float(0x7f800000);
    float p0[RPW], p1[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const float a = lane < klen ? s0[r] * scale : NEG_INF;
      const float b = lane + 32 < klen ? s1[r] * scale : NEG_INF;
      float cm = fmaxf(a, b);
#pragma unroll
      for (int off = 16; off; off >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
      const float mn = fmaxf(m[r], cm);
      const float alpha = expf(m[r] - mn);
      p0[r] = expf(a - mn);
      p1[r] = expf(b - mn);
      float ps = p0[r] + p1[r];
#pragma unroll
      for (int off = 16; off; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      l[r] = l[r] * alpha + ps;
      m[r] = mn;
#pragma unroll
      for (int u = 0; u < DPL; ++u) o[r][u] *= alpha;
    }
    const int jmax = min(klen, SM_CHUNK);
    for (int j = 0; j < jmax; ++j) {
      float vv[DPL];
#pragma unroll
      for (int u = 0; u < DPL; ++u) vv[u] = Vs[j][lane + 32 * u];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0[r] : p1[r], j & 31);
#pragma unroll
        for (int u = 0; u < DPL; ++u) o[r][u] = fmaf(pj, vv[u], o[r][u]);
      }
    }
  }
  // epilogue
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int64_t pr = row0 + warp * RPW + r;
    if (pr >= row1) continue;
    const int64_t dst = permuted ? pr : G.L.part_src(pr);
    const float inv = 1.0f / l[r];
#pragma unroll
    for (int u = 0; u < DPL; ++u) {
      const int c = lane + 32 * u;
      if (c >= d) continue;
      const float val = o[r][u] * inv;
      const int64_t off = (h * G.T + dst) * d + c;
      if (out_bf16) reinterpret_cast<__nv_bfloat16*>(out)[off] = __float2bfloat16(val);
      else reinterpret_cast<float*>(out)[off] = val;
    }
  }
}

template <typename T, int DMAX>
__global__ void __launch_bounds__(SM_THREADS)
    simt_attn_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                     int64_t qsH, int64_t qsT, int64_t ksH, int64_t ksT, int64_t vsH,
                     int64_t vsT, void* __restrict__ out, int out_bf16, AttnGeom G,
                     const uint8_t* __restrict__ mask_bits, int permuted, float scale,
                     int shard, int num_shards) {
  const int64_t tiles_per_head = G.simt_tiles_per_head();
  int64_t item = blockIdx.x;
  if (num_shards > 1) {
    if (item % num_shards != shard) return;
  }
  simt_tile<T, DMAX>(q, k, v, qsH, qsT, ksH, ksT, vsH, vsT, out, out_bf16, G, mask_bits, permuted,
                     scale, item / tiles_per_head, item % tiles_per_head);
}

// recomputes listed tensor-core items (128-row tiles: 4 SIMT tiles each)
template <typename T, int DMAX>
__global__ void __launch_bounds__(SM_THREADS)
    simt_list_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                     int64_t qsH, int64_t qsT, int64_t ksH, int64_t ksT, int64_t vsH,
                     int64_t vsT, void* __restrict__ out, int out_bf16, AttnGeom G,
                     const uint8_t* __restrict__ mask_bits, int permuted, float scale,
                     SimtList sl) {
  const int64_t n = 4 * (int64_t)*sl.count;
  const int64_t nspec_tiles = ceil_div(G.Ts, SM_ROWS);
  const int64_t sub_per_qb = ceil_div(G.bq, SM_ROWS);
  for (int64_t idx = blockIdx.x; idx < n; idx += gridDim.x) {
    const int32_t code = sl.list[idx / 4];
    const int sub = (int)(idx % 4);
    const int64_t li = code % sl.M, h = (code / sl.M) / sl.nr;
    int64_t ti;
    if (li < sl.nst) {
      ti = li * 4 + sub;
      if (ti >= nspec_tiles) continue;
    } else {
      if (sub >= sub_per_qb) continue;
      ti = nspec_tiles + (li - sl.nst) * sub_per_qb + sub;
    }
    __syncthreads();  // the previous tile's warps are done with shared memory
    simt_tile<T, DMAX>(q, k, v, qsH, qsT, ksH, ksT, vsH, vsT, out, out_bf16, G, mask_bits,
                       permuted, scale, h, ti);
  }
}

template <typename T, int DMAX>
static int launch_simt_t(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                         void* out, int out_dtype, const AttnGeom& G, const uint8_t* bits,
                         int permuted, float scale, int shard, int num_shards, cudaStream_t st) {
  const int64_t items = G.H * G.simt_tiles_per_head();
  if (items > 0x7fffffffLL) return fail(BSA_EUNSUPPORTED, "too many SIMT tiles");
  const size_t smem = sizeof(float) * (SM_ROWS * DMAX + SM_CHUNK * (DMAX + 1) + SM_CHUNK * DMAX);
  BSA_CUDA_TRY(cudaFuncSetAttribute(simt_attn_kernel<T, DMAX>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  simt_attn_kernel<T, DMAX><<<(unsigned)items, SM_THREADS, smem, st>>>(
      (const T*)q->data, (const T*)k->data, (const T*)v->data, q->stride_head, q->stride_token,
      k->stride_head, k->stride_token, v->stride_head, v->stride_token, out,
      out_dtype == BSA_BF16, G, bits, permuted, scale, shard, num_shards);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

int launch_simt_attention_list(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                               void* out, int out_dtype, const AttnGeom& G, const uint8_t* bits,
                               int permuted, float scale, const SimtList& sl, cudaStream_t st) {
  if (q->dtype != BSA_F32 || G.d != 64 || G.bq != 128)
    return fail(BSA_EUNSUPPORTED, "SIMT item repair: fp32 inputs, head_dim 64, block_q 128");
  constexpr int DMAX = 64;
  const size_t smem = sizeof(float) * (SM_ROWS * DMAX + SM_CHUNK * (DMAX + 1) + SM_CHUNK * DMAX);
  BSA_CUDA_TRY(cudaFuncSetAttribute(simt_list_kernel<float, DMAX>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)std::min<int64_t>(std::max<int64_t>(4 * sl.cap, 1), 148 * 4);
  simt_list_kernel<float, DMAX><<<grid, SM_THREADS, smem, st>>>(
      (const float*)q->data, (const float*)k->data, (const float*)v->data, q->stride_head,
      q->stride_token, k->stride_head, k->stride_token, v->stride_head, v->stride_token, out,
      out_dtype == BSA_BF16, G, bits, permuted, scale, sl);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

int launch_simt_attention(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                          void* out, int out_dtype, const AttnGeom& G, const uint8_t* bits,
                          int permuted, float scale, int shard, int num_shards, cudaStream_t st) {
  const bool bf = q->dtype == BSA_BF16;
  if (G.d <= 32)
    return bf ? launch_simt_t<__nv_bfloat16, 32>(q, k, v, out, out_dtype, G, bits, permuted, scale, shard, num_shards, st)
              : launch_simt_t<float, 32>(q, k, v, out, out_dtype, G, bits, permuted, scale, shard, num_shards, st);
  if (G.d <= 64)
    return bf ? launch_simt_t<__nv_bfloat16, 64>(q, k, v, out, out_dtype, G, bits, permuted, scale, shard, num_shards, st)
              : launch_simt_t<float, 64>(q, k, v, out, out_dtype, G, bits, permuted, scale, shard, num_shards, st);
  if (G.d <= 128)
    return bf ? launch_simt_t<__nv_bfloat16, 128>(q, k, v, out, out_dtype, G, bits, permuted, scale, shard, num_shards, st)
              : launch_simt_t<float, 128>(q, k, v, out, out_dtype, G, bits, permuted, scale, shard, num_shards, st);
  return fail(BSA_EUNSUPPORTED, "head_dim %d > 128 is not supported", G.d);
}

}  // namespace bsa
