// bsa_attn_host.cu -- attention-stage entry points of the C ABI, plus the
// small device passes around the attention kernels:
//   pack_kernel      source order (f32|bf16, any strides) -> contiguous bf16
//                    [specials | patches] order (layout.py:113-132), the TMA
//                    operand layout of the tcgen05 kernel.
//   counts_kernel    per-row popcount of the .bsm bitsets.
//   schedule_kernel  per head, an LPT (longest-first) counting sort of the
//                    work items (special-row tiles, patch q-blocks) by their
//                    key-tile count; heads stay contiguous so the K/V of one
//                    head stay L2-resident while the SMs drain it.
//   area_kernel      BlockMask.selected_area (maskpred.py:97-101).
//   csr kernels      CSR view of the mask.
#include <algorithm>
#include <cstring>
#include <cstdlib>

#include "bsa_attn.cuh"

namespace bsa {

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <typename T>
__global__ void pack_kernel(const T* __restrict__ x, int64_t sH, int64_t sT, int64_t H,
                            int64_t ntok, int d, Layout L, int permuted,
                            __nv_bfloat16* __restrict__ out, __nv_bfloat16* __restrict__ lo) {
  // one thread per 8 output elements (d % 8 == 0)
  const int64_t per_row = d / 8;
  const int64_t total = H * ntok * per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c8 = i % per_row;
    const int64_t hr = i / per_row;
    const int64_t r = hr % ntok, h = hr / ntok;
    const int64_t src = permuted ? r : L.part_src(r);
    const T* p = x + h * sH + src * sT + c8 * 8;
    float v[8];
    if constexpr (sizeof(T) == 4) {
      const float4 a = *reinterpret_cast<const float4*>(p);
      const float4 b = *reinterpret_cast<const float4*>(p + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      uint4 o;
      __nv_bfloat162 t;
      t = __floats2bfloat162_rn(v[0], v[1]); o.x = *reinterpret_cast<uint32_t*>(&t);
      t = __floats2bfloat162_rn(v[2], v[3]); o.y = *reinterpret_cast<uint32_t*>(&t);
      t = __floats2bfloat162_rn(v[4], v[5]); o.z = *reinterpret_cast<uint32_t*>(&t);
      t = __floats2bfloat162_rn(v[6], v[7]); o.w = *reinterpret_cast<uint32_t*>(&t);
      *reinterpret_cast<uint4*>(out + hr * d + c8 * 8) = o;
      if (lo) {
        // the residual x - bf16(x) (exact in fp32), rounded to bf16: hi + lo
        // carries ~16 significant bits (the X3 tensor-core path)
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
        uint32_t r[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 h = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
          t = __floats2bfloat162_rn(v[2 * e] - h.x, v[2 * e + 1] - h.y);
          r[e] = *reinterpret_cast<uint32_t*>(&t);
        }
        *reinterpret_cast<uint4*>(lo + hr * d + c8 * 8) = make_uint4(r[0], r[1], r[2], r[3]);
      }
    } else {
      *reinterpret_cast<uint4*>(out + hr * d + c8 * 8) = *reinterpret_cast<const uint4*>(p);
    }
  }
}

// per-head max |v| (as float bits: non-negative floats order like integers)
template <typename T>
__global__ void vamax_kernel(const T* __restrict__ x, int64_t sH, int64_t sT, int64_t ntok, int d,
                             unsigned int* __restrict__ amax) {
  const int64_t h = blockIdx.y;
  unsigned int m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ntok * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d, c = i - r * d;
    m = max(m, __float_as_uint(fabsf(to_f32(x[h * sH + r * sT + c]))));
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(&amax[h], m);
}

// V -> fp16 in partitioned order, scaled by 2^shift[h] so that max|v| lands in
// [2^14, 2^15) (power-of-two scaling is exact; the epilogue divides it out)
template <typename T>
__global__ void pack_v_kernel(const T* __restrict__ x, int64_t sH, int64_t sT, int64_t H,
                              int64_t ntok, int d, Layout L, int permuted,
                              const unsigned int* __restrict__ amax, int32_t* __restrict__ shift,
                              __half* __restrict__ out) {
  const int64_t per_row = d / 8;
  const int64_t total = H * ntok * per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c8 = i % per_row;
    const int64_t hr = i / per_row;
    const int64_t r = hr % ntok, h = hr / ntok;
    const unsigned int am = amax[h];
    const int e = (am >> 23) == 0 ? -126 : (int)(am >> 23) - 127;
    int sft = am == 0u ? 0 : 14 - e;
    sft = max(-100, min(100, sft));
    if (r == 0 && c8 == 0) shift[h] = sft;
    const float mul = exp2f((float)sft);
    const int64_t src = permuted ? r : L.part_src(r);
    const T* p = x + h * sH + src * sT + c8 * 8;
    uint4 o;
    uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      __half2 t = __floats2half2_rn(to_f32(p[2 * k]) * mul, to_f32(p[2 * k + 1]) * mul);
      ow[k] = *reinterpret_cast<uint32_t*>(&t);
    }
    *reinterpret_cast<uint4*>(out + hr * d + c8 * 8) = o;
  }
}

__global__ void counts_kernel(const uint8_t* __restrict__ bits, int64_t rows, int64_t row_bytes,
                              int32_t* __restrict__ counts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint8_t* b = bits + r * row_bytes;
  int c = 0;
  for (int64_t i = 0; i < row_bytes; ++i) c += __popc((unsigned)b[i]);
  counts[r] = c;
}

// ---------------------------------------------------------------------------
// LPT work list.  Row tiles per head: nst special tiles (rows of 128), then
// nq patch q-blocks.  Item code = (h * nr + r) * M + li (bsa_tc_common.cuh).
//
// Deterministic stable counting sorts by descending cost (histogram in
// parallel, placement by warp 0 walking the rows in index order, 32 at a
// time, __match_any_sync ranking equal costs).  Every rank of a multi-GPU run
// builds the same order independently:
//   1. (num_shards > 1) rows of a head in LPT order of their total cost are
//      dealt round-robin to the shards: row_shard[h][li] = position % shards.
//      All key ranges of a row stay on one shard, so its partials can be
//      merged locally.
//   2. per key range r: this shard's rows with keys in range r, LPT by their
//      range cost, appended to the head's list.
// Heads stay contiguous, then ranges within a head, so one (head, range)'s
// K/V stays L2-resident while the SMs drain it.  compact_kernel packs the
// per-head lists and leaves the item count on the device.
// ---------------------------------------------------------------------------
struct SchedGeom {
  int64_t nq, nst, M, nsc, T, Ts;
  int32_t nr, rb;
  int64_t max_cost;
  int32_t lpt;  // 0: every row costs the same (row order; BSA_FLAG_NATURAL_ORDER)
};

// chunks of row tile li of head h in key range r (0: no keys there)
__device__ __forceinline__ int64_t range_cost(const SchedGeom& S, const int32_t* counts,
                                              const int32_t* rcounts, int64_t h, int64_t li,
                                              int32_t r) {
  int64_t c;
  if (li < S.nst) {
    const int64_t rkeys = (int64_t)S.rb * 64;
    const int64_t k0 = r == 0 ? 0 : S.Ts + r * rkeys;
    const int64_t k1 = r == S.nr - 1 ? S.T : S.Ts + (r + 1) * rkeys;
    c = k1 > k0 ? (k1 - k0 + 63) / 64 : 0;
  } else {
    const int64_t row = h * S.nq + (li - S.nst);
    c = (r == 0 ? S.nsc : 0) + (S.nr == 1 ? counts[row] : rcounts[row * S.nr + r]);
  }
  return min(c, S.max_cost);
}

// stable descending counting sort of the rows with cost(i) >= 0:
// out[k] = base + i for the k-th longest; returns how many were placed
template <class CostF>
__device__ int32_t lpt_place(int64_t M, int64_t max_cost, int32_t* hist, CostF cost,
                             int32_t* out, int32_t base) {
  __shared__ int32_t total;
  for (int64_t c = threadIdx.x; c <= max_cost; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    const int64_t c = cost(i);
    if (c >= 0) atomicAdd(&hist[c], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t run = 0;  // descending cost: longest first
    for (int64_t c = max_cost; c >= 0; --c) {
      const int32_t n = hist[c];
      hist[c] = run;
      run += n;
    }
    total = run;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    for (int64_t i0 = 0; i0 < M; i0 += 32) {
      const int64_t i = i0 + lane;
      const int c = i < M ? (int)cost(i) : -1;
      const bool valid = c >= 0;
      const unsigned active = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        const unsigned same = __match_any_sync(active, c);
        const int rank = __popc(same & ((1u << lane) - 1u));
        const int32_t at = hist[c];
        out[at + rank] = base + (int32_t)i;
        __syncwarp(active);
        if (rank == 0) hist[c] = at + __popc(same);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(1024)
    schedule_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ rcounts,
                    SchedGeom S, int num_shards, int shard, int32_t* __restrict__ row_shard,
                    int32_t* __restrict__ tmp, int32_t* __restrict__ head_count) {
  extern __shared__ int32_t hist[];  // max_cost + 1 bins
  const int64_t h = blockIdx.x;
  const int64_t cap = (int64_t)S.nr * S.M;
  int32_t* list = tmp + h * cap;
  int32_t* rs = row_shard + h * S.M;
  if (num_shards > 1) {
    // 1. rows by total cost, dealt round-robin to the shards
    auto total_cost = [&](int64_t i) -> int64_t {
      int64_t c = 0;
      for (int32_t r = 0; r < S.nr; ++r) c += range_cost(S, counts, rcounts, h, i, r);
      return min(c, S.max_cost);
    };
    lpt_place(S.M, S.max_cost, hist, total_cost, list, 0);
    for (int64_t p = threadIdx.x; p < S.M; p += blockDim.x) rs[list[p]] = (int32_t)(p % num_shards);
    __syncthreads();
  }
  // 2. per key range, this shard's rows with keys there
  int32_t n = 0;
  for (int32_t r = 0; r < S.nr; ++r) {
    auto cost = [&](int64_t i) -> int64_t {
      if (num_shards > 1 && rs[i] != shard) return -1;
      const int64_t c = range_cost(S, counts, rcounts, h, i, r);
      return c > 0 ? (S.lpt ? c : 1) : -1;
    };
    n += lpt_place(S.M, S.max_cost, hist, cost, list + n, (int32_t)((h * S.nr + r) * S.M));
  }
  if (threadIdx.x == 0) head_count[h] = n;
}

// pack the per-head lists back to back; the total goes to n_items
__global__ void compact_kernel(const int32_t* __restrict__ tmp,
                               const int32_t* __restrict__ head_count, int64_t cap,
                               int32_t* __restrict__ items, int32_t* __restrict__ n_items) {
  const int64_t h = blockIdx.x;
  int64_t off = 0;
  for (int64_t j = 0; j < h; ++j) off += head_count[j];
  const int32_t n = head_count[h];
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) items[off + i] = tmp[h * cap + i];
  if (h == gridDim.x - 1 && threadIdx.x == 0) *n_items = (int32_t)(off + n);
}

// selected blocks of every (row, key range): popcount of the range's bytes
__global__ void range_counts_kernel(const uint8_t* __restrict__ bits, int64_t rows,
                                    int64_t row_bytes, int32_t nr, int32_t rb,
                                    int32_t* __restrict__ rcounts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * nr) return;
  const int64_t row = i / nr, r = i - row * nr;
  const int64_t b0 = r * (rb / 8), b1 = min(row_bytes, (r + 1) * (rb / 8));
  const uint8_t* b = bits + row * row_bytes;
  int c = 0;
  for (int64_t j = b0; j < b1; ++j) c += __popc((unsigned)b[j]);
  rcounts[i] = c;
}

// merge of the key-range partials (CombineArgs); one thread per 8 columns
__global__ void combine_kernel(AttnGeom G, CombineArgs C) {
  const int64_t nst = ceil_div(G.Ts, 128), M = nst + G.nq;
  const int nr = C.kr.nr;
  const int64_t total = G.H * G.T * 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i & 7);
    const int64_t hr = i >> 3;
    const int64_t h = hr / G.T, pr = hr - h * G.T;
    const bool spec = pr < G.Ts;
    const int64_t qb = spec ? -1 : (pr - G.Ts) / 128;
    const int64_t li = spec ? pr / 128 : nst + qb;
    if (C.row_shard && C.row_shard[h * M + li] != C.shard) continue;
    auto valid = [&](int r) -> bool {
      if (spec) return true;  // every range holds keys of a special row
      return (r == 0 && G.Ts > 0) || C.kr.rcounts[(h * G.nq + qb) * nr + r] > 0;
    };
    float L = -INFINITY;
    for (int r = 0; r < nr; ++r)
      if (valid(r)) L = fmaxf(L, C.part_lse[(r * G.H + h) * G.T + pr]);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, den = 0.f;
    for (int r = 0; r < nr; ++r) {
      if (!valid(r)) continue;
      const int64_t prow = (r * G.H + h) * G.T + pr;
      const float w = exp2f(C.part_lse[prow] - L);
      den += w;
      if (C.part_bf16) {
        const uint4 u = *reinterpret_cast<const uint4*>((const __nv_bfloat16*)C.part_out + prow * 64 + c8 * 8);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(p2[e]);
          acc[2 * e] = fmaf(w, f.x, acc[2 * e]);
          acc[2 * e + 1] = fmaf(w, f.y, acc[2 * e + 1]);
        }
      } else {
        const float4* p4 = reinterpret_cast<const float4*>((const float*)C.part_out + prow * 64 + c8 * 8);
        const float4 a0 = p4[0], a1 = p4[1];
        acc[0] = fmaf(w, a0.x, acc[0]); acc[1] = fmaf(w, a0.y, acc[1]);
        acc[2] = fmaf(w, a0.z, acc[2]); acc[3] = fmaf(w, a0.w, acc[3]);
        acc[4] = fmaf(w, a1.x, acc[4]); acc[5] = fmaf(w, a1.y, acc[5]);
        acc[6] = fmaf(w, a1.z, acc[6]); acc[7] = fmaf(w, a1.w, acc[7]);
      }
    }
    const float inv = 1.0f / den;
    const int64_t dst = C.permuted_out ? pr : G.L.part_src(pr);
    if (C.out_bf16) {
      __nv_bfloat16* orow = (__nv_bfloat16*)C.out + (h * G.T + dst) * 64;
      if (C.scatter_world > 0) {
        int r = 0;
        while (r + 1 < C.scatter_world && dst >= C.token_begin[r + 1]) ++r;
        const int64_t t0 = C.token_begin[r], tr = C.token_begin[r + 1] - t0;
        orow = (__nv_bfloat16*)C.out_ptrs[r] + (h * tr + (dst - t0)) * 64;
      }
      uint4 o;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 t = __floats2bfloat162_rn(acc[2 * e] * inv, acc[2 * e + 1] * inv);
        ow[e] = *reinterpret_cast<uint32_t*>(&t);
      }
      *reinterpret_cast<uint4*>(orow + c8 * 8) = o;
    } else {
      float4* op = reinterpret_cast<float4*>((float*)C.out + (h * G.T + dst) * 64 + c8 * 8);
      op[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      op[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
    }
  }
}

int launch_combine(const AttnGeom& G, const CombineArgs& c, cudaStream_t st) {
  const int64_t total = G.H * G.T * 8;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  combine_kernel<<<grid, 256, 0, st>>>(G, c);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

__global__ void area_kernel(const uint8_t* __restrict__ bits, int64_t H, int64_t nq, int64_t nk,
                            int64_t row_bytes, int64_t tp, int64_t bq, int64_t bk,
                            unsigned long long* __restrict__ area) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= H * nq) return;
  const int64_t h = r / nq, qb = r % nq;
  const uint8_t* b = bits + r * row_bytes;
  int64_t c = 0;
  for (int64_t i = 0; i < row_bytes; ++i) c += __popc((unsigned)b[i]);
  const int64_t last = nk - 1;
  const bool last_sel = (b[last >> 3] >> (last & 7)) & 1;
  const int64_t ktail = tp - last * bk;
  const int64_t keys = c * bk - (last_sel ? (bk - ktail) : 0);
  const int64_t qsz = min(bq, tp - qb * bq);
  atomicAdd(&area[h], (unsigned long long)(keys * qsz));
}

__global__ void __launch_bounds__(1024) csr_scan_kernel(const int32_t* __restrict__ counts,
                                                        int64_t rows, int32_t* __restrict__ row_ptr) {
  __shared__ int64_t part[1024];
  const int64_t per = (rows + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = threadIdx.x * per, b1 = min(rows, b0 + per);
  int64_t s = 0;
  for (int64_t i = b0; i < b1; ++i) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int64_t t = part[i];
      part[i] = run;
      run += t;
    }
    row_ptr[rows] = (int32_t)run;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t i = b0; i < b1; ++i) {
    row_ptr[i] = (int32_t)run;
    run += counts[i];
  }
}

__global__ void csr_fill_kernel(const uint8_t* __restrict__ bits, int64_t rows, int64_t row_bytes,
                                int64_t nk, const int32_t* __restrict__ row_ptr,
                                int32_t* __restrict__ col_idx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint8_t* b = bits + r * row_bytes;
  int32_t o = row_ptr[r];
  for (int64_t i = 0; i < row_bytes; ++i) {
    unsigned v = b[i];
    while (v) {
      const int t = __ffs(v) - 1;
      v &= v - 1;
      const int64_t kb = i * 8 + t;
      if (kb < nk) col_idx[o++] = (int32_t)kb;
    }
  }
}

static int check_qkv(const bsa_tensor* t, const char* name) {
  if (!t || !t->data) return fail(BSA_EINVAL, "%s: null tensor", name);
  if (t->dtype != BSA_F32 && t->dtype != BSA_BF16)
    return fail(BSA_EINVAL, "%s: unsupported dtype code %d", name, t->dtype);
  if (t->heads < 1 || t->tokens < 1 || t->dim < 1)
    return fail(BSA_EINVAL, "%s has a zero-sized dimension", name);
  return BSA_OK;
}

static int choose_path(const AttnGeom& G, int32_t in_dtype, int32_t flags) {
  flags &= 0xF;  // path bits; BSA_FLAG_* live above
  // bf16: the tcgen05 kernel; fp32: its X3 form (split-bf16 hi + lo
  // operands, three MMAs per product, fp32-level accuracy)
  const bool tc_ok = (in_dtype == BSA_BF16 || in_dtype == BSA_F32) && G.d == 64 && G.bq == 128 &&
                     G.bk == 64 && G.T < (1LL << 31) && G.H < 65536;
  if (flags == BSA_PATH_SIMT) return BSA_PATH_SIMT;
  if (flags == BSA_PATH_TC) return tc_ok ? BSA_PATH_TC : -BSA_EUNSUPPORTED;
  return tc_ok ? BSA_PATH_TC : BSA_PATH_SIMT;
}

// key-range split of the keys of one head (KeyRanges).  requested: 0 = auto:
// one range while a head's K+V (bf16) fits comfortably in L2, else ranges of
// about 64 MB of K+V each; else the requested number (capped at nk / 8).
static KeyRanges choose_ranges(const AttnGeom& G, int requested, bool x3) {
  KeyRanges kr;
  kr.rcounts = nullptr;
  const int64_t nk8 = ceil_div(G.nk, 8);  // whole mask bytes
  int64_t nr;
  if (requested > 0) {
    nr = requested;
  } else {
    const int64_t kv_head = 2 * G.T * G.d * 2 * (x3 ? 2 : 1);  // (X3: hi + lo)
    nr = kv_head <= (96ll << 20) ? 1 : ceil_div(kv_head, 64ll << 20);
  }
  nr = std::max<int64_t>(1, std::min<int64_t>(nr, nk8));
  const int64_t rb = 8 * ceil_div(nk8, nr);  // key blocks per range, whole bytes
  kr.nr = (int32_t)ceil_div(G.nk, rb);
  kr.rb = (int32_t)rb;
  return kr;
}

struct TcWorkspace {
  __nv_bfloat16 *qp, *kp;
  void* vp;
  __nv_bfloat16 *qp_lo, *kp_lo, *vp_lo;  // (X3) lo parts
  int32_t *items, *counter, *counts, *vshift;
  int32_t *ovf_flags, *ovf_list, *ovf_count;
  int32_t *row_shard, *tmp, *head_count, *n_items, *rcounts;
  unsigned int* vamax;
  void* part_out;
  float* part_lse;
  int64_t cap;  // item capacity: H * nr * M
  size_t bytes;
};

static TcWorkspace tc_ws_layout(void* base, const AttnGeom& G, const KeyRanges& kr,
                                bool part_bf16, bool x3) {
  TcWorkspace w;
  char* p = (char*)base;
  const size_t tens = align_up((size_t)(G.H * G.T * G.d) * 2, 256);
  const int64_t nst = ceil_div(G.Ts, 128);
  const int64_t M = nst + G.nq;
  w.cap = G.H * kr.nr * M;
  const size_t capb = align_up((size_t)w.cap * 4, 256);
  w.qp = (__nv_bfloat16*)p; p += tens;
  w.kp = (__nv_bfloat16*)p; p += tens;
  w.vp = (void*)p; p += tens;
  w.qp_lo = w.kp_lo = w.vp_lo = nullptr;
  if (x3) {
    w.qp_lo = (__nv_bfloat16*)p; p += tens;
    w.kp_lo = (__nv_bfloat16*)p; p += tens;
    w.vp_lo = (__nv_bfloat16*)p; p += tens;
  }
  w.items = (int32_t*)p; p += capb;
  w.counter = (int32_t*)p; p += 256;
  w.counts = (int32_t*)p; p += align_up((size_t)(G.H * G.nq) * 4, 256);
  w.vshift = (int32_t*)p; p += align_up((size_t)G.H * 4, 256);
  w.vamax = (unsigned int*)p; p += align_up((size_t)G.H * 4, 256);
  w.ovf_flags = (int32_t*)p; p += capb;
  w.ovf_list = (int32_t*)p; p += capb;
  w.ovf_count = (int32_t*)p; p += 256;
  w.row_shard = (int32_t*)p; p += align_up((size_t)(G.H * M) * 4, 256);
  w.tmp = (int32_t*)p; p += capb;
  w.head_count = (int32_t*)p; p += align_up((size_t)G.H * 4, 256);
  w.n_items = (int32_t*)p; p += 256;
  w.rcounts = nullptr;
  w.part_out = nullptr;
  w.part_lse = nullptr;
  if (kr.nr > 1) {
    w.rcounts = (int32_t*)p; p += align_up((size_t)(G.H * G.nq * kr.nr) * 4, 256);
    w.part_out = (void*)p;
    p += align_up((size_t)(kr.nr * G.H * G.T * G.d) * (part_bf16 ? 2 : 4), 256);
    w.part_lse = (float*)p; p += align_up((size_t)(kr.nr * G.H * G.T) * 4, 256);
  }
  w.bytes = (size_t)(p - (char*)base);
  return w;
}

int launch_pack(const bsa_tensor* x, const AttnGeom& G, int permuted, __nv_bfloat16* out,
                cudaStream_t st, __nv_bfloat16* lo) {
  const int64_t total = G.H * G.T * (G.d / 8);
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  const bool bf = x->dtype == BSA_BF16;
  const size_t es = bf ? 2 : 4;
  if ((uintptr_t)x->data % 16 || (x->stride_token * es) % 16 || (x->stride_head * es) % 16)
    return fail(BSA_EUNSUPPORTED, "q/k/v must be 16-byte aligned for the tensor-core path");
  if (bf)
    pack_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x->data,
                                                     x->stride_head, x->stride_token, G.H, G.T,
                                                     G.d, G.L, permuted, out, nullptr);
  else
    pack_kernel<float><<<grid, 256, 0, st>>>((const float*)x->data, x->stride_head,
                                             x->stride_token, G.H, G.T, G.d, G.L, permuted, out,
                                             lo);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

static int launch_pack_v(const bsa_tensor* x, const AttnGeom& G, int permuted, unsigned int* amax,
                         int32_t* shift, __half* out, cudaStream_t st) {
  const bool bf = x->dtype == BSA_BF16;
  const size_t es = bf ? 2 : 4;
  if ((uintptr_t)x->data % 16 || (x->stride_token * es) % 16 || (x->stride_head * es) % 16)
    return fail(BSA_EUNSUPPORTED, "q/k/v must be 16-byte aligned for the tensor-core path");
  BSA_CUDA_TRY(cudaMemsetAsync(amax, 0, (size_t)G.H * 4, st));
  dim3 ag((unsigned)std::min<int64_t>(ceil_div(G.T * G.d, 256), 64), (unsigned)G.H);
  const int64_t total = G.H * G.T * (G.d / 8);
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  if (bf) {
    vamax_kernel<__nv_bfloat16><<<ag, 256, 0, st>>>((const __nv_bfloat16*)x->data, x->stride_head,
                                                    x->stride_token, G.T, G.d, amax);
    pack_v_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x->data,
                                                       x->stride_head, x->stride_token, G.H, G.T,
                                                       G.d, G.L, permuted, amax, shift, out);
  } else {
    vamax_kernel<float><<<ag, 256, 0, st>>>((const float*)x->data, x->stride_head,
                                            x->stride_token, G.T, G.d, amax);
    pack_v_kernel<float><<<grid, 256, 0, st>>>((const float*)x->data, x->stride_head,
                                               x->stride_token, G.H, G.T, G.d, G.L, permuted,
                                               amax, shift, out);
  }
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

}  // namespace bsa

using namespace bsa;

extern "C" {

int bsa_sparse_attention_path(const bsa_layout* layout, int64_t dim, int32_t block_q,
                              int32_t block_k, int32_t in_dtype, int32_t flags) {
  if (!layout || dim < 1 || block_q < 1 || block_k < 1) return -BSA_EINVAL;
  const AttnGeom G = make_geom(to_layout(layout), 1, (int)dim, block_q, block_k);
  return choose_path(G, in_dtype, flags);
}

size_t bsa_sparse_attention_workspace(const bsa_layout* layout, int64_t heads, int64_t dim,
                                      int32_t block_q, int32_t block_k, int32_t in_dtype,
                                      int32_t inputs_permuted, int32_t flags) {
  (void)inputs_permuted;
  if (!layout || heads < 1 || dim < 1 || block_q < 1 || block_k < 1) return 0;
  const AttnGeom G = make_geom(to_layout(layout), heads, (int)dim, block_q, block_k);
  if (choose_path(G, in_dtype, flags) != BSA_PATH_TC) return 256;
  // fp32 partials cover either output dtype
  const bool x3 = in_dtype == BSA_F32;
  return tc_ws_layout(nullptr, G, choose_ranges(G, BSA_FLAG_RANGES_GET(flags), x3), false, x3).bytes +
         256;
}

static int sparse_attention_impl(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                                 void* out, int32_t out_dtype, const bsa_layout* layout,
                                 int32_t block_q, int32_t block_k, const uint8_t* mask_bits,
                                 const int32_t* counts, float scale, int32_t inputs_permuted,
                                 int32_t shard, int32_t num_shards, int32_t flags, void* ws,
                                 size_t ws_bytes, void* stream, const bsa_scatter* scatter) {
  int rc = check_qkv(q, "q");
  if (!rc) rc = check_qkv(k, "k");
  if (!rc) rc = check_qkv(v, "v");
  if (rc) return rc;
  if (!layout || (!out && !scatter) || !mask_bits)
    return fail(BSA_EINVAL, "sparse_attention: null pointer");
  if (q->heads != k->heads || q->heads != v->heads || q->tokens != k->tokens ||
      q->tokens != v->tokens || q->dim != k->dim || q->dim != v->dim)
    return fail(BSA_EINVAL, "q/k/v shapes differ");
  if (q->dtype != k->dtype || q->dtype != v->dtype)
    return fail(BSA_EINVAL, "q/k/v dtypes differ");
  if (out_dtype != BSA_F32 && out_dtype != BSA_BF16)
    return fail(BSA_EINVAL, "unsupported output dtype %d", out_dtype);
  const Layout L = to_layout(layout);
  if (L.frames < 1 || L.P < 1 || L.S < 0) return fail(BSA_EINVAL, "invalid layout");
  if (q->tokens != L.tokens())
    return fail(BSA_EINVAL, "inputs have %lld tokens but layout describes %lld",
                (long long)q->tokens, (long long)L.tokens());
  if (block_q < 1 || block_k < 1) return fail(BSA_EINVAL, "block sizes must be >= 1");
  if (num_shards < 1) num_shards = 1;
  if (shard < 0 || shard >= num_shards) return fail(BSA_EINVAL, "shard %d of %d", shard, num_shards);
  const AttnGeom G = make_geom(L, q->heads, (int)q->dim, block_q, block_k);
  int path = choose_path(G, q->dtype, flags);
  const bool x3 = path == BSA_PATH_TC && q->dtype == BSA_F32;
  if (x3) {
    // the split pack reads 16-byte fp32 vectors; unaligned inputs (or the
    // multi-GPU scatter, bf16-only) keep the CUDA-core path
    auto al16 = [](const bsa_tensor* t) {
      return (uintptr_t)t->data % 16 == 0 && (t->stride_token * 4) % 16 == 0 &&
             (t->stride_head * 4) % 16 == 0;
    };
    if (!al16(q) || !al16(k) || !al16(v) || scatter) {
      if ((flags & 0xF) == BSA_PATH_TC)
        return fail(BSA_EUNSUPPORTED, "fp32 tensor-core path: 16-byte aligned inputs, no scatter");
      path = BSA_PATH_SIMT;
    }
  }
  if (path < 0)
    return fail(BSA_EUNSUPPORTED,
                "tensor-core path needs bf16 or fp32 inputs, head_dim 64, block_q 128, block_k 64");
  cudaStream_t st = (cudaStream_t)stream;
  if (scatter) {
    if (path != BSA_PATH_TC || out_dtype != BSA_BF16 || inputs_permuted)
      return fail(BSA_EUNSUPPORTED,
                  "output scatter needs the tensor-core path, bf16 output, source order");
    if (scatter->world < 1 || scatter->world > 64 || !scatter->out_ptrs || !scatter->token_begin)
      return fail(BSA_EINVAL, "invalid scatter descriptor");
  }
  if (path == BSA_PATH_SIMT)
    return launch_simt_attention(q, k, v, out, out_dtype, G, mask_bits, inputs_permuted, scale,
                                 shard, num_shards, st);

  // ---------------- tensor-core path ----------------
  if (!ws) return fail(BSA_EINVAL, "sparse_attention: workspace required");
  static int env_ranges = -2;
  if (env_ranges == -2) {
    const char* e = getenv("BSA_TC_KEY_RANGES");  // experiments: force a key-range split
    env_ranges = e ? atoi(e) : -1;
  }
  const int req_ranges = BSA_FLAG_RANGES_GET(flags) ? BSA_FLAG_RANGES_GET(flags)
                                                    : (env_ranges > 0 ? env_ranges : 0);
  const KeyRanges KR = choose_ranges(G, req_ranges, x3);
  const bool part_bf16 = out_dtype == BSA_BF16;
  TcWorkspace W = tc_ws_layout(ws, G, KR, part_bf16, x3);
  if (ws_bytes < W.bytes) return fail(BSA_EINVAL, "sparse_attention: workspace too small");
  // kernel variant: exp2 split between MUFU and the FMA pipe, P/V precision
  static int env_poly = -2, env_f16 = -2;
  if (env_poly == -2) {
    const char* e = getenv("BSA_TC_EXP_POLY");
    env_poly = e ? atoi(e) : -1;
    const char* f = getenv("BSA_TC_F16P");
    env_f16 = f ? atoi(f) : -1;
  }
  const int v_f16 = x3 ? 0 : (env_f16 >= 0 ? env_f16 : 0);
  // 2 of every 8 exp2 pairs on the FMA pipe (degree-2 polynomial), the rest
  // on MUFU: the kernel is MUFU-bound at d=64 (profiles/r01_summary.md).
  // Round 1 measured 0: 90.0 ms, 2: 85.4, 3: 84.5, 4: 90.9; with the round-2
  // pipeline (power-capped, two boxes, profiles/r02c/ab_exp_poly_*):
  // 1: 85.9, 2: 81.2-82.4, 3: 84.2-86.4, 4: 88.8
  const int exp_poly = x3 ? 0 : (env_poly >= 0 ? env_poly : 2);
  // Pack passes only where the kernel cannot read the caller's tensors:
  //  * Q (read row by row by the softmax warps) is used in place whenever it
  //    is bf16 with 16-byte aligned rows: the partitioned-order gather is the
  //    row address part_src(pr);
  //  * K and V are TMA-loaded in 64-key boxes of the partitioned order, which
  //    straddle frames in source order: used in place only when the inputs
  //    are already partitioned (inputs_permuted), bf16, aligned and share
  //    strides; otherwise packed (3 bytes moved per 2 read, ~0.4 ms at N=200).
  auto aligned16 = [](const bsa_tensor* t) {
    return t->dtype == BSA_BF16 && (uintptr_t)t->data % 16 == 0 && (t->stride_token * 2) % 16 == 0 &&
           (t->stride_head * 2) % 16 == 0;
  };
  const bool q_direct = !x3 && aligned16(q);
  const bool kv_direct = !x3 && !v_f16 && inputs_permuted && aligned16(k) && aligned16(v) &&
                         k->stride_token == v->stride_token && k->stride_head == v->stride_head;
  if (!q_direct) rc = launch_pack(q, G, inputs_permuted, W.qp, st, W.qp_lo);
  if (!rc && !kv_direct) {
    rc = launch_pack(k, G, inputs_permuted, W.kp, st, W.kp_lo);
    if (!rc)
      rc = v_f16 ? launch_pack_v(v, G, inputs_permuted, W.vamax, W.vshift, (__half*)W.vp, st)
                 : launch_pack(v, G, inputs_permuted, (__nv_bfloat16*)W.vp, st, W.vp_lo);
  }
  if (rc) return rc;
  const int64_t rows = G.H * G.nq;
  if (!counts) {
    counts_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(mask_bits, rows,
                                                                 G.mask_row_bytes, W.counts);
    BSA_LAUNCH_CHECK();
    counts = W.counts;
  }
  KeyRanges kr = KR;
  if (kr.nr > 1) {
    range_counts_kernel<<<(unsigned)ceil_div(rows * kr.nr, 256), 256, 0, st>>>(
        mask_bits, rows, G.mask_row_bytes, kr.nr, kr.rb, W.rcounts);
    BSA_LAUNCH_CHECK();
    kr.rcounts = W.rcounts;
  }
  SchedGeom S;
  S.nq = G.nq;
  S.nst = ceil_div(G.Ts, 128);
  S.M = S.nst + G.nq;
  S.nsc = ceil_div(G.Ts, 64);
  S.T = G.T;
  S.Ts = G.Ts;
  S.nr = kr.nr;
  S.rb = kr.rb;
  S.max_cost = std::max<int64_t>(ceil_div(G.T, 64) + kr.nr, S.nsc + G.nk);
  S.lpt = (flags & BSA_FLAG_NATURAL_ORDER) ? 0 : 1;
  const size_t hsmem = (size_t)(S.max_cost + 1) * 4;
  if (hsmem > 200 * 1024) return fail(BSA_EUNSUPPORTED, "sequence too long for the scheduler");
  BSA_CUDA_TRY(cudaFuncSetAttribute(schedule_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)hsmem));
  schedule_kernel<<<(unsigned)G.H, 1024, hsmem, st>>>(counts, kr.rcounts, S, num_shards, shard,
                                                      W.row_shard, W.tmp, W.head_count);
  BSA_LAUNCH_CHECK();
  compact_kernel<<<(unsigned)G.H, 256, 0, st>>>(W.tmp, W.head_count, (int64_t)kr.nr * S.M, W.items,
                                                W.n_items);
  BSA_LAUNCH_CHECK();
  BSA_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 8, st));  // main + repair launch counters
  TcArgs a;
  a.kr = kr;
  a.part_out = W.part_out;
  a.part_bf16 = part_bf16;
  a.part_lse = W.part_lse;
  a.qp = q_direct ? (const __nv_bfloat16*)q->data : W.qp;
  a.q_src = q_direct ? 1 : 0;
  a.x3 = x3 ? 1 : 0;
  a.qp_lo = W.qp_lo;
  a.kp_lo = W.kp_lo;
  a.vp_lo = W.vp_lo;
  a.q_sH = q_direct ? q->stride_head : G.T * G.d;
  a.q_sT = q_direct ? q->stride_token : G.d;
  a.kp = kv_direct ? (const __nv_bfloat16*)k->data : W.kp;
  a.vp = kv_direct ? v->data : W.vp;
  a.kv_sH = kv_direct ? k->stride_head : G.T * G.d;
  a.kv_sT = kv_direct ? k->stride_token : G.d;
  a.v_shift = W.vshift;
  a.v_f16 = v_f16;
  a.exp_poly = exp_poly;
  a.out = out;
  a.out_bf16 = out_dtype == BSA_BF16;
  a.permuted_out = inputs_permuted;
  a.bits = mask_bits;
  a.counts = counts;
  a.items = W.items;
  a.n_items = (int32_t)W.cap;
  a.n_items_dev = W.n_items;
  a.work_counter = W.counter;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.shard = shard;
  a.num_shards = num_shards;
  a.timing = (flags & BSA_FLAG_TIMING) != 0;
  a.ovf_flags = W.ovf_flags;
  a.ovf_list = W.ovf_list;
  a.ovf_count = W.ovf_count;
  a.scatter_world = scatter ? scatter->world : 0;
  a.out_ptrs = scatter ? reinterpret_cast<const unsigned long long*>(scatter->out_ptrs) : nullptr;
  a.token_begin = scatter ? scatter->token_begin : nullptr;
  a.trace = nullptr;
  if (getenv("BSA_TC_TRACE")) {  // debug pipeline trace of CTA 0 (scripts/trace_analyze.py)
    static unsigned long long* tbuf = nullptr;
    const size_t tbytes = 20 * 512 * sizeof(unsigned long long);
    if (!tbuf) BSA_CUDA_TRY(cudaMalloc(&tbuf, tbytes));
    BSA_CUDA_TRY(cudaMemsetAsync(tbuf, 0, tbytes, st));
    a.trace = tbuf;
  }
  CombineArgs c;
  c.kr = kr;
  c.part_out = W.part_out;
  c.part_bf16 = part_bf16;
  c.part_lse = W.part_lse;
  c.row_shard = num_shards > 1 ? W.row_shard : nullptr;
  c.shard = shard;
  c.out = out;
  c.out_bf16 = a.out_bf16;
  c.permuted_out = inputs_permuted;
  c.scatter_world = a.scatter_world;
  c.out_ptrs = a.out_ptrs;
  c.token_begin = a.token_begin;
  SimtRepair sr;
  sr.q = q;
  sr.k = k;
  sr.v = v;
  sr.scale = scale;
  return launch_tc_attention(G, a, st, &c, x3 ? &sr : nullptr);
}

int bsa_sparse_attention(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                         void* out, int32_t out_dtype, const bsa_layout* layout,
                         int32_t block_q, int32_t block_k, const uint8_t* mask_bits,
                         const int32_t* counts, float scale, int32_t inputs_permuted,
                         int32_t shard, int32_t num_shards, int32_t flags, void* ws,
                         size_t ws_bytes, void* stream) {
  return sparse_attention_impl(q, k, v, out, out_dtype, layout, block_q, block_k, mask_bits,
                               counts, scale, inputs_permuted, shard, num_shards, flags, ws,
                               ws_bytes, stream, nullptr);
}

int bsa_sparse_attention_scatter(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                                 const bsa_layout* layout, int32_t block_q, int32_t block_k,
                                 const uint8_t* mask_bits, const int32_t* counts, float scale,
                                 int32_t shard, int32_t num_shards, int32_t flags,
                                 const bsa_scatter* scatter, void* ws, size_t ws_bytes,
                                 void* stream) {
  if (!scatter) return fail(BSA_EINVAL, "sparse_attention_scatter: null scatter descriptor");
  return sparse_attention_impl(q, k, v, nullptr, BSA_BF16, layout, block_q, block_k, mask_bits,
                               counts, scale, 0, shard, num_shards, flags, ws, ws_bytes, stream,
                               scatter);
}

int bsa_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out || bytes == 0) return fail(BSA_EINVAL, "ipc_alloc: invalid argument");
  BSA_CUDA_TRY(cudaMalloc(dev_ptr, bytes));
  cudaIpcMemHandle_t h;
  BSA_CUDA_TRY(cudaIpcGetMemHandle(&h, *dev_ptr));
  static_assert(sizeof(cudaIpcMemHandle_t) == BSA_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return BSA_OK;
}

int bsa_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(BSA_EINVAL, "ipc_open: invalid argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  BSA_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BSA_OK;
}

int bsa_ipc_close(void* dev_ptr) {
  BSA_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return BSA_OK;
}

int bsa_ipc_free(void* dev_ptr) {
  BSA_CUDA_TRY(cudaFree(dev_ptr));
  return BSA_OK;
}

int bsa_mask_selected_area(const uint8_t* mask_bits, int64_t heads, int64_t patch_tokens,
                           int32_t block_q, int32_t block_k, int64_t* area_out, void* stream) {
  if (!mask_bits || !area_out || heads < 1 || patch_tokens < 1 || block_q < 1 || block_k < 1)
    return fail(BSA_EINVAL, "mask_selected_area: invalid argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nq = ceil_div(patch_tokens, block_q), nk = ceil_div(patch_tokens, block_k);
  BSA_CUDA_TRY(cudaMemsetAsync(area_out, 0, (size_t)heads * 8, st));
  const int64_t rows = heads * nq;
  area_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(
      mask_bits, heads, nq, nk, ceil_div(nk, 8), patch_tokens, block_q, block_k,
      (unsigned long long*)area_out);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

size_t bsa_mask_to_csr_workspace(int64_t heads, int64_t nq) {
  return align_up((size_t)(heads * nq) * 4, 256);
}

int bsa_mask_to_csr(const uint8_t* mask_bits, int64_t heads, int64_t nq, int64_t nk,
                    int32_t* row_ptr, int32_t* col_idx, void* ws, size_t ws_bytes,
                    void* stream) {
  if (!mask_bits || !row_ptr || !col_idx || !ws || heads < 1 || nq < 1 || nk < 1)
    return fail(BSA_EINVAL, "mask_to_csr: invalid argument");
  if (ws_bytes < bsa_mask_to_csr_workspace(heads, nq))
    return fail(BSA_EINVAL, "mask_to_csr: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = heads * nq, rb = ceil_div(nk, 8);
  int32_t* counts = (int32_t*)ws;
  counts_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(mask_bits, rows, rb, counts);
  BSA_LAUNCH_CHECK();
  csr_scan_kernel<<<1, 1024, 0, st>>>(counts, rows, row_ptr);
  BSA_LAUNCH_CHECK();
  csr_fill_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(mask_bits, rows, rb, nk, row_ptr,
                                                                 col_idx);
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

}  // extern "C"
