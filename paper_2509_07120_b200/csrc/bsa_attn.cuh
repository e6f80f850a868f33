// bsa_attn.cuh -- geometry and key-stream helpers shared by the attention kernels.
#pragma once

#include <cuda_fp16.h>

#include "bsa_common.cuh"

namespace bsa {

// Attention geometry in partitioned order: [specials (Ts) | patches (Tp)].
struct AttnGeom {
  Layout L;
  int64_t H, T, Ts, Tp;
  int d;
  int64_t bq, bk, nq, nk, mask_row_bytes;
  __host__ __device__ int64_t simt_tiles_per_head() const {
    return ceil_div(Ts, 32) + nq * ceil_div(bq, 32);
  }
};

inline AttnGeom make_geom(const Layout& L, int64_t H, int d, int64_t bq, int64_t bk) {
  AttnGeom G;
  G.L = L;
  G.H = H;
  G.T = L.tokens();
  G.Ts = L.n_spec();
  G.Tp = L.n_patch();
  G.d = d;
  G.bq = bq;
  G.bk = bk;
  G.nq = ceil_div(G.Tp, bq);
  G.nk = ceil_div(G.Tp, bk);
  G.mask_row_bytes = ceil_div(G.nk, 8);
  return G;
}

// Key stream of one query row group, as chunks of <= CH consecutive
// partitioned-order keys: special query rows (qb < 0) see [0, T); patch
// q-block rows see the special strip [0, Ts) and then each selected key
// block ascending (sparse.py:101-119, :122-131).
struct KeyChunker {
  int64_t Ts, Tp, T, bk, nk;
  const uint8_t* row;   // mask row bits (nullptr for special rows)
  int CH;
  int phase;            // 0: contiguous range, 1: mask blocks, 2: done
  int64_t pos, end;     // current contiguous range [pos, end)
  int64_t byte_idx;     // mask iteration
  unsigned int cur;     // remaining bits of the current byte
  int64_t byte_end;     // mask bytes [.., byte_end) (a key range's slice of the row)
  __device__ KeyChunker(const AttnGeom& G, int64_t qb, const uint8_t* mask_row, int ch)
      : Ts(G.Ts), Tp(G.Tp), T(G.T), bk(G.bk), nk(G.nk), row(qb < 0 ? nullptr : mask_row),
        CH(ch), phase(0), pos(0), end(qb < 0 ? G.T : G.Ts), byte_idx(-1), cur(0),
        byte_end(G.mask_row_bytes) {}
  // key-range form: contiguous keys [pos0, end0), then the selected blocks
  // of mask bytes [byte0, byte1)
  __device__ KeyChunker(const AttnGeom& G, int64_t qb, const uint8_t* mask_row, int ch,
                        int64_t pos0, int64_t end0, int64_t byte0, int64_t byte1)
      : Ts(G.Ts), Tp(G.Tp), T(G.T), bk(G.bk), nk(G.nk), row(qb < 0 ? nullptr : mask_row),
        CH(ch), phase(0), pos(pos0), end(end0), byte_idx(byte0 - 1), cur(0), byte_end(byte1) {}

  // next selected key block (>= 0) or -1
  __device__ __forceinline__ int64_t next_block() {
    while (cur == 0) {
      ++byte_idx;
      if (byte_idx * 8 >= nk || byte_idx >= byte_end) return -1;
      cur = row[byte_idx];
    }
    const int b = __ffs(cur) - 1;
    cur &= cur - 1;
    return byte_idx * 8 + b;
  }

  __device__ __forceinline__ bool next(int64_t& start, int& len) {
    while (true) {
      if (pos < end) {
        start = pos;
        const int64_t n = end - pos;
        len = (int)(n < CH ? n : CH);
        pos += len;
        return true;
      }
      if (phase == 0 && row) {
        phase = 1;
      }
      if (phase == 1) {
        const int64_t kb = next_block();
        if (kb < 0) { phase = 2; return false; }
        pos = Ts + kb * bk;
        const int64_t e = (kb + 1) * bk;
        end = Ts + (e < Tp ? e : Tp);
        continue;
      }
      phase = 2;
      return false;
    }
  }
};

int launch_simt_attention(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                          void* out, int out_dtype, const AttnGeom& G, const uint8_t* bits,
                          int permuted, float scale, int shard, int num_shards, cudaStream_t st);
// SIMT recomputation of listed tensor-core work items (whole rows, exact
// online softmax): list[0..*count) of item codes (h * nr + r) * M + li,
// li < nst special-row tiles, else patch q-block li - nst; 128-row items.
struct SimtList {
  const int32_t* list;
  const int32_t* count;
  int64_t M, nst;
  int32_t nr;
  int64_t cap;
};
// the caller's fp32 inputs, for the X3 launch's SIMT repair of overflowed items
struct SimtRepair {
  const bsa_tensor *q, *k, *v;
  float scale;
};
int launch_simt_attention_list(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                               void* out, int out_dtype, const AttnGeom& G, const uint8_t* bits,
                               int permuted, float scale, const SimtList& sl, cudaStream_t st);

// Key-range split (long sequences): the keys of a head are cut into `nr`
// ranges of `rb` key blocks (rb % 8 == 0, so a range is a byte range of the
// .bsm mask row).  Work item (head, row tile, range r) streams only range r's
// keys: the special strip (range 0) or its slice of [0, T) for special rows,
// then the row's selected blocks inside the range.  Items of one (head,
// range) run together, so their K/V (1/nr of the head's) stays L2-resident.
// The ranges of a row are merged afterwards by their log-sum-exp.
struct KeyRanges {
  int32_t nr, rb;          // ranges, key blocks per range (nr == 1: rb >= nk)
  const int32_t* rcounts;  // (H * nq, nr) selected blocks per row and range (nr > 1)
};

struct TcArgs {
  // key-range split (bsa_tc_common.cuh KeyRanges); nr > 1: the kernel writes
  // per-range partials (O / l and log2-sum-exp, rows in partitioned order)
  // that combine_kernel merges into out
  KeyRanges kr;
  void* part_out;             // (nr, H, T, 64) bf16 (part_bf16) or fp32
  int part_bf16;
  float* part_lse;            // (nr, H, T): offset + log2(l)
  const __nv_bfloat16* qp;   // Q: packed partitioned (H, T, 64), or (q_src) the caller's
                             // bf16 q in its own token order and strides
  const __nv_bfloat16* qp_lo; // (x3) Q lo, packed beside qp (fp32 inputs split into bf16 hi + lo)
  int x3;                    // fp32 inputs: three-MMA split-bf16 products (kp/vp hi, kp_lo/vp_lo lo)
  const __nv_bfloat16* kp_lo;
  const __nv_bfloat16* vp_lo;
  int q_src;                 // 1: qp is the caller's q; row = permuted ? pr : part_src(pr)
  int64_t q_sH, q_sT;        // element strides of qp (packed: T*64, 64)
  int64_t kv_sH, kv_sT;      // element strides of kp / vp (packed: T*64, 64)
  const __nv_bfloat16* kp;
  const void* vp;             // V: bf16, or fp16 scaled by 2^v_shift[h] (v_f16)
  const int32_t* v_shift;
  int v_f16;                  // fp16 P x fp16 V variant
  int exp_poly;               // pairs of every 8 computed by the FMA-pipe exp2
  void* out;
  int out_bf16;
  int permuted_out;          // write rows in partitioned order
  const uint8_t* bits;
  const int32_t* counts;     // per (h, qb) selected blocks
  const int32_t* items;      // LPT-ordered work items of this shard (schedule_kernel)
  int32_t n_items;            // capacity of items / ovf_flags (H * nr * M)
  int32_t* work_counter;
  float scale_log2;          // scale * log2(e)
  int shard, num_shards;
  int timing;                // record events around the launch (bsa_last_kernel_ms)
  unsigned long long* trace; // debug: clock64 per pipeline event of CTA 0 (BSA_TC_TRACE), or null
  // stale-max overflow repair: items whose P exceeded the limit are listed
  // (ovf_flags dedups) and recomputed by the exact-max launch
  int32_t* ovf_flags;         // [n_items] zeroed per call
  int32_t* ovf_list;          // [n_items]
  int32_t* ovf_count;         // [1]
  const int32_t* n_items_dev; // exact-max launch: item count on the device (else null)
  // multi-GPU output scatter (shard.py combine="scatter"): rows of token t
  // go to out_ptrs[r] for token_begin[r] <= t < token_begin[r+1] (peer
  // pointers: the epilogue writes over NVLink); scatter_world 0 = local out
  int32_t scatter_world;
  const unsigned long long* out_ptrs;
  const int64_t* token_begin;
};

// merge of the key-range partials (bsa_attn_host.cu combine_kernel): per row
// L = max_r lse_r, out = sum_r 2^(lse_r - L) O_r / sum_r 2^(lse_r - L) over the
// ranges the row has keys in, written like the kernel epilogue would
struct CombineArgs {
  KeyRanges kr;
  const void* part_out;
  int part_bf16;
  const float* part_lse;
  const int32_t* row_shard;  // (H, M) shard of each row tile, or null (all rows)
  int shard;
  void* out;
  int out_bf16;
  int permuted_out;
  int32_t scatter_world;
  const unsigned long long* out_ptrs;
  const int64_t* token_begin;
};
int launch_combine(const AttnGeom& G, const CombineArgs& c, cudaStream_t st);
struct SimtRepair;
int launch_tc_attention(const AttnGeom& G, const TcArgs& a, cudaStream_t st,
                        const CombineArgs* comb, const SimtRepair* rep = nullptr);
cudaEvent_t timing_events(int which);
size_t tc_smem_bytes();
// source-order (f32|bf16) Q/K/V -> contiguous bf16 [specials | patches]
// (bsa_attn_host.cu; also used by the dense-statistics kernels)
// (fp32 x, lo != null: also the residual x - bf16(x) rounded to bf16)
int launch_pack(const bsa_tensor* x, const AttnGeom& G, int permuted, __nv_bfloat16* out,
                cudaStream_t st, __nv_bfloat16* lo = nullptr);

}  // namespace bsa
