/*
 * bsa.h -- C ABI of the B200-native block-sparse global-attention library
 * (libbsa.so, sm_100a).  Plain pointers and sizes only: no torch, no CUDA
 * types.  Streams are passed as `void*` (a cudaStream_t); all device memory,
 * including workspace, is owned and allocated by the caller.
 *
 * Every entry point replaces one operator of the reference package `bsattn`
 * (/root/reference/pkg/src/bsattn, the Python API re-exported by
 * __init__.py:8-59).  The reference has no FFI; its operator boundary is the
 * Python call, so the binding a maintainer adds is a ctypes stub (see
 * INTEGRATION.md) and the Python mirror paper_2509_07120_b200/ keeps the
 * reference's names, argument meaning and ValueError behaviour.
 *
 * Conventions
 *   - Asynchronous on `stream`; no host synchronisation; re-entrant.
 *   - Return codes: BSA_OK, BSA_EINVAL (bad argument -> ValueError in Python),
 *     BSA_EUNSUPPORTED (valid but not implemented on this device path),
 *     BSA_ECUDA (CUDA error -> RuntimeError).  bsa_last_error() gives a
 *     thread-local message for the last failure.
 *   - Tensors are (heads, tokens, dim) with unit stride on dim.
 *   - Block masks use the reference .bsm row layout (maskpred.py:17-19): one
 *     bitset per (head, query block) row, ceil(nk/8) bytes, LSB-first.
 */
#ifndef BSA_H_
#define BSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSA_OK 0
#define BSA_EINVAL 1
#define BSA_EUNSUPPORTED 2
#define BSA_ECUDA 3

#define BSA_F32 0
#define BSA_BF16 1

/* attention path selection (bsa_sparse_attention `flags`) */
#define BSA_PATH_AUTO 0     /* tcgen05 kernel when bf16/d64/128x64, else SIMT */
#define BSA_PATH_SIMT 1     /* force the CUDA-core kernel (fp32 math)        */
#define BSA_PATH_TC 2       /* require the tcgen05 kernel (EUNSUPPORTED if not) */
#define BSA_FLAG_TIMING 16  /* bracket the attention kernel with CUDA events */
/* key-range split of the tensor-core path (bits 8-15): 0 = auto (split when a
 * head's K+V outgrows L2, e.g. N=1000 frames), n = n ranges whose partials
 * are merged by log-sum-exp (results equal within rounding) */
#define BSA_FLAG_RANGES(n) (((n) & 0xFF) << 8)
/* tensor-core path: keep each head's work items in row order instead of the
 * LPT (longest-first) order -- for measuring what the LPT order buys */
#define BSA_FLAG_NATURAL_ORDER 32
#define BSA_FLAG_RANGES_GET(f) (((f) >> 8) & 0xFF)

/* TokenLayout (layout.py:27-66): F frames of S specials + P patches. */
typedef struct {
  int64_t frames;
  int64_t patches_per_frame;
  int64_t specials_per_frame;
  int32_t specials_first; /* 1: [s0..sS-1, p0..pP-1] per frame (layout.py:35) */
} bsa_layout;

/* (heads, tokens, dim) device tensor, dim contiguous; strides in elements. */
typedef struct {
  const void* data;
  int32_t dtype; /* BSA_F32 | BSA_BF16 */
  int64_t heads, tokens, dim;
  int64_t stride_head, stride_token;
} bsa_tensor;

/* Library version (major*10000 + minor*100 + patch). */
int bsa_version(void);
/* Message for the last failing call on this thread ("" if none). */
const char* bsa_last_error(void);
/* Number of SMs of the current device (for persistent grids / sharding). */
int bsa_device_sm_count(void);

/* Input validation of the reference's as_f32 (tensorio.py:47-59), on the
 * device: sets *flag (device int32, caller-zeroed) to 1 if x holds a NaN or
 * an infinity.  Asynchronous; several tensors may share one flag. */
int bsa_check_finite(const bsa_tensor* x, int32_t* flag, void* stream);

/* ------------------------------------------------------------------ */
/* Scoring stage                                                      */
/* ------------------------------------------------------------------ */

/* block_pool (maskpred.py:104-120).  Mean over token blocks of `block` rows,
 * ragged tail over its true length, reference fp32 summation order.
 * If `patch_gather` is non-NULL, `x` holds the full interleaved sequence
 * (tokens == layout total) and only its patch rows are pooled, in patch order
 * (the caller's patch_token_indices gather, README:127-128, folded into the
 * addressing).  out: (heads, ceil(n/block), dim) fp32 contiguous. */
int bsa_block_pool(const bsa_tensor* x, const bsa_layout* patch_gather, int32_t block,
                   float* out, void* stream);

/* pooled_scores (maskpred.py:123-139 + tensorio.py:73-87): per head
 * row_softmax(qp @ kp^T, scale).  qp (H,nq,d), kp (H,nk,d), probs (H,nq,nk),
 * all fp32 contiguous.  Bit-exact with the reference's numpy/OpenBLAS order.
 * ws: bsa_pooled_scores_workspace() bytes. */
size_t bsa_pooled_scores_workspace(int64_t heads, int64_t nq, int64_t nk);
int bsa_pooled_scores(const float* qp, const float* kp, int64_t heads, int64_t nq, int64_t nk,
                      int64_t dim, float scale, float* probs, void* ws, size_t ws_bytes,
                      void* stream);

/* row_softmax (tensorio.py:73-87): out = softmax(a * scale) per row of a
 * (rows, cols) fp32 matrix, reference arithmetic (numpy exp, pairwise sum). */
size_t bsa_row_softmax_workspace(int64_t rows, int64_t cols);
int bsa_row_softmax(const float* a, int64_t rows, int64_t cols, float scale, float* out,
                    void* ws, size_t ws_bytes, void* stream);

/* select_blocks (maskpred.py:142-174).  probs (H,nq,nk) fp32 contiguous ->
 * mask_bits (H*nq rows of ceil(nk/8) bytes) and counts[H*nq] (selected
 * blocks per row).  k_floor = MaskPolicy.min_blocks (maskpred.py:52-57),
 * computed by the caller.  ws: bsa_select_workspace() bytes. */
size_t bsa_select_workspace(int64_t heads, int64_t nq, int64_t nk);
int bsa_select_blocks(const float* probs, int64_t heads, int64_t nq, int64_t nk, double tau,
                      int64_t k_floor, uint8_t* mask_bits, int32_t* counts, void* ws,
                      size_t ws_bytes, void* stream);

/* predict_mask (maskpred.py:177-194): pool -> score -> select in one call.
 * q,k: patch-only (H,Tp,d) when patch_gather == NULL, else full interleaved
 * sequences described by patch_gather.  probs_out (H,nq,nk) fp32 is
 * optional (NULL to skip).  ws: bsa_predict_mask_workspace() bytes. */
size_t bsa_predict_mask_workspace(int64_t heads, int64_t patch_tokens, int64_t dim,
                                  int32_t block_q, int32_t block_k);
int bsa_predict_mask(const bsa_tensor* q, const bsa_tensor* k, const bsa_layout* patch_gather,
                     int32_t block_q, int32_t block_k, float scale, double tau,
                     int64_t k_floor, uint8_t* mask_bits, int32_t* counts, float* probs_out,
                     void* ws, size_t ws_bytes, void* stream);

/* predict_mask from pooled inputs: score -> select on (H,nq,d) / (H,nk,d)
 * fp32 block means (e.g. from bsa_qkv_project_pooled's epilogue), the
 * second half of maskpred.py:177-194.  Same masks, counts and probabilities
 * as bsa_predict_mask on the tensors those means were pooled from.
 * ws: bsa_predict_mask_pooled_workspace() bytes. */
size_t bsa_predict_mask_pooled_workspace(int64_t heads, int64_t nq, int64_t nk, int64_t dim);
int bsa_predict_mask_pooled(const float* q_pooled, const float* k_pooled, int64_t heads,
                            int64_t nq, int64_t nk, int64_t dim, float scale, double tau,
                            int64_t k_floor, uint8_t* mask_bits, int32_t* counts, float* probs_out,
                            void* ws, size_t ws_bytes, void* stream);

/* The step before the path, fused (the reference has no
 * model code, SPEC.md:8 -- the harness's QKV projection is the caller of
 * predict_mask, maskpred.py:177, and sparse_attention, sparse.py:182).
 * q/k/v (H,T,64) bf16 = x W^T + bias on the tensor cores (fp32 accumulate),
 * x (T, C=H*64) bf16 with rows in partitioned order [special_rows | patches]
 * (layout.py:113-138), W (3C, C) bf16 [Q | K | V] x C, bias (3C) bf16 or
 * NULL.  Outputs are head-major in the same row order, the layout
 * bsa_sparse_attention reads in place with inputs_permuted = 1.  The
 * epilogue also writes q_pooled (H, ceil(Tp/128), 64) and k_pooled
 * (H, ceil(Tp/64), 64) fp32 -- block_pool (maskpred.py:104-120) of the
 * bf16 patch rows, bit-identical to bsa_block_pool -- unless NULL.
 * C % 256 == 0, block_q 128 / block_k 64 (else BSA_EUNSUPPORTED). */
int bsa_qkv_project_pooled(const void* x, int64_t tokens, int64_t dim_in, const void* weight,
                           const void* bias, int64_t heads, int64_t head_dim, int64_t special_rows,
                           int32_t block_q, int32_t block_k, void* q, void* k, void* v,
                           float* q_pooled, float* k_pooled, void* stream);

/* The step after the path, fused (the harness's caller side of
 * sparse_attention, sparse.py:182): out (T, C) = residual + o W^T + bias, o
 * the attention output (H, T, 64) bf16 head-major as bsa_sparse_attention
 * writes it -- read in place as the GEMM's A operand, no transpose --,
 * W (C, C) bf16, residual and out (T, C) bf16 (out may alias residual),
 * bias (C) bf16 or NULL; fp32 accumulation, one rounding to bf16.
 * C = H*64, C % 256 == 0 (else BSA_EUNSUPPORTED). */
int bsa_proj_residual(const void* o, int64_t heads, int64_t tokens, const void* weight,
                      const void* bias, const void* residual, void* out, void* stream);

/* Token-order conversion by the copy engines: (heads, T, row_bytes) between
 * the interleaved source order and the partitioned order [specials |
 * patches] (layout.py:113-138, partition_permutation), two strided copies
 * per head (cudaMemcpy2DAsync, any host/device combination).
 * to_partitioned = 1: src interleaved -> dst partitioned; 0: the inverse.
 * Used by pipeline.HostLayerPipeline so host-resident layers arrive in the
 * layout bsa_sparse_attention reads in place (inputs_permuted = 1). */
int bsa_copy_tokens(void* dst, const void* src, const bsa_layout* layout, int64_t heads,
                    int64_t row_bytes, int32_t to_partitioned, void* stream);

/* Which scoring kernel predict_mask runs for nk key blocks of head_dim
 * dim: the fused score+softmax+select kernel's rows per CTA (8 or 4), or 0
 * for the three-kernel path (rows longer than shared memory holds, head_dim
 * not a multiple of 32, or BSA_SCORESEL=0 in the environment). */
int bsa_scoring_rows_per_cta(int64_t nk, int64_t dim);
/* Diagnostics: with BSA_SCORESEL_DEBUG=2 the fused scoring kernel records
 * clock64 per K stage of its first CTA (issue, ready, consumed; 512 each);
 * copies them (synchronously) to host.  Returns 0, or -1 if none recorded. */
int bsa_debug_scoring_trace(void* host, size_t bytes);

/* ------------------------------------------------------------------ */
/* Attention stage                                                    */
/* ------------------------------------------------------------------ */

/* sparse_attention (sparse.py:157-205).  q,k,v: (H,T,d) in interleaved
 * source order (or [specials|patches] order when inputs_permuted != 0).
 * out: (H,T,d) contiguous, out_dtype BSA_F32|BSA_BF16, same order as the
 * inputs.  Special query rows attend every key; patch query rows attend all
 * special keys plus the key blocks set in their mask row, ascending.
 * `counts` may be NULL (recomputed on device).  `shard`/`num_shards` split
 * the LPT-ordered work list for multi-GPU runs (0/1 = everything); rows of
 * other shards are not written.  ws: bsa_sparse_attention_workspace(). */
size_t bsa_sparse_attention_workspace(const bsa_layout* layout, int64_t heads, int64_t dim,
                                      int32_t block_q, int32_t block_k, int32_t in_dtype,
                                      int32_t inputs_permuted, int32_t flags);
int bsa_sparse_attention(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                         void* out, int32_t out_dtype, const bsa_layout* layout,
                         int32_t block_q, int32_t block_k, const uint8_t* mask_bits,
                         const int32_t* counts, float scale, int32_t inputs_permuted,
                         int32_t shard, int32_t num_shards, int32_t flags, void* ws,
                         size_t ws_bytes, void* stream);

/* Multi-GPU output scatter (the fused compute + collective of the sharded
 * path, paper_2509_07120_b200/shard.py).  Instead of writing a local
 * (H, T, d) output, the attention epilogue writes the row of interleaved
 * token t to the buffer of the rank that owns t:
 *     out_ptrs[r] + (h * (token_begin[r+1] - token_begin[r]) + t - token_begin[r]) * d
 * for token_begin[r] <= t < token_begin[r+1].  out_ptrs are peer pointers
 * (bsa_ipc_open) so the stores go over NVLink as each tile finishes; no
 * output all-reduce is needed.  out_ptrs (u64[world]) and token_begin
 * (i64[world+1]) are DEVICE arrays.  Tensor-core path, bf16 output only.
 * Replaces the reference's in-process result assembly (sparse.py:186-205). */
typedef struct {
  int32_t world;
  const uint64_t* out_ptrs;
  const int64_t* token_begin;
} bsa_scatter;
int bsa_sparse_attention_scatter(const bsa_tensor* q, const bsa_tensor* k, const bsa_tensor* v,
                                 const bsa_layout* layout, int32_t block_q, int32_t block_k,
                                 const uint8_t* mask_bits, const int32_t* counts, float scale,
                                 int32_t shard, int32_t num_shards, int32_t flags,
                                 const bsa_scatter* scatter, void* ws, size_t ws_bytes,
                                 void* stream);

/* CUDA IPC for the scatter buffers: allocate a device buffer and export its
 * handle (BSA_IPC_HANDLE_BYTES opaque bytes); open a peer's handle (enables
 * peer access); close / free. */
#define BSA_IPC_HANDLE_BYTES 64
int bsa_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
int bsa_ipc_open(const void* handle, void** dev_ptr);
int bsa_ipc_close(void* dev_ptr);
int bsa_ipc_free(void* dev_ptr);

/* Device time (ms) of the last tensor-core attention kernel launched on this
 * host thread with BSA_FLAG_TIMING set (waits for it); -1 on error. */
float bsa_last_kernel_ms(void);
/* Durations (ms) of the n most recent BSA_FLAG_TIMING launches of the
 * tensor-core kernel on this thread, oldest first (a ring of 64 event
 * pairs: a timed loop needs no host sync inside it); synchronises on them.
 * Returns n (<= max_n, <= 64) or -1 on a CUDA error; reset != 0 clears the
 * count. */
int bsa_kernel_times(float* out, int32_t max_n, int32_t reset);

/* Which path bsa_sparse_attention would take for these arguments:
 * BSA_PATH_SIMT or BSA_PATH_TC (or <0 on invalid arguments). */
int bsa_sparse_attention_path(const bsa_layout* layout, int64_t dim, int32_t block_q,
                              int32_t block_k, int32_t in_dtype, int32_t flags);

/* Selected patch-patch area per head (BlockMask.selected_area,
 * maskpred.py:97-101), int64[heads]: sum of |q block| * |k block| over set
 * bits with ragged tails weighted by their true length. */
int bsa_mask_selected_area(const uint8_t* mask_bits, int64_t heads, int64_t patch_tokens,
                           int32_t block_q, int32_t block_k, int64_t* area_out,
                           void* stream);

/* CSR view of a mask: row_ptr[H*nq+1] (int32, exclusive scan of per-row
 * counts) and col_idx (int32, ascending key blocks per row). */
int bsa_mask_to_csr(const uint8_t* mask_bits, int64_t heads, int64_t nq, int64_t nk,
                    int32_t* row_ptr, int32_t* col_idx, void* ws, size_t ws_bytes,
                    void* stream);
size_t bsa_mask_to_csr_workspace(int64_t heads, int64_t nq);

/* ---- dense attention statistics without the (H, T, T) map ----------------
 * the reference materialises the post-softmax map
 * (dense_attention_map, dense.py:79-102) and reduces it on the CPU
 * (quadrant_stats, analysis.py:47-74).  These stream S = Q K^T through the
 * tensor cores instead (bf16 q/k in source token order, head_dim 64).
 *
 * bsa_attention_row_stats: row_stats (H, T, 5) fp32 in source token order,
 *   per query row with x = s * scale * log2(e) over all T keys:
 *   [0] m = max x, [1] sum over special keys of 2^(x - m), [2] the same over
 *   patch keys, [3] max x over special keys, [4] max x over patch keys.
 *   So p(row, key) = 2^(x - m) / ([1] + [2]).
 * bsa_block_attention_map: from those row stats, block_map (H, nq, nk) fp32
 *   (block_q 128, block_k 64 over the patch tokens, the BlockMask geometry):
 *   the attention mass of patch q-block qb on patch k-block kb, i.e. the
 *   mean over the q-block's rows of the summed probabilities of the
 *   k-block's keys.  Deterministic (fixed reduction order).
 * Both pack q/k into the workspace (bsa_attention_stats_workspace bytes). */
size_t bsa_attention_stats_workspace(const bsa_layout* layout, int64_t heads);
int bsa_attention_row_stats(const bsa_tensor* q, const bsa_tensor* k, const bsa_layout* layout,
                            float scale, float* row_stats, void* ws, size_t ws_bytes,
                            void* stream);
int bsa_block_attention_map(const bsa_tensor* q, const bsa_tensor* k, const bsa_layout* layout,
                            float scale, const float* row_stats, float* block_map, void* ws,
                            size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BSA_H_ */
