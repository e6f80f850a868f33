// bsa_capi.cu -- error state and small utilities of the C ABI (include/bsa.h).
#include <algorithm>
#include <cstdarg>
#include <cstdio>

#include "bsa_common.cuh"

namespace bsa {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace bsa

namespace bsa { extern unsigned long long* g_scoresel_trace; }
extern "C" {
int bsa_debug_scoring_trace(void* host, size_t bytes) {
  if (!bsa::g_scoresel_trace) return -1;
  return cudaMemcpy(host, bsa::g_scoresel_trace, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}

int bsa_version(void) { return 100; }

const char* bsa_last_error(void) { return bsa::g_err; }

int bsa_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// non-finite scan (as_f32's isfinite check, tensorio.py:47-59, on the device):
// one HBM-bound pass with 16-byte loads; any NaN/Inf sets *flag to 1.
// ---------------------------------------------------------------------------
namespace bsa {

__device__ __forceinline__ bool bad_f32(uint32_t w) { return (w & 0x7F800000u) == 0x7F800000u; }
__device__ __forceinline__ bool bad_bf16x2(uint32_t w) {
  return (w & 0x7F80u) == 0x7F80u || (w & 0x7F800000u) == 0x7F800000u;
}

template <bool BF16>
__global__ void __launch_bounds__(256) nonfinite_kernel(const void* __restrict__ x, int64_t H,
                                                        int64_t T, int64_t d, int64_t sH,
                                                        int64_t sT, int32_t* __restrict__ flag) {
  const int es = BF16 ? 2 : 4;
  const int64_t per = d * es / 16;  // 16-byte vectors per row (d * es % 16 == 0 here)
  const int64_t total = H * T * per;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % per, ht = i / per, t = ht % T, h = ht / T;
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(
        (const char*)x + ((h * sH + t * sT) * es) + c * 16));
    if (BF16)
      bad |= bad_bf16x2(u.x) | bad_bf16x2(u.y) | bad_bf16x2(u.z) | bad_bf16x2(u.w);
    else
      bad |= bad_f32(u.x) | bad_f32(u.y) | bad_f32(u.z) | bad_f32(u.w);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
__global__ void nonfinite_scalar_kernel(const T* __restrict__ x, int64_t H, int64_t Tn, int64_t d,
                                        int64_t sH, int64_t sT, int32_t* __restrict__ flag) {
  const int64_t total = H * Tn * d;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % d, ht = i / d, t = ht % Tn, h = ht / Tn;
    bad |= !isfinite(to_f32(x[h * sH + t * sT + c]));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace bsa

extern "C" int bsa_check_finite(const bsa_tensor* x, int32_t* flag, void* stream) {
  using namespace bsa;
  if (!x || !x->data || !flag) return fail(BSA_EINVAL, "check_finite: null argument");
  if (x->dtype != BSA_F32 && x->dtype != BSA_BF16)
    return fail(BSA_EINVAL, "check_finite: unsupported dtype code %d", x->dtype);
  if (x->heads < 1 || x->tokens < 1 || x->dim < 1) return BSA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool bf = x->dtype == BSA_BF16;
  const int64_t es = bf ? 2 : 4;
  const bool vec = (x->dim * es) % 16 == 0 && (uintptr_t)x->data % 16 == 0 &&
                   (x->stride_token * es) % 16 == 0 && (x->stride_head * es) % 16 == 0;
  const int64_t work = x->heads * x->tokens * (vec ? x->dim * es / 16 : x->dim);
  const int grid = (int)std::min<int64_t>(ceil_div(work, 256), 148 * 8);
  if (vec) {
    if (bf)
      nonfinite_kernel<true><<<grid, 256, 0, st>>>(x->data, x->heads, x->tokens, x->dim,
                                                   x->stride_head, x->stride_token, flag);
    else
      nonfinite_kernel<false><<<grid, 256, 0, st>>>(x->data, x->heads, x->tokens, x->dim,
                                                    x->stride_head, x->stride_token, flag);
  } else if (bf) {
    nonfinite_scalar_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        (const __nv_bfloat16*)x->data, x->heads, x->tokens, x->dim, x->stride_head,
        x->stride_token, flag);
  } else {
    nonfinite_scalar_kernel<float><<<grid, 256, 0, st>>>((const float*)x->data, x->heads,
                                                         x->tokens, x->dim, x->stride_head,
                                                         x->stride_token, flag);
  }
  BSA_LAUNCH_CHECK();
  return BSA_OK;
}

// Token-order conversion on the copy engines (host <-> device, or device <->
// device): (heads, T, row) in the interleaved source order <-> the
// partitioned order [specials | patches] (layout.py:113-138), as two strided
// copies per head (a frame's specials and its patches are contiguous runs).
// A host-resident layer then lands in HBM already partitioned -- the layout
// the attention kernel reads in place -- and its output leaves the same way.
extern "C" int bsa_copy_tokens(void* dst, const void* src, const bsa_layout* layout, int64_t heads,
                               int64_t row_bytes, int32_t to_partitioned, void* stream) {
  using namespace bsa;
  if (!dst || !src || !layout) return fail(BSA_EINVAL, "copy_tokens: null argument");
  const Layout L = to_layout(layout);
  if (L.frames < 1 || L.P < 1 || L.S < 0 || heads < 1 || row_bytes < 1)
    return fail(BSA_EINVAL, "copy_tokens: bad shape");
  const int64_t T = L.tokens(), F = L.frames, S = L.S, P = L.P, Ts = L.n_spec();
  const size_t frame = (size_t)(S + P) * row_bytes;
  const size_t spec_off = (size_t)(L.specials_first ? 0 : P) * row_bytes;
  const size_t patch_off = (size_t)(L.specials_first ? S : 0) * row_bytes;
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t h = 0; h < heads; ++h) {
    char* d = (char*)dst + (size_t)h * T * row_bytes;
    const char* s = (const char*)src + (size_t)h * T * row_bytes;
    if (to_partitioned) {
      if (S > 0)
        BSA_CUDA_TRY(cudaMemcpy2DAsync(d, (size_t)S * row_bytes, s + spec_off, frame,
                                       (size_t)S * row_bytes, (size_t)F, cudaMemcpyDefault, st));
      BSA_CUDA_TRY(cudaMemcpy2DAsync(d + (size_t)Ts * row_bytes, (size_t)P * row_bytes,
                                     s + patch_off, frame, (size_t)P * row_bytes, (size_t)F,
                                     cudaMemcpyDefault, st));
    } else {
      if (S > 0)
        BSA_CUDA_TRY(cudaMemcpy2DAsync(d + spec_off, frame, s, (size_t)S * row_bytes,
                                       (size_t)S * row_bytes, (size_t)F, cudaMemcpyDefault, st));
      BSA_CUDA_TRY(cudaMemcpy2DAsync(d + patch_off, frame, s + (size_t)Ts * row_bytes,
                                     (size_t)P * row_bytes, (size_t)P * row_bytes, (size_t)F,
                                     cudaMemcpyDefault, st));
    }
  }
  return BSA_OK;
}
