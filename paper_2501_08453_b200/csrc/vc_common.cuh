// Shared helpers for the vchitect_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>

#include "../../include/vchitect_b200.h"

namespace vc {

// Thread-local last error (vc_last_error()).
void set_error(const char* fmt, ...);

#define VC_CHECK_CUDA(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::vc::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                      cudaGetErrorString(_e));                                \
      return VC_ECUDA;                                                        \
    }                                                                         \
  } while (0)

#define VC_CHECK_LAUNCH()                                                     \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      ::vc::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__,          \
                      cudaGetErrorString(_e));                                \
      return VC_ECUDA;                                                        \
    }                                                                         \
  } while (0)

#define VC_TRY(expr)                                                          \
  do {                                                                        \
    int _r = (expr);                                                          \
    if (_r != VC_OK) return _r;                                               \
  } while (0)

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Generic strided attention problem (SIMT kernels; see vc_attn_simt.cu).
// Token t of sequence s lives at row s*seq_stride + t*tok_stride of its
// buffer; head h occupies columns [col + h*dh, col + (h+1)*dh).
// Keys are the concatenation of an optional shared segment A (rows 0..na-1
// of ka/va, every key's logit biased by log(weight_a): the deduplicated
// anchored text) and the per-sequence segment B.
// Pointers are pre-offset to the head-0 column.
template <typename T, typename OutT>
struct AttnArgs {
  const T* q; int64_t ldq; int64_t q_seq_stride, q_tok_stride;
  const T* k; const T* v; int64_t ldk; int64_t k_seq_stride, k_tok_stride;
  const T* ka; const T* va; int64_t lda; int32_t na; float log2_weight_a;
  OutT* o; int64_t ldo; int64_t o_seq_stride, o_tok_stride;
  int32_t n_seq, len_q, len_k, heads, dh;
  float scale_log2;  // log2(e)/sqrt(dh)
};

}  // namespace vc
