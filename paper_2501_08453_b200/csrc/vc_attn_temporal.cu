// Temporal-branch attention (model.py:238-244): one sequence per spatial
// position l, made of the F tokens {f*Lv + l}; numerics.py:87-107 per head.
//
// The sequences are short (F = 16..160 frames), so the whole (position,
// head group) problem lives in shared memory: one CTA stages the F rows of
// q, k, v for HG heads (16-byte loads of one contiguous row segment per frame,
// converted to fp32 once), forms the F x F logits (each thread two keys of one
// query row, 8-byte shared loads), softmaxes each row and writes o = P v (two
// adjacent columns per thread, bf16x2 / float2 stores).  The work is ~F/2
// flop per byte read, so the kernel is judged against HBM bandwidth (SURVEY
// 8(d)).
//
// In : qkv [rows][ld] (q at col 0, k at col D, v at col 2D of each row)
// Out: o   [rows][ldo] at head columns h*dh (pointer pre-offset to the branch)
#include "vc_kernels.h"
#include "vc_ptx.cuh"

namespace vc {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void st_out2(float* o, float a, float b) {
  *reinterpret_cast<float2*>(o) = make_float2(a, b);
}
__device__ __forceinline__ void st_out2(__nv_bfloat16* o, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(o) = __floats2bfloat162_rn(a, b);
}

__device__ __forceinline__ void unpack8(const uint4& u, float* d, const float*) {
  // 4 fp32 in a 16-byte vector
  d[0] = __uint_as_float(u.x); d[1] = __uint_as_float(u.y);
  d[2] = __uint_as_float(u.z); d[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack8(const uint4& u, float* d, const __nv_bfloat16*) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    d[2 * i] = f.x;
    d[2 * i + 1] = f.y;
  }
}

// dh even; W = hg*dh columns; K rows padded to W+2 floats (odd 8-byte stride)
template <typename T, typename OutT>
__global__ void __launch_bounds__(kThreads)
    temporal_attn_kernel(const T* __restrict__ qkv, int64_t ld, int64_t D, OutT* __restrict__ o,
                         int64_t ldo, int F, int Lv, int H, int dh, int HG, float scale_log2, int vec) {
  extern __shared__ __align__(16) float smem[];
  constexpr int E = 16 / sizeof(T);  // elements per 16-byte vector
  const int l = blockIdx.x;
  const int h0 = blockIdx.y * HG;
  const int hg = min(HG, H - h0);
  const int W = hg * dh, WK = W + 2;
  float* sq = smem;               // [F][W]
  float* sv = sq + F * W;         // [F][W]
  float* sk = sv + F * W;         // [F][WK]
  float* sS = sk + F * WK;        // [hg][F][F+1]
  const int tid = threadIdx.x;

  // ---- stage q, k, v rows of the F frames (fp32 in smem) ----
  if (vec) {
    const int WV = W / E;
    for (int e = tid; e < F * WV; e += kThreads) {
      const int f = e / WV, cv = e - f * WV;
      const uint4* row = reinterpret_cast<const uint4*>(qkv + ((int64_t)f * Lv + l) * ld + (int64_t)h0 * dh) + cv;
      const uint4 a = __ldg(row), b = __ldg(row + D / E), c = __ldg(row + 2 * D / E);
      float t[E];
      unpack8(a, t, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < E; ++i) sq[f * W + cv * E + i] = t[i];
      unpack8(b, t, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < E; ++i) sk[f * WK + cv * E + i] = t[i];
      unpack8(c, t, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < E; ++i) sv[f * W + cv * E + i] = t[i];
    }
  } else {
    for (int e = tid; e < F * W; e += kThreads) {
      const int f = e / W, c = e - f * W;
      const T* row = qkv + ((int64_t)f * Lv + l) * ld + (int64_t)h0 * dh + c;
      sq[f * W + c] = to_f32(row[0]);
      sk[f * WK + c] = to_f32(row[D]);
      sv[f * W + c] = to_f32(row[2 * D]);
    }
  }
  __syncthreads();

  // ---- logits: S[h][i][j], j and j + F/2 per thread (F even) or one j ----
  const int half = (F + 1) / 2;
  const int nS = hg * F * half;
  for (int e = tid; e < nS; e += kThreads) {
    const int hh = e / (F * half), r = e - hh * F * half, i = r / half, j = r - i * half;
    const int j2 = j + half;
    const float2* qi = reinterpret_cast<const float2*>(sq + i * W + hh * dh);
    const float2* k1 = reinterpret_cast<const float2*>(sk + j * WK + hh * dh);
    const float2* k2 = reinterpret_cast<const float2*>(sk + (j2 < F ? j2 : j) * WK + hh * dh);
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 4
    for (int d = 0; d < dh / 2; ++d) {
      const float2 q = qi[d], x = k1[d], y = k2[d];
      a0 = fmaf(q.x, x.x, a0); a1 = fmaf(q.y, x.y, a1);
      b0 = fmaf(q.x, y.x, b0); b1 = fmaf(q.y, y.y, b1);
    }
    float* srow = sS + (hh * F + i) * (F + 1);
    srow[j] = (a0 + a1) * scale_log2;
    if (j2 < F) srow[j2] = (b0 + b1) * scale_log2;
  }
  __syncthreads();

  // ---- row softmax (one thread per (head, query) row) ----
  for (int rr = tid; rr < hg * F; rr += kThreads) {
    float* srow = sS + rr * (F + 1);
    float m = -INFINITY;
    for (int j = 0; j < F; ++j) m = fmaxf(m, srow[j]);
    float sum = 0.f;
    for (int j = 0; j < F; ++j) {
      const float pj = ptx::ex2(srow[j] - m);
      srow[j] = pj;
      sum += pj;
    }
    const float inv = 1.f / sum;
    for (int j = 0; j < F; ++j) srow[j] *= inv;
  }
  __syncthreads();

  // ---- o[i][h*dh + c] = sum_j P[h][i][j] v[j][h*dh + c], two columns per thread ----
  const int W2 = W / 2;
  for (int e = tid; e < F * W2; e += kThreads) {
    const int i = e / W2, c = 2 * (e - i * W2);
    const int hh = c / dh;  // dh even: c, c+1 share the head
    const float* prow = sS + (hh * F + i) * (F + 1);
    float a0 = 0.f, a1 = 0.f;
    for (int j = 0; j < F; ++j) {
      const float pj = prow[j];
      const float2 v = *reinterpret_cast<const float2*>(sv + j * W + c);
      a0 = fmaf(pj, v.x, a0);
      a1 = fmaf(pj, v.y, a1);
    }
    st_out2(o + ((int64_t)i * Lv + l) * ldo + (int64_t)h0 * dh + c, a0, a1);
  }
}

inline size_t smem_for(int F, int W, int hg) {
  return (size_t)4 * ((size_t)F * W * 2 + (size_t)F * (W + 2) + (size_t)hg * F * (F + 1));
}

}  // namespace

template <typename T, typename OutT>
int launch_temporal_attn(const T* qkv, int64_t ld, int64_t D, OutT* o, int64_t ldo, int F, int Lv,
                         int H, int dh, cudaStream_t st) {
  if (F <= 0 || Lv <= 0) return VC_OK;
  if (dh % 2 != 0 || (ldo % 2) != 0) {
    set_error("temporal attention needs an even head dim and output pitch (dh %d)", dh);
    return VC_ENOTSUP;
  }
  constexpr size_t kMaxSmem = 200 * 1024, kTarget = 56 * 1024;  // ~4 CTAs per SM
  const size_t es = sizeof(T);
  // head-group size: a multiple of u keeps every group's first column 16-byte aligned
  int u = 1;
  while (((int64_t)u * dh * es) % 16 != 0 && u < 16) ++u;
  const bool vec_ok = ((int64_t)u * dh * es) % 16 == 0 && (ld * es) % 16 == 0 && (D * es) % 16 == 0 &&
                      ((uintptr_t)qkv % 16) == 0;
  int HG = 0;
  if (vec_ok) {
    for (int c = u; c <= std::min(H, 8); c += u)
      if (smem_for(F, c * dh, c) <= kTarget) HG = c;
    if (HG == 0 && u <= H && smem_for(F, u * dh, u) <= kMaxSmem) HG = u;
  }
  const int vec = HG > 0 ? 1 : 0;
  if (!vec) {  // scalar staging, any head-group size
    HG = std::min(H, 8);
    while (HG > 1 && smem_for(F, HG * dh, HG) > kTarget) --HG;
  }
  const size_t smem = smem_for(F, HG * dh, HG);
  if (smem > kMaxSmem) {
    set_error("temporal attention: %d frames x head dim %d does not fit in shared memory", F, dh);
    return VC_ENOTSUP;
  }
  if ((H + HG - 1) / HG > 65535) { set_error("temporal grid too large"); return VC_ENOTSUP; }
  VC_CHECK_CUDA(cudaFuncSetAttribute(temporal_attn_kernel<T, OutT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
  dim3 grid((unsigned)Lv, (unsigned)((H + HG - 1) / HG));
  temporal_attn_kernel<T, OutT><<<grid, kThreads, smem, st>>>(
      qkv, ld, D, o, ldo, F, Lv, H, dh, HG, (float)(1.4426950408889634 / sqrt((double)dh)), vec);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

template int launch_temporal_attn<float, float>(const float*, int64_t, int64_t, float*, int64_t, int,
                                                int, int, int, cudaStream_t);
template int launch_temporal_attn<__nv_bfloat16, __nv_bfloat16>(const __nv_bfloat16*, int64_t, int64_t,
                                                                __nv_bfloat16*, int64_t, int, int, int,
                                                                int, cudaStream_t);

}  // namespace vc
