// Temporal-branch attention (model.py:238-244): one sequence per spatial
// position l, made of the F tokens {f*Lv + l}; numerics.py:87-107 per head.
//
// The sequences are short (F = 16..160 frames), so the whole (position,
// head group) problem lives in shared memory: one CTA stages the F rows of
// q, k, v for HG heads (one coalesced row segment per frame), forms the F x F
// logits, softmaxes each row and writes o = P v.  The work is ~F/2 flop per
// byte read, so the kernel is judged against HBM bandwidth.
//
// In : qkv [rows][ld] (q at col 0, k at col D, v at col 2D of each row)
// Out: o   [rows][ldo] at head columns h*dh (pointer pre-offset to the branch)
#include "vc_kernels.h"
#include "vc_ptx.cuh"

namespace vc {

namespace {

constexpr int kThreads = 256;

template <typename T, typename OutT>
__global__ void __launch_bounds__(kThreads)
    temporal_attn_kernel(const T* __restrict__ qkv, int64_t ld, int64_t D, OutT* __restrict__ o,
                         int64_t ldo, int F, int Lv, int H, int dh, int HG, float scale_log2, int vec) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int KP = sizeof(T) == 2 ? 2 : 1;  // K row padding: odd 32-bit word stride
  constexpr int E = 16 / sizeof(T);           // elements per 16-byte vector
  const int l = blockIdx.x;
  const int h0 = blockIdx.y * HG;
  const int hg = min(HG, H - h0);
  const int W = hg * dh;  // columns of this head group
  float* sS = reinterpret_cast<float*>(smem);                                   // [hg][F][F+1]
  T* sq = reinterpret_cast<T*>(smem + ((hg * F * (F + 1) * 4 + 15) & ~15));    // [F][W]
  T* sv = sq + F * W;                                                            // [F][W]
  T* sk = sv + F * W;                                                            // [F][W+KP]
  const int tid = threadIdx.x;

  // ---- stage q, k, v rows of the F frames ----
  if (vec) {  // 16-byte global loads (head group start and row pitch 16-byte aligned)
    const int WV = W / E;
    for (int e = tid; e < F * WV; e += kThreads) {
      const int f = e / WV, cv = e - f * WV;
      const uint4* row = reinterpret_cast<const uint4*>(qkv + ((int64_t)f * Lv + l) * ld + (int64_t)h0 * dh) + cv;
      const uint4 a = __ldg(row), b = __ldg(row + D / E), c = __ldg(row + 2 * D / E);
      *reinterpret_cast<uint4*>(sq + f * W + cv * E) = a;
      *reinterpret_cast<uint4*>(sv + f * W + cv * E) = c;
      uint32_t* kd = reinterpret_cast<uint32_t*>(sk + f * (W + KP) + cv * E);
      kd[0] = b.x; kd[1] = b.y; kd[2] = b.z; kd[3] = b.w;
    }
  } else {
    for (int e = tid; e < F * W; e += kThreads) {
      const int f = e / W, c = e - f * W;
      const T* row = qkv + ((int64_t)f * Lv + l) * ld + (int64_t)h0 * dh + c;
      sq[f * W + c] = row[0];
      sk[f * (W + KP) + c] = row[D];
      sv[f * W + c] = row[2 * D];
    }
  }
  __syncthreads();

  // ---- logits: S[h][i][j] = q_i . k_j (log2 domain) ----
  const int nS = hg * F * F;
  for (int e = tid; e < nS; e += kThreads) {
    const int hh = e / (F * F), r = e - hh * F * F, i = r / F, j = r - i * F;
    const T* qi = sq + i * W + hh * dh;
    const T* kj = sk + j * (W + KP) + hh * dh;
    float acc = 0.f;
#pragma unroll 4
    for (int d = 0; d < dh; ++d) acc = fmaf(to_f32(qi[d]), to_f32(kj[d]), acc);
    sS[(hh * F + i) * (F + 1) + j] = acc * scale_log2;
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

  // ---- o[i][h*dh + d] = sum_j P[h][i][j] v[j][h*dh + d] ----
  for (int e = tid; e < F * W; e += kThreads) {
    const int i = e / W, c = e - i * W;
    const int hh = c / dh;
    const float* prow = sS + (hh * F + i) * (F + 1);
    float acc = 0.f;
    for (int j = 0; j < F; ++j) acc = fmaf(prow[j], to_f32(sv[j * W + c]), acc);
    o[((int64_t)i * Lv + l) * ldo + (int64_t)h0 * dh + c] = from_f32<OutT>(acc);
  }
}

inline size_t smem_for(int F, int W, int hg, size_t es) {
  const int KP = es == 2 ? 2 : 1;
  return (((size_t)4 * hg * F * (F + 1) + 15) & ~(size_t)15) + es * ((size_t)F * W * 2 + (size_t)F * (W + KP));
}

}  // namespace

template <typename T, typename OutT>
int launch_temporal_attn(const T* qkv, int64_t ld, int64_t D, OutT* o, int64_t ldo, int F, int Lv,
                         int H, int dh, cudaStream_t st) {
  if (F <= 0 || Lv <= 0) return VC_OK;
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
      if (smem_for(F, c * dh, c, es) <= kTarget) HG = c;
    if (HG == 0 && u <= H && smem_for(F, u * dh, u, es) <= kMaxSmem) HG = u;
  }
  const int vec = HG > 0 ? 1 : 0;
  if (!vec) {  // scalar staging, any head-group size
    HG = std::min(H, 8);
    while (HG > 1 && smem_for(F, HG * dh, HG, es) > kTarget) --HG;
  }
  const size_t smem = (smem_for(F, HG * dh, HG, es) + 15) / 16 * 16;
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
