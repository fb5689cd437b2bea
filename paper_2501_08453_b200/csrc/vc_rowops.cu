// Memory-bound row kernels: LayerNorm row statistics, patch embed /
// unembed, and the one-time weight pack.  Judged against HBM bandwidth.
#include "vc_kernels.h"

namespace vc {

// ---------------------------------------------------------------------------
// LayerNorm without affine, model.py:89-92: (x - mean) / sqrt(var + 1e-5),
// biased variance.  The per-branch affine (gamma, beta) is folded into the
// projection weights / bias at pack time, so one normalised copy of the rows
// feeds all three branches' Q/K/V projections.  Rows come from two sources:
// the visual tokens then the (anchored, deduplicated) prompt rows.
// One warp per row; the row is held in registers between the passes.
// ---------------------------------------------------------------------------
// MOD (north-star AdaLN extension, oracle/vchitect_ext_oracle.py): the
// normalised row is modulated, LN(x) * (1 + scale) + shift, before the store.
template <typename OutT, int VPL, bool MOD = false>
__global__ void __launch_bounds__(256) ln_rows_kernel(const float* __restrict__ x, int64_t n_x,
                                                      const float* __restrict__ p, int64_t n_p,
                                                      int D, OutT* __restrict__ out,
                                                      const float* __restrict__ shift = nullptr,
                                                      const float* __restrict__ scale = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_x + n_p) return;
  const float* src = row < n_x ? x + row * D : p + (row - n_x) * D;
  float v[VPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    int d = lane + 32 * i;
    v[i] = d < D ? src[d] : 0.f;
    s += v[i];
  }
  const float mean = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    int d = lane + 32 * i;
    float c = d < D ? v[i] - mean : 0.f;
    q = fmaf(c, c, q);
  }
  const float rstd = rsqrtf(warp_sum(q) / D + 1e-5f);
  OutT* dst = out + row * D;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    int d = lane + 32 * i;
    if (d < D) {
      float y = (v[i] - mean) * rstd;
      if constexpr (MOD) y = fmaf(y, 1.f + __ldg(scale + d), __ldg(shift + d));
      dst[d] = from_f32<OutT>(y);
    }
  }
}

// bf16 output, D % 4 == 0: 16-byte loads and 8-byte stores (the row kernel
// above issues 4-byte loads; this one keeps 4x more bytes in flight per load).
template <int NV, bool MOD>
__global__ void __launch_bounds__(256) ln_rows_v4_kernel(const float* __restrict__ x, int64_t n_x,
                                                         const float* __restrict__ p, int64_t n_p, int D,
                                                         __nv_bfloat16* __restrict__ out,
                                                         const float* __restrict__ shift,
                                                         const float* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_x + n_p) return;
  const float4* src = reinterpret_cast<const float4*>(row < n_x ? x + row * D : p + (row - n_x) * D);
  const int D4 = D >> 2;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < D4 ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (lane + 32 * i < D4) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
      q = fmaf(a, a, fmaf(b, b, fmaf(c, c, fmaf(d, d, q))));
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / D + 1e-5f);
  uint2* dst = reinterpret_cast<uint2*>(out + row * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < D4) {
      float y0 = (v[i].x - mean) * rstd, y1 = (v[i].y - mean) * rstd;
      float y2 = (v[i].z - mean) * rstd, y3 = (v[i].w - mean) * rstd;
      if constexpr (MOD) {
        const float4 sc = __ldg(reinterpret_cast<const float4*>(scale) + c);
        const float4 sh = __ldg(reinterpret_cast<const float4*>(shift) + c);
        y0 = fmaf(y0, 1.f + sc.x, sh.x); y1 = fmaf(y1, 1.f + sc.y, sh.y);
        y2 = fmaf(y2, 1.f + sc.z, sh.z); y3 = fmaf(y3, 1.f + sc.w, sh.w);
      }
      __nv_bfloat162 lo = __floats2bfloat162_rn(y0, y1), hi = __floats2bfloat162_rn(y2, y3);
      dst[c] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
}

template <bool MOD>
int launch_ln_rows_v4(const float* x, int64_t n_x, const float* p, int64_t n_p, int D, __nv_bfloat16* out,
                      const float* shift, const float* scale, cudaStream_t st) {
  const int64_t rows = n_x + n_p;
  if (rows <= 0) return VC_OK;
  dim3 grid((unsigned)cdiv(rows, 8));
  const int nv = (int)cdiv(D / 4, 32);
  if (nv <= 4) ln_rows_v4_kernel<4, MOD><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else if (nv <= 13) ln_rows_v4_kernel<13, MOD><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else if (nv <= 24) ln_rows_v4_kernel<24, MOD><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else {
    set_error("LayerNorm supports dim <= 3072, got %d", D);
    return VC_ENOTSUP;
  }
  VC_CHECK_LAUNCH();
  return VC_OK;
}

template <typename OutT>
int launch_ln_rows(const float* x, int64_t n_x, const float* p, int64_t n_p, int D, OutT* out,
                   cudaStream_t st) {
  int64_t rows = n_x + n_p;
  if (rows <= 0) return VC_OK;
  if constexpr (sizeof(OutT) == 2) {
    if (D % 4 == 0) return launch_ln_rows_v4<false>(x, n_x, p, n_p, D, out, nullptr, nullptr, st);
  }
  dim3 grid((unsigned)cdiv(rows, 8));
  int vpl = (int)cdiv(D, 32);
  if (vpl <= 4) ln_rows_kernel<OutT, 4><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out);
  else if (vpl <= 16) ln_rows_kernel<OutT, 16><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out);
  else if (vpl <= 50) ln_rows_kernel<OutT, 50><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out);
  else if (vpl <= 96) ln_rows_kernel<OutT, 96><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out);
  else {
    set_error("LayerNorm supports dim <= 3072, got %d", D);
    return VC_ENOTSUP;
  }
  VC_CHECK_LAUNCH();
  return VC_OK;
}
template int launch_ln_rows<float>(const float*, int64_t, const float*, int64_t, int, float*, cudaStream_t);
template int launch_ln_rows<__nv_bfloat16>(const float*, int64_t, const float*, int64_t, int, __nv_bfloat16*, cudaStream_t);

int launch_ln_rows_mod(const float* x, int64_t n_x, const float* p, int64_t n_p, int D,
                       const float* shift, const float* scale, __nv_bfloat16* out, cudaStream_t st) {
  int64_t rows = n_x + n_p;
  if (rows <= 0) return VC_OK;
  if (D % 4 == 0) return launch_ln_rows_v4<true>(x, n_x, p, n_p, D, out, shift, scale, st);
  dim3 grid((unsigned)cdiv(rows, 8));
  int vpl = (int)cdiv(D, 32);
  typedef __nv_bfloat16 bf;
  if (vpl <= 4) ln_rows_kernel<bf, 4, true><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else if (vpl <= 16) ln_rows_kernel<bf, 16, true><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else if (vpl <= 50) ln_rows_kernel<bf, 50, true><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else if (vpl <= 96) ln_rows_kernel<bf, 96, true><<<grid, 256, 0, st>>>(x, n_x, p, n_p, D, out, shift, scale);
  else {
    set_error("LayerNorm supports dim <= 3072, got %d", D);
    return VC_ENOTSUP;
  }
  VC_CHECK_LAUNCH();
  return VC_OK;
}

// ---------------------------------------------------------------------------
// Patch embed, model.py:303-314 with patchify model.py:53-64 and
// sinusoidal_embedding model.py:79-86.  x[f][i][d] = patch(f,i) . w_in[:,d]
// + sinus(f*Lv + i)[d] + sinus(t)[d].  Angles and sin/cos in fp64 (the
// global token index reaches 1e5-1e6 where an fp32 angle would be off by
// 1e-2), the patch dot in fp64, stored fp32 (the residual stream).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sinus(double pos, int d, int D) {
  const int half = D >> 1;
  const int k = d < half ? d : d - half;
  const double freq = exp(-9.210340371976184 * (double)k / (double)half);  // -ln(1e4)
  const double ang = pos * freq;
  return d < half ? sin(ang) : cos(ang);
}

__global__ void embed_kernel(const float* __restrict__ lat, const float* __restrict__ w_in,
                             float* __restrict__ x, int F, int first_frame, int tok0, int ntok, int h,
                             int w, int c, int p, int D, double t) {
  // x[f][k][d] for tokens i = tok0 + k of each frame (a sequence-parallel rank
  // embeds only its own rows; model.py:303-314 is position-wise, so the rows
  // equal the single-device ones exactly)
  const int gh = (h + p - 1) / p, gw = (w + p - 1) / p;
  const int Lv = gh * gw, pd = p * p * c;
  const int64_t total = (int64_t)F * ntok * D;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const int64_t r = e / D;  // f*ntok + k
    const int f = (int)(r / ntok), i = tok0 + (int)(r % ntok);
    const int gy = i / gw, gx = i % gw;
    double acc = 0.0;
    for (int j = 0; j < pd; ++j) {
      const int py = j / (p * c), px = (j / c) % p, ch = j % c;
      const int yy = gy * p + py, xx = gx * p + px;
      if (yy < h && xx < w)
        acc += (double)lat[(((int64_t)f * h + yy) * w + xx) * c + ch] * (double)w_in[(int64_t)j * D + d];
    }
    acc += sinus((double)((int64_t)(first_frame + f) * Lv + i), d, D);
    acc += sinus(t, d, D);
    x[e] = (float)acc;
  }
}

// Unembed, model.py:331-333 + unpatchify model.py:67-76: one warp per token
// computes its p*p*c outputs (x_tok . w_out) and scatters the in-bounds
// pixels (the crop).
template <int PD>
__global__ void unembed_kernel(const float* __restrict__ x, const float* __restrict__ w_out,
                               float* __restrict__ eps, int F, int h, int w, int c, int p, int D,
                               ReverseStep rs) {
  const int gh = (h + p - 1) / p, gw = (w + p - 1) / p;
  const int Lv = gh * gw, pd = p * p * c;
  const int lane = threadIdx.x & 31;
  const int64_t tok = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tok >= (int64_t)F * Lv) return;
  float acc[PD];
#pragma unroll
  for (int j = 0; j < PD; ++j) acc[j] = 0.f;
  const float* xr = x + tok * D;
  for (int d = lane; d < D; d += 32) {
    const float xv = xr[d];
#pragma unroll
    for (int j = 0; j < PD; ++j)
      if (j < pd) acc[j] = fmaf(xv, w_out[(int64_t)d * pd + j], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < PD; ++j) acc[j] = warp_sum(acc[j]);
  const int f = (int)(tok / Lv), i = (int)(tok % Lv);
  const int gy = i / gw, gx = i % gw;
#pragma unroll
  for (int j = 0; j < PD; ++j) {
    if (j >= pd || lane != (j & 31)) continue;
    const int py = j / (p * c), px = (j / c) % p, ch = j % c;
    const int yy = gy * p + py, xx = gx * p + px;
    if (yy < h && xx < w) {
      const int64_t px_i = (((int64_t)f * h + yy) * w + xx) * c + ch;
      if (eps) eps[px_i] = acc[j];
      if (rs.x_prev) {  // fused ancestral step, diffusion.py:95-116
        float v = (rs.x_t[px_i] - rs.coef_eps * acc[j]) * rs.inv_sqrt_alpha;
        if (rs.noise) v = fmaf(rs.sqrt_beta, rs.noise[px_i], v);
        rs.x_prev[px_i] = v;
      }
    }
  }
}

int launch_embed(const float* lat, const float* w_in, float* x, int F, int first_frame, int tok0,
                 int ntok, int h, int w, int c, int p, int D, double t, cudaStream_t st) {
  const int Lv = ((h + p - 1) / p) * ((w + p - 1) / p);
  if (ntok < 0) ntok = Lv - tok0;
  if (tok0 < 0 || tok0 + ntok > Lv) { set_error("token range [%d, %d) outside %d tokens", tok0, tok0 + ntok, Lv); return VC_EINVAL; }
  const int64_t total = (int64_t)F * ntok * D;
  if (total <= 0) return VC_OK;
  const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  embed_kernel<<<blocks, 256, 0, st>>>(lat, w_in, x, F, first_frame, tok0, ntok, h, w, c, p, D, t);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

int launch_unembed(const float* x, const float* w_out, float* eps, int F, int h, int w, int c,
                   int p, int D, cudaStream_t st, ReverseStep rs) {
  const int64_t toks = (int64_t)F * ((h + p - 1) / p) * ((w + p - 1) / p);
  const int pd = p * p * c;
  if (toks <= 0) return VC_OK;
  dim3 grid((unsigned)cdiv(toks, 8));
  if (pd <= 16) unembed_kernel<16><<<grid, 256, 0, st>>>(x, w_out, eps, F, h, w, c, p, D, rs);
  else if (pd <= 64) unembed_kernel<64><<<grid, 256, 0, st>>>(x, w_out, eps, F, h, w, c, p, D, rs);
  else {
    set_error("unembed supports patch*patch*channels <= 64, got %d", pd);
    return VC_ENOTSUP;
  }
  VC_CHECK_LAUNCH();
  return VC_OK;
}

// ---------------------------------------------------------------------------
// Weight pack (one-time).  raw = 3 branches x {gamma[D], beta[D], wq, wk, wv,
// wo [D][D] row-major}.  Folding: (xhat*gamma + beta) @ W
//   = xhat @ (diag(gamma) W) + beta @ W.
// fp32 layout : Wqkv [D][9D] (x @ W orientation), bias [9D], Wo [3D][D];
//               column n of the 9D space = branch*3D + {q,k,v}*D + c.
// bf16 layout : Wqkv^T [Npad][D] (K-major for tcgen05) in the head-padded
//               column space of QkvPad (zero rows for the pad columns, so
//               the GEMM writes exact zeros there), bias [Npad] fp32,
//               Wo^T [D][3D].
// ---------------------------------------------------------------------------
__device__ __forceinline__ const float* raw_branch(const float* raw, int b, int D) {
  return raw + (int64_t)b * (2 * (int64_t)D + 4 * (int64_t)D * D);
}
__device__ __forceinline__ const float* raw_w(const float* raw, int b, int which, int D) {
  return raw_branch(raw, b, D) + 2 * (int64_t)D + (int64_t)which * D * D;  // which: 0 q,1 k,2 v,3 o
}

// Packed QKV column n -> (branch, which, source column c); false for a pad column.
__device__ __forceinline__ bool qkv_source(int64_t n, int D, int H, bool padded, QkvPad q, int& b,
                                           int& which, int& c) {
  if (!padded) {
    b = (int)(n / (3 * D)); which = (int)((n / D) % 3); c = (int)(n % D);
    return true;
  }
  const int dh = D / H;
  int64_t j;
  if (n < 3 * q.SEG) { b = 0; which = (int)(n / q.SEG); j = n % q.SEG; }
  else if (n < q.fs_base()) {
    b = 1; j = n - 3 * q.SEG;
    if (j >= 3 * D) return false;
    which = (int)(j / D); c = (int)(j % D);
    return true;
  } else { b = 2; const int64_t r = n - q.fs_base(); which = (int)(r / q.SEG); j = r % q.SEG; }
  if (q.compact) {  // [h: d 0..63] x H, then the (h, 64), (h, 65) tail pairs (vc_kernels.h)
    int h, d;
    if (j < q.MAIN) { h = (int)(j / q.HW); d = (int)(j % q.HW); }
    else { const int t = (int)(j - q.MAIN); h = t / (dh - q.HW); d = q.HW + t % (dh - q.HW); }
    if (h >= H) { c = -2; return false; }
    c = h * dh + d;
    return true;
  }
  const int h = (int)(j / q.DP), d = (int)(j % q.DP);
  if (h >= H || d >= dh) {
    c = (h < H && d == dh) ? -1 : -2;  // -1: first V pad column (the ones column, see below)
    return false;
  }
  c = h * dh + d;
  return true;
}

// The first padding column of every head's V (d == dh < DP) is a constant 1.0
// (zero weights, bias 1): the P.V MMA then accumulates the softmax row sum
// in O[:, dh] for free, in the same bf16 P the numerator uses.
__device__ __forceinline__ bool is_ones_column(int64_t n, int D, int H, QkvPad q) {
  if (q.compact) return false;  // compact: fill_vt_pad_kernel writes the ones row
  int b, which, c;
  if (qkv_source(n, D, H, true, q, b, which, c)) return false;
  return b != 1 && which == 2 && c == -1;
}

template <typename T, bool KMAJOR>
__global__ void pack_qkv_kernel(const float* __restrict__ raw, T* __restrict__ wqkv, int D, int H,
                                int64_t N, QkvPad q) {
  // one thread per (k, n) of the N x D matrix
  const int64_t total = N * D;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t n, k;
    if (KMAJOR) { n = e / D; k = e % D; }  // output [N][D], k fastest
    else { k = e / N; n = e % N; }         // output [D][N]
    int b, which, c;
    float v = 0.f;
    if (qkv_source(n, D, H, KMAJOR, q, b, which, c))
      v = raw_branch(raw, b, D)[k] * raw_w(raw, b, which, D)[k * D + c];
    wqkv[e] = from_f32<T>(v);
  }
}

__global__ void pack_bias_kernel(const float* __restrict__ raw, float* __restrict__ bias, int D,
                                 int H, int64_t N, bool padded, QkvPad q) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  int b, which, c;
  if (!qkv_source(n, D, H, padded, q, b, which, c)) {
    bias[n] = (padded && is_ones_column(n, D, H, q)) ? 1.f : 0.f;
    return;
  }
  const float* beta = raw_branch(raw, b, D) + D;
  const float* W = raw_w(raw, b, which, D);
  double acc = 0.0;
  for (int k = 0; k < D; ++k) acc += (double)beta[k] * (double)W[(int64_t)k * D + c];
  bias[n] = (float)acc;
}

template <typename T, bool KMAJOR>
__global__ void pack_o_kernel(const float* __restrict__ raw, T* __restrict__ wo, int D) {
  const int64_t total = (int64_t)3 * D * D;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t kk, n;  // kk in [0, 3D): branch*D + k
    if (KMAJOR) { n = e / (3 * (int64_t)D); kk = e % (3 * (int64_t)D); }  // [D][3D]
    else { kk = e / D; n = e % D; }                                      // [3D][D]
    const int b = (int)(kk / D), k = (int)(kk % D);
    wo[e] = from_f32<T>(raw_w(raw, b, 3, D)[(int64_t)k * D + n]);
  }
}

// Wo^T for the head-slot layout of the O-GEMM A operand (acat [Nv][3][H][S],
// AttnTcParams.head_slot = S): [D][3*H*S] bf16, zero for the slot padding.
__global__ void pack_o_slot_kernel(const float* __restrict__ raw, __nv_bfloat16* __restrict__ wo, int D, int H,
                                   int S) {
  const int dh = D / H;
  const int64_t K = 3 * (int64_t)H * S;
  const int64_t total = (int64_t)D * K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / K, kk = e % K;
    const int b = (int)(kk / ((int64_t)H * S));
    const int r = (int)(kk % ((int64_t)H * S));
    const int h = r / S, d = r % S;
    wo[e] = __float2bfloat16_rn(d < dh ? raw_w(raw, b, 3, D)[(int64_t)(h * dh + d) * D + n] : 0.f);
  }
}

int launch_pack(const float* raw, void* wqkv, float* bias, void* wo, int D, int H, bool bf16,
                cudaStream_t st, void* wqkv_c, float* bias_c, void* wo_s) {
  const int blocks = 148 * 8;
  const QkvPad q = qkv_pad_layout(D, H);
  const int64_t N = bf16 ? q.Npad : 9 * (int64_t)D;
  if (bf16) {
    if (q.DP == 0) { set_error("head dim %d unsupported on the bf16 path", D / H); return VC_ENOTSUP; }
    pack_qkv_kernel<__nv_bfloat16, true><<<blocks, 256, 0, st>>>(raw, (__nv_bfloat16*)wqkv, D, H, N, q);
    pack_o_kernel<__nv_bfloat16, true><<<blocks, 256, 0, st>>>(raw, (__nv_bfloat16*)wo, D);
    if (wqkv_c && bias_c && qkv_compact_ok(D, H)) {
      const QkvPad qc = qkv_compact_layout(D, H);
      pack_qkv_kernel<__nv_bfloat16, true><<<blocks, 256, 0, st>>>(raw, (__nv_bfloat16*)wqkv_c, D, H, qc.Npad, qc);
      pack_bias_kernel<<<(unsigned)cdiv(qc.Npad, 128), 128, 0, st>>>(raw, bias_c, D, H, qc.Npad, true, qc);
    }
    if (wo_s && qkv_compact_ok(D, H))
      pack_o_slot_kernel<<<blocks, 256, 0, st>>>(raw, (__nv_bfloat16*)wo_s, D, H, qkv_pad_layout(D, H).DP);
  } else {
    pack_qkv_kernel<float, false><<<blocks, 256, 0, st>>>(raw, (float*)wqkv, D, H, N, q);
    pack_o_kernel<float, false><<<blocks, 256, 0, st>>>(raw, (float*)wo, D);
  }
  pack_bias_kernel<<<(unsigned)cdiv(N, 128), 128, 0, st>>>(raw, bias, D, H, N, bf16, q);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

// V^T rows [dh, DP) of every (sequence, head) slot for keys [0, keys): the
// ones column (row dh) and zeros.  The compact QKV GEMM writes rows < dh only.
// 16-byte stores over whole rows when the pitch allows (keys past `keys` up
// to the pitch are never read: the attention's V map ends at Lk).
template <bool V16>
__global__ void fill_vt_pad_kernel(__nv_bfloat16* __restrict__ vt, int64_t nslots, int DP, int dh, int64_t ld,
                                   int64_t keys) {
  const int rows = DP - dh;
  const int64_t kw = V16 ? ld / 8 : (keys + 1) / 2;  // vectors per row
  const int64_t total = nslots * rows * kw;
  const uint32_t one2 = 0x3f803f80u;  // bf16x2 (1, 1)
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = e % kw;
    const int64_t sr = e / kw;
    const int r = (int)(sr % rows);
    const int64_t slot = sr / rows;
    const uint32_t x = r == 0 ? one2 : 0u;
    if (V16) reinterpret_cast<uint4*>(vt + (slot * DP + dh + r) * ld)[w] = make_uint4(x, x, x, x);
    else reinterpret_cast<uint32_t*>(vt + (slot * DP + dh + r) * ld)[w] = x;
  }
}

int launch_fill_vt_pad(__nv_bfloat16* vt, int64_t nslots, int DP, int dh, int64_t ld, int64_t keys,
                       cudaStream_t st) {
  if (nslots <= 0 || keys <= 0 || dh >= DP) return VC_OK;
  if (ld % 2) { set_error("V^T pitch must be even"); return VC_EINVAL; }
  const bool v16 = ld % 8 == 0 && ((uintptr_t)vt % 16) == 0;
  const int64_t total = nslots * (DP - dh) * (v16 ? ld / 8 : (keys + 1) / 2);
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  if (v16) fill_vt_pad_kernel<true><<<blocks, 256, 0, st>>>(vt, nslots, DP, dh, ld, keys);
  else fill_vt_pad_kernel<false><<<blocks, 256, 0, st>>>(vt, nslots, DP, dh, ld, keys);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

}  // namespace vc
