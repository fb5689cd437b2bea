// North-star extensions of the block (BASELINE.json north_star; SURVEY.md §8
// "a-ext"): AdaLN timestep modulation, QK-RMSNorm + 3D RoPE, gated residual
// and the gated GELU FFN.  The reference `spsim` has none of them, so their
// semantics are defined by oracle/vchitect_ext_oracle.py (parity unpinned) and
// checked against it by tests/test_gpu_ext.py.
//
// Per forward (vc_ext_block_forward):
//   adaln_mod_kernel    mod[6][D] = silu(sinus(t)) @ w_ada + b_ada   (tiny GEMV)
//   rope_table_kernel   (cos, sin) per frame / grid row / grid column  (tiny)
//   then block_forward_bf16 with ExtArgs: modulated LN, QKV GEMM with the
//   RMSNorm + RoPE epilogue (EPI_QKVN), the three attentions, the O GEMM with
//   the gated residual (EPI_F32G), modulated LN of h, FFN up (EPI_GELU) and
//   FFN down with the gated residual (EPI_F32G).
#include <math.h>

#include "vc_kernels.h"

namespace vc {

namespace {
inline size_t aup(size_t v) { return (v + 1023) / 1024 * 1024; }

struct ExtDims {
  int64_t F, Lv, Lt, D, H, dh, Nv, gh, gw, Dff;
};

struct ExtLayout {  // packed extension weights (bytes)
  size_t w_ada, b_ada, qn, kn, w1, b1, w2, b2, total;
};
ExtLayout ext_layout(const ExtDims& d) {
  ExtLayout l;
  size_t o = 0;
  l.w_ada = o; o = aup(o + (size_t)d.D * 6 * d.D * 4);
  l.b_ada = o; o = aup(o + (size_t)6 * d.D * 4);
  l.qn = o; o = aup(o + (size_t)2 * d.dh * 4);
  l.kn = o; o = aup(o + (size_t)2 * d.dh * 4);
  l.w1 = o; o = aup(o + (size_t)d.Dff * d.D * 2);
  l.b1 = o; o = aup(o + (size_t)d.Dff * 4);
  l.w2 = o; o = aup(o + (size_t)d.D * d.Dff * 2);
  l.b2 = o; o = aup(o + (size_t)d.D * 4);
  l.total = o;
  return l;
}

void rope_split(int64_t dh, int32_t& nt, int32_t& ny, int32_t& nx) {
  const int32_t p = (int32_t)(dh / 2);
  ny = nx = p / 3;
  nt = p - ny - nx;
}

struct ExtWs {  // workspace after the bf16 block's own
  size_t block, mod, rope, u, total;
  int64_t rope_off_y, rope_off_x, rope_n;
};
ExtWs ext_ws(const ExtDims& d) {
  ExtWs w;
  int32_t nt, ny, nx;
  rope_split(d.dh, nt, ny, nx);
  w.rope_off_y = d.F * nt;
  w.rope_off_x = w.rope_off_y + d.gh * ny;
  w.rope_n = w.rope_off_x + d.gw * nx;
  size_t o = aup(bf16_workspace_bytes(d.F, d.Lv, d.Lt, d.D, d.H));
  w.block = 0;
  w.mod = o; o = aup(o + (size_t)6 * d.D * 4);
  w.rope = o; o = aup(o + (size_t)w.rope_n * 8);
  if (d.Dff > 3 * d.D) { w.u = o; o = aup(o + (size_t)d.Nv * d.Dff * 2); }
  else w.u = bf16_workspace_acat_offset(d.F, d.Lv, d.Lt, d.D, d.H);  // free after the O GEMM
  w.total = o;
  return w;
}

int check_ext(const vc_ext_shape* s, ExtDims* d) {
  if (!s) { set_error("null shape"); return VC_EINVAL; }
  VC_TRY(vc_block_shape_check(&s->block));
  const vc_block_shape& b = s->block;
  if (b.dtype != VC_DTYPE_BF16) { set_error("the extended block runs on the bf16 path only"); return VC_EINVAL; }
  const int64_t dh = b.dim / b.heads;
  if (dh % 2) { set_error("3D RoPE needs an even head dim, got %lld", (long long)dh); return VC_EINVAL; }
  if (qkv_head_pad(dh) == 0) { set_error("head dim %lld unsupported on the tensor-core path", (long long)dh); return VC_ENOTSUP; }
  if (s->grid_h < 1 || s->grid_w < 1 || (int64_t)s->grid_h * s->grid_w != b.visual_len) {
    set_error("patch grid %dx%d does not hold %d visual tokens", s->grid_h, s->grid_w, b.visual_len);
    return VC_EINVAL;
  }
  if (s->ffn_dim < 8 || s->ffn_dim % 8) { set_error("ffn_dim must be a positive multiple of 8, got %d", s->ffn_dim); return VC_EINVAL; }
  if (d) {
    d->F = b.frames; d->Lv = b.visual_len; d->Lt = b.text_len; d->D = b.dim; d->H = b.heads;
    d->dh = dh; d->Nv = d->F * d->Lv; d->gh = s->grid_h; d->gw = s->grid_w; d->Dff = s->ffn_dim;
  }
  return VC_OK;
}

__device__ __forceinline__ double sinus_t(double pos, int d, int D) {  // model.py:79-86
  const int half = D >> 1;
  const int k = d < half ? d : d - half;
  const double ang = pos * exp(-9.210340371976184 * (double)k / (double)half);
  return d < half ? sin(ang) : cos(ang);
}

// mod[c] = sum_k silu(sinus(t)[k]) * w_ada[k][c] + b_ada[c]; 32 columns per
// block (one coalesced 128-byte row segment per warp load), 32 K slices (one
// per warp) reduced through shared memory.  HBM-bound: w_ada is read once.
constexpr int kModSlices = 32;
__global__ void __launch_bounds__(1024) adaln_mod_kernel(double t, int D, const float* __restrict__ w,
                                                        const float* __restrict__ b, float* __restrict__ mod) {
  extern __shared__ float se[];  // [D] silu(temb), then [kModSlices][32] partials
  for (int k = threadIdx.x; k < D; k += blockDim.x) {
    const double e = sinus_t(t, k, D);
    se[k] = (float)(e / (1.0 + exp(-e)));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, ks = threadIdx.x >> 5;
  const int64_t N = 6 * (int64_t)D;
  const int64_t col = (int64_t)blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (col < N)
#pragma unroll 4
    for (int k = ks; k < D; k += kModSlices) acc = fmaf(se[k], __ldg(w + (int64_t)k * N + col), acc);
  float* red = se + D;
  red[ks * 32 + lane] = acc;
  __syncthreads();
  if (ks == 0 && col < N) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kModSlices; ++i) s += red[i * 32 + lane];
    mod[col] = s + b[col];
  }
}

// (cos, sin) of pos * 1e4^(-j / n) per axis, fp64 angles.
__global__ void rope_table_kernel(float2* __restrict__ tab, int64_t F, int64_t gh, int64_t gw, int nt,
                                  int ny, int nx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t oy = F * nt, ox = oy + gh * ny, n = ox + gw * nx;
  if (i >= n) return;
  int64_t pos, j, na;
  if (i < oy) { pos = i / nt; j = i - pos * nt; na = nt; }
  else if (i < ox) { pos = (i - oy) / ny; j = (i - oy) - pos * ny; na = ny; }
  else { pos = (i - ox) / nx; j = (i - ox) - pos * nx; na = nx; }
  const double ang = (double)pos * pow(10000.0, -(double)j / (double)na);
  tab[i] = make_float2((float)cos(ang), (float)sin(ang));
}

// dst[c][r] = bf16(src[r][c]): x @ W weights -> the K-major B operand.
__global__ void transpose_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                      int64_t R, int64_t C) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < R && c < C) ? src[r * C + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (c < C && r < R) dst[c * R + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

int launch_transpose_bf16(const float* src, void* dst, int64_t R, int64_t C, cudaStream_t st) {
  dim3 grid((unsigned)cdiv(C, 32), (unsigned)cdiv(R, 32)), block(32, 8);
  transpose_bf16_kernel<<<grid, block, 0, st>>>(src, (__nv_bfloat16*)dst, R, C);
  VC_CHECK_LAUNCH();
  return VC_OK;
}
}  // namespace

}  // namespace vc

using namespace vc;

extern "C" {

size_t vc_ext_raw_weight_floats(const vc_ext_shape* shape) {
  ExtDims d;
  if (check_ext(shape, &d) != VC_OK) return 0;
  return (size_t)(d.D * 6 * d.D + 6 * d.D + 4 * d.dh + d.D * d.Dff + d.Dff + d.Dff * d.D + d.D);
}

size_t vc_ext_packed_weight_bytes(const vc_ext_shape* shape) {
  ExtDims d;
  if (check_ext(shape, &d) != VC_OK) return 0;
  return ext_layout(d).total;
}

size_t vc_ext_workspace_bytes(const vc_ext_shape* shape) {
  ExtDims d;
  if (check_ext(shape, &d) != VC_OK) return 0;
  return ext_ws(d).total;
}

int vc_ext_block_launches(const vc_ext_shape* shape) {
  ExtDims d;
  if (check_ext(shape, &d) != VC_OK) return -1;
  // mod, rope, ln, 2 QKV, [text K/V], 3 attention, O, ln, 2 FFN
  return d.Lt > 0 ? 13 : 12;
}

int vc_pack_ext_weights(const vc_ext_shape* shape, const float* raw_dev, void* packed_dev, void* stream) {
  ExtDims d;
  VC_TRY(check_ext(shape, &d));
  if (!raw_dev || !packed_dev) { set_error("null weight pointer"); return VC_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  const ExtLayout l = ext_layout(d);
  char* p = (char*)packed_dev;
  const float* r = raw_dev;
  auto copy = [&](size_t off, int64_t n) -> int {
    VC_CHECK_CUDA(cudaMemcpyAsync(p + off, r, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    r += n;
    return VC_OK;
  };
  VC_TRY(copy(l.w_ada, d.D * 6 * d.D));
  VC_TRY(copy(l.b_ada, 6 * d.D));
  VC_TRY(copy(l.qn, 2 * d.dh));
  VC_TRY(copy(l.kn, 2 * d.dh));
  VC_TRY(launch_transpose_bf16(r, p + l.w1, d.D, d.Dff, st));  // w1 [D][Dff] -> [Dff][D]
  r += d.D * d.Dff;
  VC_TRY(copy(l.b1, d.Dff));
  VC_TRY(launch_transpose_bf16(r, p + l.w2, d.Dff, d.D, st));  // w2 [Dff][D] -> [D][Dff]
  r += d.Dff * d.D;
  VC_TRY(copy(l.b2, d.D));
  return VC_OK;
}

int vc_ext_block_forward(const vc_ext_shape* shape, const void* block_packed_dev, const void* ext_packed_dev,
                         const float* visual_dev, const float* prompt_dev, double timestep, float* out_dev,
                         void* workspace_dev, size_t workspace_bytes, void* stream) {
  ExtDims d;
  VC_TRY(check_ext(shape, &d));
  if (!block_packed_dev || !ext_packed_dev || !visual_dev || !out_dev || !workspace_dev ||
      (d.Lt > 0 && !prompt_dev)) {
    set_error("null pointer argument");
    return VC_EINVAL;
  }
  if ((const void*)out_dev == (const void*)visual_dev) {
    set_error("out must not alias visual (the O GEMM reads x while writing h)");
    return VC_EINVAL;
  }
  const ExtWs w = ext_ws(d);
  if (workspace_bytes < w.total) {
    set_error("workspace too small: %zu < %zu", workspace_bytes, w.total);
    return VC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace_dev;
  const char* ep = (const char*)ext_packed_dev;
  const ExtLayout l = ext_layout(d);
  float* mod = (float*)(ws + w.mod);
  float2* rope = (float2*)(ws + w.rope);
  int32_t nt, ny, nx;
  rope_split(d.dh, nt, ny, nx);

  profile_begin(st);
  const size_t smem = (size_t)(d.D + kModSlices * 32) * 4;
  adaln_mod_kernel<<<(unsigned)cdiv(6 * d.D, 32), kModSlices * 32, smem, st>>>(timestep, (int)d.D,
                                                                   (const float*)(ep + l.w_ada),
                                                                   (const float*)(ep + l.b_ada), mod);
  VC_CHECK_LAUNCH();
  rope_table_kernel<<<(unsigned)cdiv(w.rope_n, 256), 256, 0, st>>>(rope, d.F, d.gh, d.gw, nt, ny, nx);
  VC_CHECK_LAUNCH();
  profile_mark(st, "mod_rope");

  ExtArgs e{};
  e.mod = mod;
  e.qn[0] = (const float*)(ep + l.qn); e.qn[1] = e.qn[0] + d.dh;
  e.kn[0] = (const float*)(ep + l.kn); e.kn[1] = e.kn[0] + d.dh;
  e.rope = rope; e.rope_nt = nt; e.rope_ny = ny; e.rope_nx = nx; e.gw = (int32_t)d.gw;
  e.rope_off_y = w.rope_off_y; e.rope_off_x = w.rope_off_x;
  e.Dff = d.Dff;
  e.w1 = ep + l.w1; e.b1 = (const float*)(ep + l.b1);
  e.w2 = ep + l.w2; e.b2 = (const float*)(ep + l.b2);
  e.u = (__nv_bfloat16*)(ws + w.u);

  size_t wqkv, bias, wo, tot;
  packed_offsets(d.D, d.H, true, &wqkv, &bias, &wo, &tot);
  const char* bp = (const char*)block_packed_dev;
  int rc = block_forward_bf16(d.F, d.Lv, d.Lt, d.D, d.H, bp + wqkv, (const float*)(bp + bias), bp + wo,
                              visual_dev, prompt_dev, out_dev, 1, ws, st, &e);
  profile_end();
  return rc;
}

}  // extern "C"
