// Block-forward orchestration and the exported C ABI (include/vchitect_b200.h).
//
// One parallel MM-DiT block (model.py:263-271):
//   1. LN row stats of the visual rows and the Lt prompt rows  -> xhat
//   2. one projection GEMM for all three branches' Q/K/V (N = 9D), gamma
//      folded into W, beta@W as the epilogue bias (model.py:181-184)
//   3. attention: spatial (per frame), temporal (per position, F tokens),
//      full sequence (all visual queries vs deduplicated text + all visual
//      keys, text logits + log F)                     (model.py:230-260)
//   4. one O-projection GEMM with K = 3D over [A_sp | A_tm | A_fs] against
//      [Wo_sp; Wo_tm; Wo_fs]: the branch sum happens inside the K reduction
//      (model.py:190, :267-271); the residual (model.py:324) is the epilogue.
#include <stdarg.h>
#include <math.h>
#include <string.h>

#include "vc_common.cuh"
#include "vc_kernels.h"
#include "vc_gemm_tc.h"

namespace vc {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Dims {
  int64_t F, Lv, Lt, D, H, dh, Nv;
  bool bf16;
};

static int check_shape(const vc_block_shape* s, Dims* d) {
  if (!s) { set_error("null shape"); return VC_EINVAL; }
  if (s->frames < 1 || s->visual_len < 1 || s->text_len < 0 || s->dim < 1 || s->heads < 1) {
    set_error("bad block shape (F=%d, Lv=%d, Lt=%d, D=%d, H=%d)", s->frames, s->visual_len,
              s->text_len, s->dim, s->heads);
    return VC_EINVAL;
  }
  if (s->dim % s->heads != 0) {  // numerics.py:97-98
    set_error("feature dim %d not divisible by %d heads", s->dim, s->heads);
    return VC_EINVAL;
  }
  if (s->dtype != VC_DTYPE_F32 && s->dtype != VC_DTYPE_BF16) {
    set_error("unknown dtype %d", s->dtype);
    return VC_EINVAL;
  }
  if (s->dim % 2 != 0 && s->dtype == VC_DTYPE_BF16) {
    set_error("bf16 path needs an even dim, got %d", s->dim);
    return VC_EINVAL;
  }
  if (s->dim > 3072) {
    set_error("dim %d > 3072 not supported", s->dim);
    return VC_ENOTSUP;
  }
  if (s->dim / s->heads > 128) {
    set_error("head dim %d > 128 not supported", s->dim / s->heads);
    return VC_ENOTSUP;
  }
  if (s->dtype == VC_DTYPE_BF16 && s->dim % 8 != 0) {
    set_error("bf16 path needs dim %% 8 == 0 (TMA row pitch), got %d", s->dim);
    return VC_EINVAL;
  }
  if (d) {
    d->F = s->frames; d->Lv = s->visual_len; d->Lt = s->text_len; d->D = s->dim;
    d->H = s->heads; d->dh = s->dim / s->heads; d->Nv = d->F * d->Lv;
    d->bf16 = s->dtype == VC_DTYPE_BF16;
  }
  return VC_OK;
}

// ---- packed weight layout --------------------------------------------------
struct PackedLayout {
  size_t wqkv, bias, wo, total, wqkv_c, bias_c, wo_s;
};
void packed_offsets(int64_t D, int64_t H, bool bf16, size_t* wqkv, size_t* bias, size_t* wo,
                    size_t* total, size_t* wqkv_c, size_t* bias_c, size_t* wo_s) {
  const size_t es = bf16 ? 2 : 4;
  // bf16: head-padded QKV column space (vc_kernels.h QkvPad); fp32: plain 9D
  const int64_t nq = bf16 ? qkv_pad_layout(D, H).Npad : 9 * D;
  *wqkv = 0;
  *bias = align_up(*wqkv + (size_t)nq * D * es, 1024);
  *wo = align_up(*bias + (size_t)nq * 4, 1024);
  *total = align_up(*wo + (size_t)3 * D * D * es, 1024);
  size_t wc = *wqkv, bc = *bias, ws = *wo;
  if (bf16 && qkv_compact_ok(D, H)) {  // + the compact QKV space and the head-slot Wo of the single-GPU block
    const int64_t nc = qkv_compact_layout(D, H).Npad;
    wc = *total;
    bc = align_up(wc + (size_t)nc * D * es, 1024);
    ws = align_up(bc + (size_t)nc * 4, 1024);
    *total = align_up(ws + (size_t)3 * H * qkv_pad_layout(D, H).DP * D * es, 1024);
  }
  if (wqkv_c) *wqkv_c = wc;
  if (bias_c) *bias_c = bc;
  if (wo_s) *wo_s = ws;
}
static PackedLayout packed_layout(const Dims& d) {
  PackedLayout p;
  packed_offsets(d.D, d.H, d.bf16, &p.wqkv, &p.bias, &p.wo, &p.total, &p.wqkv_c, &p.bias_c, &p.wo_s);
  return p;
}

// ---- workspace layout --------------------------------------------------------
struct WsF32 {
  size_t xhat, qkv, acat, total;
};
static WsF32 ws_f32(const Dims& d) {
  WsF32 w;
  const int64_t rows = d.Nv + d.Lt;
  w.xhat = 0;
  w.qkv = align_up(w.xhat + (size_t)rows * d.D * 4, 1024);
  w.acat = align_up(w.qkv + (size_t)rows * 9 * d.D * 4, 1024);
  w.total = align_up(w.acat + (size_t)d.Nv * 3 * d.D * 4, 1024);
  return w;
}

static size_t workspace_bytes(const Dims& d) {
  if (d.bf16) return bf16_workspace_bytes(d.F, d.Lv, d.Lt, d.D, d.H);
  return ws_f32(d).total;
}

static int block_forward_f32(const Dims& d, const char* packed, const float* x,
                             const float* prompt, float* out, int add_residual, char* ws,
                             cudaStream_t st) {
  const PackedLayout pl = packed_layout(d);
  const WsF32 wl = ws_f32(d);
  const float* Wqkv = (const float*)(packed + pl.wqkv);
  const float* bias = (const float*)(packed + pl.bias);
  const float* Wo = (const float*)(packed + pl.wo);
  float* xhat = (float*)(ws + wl.xhat);
  float* qkv = (float*)(ws + wl.qkv);
  float* acat = (float*)(ws + wl.acat);
  const int64_t D = d.D, rows = d.Nv + d.Lt;

  VC_TRY(launch_ln_rows<float>(x, d.Nv, prompt, d.Lt, (int)D, xhat, st));
  profile_mark(st, "ln");
  {
    GemmF32Args g{xhat, D, Wqkv, 9 * D, bias, nullptr, 0, qkv, 9 * D, rows, (int)(9 * D), (int)D};
    VC_TRY(launch_gemm_f32(g, st));
  }
  profile_mark(st, "qkv_gemm");
  const float scale_log2 = (float)(1.4426950408889634 / sqrt((double)d.dh));
  const int64_t ld = 9 * D;
  // spatial: sequence f = rows f*Lv .. f*Lv+Lv-1
  {
    AttnArgs<float, float> a{};
    a.q = qkv + 0 * D; a.ldq = ld; a.q_seq_stride = d.Lv; a.q_tok_stride = 1;
    a.k = qkv + 1 * D; a.v = qkv + 2 * D; a.ldk = ld; a.k_seq_stride = d.Lv; a.k_tok_stride = 1;
    a.na = 0;
    a.o = acat + 0 * D; a.ldo = 3 * D; a.o_seq_stride = d.Lv; a.o_tok_stride = 1;
    a.n_seq = (int)d.F; a.len_q = (int)d.Lv; a.len_k = (int)d.Lv; a.heads = (int)d.H; a.dh = (int)d.dh;
    a.scale_log2 = scale_log2;
    VC_TRY(launch_attn_simt(a, st));
  }
  profile_mark(st, "attn_spatial");
  // temporal: sequence l = rows l, l+Lv, ..., l+(F-1)Lv
  int trc = VC_ENOTSUP;
  if (d.dh % 2 == 0)
    trc = launch_temporal_attn<float, float>(qkv + 3 * D, ld, D, acat + D, 3 * D, (int)d.F, (int)d.Lv,
                                             (int)d.H, (int)d.dh, st);
  if (trc != VC_OK && trc != VC_ENOTSUP) return trc;
  if (trc == VC_ENOTSUP) {  // odd head dims / very long clips: generic strided kernel
    AttnArgs<float, float> a{};
    a.q = qkv + 3 * D; a.ldq = ld; a.q_seq_stride = 1; a.q_tok_stride = d.Lv;
    a.k = qkv + 4 * D; a.v = qkv + 5 * D; a.ldk = ld; a.k_seq_stride = 1; a.k_tok_stride = d.Lv;
    a.o = acat + 1 * D; a.ldo = 3 * D; a.o_seq_stride = 1; a.o_tok_stride = d.Lv;
    a.n_seq = (int)d.Lv; a.len_q = (int)d.F; a.len_k = (int)d.F; a.heads = (int)d.H; a.dh = (int)d.dh;
    a.scale_log2 = scale_log2;
    VC_TRY(launch_attn_simt(a, st));
  }
  profile_mark(st, "attn_temporal");
  // full sequence: queries = all visual rows; keys = Lt text rows (weight F) + all visual rows
  {
    AttnArgs<float, float> a{};
    a.q = qkv + 6 * D; a.ldq = ld; a.q_seq_stride = 0; a.q_tok_stride = 1;
    a.k = qkv + 7 * D; a.v = qkv + 8 * D; a.ldk = ld; a.k_seq_stride = 0; a.k_tok_stride = 1;
    a.ka = qkv + d.Nv * ld + 7 * D; a.va = qkv + d.Nv * ld + 8 * D; a.lda = ld; a.na = (int)d.Lt;
    a.log2_weight_a = (float)log2((double)d.F);
    a.o = acat + 2 * D; a.ldo = 3 * D; a.o_seq_stride = 0; a.o_tok_stride = 1;
    a.n_seq = 1; a.len_q = (int)d.Nv; a.len_k = (int)d.Nv; a.heads = (int)d.H; a.dh = (int)d.dh;
    a.scale_log2 = scale_log2;
    VC_TRY(launch_attn_simt(a, st));
  }
  profile_mark(st, "attn_fullseq");
  {
    GemmF32Args g{acat, 3 * D, Wo, D, nullptr, add_residual ? x : nullptr, D, out, D, d.Nv,
                  (int)D, (int)(3 * D)};
    VC_TRY(launch_gemm_f32(g, st));
  }
  profile_mark(st, "oproj_gemm");
  return VC_OK;
}

}  // namespace vc

using namespace vc;

extern "C" {

const char* vc_version(void) {
  return "vchitect_b200 0.1 (sm_100a; fp32 SIMT + bf16 tcgen05/TMA paths)";
}

const char* vc_last_error(void) { return g_err; }

int vc_block_shape_check(const vc_block_shape* shape) { return check_shape(shape, nullptr); }

size_t vc_block_raw_weight_floats(const vc_block_shape* shape) {
  Dims d;
  if (check_shape(shape, &d) != VC_OK) return 0;
  return (size_t)3 * (2 * d.D + 4 * d.D * d.D);
}

size_t vc_block_packed_weight_bytes(const vc_block_shape* shape) {
  Dims d;
  if (check_shape(shape, &d) != VC_OK) return 0;
  return packed_layout(d).total;
}

size_t vc_block_workspace_bytes(const vc_block_shape* shape) {
  Dims d;
  if (check_shape(shape, &d) != VC_OK) return 0;
  return workspace_bytes(d);
}

size_t vc_block_host_workspace_bytes(const vc_block_shape* shape) {
  Dims d;
  if (check_shape(shape, &d) != VC_OK) return 0;
  size_t b = align_up(workspace_bytes(d), 1024);
  b += align_up((size_t)d.Nv * d.D * 4, 1024) * 2 + align_up((size_t)(d.Lt > 0 ? d.Lt : 1) * d.D * 4, 1024);
  return b;
}

int vc_pack_block_weights(const vc_block_shape* shape, const float* raw_dev, void* packed_dev,
                          void* stream) {
  Dims d;
  VC_TRY(check_shape(shape, &d));
  if (!raw_dev || !packed_dev) { set_error("null weight pointer"); return VC_EINVAL; }
  const PackedLayout pl = packed_layout(d);
  char* p = (char*)packed_dev;
  return launch_pack(raw_dev, p + pl.wqkv, (float*)(p + pl.bias), p + pl.wo, (int)d.D, (int)d.H,
                     d.bf16, (cudaStream_t)stream, pl.wqkv_c != pl.wqkv ? p + pl.wqkv_c : nullptr, pl.wqkv_c != pl.wqkv ? (float*)(p + pl.bias_c) : nullptr,
                     pl.wqkv_c != pl.wqkv ? p + pl.wo_s : nullptr);
}

int vc_block_forward(const vc_block_shape* shape, const void* packed_dev, const float* visual_dev,
                     const float* prompt_dev, float* out_dev, int add_residual,
                     void* workspace_dev, size_t workspace_bytes_, void* stream) {
  Dims d;
  VC_TRY(check_shape(shape, &d));
  if (!packed_dev || !visual_dev || !out_dev || !workspace_dev || (d.Lt > 0 && !prompt_dev)) {
    set_error("null pointer argument");
    return VC_EINVAL;
  }
  if (workspace_bytes_ < workspace_bytes(d)) {
    set_error("workspace too small: %zu < %zu", workspace_bytes_, workspace_bytes(d));
    return VC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  profile_begin(st);
  int rc;
  if (d.bf16) {
    const PackedLayout pl = packed_layout(d);
    const char* p = (const char*)packed_dev;
    const bool cpt = pl.wqkv_c != pl.wqkv;
    rc = block_forward_bf16(d.F, d.Lv, d.Lt, d.D, d.H, p + pl.wqkv, (const float*)(p + pl.bias),
                            p + pl.wo, visual_dev, prompt_dev, out_dev, add_residual,
                            (char*)workspace_dev, st, nullptr, cpt ? p + pl.wqkv_c : nullptr,
                            cpt ? (const float*)(p + pl.bias_c) : nullptr, cpt ? p + pl.wo_s : nullptr);
  } else {
    rc = block_forward_f32(d, (const char*)packed_dev, visual_dev, prompt_dev, out_dev,
                           add_residual, (char*)workspace_dev, st);
  }
  profile_end();
  return rc;
}

int vc_block_forward_host(const vc_block_shape* shape, const void* packed_dev,
                          const float* visual_host, const float* prompt_host, float* out_host,
                          void* workspace_dev, size_t workspace_bytes_, void* stream) {
  Dims d;
  VC_TRY(check_shape(shape, &d));
  if (workspace_bytes_ < vc_block_host_workspace_bytes(shape)) {
    set_error("workspace too small for host staging");
    return VC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace_dev;
  size_t off = align_up(workspace_bytes(d), 1024);
  float* xin = (float*)(ws + off);
  off += align_up((size_t)d.Nv * d.D * 4, 1024);
  float* yout = (float*)(ws + off);
  off += align_up((size_t)d.Nv * d.D * 4, 1024);
  float* pin = (float*)(ws + off);
  VC_CHECK_CUDA(cudaMemcpyAsync(xin, visual_host, (size_t)d.Nv * d.D * 4, cudaMemcpyHostToDevice, st));
  if (d.Lt > 0)
    VC_CHECK_CUDA(cudaMemcpyAsync(pin, prompt_host, (size_t)d.Lt * d.D * 4, cudaMemcpyHostToDevice, st));
  VC_TRY(vc_block_forward(shape, packed_dev, xin, pin, yout, 0, workspace_dev, workspace_bytes(d), stream));
  VC_CHECK_CUDA(cudaMemcpyAsync(out_host, yout, (size_t)d.Nv * d.D * 4, cudaMemcpyDeviceToHost, st));
  return VC_OK;
}

size_t vc_block_stream_workspace_bytes(const vc_block_shape* shape) {
  Dims d;
  if (check_shape(shape, &d) != VC_OK) return 0;
  return align_up(workspace_bytes(d), 1024) + 4 * align_up((size_t)d.Nv * d.D * 4, 1024) +
         align_up((size_t)(d.Lt > 0 ? d.Lt : 1) * d.D * 4, 1024);
}

int vc_block_forward_host_batched(const vc_block_shape* shape, const void* packed_dev, int32_t n,
                                  const float* const* visual_host, const float* prompt_host,
                                  float* const* out_host, void* workspace_dev, size_t workspace_bytes_,
                                  void* compute_stream, void* h2d_stream, void* d2h_stream) {
  Dims d;
  VC_TRY(check_shape(shape, &d));
  if (n < 0 || (n > 0 && (!visual_host || !out_host))) { set_error("bad batch arguments"); return VC_EINVAL; }
  if (workspace_bytes_ < vc_block_stream_workspace_bytes(shape)) {
    set_error("workspace too small for the streamed host path");
    return VC_EINVAL;
  }
  cudaStream_t sc = (cudaStream_t)compute_stream, si = (cudaStream_t)h2d_stream, so = (cudaStream_t)d2h_stream;
  const size_t xbytes = (size_t)d.Nv * d.D * 4;
  char* ws = (char*)workspace_dev;
  size_t off = align_up(workspace_bytes(d), 1024);
  float* xin[2];
  float* yout[2];
  for (int b = 0; b < 2; ++b) { xin[b] = (float*)(ws + off); off += align_up(xbytes, 1024); }
  for (int b = 0; b < 2; ++b) { yout[b] = (float*)(ws + off); off += align_up(xbytes, 1024); }
  float* pin = (float*)(ws + off);
  // events: inputs landed / compute done / result copied out, per staging buffer
  cudaEvent_t ev[7];
  for (int i = 0; i < 7; ++i) VC_CHECK_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  cudaEvent_t *in_ready = ev, *done = ev + 2, *out_free = ev + 4, start = ev[6];
  int rc = VC_OK;
  // the copy streams start after everything already queued on the compute stream
  cudaEventRecord(start, sc);
  cudaStreamWaitEvent(si, start, 0);
  cudaStreamWaitEvent(so, start, 0);
  if (d.Lt > 0) cudaMemcpyAsync(pin, prompt_host, (size_t)d.Lt * d.D * 4, cudaMemcpyHostToDevice, sc);
  for (int i = 0; i < n && rc == VC_OK; ++i) {
    const int b = i & 1;
    // H2D of batch i may overwrite xin[b] once batch i-2's compute has read it
    if (i >= 2) cudaStreamWaitEvent(si, done[b], 0);
    cudaMemcpyAsync(xin[b], visual_host[i], xbytes, cudaMemcpyHostToDevice, si);
    cudaEventRecord(in_ready[b], si);
    cudaStreamWaitEvent(sc, in_ready[b], 0);
    if (i >= 2) cudaStreamWaitEvent(sc, out_free[b], 0);  // D2H of batch i-2 done with yout[b]
    rc = vc_block_forward(shape, packed_dev, xin[b], pin, yout[b], 0, workspace_dev, workspace_bytes(d), sc);
    cudaEventRecord(done[b], sc);
    cudaStreamWaitEvent(so, done[b], 0);
    cudaMemcpyAsync(out_host[i], yout[b], xbytes, cudaMemcpyDeviceToHost, so);
    cudaEventRecord(out_free[b], so);
  }
  // join: the compute stream completes after the last copy out
  cudaEventRecord(start, so);
  cudaStreamWaitEvent(sc, start, 0);
  for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);  // deferred until the events complete
  if (rc != VC_OK) return rc;
  VC_CHECK_CUDA(cudaGetLastError());
  return VC_OK;
}

int vc_attention_f32(const float* q, const float* k, const float* v, float* out, int32_t sq,
                     int32_t sk, int32_t dim, int32_t heads, void* stream) {
  if (heads < 1 || dim % heads != 0) {
    set_error("feature dim %d not divisible by %d heads", dim, heads);
    return VC_EINVAL;
  }
  if (sq < 0 || sk < 1) { set_error("bad attention lengths sq=%d sk=%d", sq, sk); return VC_EINVAL; }
  AttnArgs<float, float> a{};
  a.q = q; a.ldq = dim; a.q_seq_stride = 0; a.q_tok_stride = 1;
  a.k = k; a.v = v; a.ldk = dim; a.k_seq_stride = 0; a.k_tok_stride = 1;
  a.na = 0;
  a.o = out; a.ldo = dim; a.o_seq_stride = 0; a.o_tok_stride = 1;
  a.n_seq = 1; a.len_q = sq; a.len_k = sk; a.heads = heads; a.dh = dim / heads;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)(dim / heads)));
  return launch_attn_simt(a, (cudaStream_t)stream);
}

int vc_layer_norm_f32(const float* x, float* out, int64_t rows, int32_t dim, void* stream) {
  return launch_ln_rows<float>(x, rows, nullptr, 0, dim, out, (cudaStream_t)stream);
}

int vc_embed_frames(const float* lat, const float* w_in, float* x, int32_t F, int32_t first_frame,
                    int32_t h, int32_t w, int32_t c, int32_t patch, int32_t dim, double t,
                    void* stream) {
  if (dim % 2 != 0) { set_error("embedding dim must be even, got %d", dim); return VC_EINVAL; }
  if (F < 1 || h < 1 || w < 1 || c < 1 || patch < 1) { set_error("bad latent shape"); return VC_EINVAL; }
  return launch_embed(lat, w_in, x, F, first_frame, 0, -1, h, w, c, patch, dim, t, (cudaStream_t)stream);
}

int vc_embed_frames_rows(const float* lat, const float* w_in, float* x, int32_t F, int32_t first_frame,
                         int32_t tok0, int32_t ntok, int32_t h, int32_t w, int32_t c, int32_t patch,
                         int32_t dim, double t, void* stream) {
  if (dim % 2 != 0) { set_error("embedding dim must be even, got %d", dim); return VC_EINVAL; }
  if (F < 1 || h < 1 || w < 1 || c < 1 || patch < 1 || ntok < 0) { set_error("bad latent shape"); return VC_EINVAL; }
  return launch_embed(lat, w_in, x, F, first_frame, tok0, ntok, h, w, c, patch, dim, t, (cudaStream_t)stream);
}

int vc_unembed_frames(const float* x, const float* w_out, float* eps, int32_t F, int32_t h,
                      int32_t w, int32_t c, int32_t patch, int32_t dim, void* stream) {
  if (F < 1 || h < 1 || w < 1 || c < 1 || patch < 1) { set_error("bad latent shape"); return VC_EINVAL; }
  return launch_unembed(x, w_out, eps, F, h, w, c, patch, dim, (cudaStream_t)stream);
}

int vc_unembed_reverse_step(const float* x, const float* w_out, const float* x_t, const float* noise,
                            float* eps, float* x_prev, int32_t F, int32_t h, int32_t w, int32_t c,
                            int32_t patch, int32_t dim, double coef_eps, double inv_sqrt_alpha,
                            double sqrt_beta, void* stream) {
  if (F < 1 || h < 1 || w < 1 || c < 1 || patch < 1) { set_error("bad latent shape"); return VC_EINVAL; }
  if (!x_t || !x_prev) { set_error("reverse step needs x_t and x_prev"); return VC_EINVAL; }
  ReverseStep rs{x_t, noise, x_prev, (float)coef_eps, (float)inv_sqrt_alpha, (float)sqrt_beta};
  return launch_unembed(x, w_out, eps, F, h, w, c, patch, dim, (cudaStream_t)stream, rs);
}

int vc_gemm_bf16(const void* a, int64_t lda, const void* b, int64_t ldb, const float* bias,
                 const float* resid, float* out, int64_t ldo, int64_t M, int32_t N, int32_t K,
                 void* stream) {
  if (M < 0 || N < 0 || K < 1) { set_error("bad GEMM shape"); return VC_EINVAL; }
  GemmTcParams g{};
  g.M = M; g.N = N; g.K = K; g.bias = bias; g.out_f32 = out; g.ldo = ldo; g.R = resid; g.ldr = ldo;
  return launch_gemm_tc(a, lda, b, ldb, g, EPI_F32, (cudaStream_t)stream);
}

int vc_block_forward_launches(const vc_block_shape* shape) {
  Dims d;
  if (check_shape(shape, &d) != VC_OK) return -1;
  return d.bf16 ? bf16_launch_count(d.F, d.Lv, d.Lt, d.D, d.H) : 6;
}

}  // extern "C"
