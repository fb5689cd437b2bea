// bf16 block forward: tcgen05 projection GEMMs around the attention cores.
// See vc_block.cu for the step list; this file owns the bf16 workspace.
#include <math.h>

#include "vc_gemm_tc.h"
#include "vc_kernels.h"

namespace vc {

namespace {
inline size_t aup(size_t v) { return (v + 1023) / 1024 * 1024; }

struct WsBf16 {
  size_t xhat, qkv, acat, total;
};
WsBf16 ws_layout(int64_t F, int64_t Lv, int64_t Lt, int64_t D) {
  const int64_t Nv = F * Lv, rows = Nv + Lt;
  WsBf16 w;
  w.xhat = 0;
  w.qkv = aup(w.xhat + (size_t)rows * D * 2);
  w.acat = aup(w.qkv + (size_t)rows * 9 * D * 2);
  w.total = aup(w.acat + (size_t)Nv * 3 * D * 2);
  return w;
}
}  // namespace

size_t bf16_workspace_bytes(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H) {
  (void)H;
  return ws_layout(F, Lv, Lt, D).total;
}

int bf16_launch_count(int64_t, int64_t, int64_t, int64_t, int64_t) { return 6; }

int block_forward_bf16(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H, const void* wqkv,
                       const float* bias, const void* wo, const float* x, const float* prompt,
                       float* out, int add_residual, char* ws, cudaStream_t st) {
  const WsBf16 wl = ws_layout(F, Lv, Lt, D);
  const int64_t Nv = F * Lv, rows = Nv + Lt, dh = D / H;
  __nv_bfloat16* xhat = (__nv_bfloat16*)(ws + wl.xhat);
  __nv_bfloat16* qkv = (__nv_bfloat16*)(ws + wl.qkv);
  __nv_bfloat16* acat = (__nv_bfloat16*)(ws + wl.acat);

  VC_TRY(launch_ln_rows<__nv_bfloat16>(x, Nv, prompt, Lt, (int)D, xhat, st));
  profile_mark(st, "ln");
  {
    GemmTcParams g{};
    g.M = rows; g.N = (int)(9 * D); g.K = (int)D;
    g.bias = bias; g.out_bf16 = qkv; g.ldo = 9 * D;
    VC_TRY(launch_gemm_tc(xhat, D, wqkv, D, g, EPI_BF16, st));
  }
  profile_mark(st, "qkv_gemm");
  const float scale_log2 = (float)(1.4426950408889634 / sqrt((double)dh));
  const int64_t ld = 9 * D;
  typedef AttnArgs<__nv_bfloat16, __nv_bfloat16> A;
  {
    A a{};
    a.q = qkv + 0 * D; a.ldq = ld; a.q_seq_stride = Lv; a.q_tok_stride = 1;
    a.k = qkv + 1 * D; a.v = qkv + 2 * D; a.ldk = ld; a.k_seq_stride = Lv; a.k_tok_stride = 1;
    a.o = acat + 0 * D; a.ldo = 3 * D; a.o_seq_stride = Lv; a.o_tok_stride = 1;
    a.n_seq = (int)F; a.len_q = (int)Lv; a.len_k = (int)Lv; a.heads = (int)H; a.dh = (int)dh;
    a.scale_log2 = scale_log2;
    VC_TRY(launch_attn_simt(a, st));
  }
  profile_mark(st, "attn_spatial");
  {
    A a{};
    a.q = qkv + 3 * D; a.ldq = ld; a.q_seq_stride = 1; a.q_tok_stride = Lv;
    a.k = qkv + 4 * D; a.v = qkv + 5 * D; a.ldk = ld; a.k_seq_stride = 1; a.k_tok_stride = Lv;
    a.o = acat + 1 * D; a.ldo = 3 * D; a.o_seq_stride = 1; a.o_tok_stride = Lv;
    a.n_seq = (int)Lv; a.len_q = (int)F; a.len_k = (int)F; a.heads = (int)H; a.dh = (int)dh;
    a.scale_log2 = scale_log2;
    VC_TRY(launch_attn_simt(a, st));
  }
  profile_mark(st, "attn_temporal");
  {
    A a{};
    a.q = qkv + 6 * D; a.ldq = ld; a.q_seq_stride = 0; a.q_tok_stride = 1;
    a.k = qkv + 7 * D; a.v = qkv + 8 * D; a.ldk = ld; a.k_seq_stride = 0; a.k_tok_stride = 1;
    a.ka = qkv + Nv * ld + 7 * D; a.va = qkv + Nv * ld + 8 * D; a.lda = ld; a.na = (int)Lt;
    a.log2_weight_a = (float)log2((double)F);
    a.o = acat + 2 * D; a.ldo = 3 * D; a.o_seq_stride = 0; a.o_tok_stride = 1;
    a.n_seq = 1; a.len_q = (int)Nv; a.len_k = (int)Nv; a.heads = (int)H; a.dh = (int)dh;
    a.scale_log2 = scale_log2;
    VC_TRY(launch_attn_simt(a, st));
  }
  profile_mark(st, "attn_fullseq");
  {
    GemmTcParams g{};
    g.M = Nv; g.N = (int)D; g.K = (int)(3 * D);
    g.out_f32 = out; g.ldo = D; g.R = add_residual ? x : nullptr; g.ldr = D;
    VC_TRY(launch_gemm_tc(acat, 3 * D, wo, 3 * D, g, EPI_F32, st));
  }
  profile_mark(st, "oproj_gemm");
  return VC_OK;
}

}  // namespace vc
