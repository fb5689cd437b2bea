// bf16 block forward on tensor cores (see vc_block.cu for the step list).
//
//   ln (visual + prompt rows) -> xhat bf16
//   QKV GEMM (tcgen05, N = 9D) whose epilogue scatters into the attention
//     layouts: spatial / full-seq Q,K [row][H][DP] and V^T [seq][H][DP][key],
//     temporal plain [row][3D]
//   text K/V GEMM: the Lt prompt rows against the full-seq K,V columns only
//   attention: spatial + full sequence on tcgen05 (vc_attn_tc.cu), temporal
//     (F-token sequences, HBM-bound) on the SIMT kernel
//   O GEMM (tcgen05, K = 3D) with the residual fused in the epilogue.
#include <math.h>

#include "vc_attn_tc.h"
#include "vc_gemm_tc.h"
#include "vc_kernels.h"
#include "vc_tuning.h"

namespace vc {

namespace {
inline size_t aup(size_t v) { return (v + 1023) / 1024 * 1024; }

struct WsBf16 {
  int64_t DP, Lv_ld, Lk_ld;
  size_t xhat, qsp, ksp, vtsp, tm, qfs, kfs, vtfs, acat, total;
};
WsBf16 ws_layout(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H) {
  const int64_t Nv = F * Lv, dh = D / H;
  WsBf16 w;
  w.DP = qkv_head_pad(dh);
  w.Lv_ld = round_up(Lv, 8);
  w.Lk_ld = round_up(Lt + Nv, 8);
  const size_t qk = (size_t)H * w.DP * 2;
  size_t o = 0;
  w.xhat = o; o = aup(o + (size_t)(Nv + Lt) * D * 2);
  w.qsp = o; o = aup(o + (size_t)Nv * qk);
  w.ksp = o; o = aup(o + (size_t)Nv * qk);
  w.vtsp = o; o = aup(o + (size_t)F * H * w.DP * w.Lv_ld * 2);
  w.tm = o; o = aup(o + (size_t)Nv * 3 * D * 2);
  w.qfs = o; o = aup(o + (size_t)Nv * qk);
  w.kfs = o; o = aup(o + (size_t)(Lt + Nv) * qk);
  w.vtfs = o; o = aup(o + (size_t)H * w.DP * w.Lk_ld * 2);
  // [Nv][3D], or [Nv][3][H][DP] in the head-slot layout (DP >= dh)
  w.acat = o; o = aup(o + (size_t)Nv * 3 * std::max<int64_t>(D, H * w.DP) * 2);
  w.total = o;
  return w;
}

// The text K/V GEMM and the temporal branch run on a side stream forked
// after the QKV GEMM (joined before the full-sequence attention / the O
// GEMM), so their CTAs fill the SMs the attention kernels leave idle in their
// last waves. One side stream and two
// events per host thread and device (fork / join by events: stream-capture
// safe). Sequential while the stage profiler runs (per-stage times).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, text = nullptr, join = nullptr;
  int dev = -1;
};
int side_stream(SideStream** out) {
  static thread_local SideStream ss[16];
  int dev = 0;
  VC_CHECK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) { set_error("device %d out of range", dev); return VC_EINVAL; }
  SideStream& x = ss[dev];
  if (!x.s) {
    VC_CHECK_CUDA(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
    VC_CHECK_CUDA(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming));
    VC_CHECK_CUDA(cudaEventCreateWithFlags(&x.text, cudaEventDisableTiming));
    VC_CHECK_CUDA(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming));
    x.dev = dev;
  }
  *out = &x;
  return VC_OK;
}
}  // namespace

size_t bf16_workspace_bytes(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H) {
  return ws_layout(F, Lv, Lt, D, H).total;
}

size_t bf16_workspace_acat_offset(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H) {
  return ws_layout(F, Lv, Lt, D, H).acat;
}

int bf16_launch_count(int64_t, int64_t, int64_t Lt, int64_t D, int64_t H) {
  return (Lt > 0 ? 7 : 6) + (qkv_compact_ok(D, H) ? 2 : 0);  // + the two V^T pad fills
}

int block_forward_bf16(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H, const void* wqkv,
                       const float* bias, const void* wo, const float* x, const float* prompt,
                       float* out, int add_residual, char* ws, cudaStream_t st, const ExtArgs* ext,
                       const void* wqkv_c, const float* bias_c, const void* wo_s) {
  const WsBf16 wl = ws_layout(F, Lv, Lt, D, H);
  const int64_t Nv = F * Lv, dh = D / H;
  if (wl.DP == 0) { set_error("head dim %lld unsupported on the tensor-core path", (long long)dh); return VC_ENOTSUP; }
  typedef __nv_bfloat16 bf;
  bf* xhat = (bf*)(ws + wl.xhat);
  bf* acat = (bf*)(ws + wl.acat);
  bf* tm = (bf*)(ws + wl.tm);

  if (ext) VC_TRY(launch_ln_rows_mod(x, Nv, prompt, Lt, (int)D, ext->mod, ext->mod + D, xhat, st));
  else VC_TRY(launch_ln_rows<bf>(x, Nv, prompt, Lt, (int)D, xhat, st));
  profile_mark(st, "ln");

  // the compact column space (dh 66; no padding columns in the GEMM) unless the
  // extension's head-aligned QK-norm epilogue needs the padded one
  const bool compact = !ext && wqkv_c && bias_c && qkv_compact_ok(D, H);
  if (compact) { wqkv = wqkv_c; bias = bias_c; }
  const QkvPad pad = compact ? qkv_compact_layout(D, H) : qkv_pad_layout(D, H);
  QkvScatter sc{};
  sc.pad = pad; sc.D = D; sc.Lv = Lv; sc.Lt = Lt; sc.H = (int)H;
  sc.sp = BranchOut{(bf*)(ws + wl.qsp), (bf*)(ws + wl.ksp), (bf*)(ws + wl.vtsp), wl.Lv_ld};
  sc.fs = BranchOut{(bf*)(ws + wl.qfs), (bf*)(ws + wl.kfs), (bf*)(ws + wl.vtfs), wl.Lk_ld};
  sc.tm = tm;
  sc.tm_F = (int)F;  // temporal q/k/v position-major: each position's F frames are consecutive rows
  const int qkv_epi = ext ? EPI_QKVN : EPI_QKV;
  if (ext) {
    sc.qn[0] = ext->qn[0]; sc.qn[1] = ext->qn[1]; sc.kn[0] = ext->kn[0]; sc.kn[1] = ext->kn[1];
    sc.rope = ext->rope; sc.dh = (int)dh; sc.gw = ext->gw;
    sc.rope_nt = ext->rope_nt; sc.rope_ny = ext->rope_ny; sc.rope_nx = ext->rope_nx;
    sc.rope_off_y = ext->rope_off_y; sc.rope_off_x = ext->rope_off_x;
    // two launches so each starts on a segment base (head-aligned tiles):
    // [sp.q sp.k sp.v | tm] and [fs.q fs.k fs.v]
    GemmTcParams g{};
    g.M = Nv; g.N = (int)pad.fs_base(); g.K = (int)D; g.bias = bias;
    g.qkv = sc; g.qkv.n_base = 0; g.qkv.text_rows = 0;
    VC_TRY(launch_gemm_tc(xhat, D, wqkv, D, g, EPI_QKVN, st));
    g.N = (int)(3 * pad.SEG); g.bias = bias + pad.fs_base(); g.qkv.n_base = pad.fs_base();
    VC_TRY(launch_gemm_tc(xhat, D, (const bf*)wqkv + pad.fs_base() * D, D, g, EPI_QKVN, st));
  } else {
    GemmTcParams g{};
    g.M = Nv; g.N = (int)pad.Npad; g.K = (int)D; g.bias = bias;
    g.qkv = sc; g.qkv.n_base = 0; g.qkv.text_rows = 0;
    // compact: 256-column tiles (the least-padding pick would be 176, whose
    // smaller tiles cost more than the 80 padding columns of 256)
    static const int qkv_bn = tuning_int("VC_QKV_BN", 256);  // A/B
    VC_TRY(launch_gemm_tc(xhat, D, wqkv, D, g, EPI_QKV, st, compact ? qkv_bn : 0));
  }
  if (compact) {  // V^T rows dh..DP-1 (ones column, zeros) the compact GEMM does not write
    VC_TRY(launch_fill_vt_pad(sc.sp.vt, F * H, (int)wl.DP, (int)dh, wl.Lv_ld, Lv, st));
    VC_TRY(launch_fill_vt_pad(sc.fs.vt, H, (int)wl.DP, (int)dh, wl.Lk_ld, Lt + Nv, st));
  }
  profile_mark(st, "qkv_gemm");
  const float scale_log2 = (float)(1.4426950408889634 / sqrt((double)dh));
  // O-GEMM A operand: the three branches' outputs [Nv][3D], or, with the
  // head-slot Wo (dh 66), [Nv][3][H][DP] written as whole 16-byte sectors
  const int slot = (!ext && wo_s) ? (int)wl.DP : 0;
  if (slot) wo = wo_s;
  const int64_t bw = slot ? H * slot : D;  // columns per branch in acat
  const int64_t lda = 3 * bw;
  // text K/V GEMM and temporal branch on the side stream (forked here)
  static const int fork_on = tuning_int("VC_TEMPORAL_FORK", 1);
  SideStream* side = nullptr;
  if (fork_on && !profile_on()) {
    VC_TRY(side_stream(&side));
    VC_CHECK_CUDA(cudaEventRecord(side->fork, st));
    VC_CHECK_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
  }
  cudaStream_t sx = side ? side->s : st;
  if (Lt > 0) {  // prompt rows: only the full-sequence K and V segments
    const int64_t n0 = pad.fs_base() + pad.SEG;
    GemmTcParams g{};
    g.M = Lt; g.N = (int)(2 * pad.SEG); g.K = (int)D; g.bias = bias + n0;
    g.qkv = sc; g.qkv.n_base = n0; g.qkv.text_rows = 1;
    VC_TRY(launch_gemm_tc(xhat + Nv * D, D, (const bf*)wqkv + n0 * D, D, g, qkv_epi, sx));
    if (!side) profile_mark(st, "text_kv_gemm");
  }
  if (side) {
    VC_CHECK_CUDA(cudaEventRecord(side->text, side->s));
    VC_TRY(launch_temporal_bf16(tm, 3 * D, D, acat + bw, lda, (int)F, (int)Lv, (int)H, (int)dh, side->s, slot, 1));
    VC_CHECK_CUDA(cudaEventRecord(side->join, side->s));
  }
  {
    AttnTcParams a{};
    a.Lq = (int)Lv; a.Lk = (int)Lv; a.H = (int)H; a.dh = (int)dh;
    a.n_bias = 0; a.bias_log2 = 0.f; a.scale_log2 = scale_log2;
    a.out = acat; a.ld_out = lda; a.col_off = 0; a.out_seq_rows = Lv; a.head_slot = slot;
    VC_TRY(launch_attn_tc(a, sc.sp.q, sc.sp.k, sc.sp.vt, (int)F, Lv, Lv, wl.Lv_ld, (int)wl.DP, st));
  }
  profile_mark(st, "attn_spatial");
  if (side) VC_CHECK_CUDA(cudaStreamWaitEvent(st, side->text, 0));  // the text keys of the full sequence
  if (!side) {
    VC_TRY(launch_temporal_bf16(tm, 3 * D, D, acat + bw, lda, (int)F, (int)Lv, (int)H, (int)dh, st, slot, 1));
    profile_mark(st, "attn_temporal");
  }
  {
    AttnTcParams a{};
    a.Lq = (int)Nv; a.Lk = (int)(Lt + Nv); a.H = (int)H; a.dh = (int)dh;
    a.n_bias = (int)Lt; a.bias_log2 = (float)log2((double)F); a.scale_log2 = scale_log2;
    a.out = acat; a.ld_out = lda; a.col_off = 2 * bw; a.out_seq_rows = 0; a.head_slot = slot;
    VC_TRY(launch_attn_tc(a, sc.fs.q, sc.fs.k, sc.fs.vt, 1, Nv, Lt + Nv, wl.Lk_ld, (int)wl.DP, st));
  }
  profile_mark(st, "attn_fullseq");
  if (side) VC_CHECK_CUDA(cudaStreamWaitEvent(st, side->join, 0));
  if (ext) {  // h = x + gate_msa * (branch sum)  -> out
    GemmTcParams g{};
    g.M = Nv; g.N = (int)D; g.K = (int)(3 * D);
    g.out_f32 = out; g.ldo = D; g.R = x; g.ldr = D; g.gate = ext->mod + 2 * D;
    VC_TRY(launch_gemm_tc(acat, 3 * D, wo, 3 * D, g, EPI_F32G, st));
    profile_mark(st, "oproj_gemm");
    // FFN: n2 = LN(h)(1 + scale_mlp) + shift_mlp; u = gelu(n2 W1 + b1);
    // out = h + gate_mlp * (u W2 + b2)
    VC_TRY(launch_ln_rows_mod(out, Nv, nullptr, 0, (int)D, ext->mod + 3 * D, ext->mod + 4 * D, xhat, st));
    profile_mark(st, "ln_mlp");
    GemmTcParams g1{};
    g1.M = Nv; g1.N = (int)ext->Dff; g1.K = (int)D; g1.bias = ext->b1;
    g1.out_bf16 = ext->u; g1.ldo = ext->Dff;
    VC_TRY(launch_gemm_tc(xhat, D, ext->w1, D, g1, EPI_GELU, st));
    profile_mark(st, "ffn1_gemm");
    GemmTcParams g2{};
    g2.M = Nv; g2.N = (int)D; g2.K = (int)ext->Dff; g2.bias = ext->b2;
    g2.out_f32 = out; g2.ldo = D; g2.R = out; g2.ldr = D; g2.gate = ext->mod + 5 * D;
    VC_TRY(launch_gemm_tc(ext->u, ext->Dff, ext->w2, ext->Dff, g2, EPI_F32G, st));
    profile_mark(st, "ffn2_gemm");
    return VC_OK;
  }
  {
    GemmTcParams g{};
    g.M = Nv; g.N = (int)D; g.K = (int)lda;
    g.out_f32 = out; g.ldo = D; g.R = add_residual ? x : nullptr; g.ldr = D;
    VC_TRY(launch_gemm_tc(acat, lda, wo, lda, g, EPI_F32, st));
  }
  profile_mark(st, "oproj_gemm");
  return VC_OK;
}

}  // namespace vc
