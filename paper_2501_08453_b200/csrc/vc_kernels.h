// Internal launcher declarations shared between the .cu files.
#pragma once
#include "vc_common.cuh"

namespace vc {

struct GemmF32Args {
  const float* A; int64_t lda;
  const float* B; int64_t ldb;
  const float* bias;
  const float* R; int64_t ldr;
  float* out; int64_t ldo;
  int64_t M; int32_t N, K;
};
int launch_gemm_f32(const GemmF32Args& g, cudaStream_t st);

template <typename T, typename OutT>
int launch_attn_simt(const AttnArgs<T, OutT>& a, cudaStream_t st);

// Temporal branch: q/k/v of row r at qkv[r*ld + {0, D, 2D}], sequence l =
// rows {f*Lv + l}; output o[r*ldo + h*dh + d].  (vc_attn_temporal.cu)
template <typename T, typename OutT>
int launch_temporal_attn(const T* qkv, int64_t ld, int64_t D, OutT* o, int64_t ldo, int F, int Lv,
                         int H, int dh, cudaStream_t st);

// bf16 temporal branch on warp-level tensor-core MMAs (vc_attn_temporal_mma.cu)
// pos_major: q/k/v row of (frame f, position l) is l*F + f (else f*Lv + l)
int launch_temporal_mma(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo,
                        int F, int Lv, int H, int dh, cudaStream_t st, int head_slot = 0, int pos_major = 0);
// bf16 temporal branch on tcgen05 + TMA (vc_attn_temporal_tc.cu), F <= 176, dh <= 128
bool temporal_tc_supported(int64_t ld, int64_t D, int F, int dh, const void* qkv);
int launch_temporal_tc(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F,
                       int Lv, int H, int dh, cudaStream_t st, int head_slot = 0, int pos_major = 0);
// the bf16 temporal branch: tcgen05 kernel where it applies, else the mma.sync one
int launch_temporal_bf16(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F,
                         int Lv, int H, int dh, cudaStream_t st, int head_slot = 0, int pos_major = 0);

template <typename OutT>
int launch_ln_rows(const float* x, int64_t n_x, const float* p, int64_t n_p, int D, OutT* out,
                   cudaStream_t st);

// AdaLN-modulated LayerNorm rows (north-star extension): LN(x)*(1+scale)+shift
int launch_ln_rows_mod(const float* x, int64_t n_x, const float* p, int64_t n_p, int D,
                       const float* shift, const float* scale, __nv_bfloat16* out, cudaStream_t st);

int launch_embed(const float* lat, const float* w_in, float* x, int F, int first_frame, int tok0,
                 int ntok, int h, int w, int c, int p, int D, double t, cudaStream_t st);
// Optional DDPM reverse step fused into the unembed (diffusion.py:95-116):
// x_prev = (x_t - coef_eps * eps) * inv_sqrt_alpha (+ sqrt_beta * noise)
struct ReverseStep {
  const float* x_t;
  const float* noise;  // null: mean only (t == 1 or no injected noise)
  float* x_prev;       // null: plain unembed
  float coef_eps, inv_sqrt_alpha, sqrt_beta;
};
int launch_unembed(const float* x, const float* w_out, float* eps, int F, int h, int w, int c,
                   int p, int D, cudaStream_t st, ReverseStep rs = ReverseStep{});
// Column space of the bf16 QKV GEMM: the spatial / full-sequence Q, K, V
// segments are head-padded (H heads x DP columns, dh real + DP-dh zero
// weight columns) so every 16-column chunk of the GEMM tile lies inside one
// head and is stored as one contiguous 32-byte run of the attention layout;
// the temporal segment is the plain 3D columns.  Segment order:
//   sp.q sp.k sp.v | tm (3D) | fs.q fs.k fs.v
//
// Compact variant (dh = 66, the 2B head dim; single-GPU block only): the GEMM
// computes no padding columns.  Each sp / fs segment is
//   [head h: columns 0..63, 64-column runs, h = 0..H-1] [tail: (h, 64), (h, 65) pairs]
// (HW = 64 columns per head in the main part, MAIN = 64 H; the tail packs 8
// heads per 16-column chunk, rounded up to 16).  The destination layouts keep
// the DP = 80 head slots: the tail chunk writes d = 64..79 of Q/K rows (the
// real pair and the zero padding) and V^T rows 64, 65; V^T rows 66..79 (the
// ones column and zeros) are written by fill_vt_pad_kernel.  12% fewer MMA
// columns than the padded space for the same stores.
struct QkvPad {
  int32_t DP;       // head slot of the destination layouts (64, 80 or 128)
  int64_t SEG;      // columns per sp / fs Q, K or V segment: H*DP (padded) or MAIN + tail (compact)
  int64_t TMSEG;    // round_up(3D, 16)
  int64_t Npad;     // 6*SEG + TMSEG
  int32_t HW;       // columns per head in the main part: DP (padded) or 64 (compact)
  int32_t compact;  // 1: compact column space (tail chunks after MAIN)
  int64_t MAIN;     // H*HW
  __host__ __device__ int64_t fs_base() const { return 3 * SEG + TMSEG; }
};
inline int qkv_head_pad(int64_t dh) { return dh <= 64 ? 64 : dh <= 80 ? 80 : dh <= 128 ? 128 : 0; }
inline QkvPad qkv_pad_layout(int64_t D, int64_t H) {
  QkvPad q;
  q.DP = qkv_head_pad(D / H);
  q.SEG = H * q.DP;
  q.TMSEG = (3 * D + 15) / 16 * 16;
  q.Npad = 6 * q.SEG + q.TMSEG;
  q.HW = q.DP;
  q.compact = 0;
  q.MAIN = q.SEG;
  return q;
}
inline bool qkv_compact_ok(int64_t D, int64_t H) { return H > 0 && D % H == 0 && D / H == 66; }
inline QkvPad qkv_compact_layout(int64_t D, int64_t H) {
  if (!qkv_compact_ok(D, H)) return qkv_pad_layout(D, H);
  QkvPad q = qkv_pad_layout(D, H);
  q.HW = 64;
  q.compact = 1;
  q.MAIN = H * 64;
  q.SEG = q.MAIN + (2 * H + 15) / 16 * 16;
  q.Npad = 6 * q.SEG + q.TMSEG;
  return q;
}

int launch_pack(const float* raw, void* wqkv, float* bias, void* wo, int D, int H, bool bf16,
                cudaStream_t st, void* wqkv_c = nullptr, float* bias_c = nullptr, void* wo_s = nullptr);
// Byte offsets inside the packed weight buffer (vc_block.cu).  wqkv_c /
// bias_c: the compact QKV column space (qkv_compact_layout; == wqkv / bias
// when the shape has none).
void packed_offsets(int64_t D, int64_t H, bool bf16, size_t* wqkv, size_t* bias, size_t* wo,
                    size_t* total, size_t* wqkv_c = nullptr, size_t* bias_c = nullptr,
                    size_t* wo_s = nullptr);
// V^T rows [dh, DP) of the compact layout: the ones column (row dh) and zeros
int launch_fill_vt_pad(__nv_bfloat16* vt, int64_t nslots, int DP, int dh, int64_t ld, int64_t keys,
                       cudaStream_t st);

// stage profiler (vc_profile.cu)
bool profile_on();
void profile_begin(cudaStream_t st);
void profile_mark(cudaStream_t st, const char* name);
void profile_end();

// bf16 tensor-core path (vc_block_bf16.cu)
size_t bf16_workspace_bytes(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H);
int bf16_launch_count(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H);
// North-star extensions of the bf16 block (vc_ext.cu; parity unpinned,
// oracle/vchitect_ext_oracle.py): AdaLN modulation, QK-RMSNorm + 3D RoPE in
// the QKV epilogue, gated residual, gated GELU FFN.
struct ExtArgs {
  const float* mod;     // [6][D] shift_msa, scale_msa, gate_msa, shift_mlp, scale_mlp, gate_mlp
  const float* qn[2];   // RMSNorm weights [dh]: spatial, full sequence
  const float* kn[2];
  const float2* rope;   // (cos, sin) tables, layout in QkvScatter
  int32_t rope_nt, rope_ny, rope_nx, gw;
  int64_t rope_off_y, rope_off_x;
  int64_t Dff;
  const void* w1;       // bf16 [Dff][D] (K-major B operand)
  const float* b1;      // [Dff]
  const void* w2;       // bf16 [D][Dff]
  const float* b2;      // [D]
  __nv_bfloat16* u;     // FFN hidden [Nv][Dff] (workspace)
};
int block_forward_bf16(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H, const void* wqkv,
                       const float* bias, const void* wo, const float* x, const float* prompt,
                       float* out, int add_residual, char* ws, cudaStream_t st,
                       const ExtArgs* ext = nullptr, const void* wqkv_c = nullptr,
                       const float* bias_c = nullptr, const void* wo_s = nullptr);
// bytes of the bf16 block workspace region holding the O-GEMM A operand
// (acat, [Nv][3D] bf16), reused by the extension as the FFN hidden when Dff <= 3D
size_t bf16_workspace_acat_offset(int64_t F, int64_t Lv, int64_t Lt, int64_t D, int64_t H);

}  // namespace vc
