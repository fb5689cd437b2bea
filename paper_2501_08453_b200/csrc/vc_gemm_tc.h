// tcgen05 GEMM interface (vc_gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "vc_kernels.h"

namespace vc {

enum {
  EPI_F32 = 0, EPI_BF16 = 1, EPI_QKV = 2,
  // north-star extensions (vc_ext.cu; parity unpinned, see oracle/vchitect_ext_oracle.py)
  EPI_QKVN = 3,  // EPI_QKV + per-head QK-RMSNorm and 3D RoPE on the spatial / full-seq Q, K
  EPI_GELU = 4,  // out bf16 = gelu_tanh(acc + bias[n])                  (FFN up-projection)
  EPI_F32G = 5,  // out fp32 = R[m][n] + gate[n] * (acc + bias[n])        (gated residual)
};

// Attention-layout destination of one branch (spatial or full-sequence).
struct BranchOut {
  __nv_bfloat16* q;   // [q rows][H][DP]
  __nv_bfloat16* k;   // [k rows][H][DP]
  __nv_bfloat16* vt;  // [seq][H][DP][ld_key]
  int64_t ld_key;
};

struct QkvScatter {
  QkvPad pad;         // head-padded column space (vc_kernels.h)
  int64_t D, Lv, Lt;
  int32_t H;          // heads of the destination layout
  int32_t head_base;  // first head of this GEMM's columns (stored as h - head_base)
  int64_t n_base;     // column of this GEMM's n=0 in the padded space
  int32_t text_rows;  // rows are prompt rows (full-sequence keys 0..Lt-1)
  BranchOut sp, fs;
  __nv_bfloat16* tm;  // temporal branch, plain [row][3D]
  // 0: tm rows in GEMM row order (frame-major f*Lv + l); F > 0: position-major
  // rows l*F + f, so a position's F frames are consecutive rows (the
  // temporal attention's sequences, read as whole boxes)
  int32_t tm_F;
  // GEMM rows per frame (0: Lv). The sequence-parallel stage 1 runs on a
  // rank's local rows m = f * vc + l, so its frames are vc rows long.
  int32_t Lf;
  // mode 1 (sequence-parallel send): spatial / full-seq Q, K, V of local row m
  // and head h go to send[b'][g][which][m][h % Hg][DP], g = h / Hg (head group
  // owner), b' = 0 spatial / 1 full sequence (branch-major, so each branch's
  // all-to-all #1 (executor.py:344) can go on its own); P = H / Hg.
  int32_t mode;
  int32_t Hg;
  int64_t send_rows;  // local rows M_r
  __nv_bfloat16* send;
  // mode 1: self_g = this rank's own head group + 1 (0: every group is
  // sent). The own group is not sent: its q, k, V^T go straight into the
  // attention layouts sp / fs (H = Hg heads), local row m = f * Lf + l ->
  // visual token f * Lv + self_v0 + l; send holds the other P - 1 groups in
  // rank order.
  int32_t self_g;
  int32_t self_v0;
  // EPI_QKVN: RMSNorm weights [dh] per branch (0 spatial, 1 full sequence),
  // RoPE (cos, sin) tables: rope[pos_t * nt + j] (frames), then
  // rope[rope_off_y + y * ny + j] and rope[rope_off_x + x * nx + j] (patch
  // grid rows / columns, gw columns); pair i < nt is temporal, i < nt + ny row,
  // else column.  Text rows carry no position (no rotation).
  const float* qn[2];
  const float* kn[2];
  const float2* rope;
  int32_t dh, rope_nt, rope_ny, rope_nx, gw;
  int64_t rope_off_y, rope_off_x;
};

struct GemmTcParams {
  int64_t M;
  int32_t N, K;
  const float* bias;  // [N] (indexed by local n) or null
  float* out_f32; const float* R; int64_t ldr;
  __nv_bfloat16* out_bf16;
  int64_t ldo;
  const float* gate;  // EPI_F32G: [N]
  QkvScatter qkv;
  int32_t group_m;    // M tiles per rasterization group (0: the default, kGroupM)
};

// C = A[M][K] . B[N][K]^T with the selected epilogue.  A/B bf16 K-major.
// bn: N tile width (0 = pick the least padding among 256/240/176/128).
int launch_gemm_tc(const void* A, int64_t lda, const void* B, int64_t ldb, const GemmTcParams& p,
                   int epi, cudaStream_t st, int bn = 0);

int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                      CUtensorMapSwizzle swz);
int make_tmap_4d_bf16(CUtensorMap* map, const void* base, const uint64_t dims[4],
                      const uint64_t strides_bytes[3], const uint32_t box[4],
                      CUtensorMapSwizzle swz);
int num_sms();

}  // namespace vc
