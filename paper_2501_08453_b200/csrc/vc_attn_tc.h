// tcgen05 flash attention interface (vc_attn_tc.cu).
#pragma once
#include "vc_common.cuh"

namespace vc {

// Sequence-parallel output remap (all-to-all #2 send layout, executor.py:395-412):
// query (frame f, position l) is owned by rank r with vb[r] <= l < vb[r+1]; its
// head-group output row goes to send2[base[r] + (f*vc_r + l - vb[r]) * Dg], base[r]
// = the (branch, r) block of the branch-major send2 [b'][r][M_r][Dg].
struct SpOutMap {
  int32_t P;         // 0: disabled (plain output rows)
  int32_t branch;    // 0 spatial, 1 full sequence
  int32_t F, Lv;
  int64_t Dg;        // Hg * dh
  int32_t vb[17];
  int64_t base[17];
  // own rank + 1 (0: none): rows this rank owns skip the exchange and go to
  // self_out[row * self_ld] (the O GEMM's input; row = f * vc + l - vb[r])
  int32_t self_r1;
  int64_t self_ld;
  __nv_bfloat16* self_out;
};

struct AttnTcParams {
  int32_t Lq, Lk, H, dh;
  int32_t n_bias;       // keys [0, n_bias) get + bias_log2 (deduplicated anchored text)
  float bias_log2;      // log2(F)
  float scale_log2;     // log2(e) / sqrt(dh)
  __nv_bfloat16* out;   // [seq * out_seq_rows + q][ld_out], head h at col_off + h*dh
  int64_t ld_out;
  int64_t col_off;
  int64_t out_seq_rows;
  SpOutMap spo;
  // 0: head h at col_off + h*dh (dh columns).  Else head h at col_off +
  // h*head_slot, written as whole 16-column chunks with zeros past dh (full
  // 32-byte sectors: partial-sector row stores cost ~14% of a 1350-key
  // attention, profiles/r01/attn_study); the O GEMM's weights have zero rows
  // for the slot padding.
  int32_t head_slot;
};

// Split-row variant: each tile's softmax on two warpgroups (vc_attn_tc3.cu).
template <int DP>
int launch_attn_tc3(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st);

// P-in-TMEM variant (112-key blocks; vc_attn_tp.cu), the default for DP <= 80.
template <int DP>
int launch_attn_tp(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                   int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st);

// Padded head dim the tensor-core kernel uses for dh (0: unsupported).
int attn_tc_head_pad(int dh);

// q: [nseq][q_rows_per_seq][H][DP], k: [nseq][k_rows_per_seq][H][DP],
// vt: [nseq][H][DP][ld_key] (bf16).
int launch_attn_tc(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                   int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, int DP,
                   cudaStream_t st);

}  // namespace vc
