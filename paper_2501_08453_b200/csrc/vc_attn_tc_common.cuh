// Shared pieces of the tcgen05 attention kernels (vc_attn_tc.cu, vc_attn_tc3.cu):
// Q/K smem descriptors, the per-row online-softmax step, O rescale, P store
// and the output epilogue.  Thread = query row = TMEM lane throughout.
#pragma once
#include <math.h>

#include "vc_attn_tc.h"
#include "vc_gemm_tc.h"
#include "vc_ptx.cuh"
#include "vc_sp_maps.cuh"

namespace vc {
namespace attn {

constexpr int BQ = 128, BKV = 128;
constexpr float kRescaleThreshold = 8.0f;
// Fixed-offset softmax (attn_tp_kernel FIXM): the row's exponent offset is
// set once, from the exact max of the first key block, to max + this margin
// (log2 units), and never moves: P = 2^(x - m) <= 1 for every key within the
// margin of that max, P <= 2^127 (no overflow) for any key up to 187 above
// it, and the first block's max element keeps P = 2^-60 (far from fp32 / bf16
// subnormals). softmax is shift-invariant, so O / l is unchanged; no per-block
// row max, exchange or rescale.
constexpr float kFixedMaxMargin = 60.0f;

// smem descriptor of head-dim 16-chunk c of a [128 rows][DP] Q/K tile laid out
// as N64 SW128 sub-tiles [128][128 B] followed by the SW32 tail [128][32 B]
template <int DP, int ROWS = BQ>
__device__ __forceinline__ uint64_t qk_desc(uint32_t tile_addr, int c) {
  constexpr int N64 = DP / 64;
  if (c < 4 * N64) {
    const uint32_t a = tile_addr + (c >> 2) * (ROWS * 128) + (c & 3) * 32;
    return ptx::smem_desc(a, 0, 1024, ptx::kLayoutSW128);
  }
  return ptx::smem_desc(tile_addr + N64 * (ROWS * 128), 0, 256, ptx::kLayoutSW32);
}

// Load the row's 128 logits of S from TMEM (s_addr includes the lane offset).
__device__ __forceinline__ void load_s(uint32_t s_addr, float (&v)[BKV]) {
  uint32_t r[BKV];
#pragma unroll
  for (int c = 0; c < BKV / 32; ++c)
    ptx::tmem_ld32(s_addr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
  ptx::tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < BKV; ++i) v[i] = __uint_as_float(r[i]);
}

// One online-softmax step on the row's logits of key tile k0: v <- 2^(s*scale
// (+ log2 F on text keys) - m), returns alpha (the factor O and l must be
// rescaled by; 1 when the lazily tracked max m_used did not move).
__device__ __forceinline__ float softmax_step(float (&v)[BKV], int k0, const AttnTcParams& p,
                                              float& m_used, float& l) {
  float scale = p.scale_log2;
  if (k0 < p.n_bias || k0 + BKV > p.Lk) {  // warp-uniform slow path: text keys / tail mask
#pragma unroll
    for (int i = 0; i < BKV; ++i) {
      float t = v[i] * p.scale_log2;
      if (k0 + i < p.n_bias) t += p.bias_log2;
      if (k0 + i >= p.Lk) t = -INFINITY;
      v[i] = t;
    }
    scale = 1.f;
  }
  float m8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m8[i] = v[i];
#pragma unroll
  for (int i = 8; i < BKV; ++i) m8[i & 7] = fmaxf(m8[i & 7], v[i]);
  const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * scale;
  float alpha = 1.f;
  if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
    alpha = ptx::ex2(m_used - mx);         // 0 on the first tile
    m_used = mx;
  }
  const float2 sc2 = make_float2(scale, scale), nm2 = make_float2(-m_used, -m_used);
  float2 s4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) s4[i] = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < BKV; i += 2) {
    float2 t = ptx::ffma2(make_float2(v[i], v[i + 1]), sc2, nm2);
    t.x = ptx::ex2(t.x);
    t.y = ptx::ex2(t.y);
    v[i] = t.x;
    v[i + 1] = t.y;
    s4[(i >> 1) & 3] = ptx::fadd2(s4[(i >> 1) & 3], t);
  }
  const float2 s2 = ptx::fadd2(ptx::fadd2(s4[0], s4[1]), ptx::fadd2(s4[2], s4[3]));
  l = l * alpha + (s2.x + s2.y);
  return alpha;
}

// O (TMEM, DP fp32 columns of this lane) *= alpha; ON < DP: O holds only
// ON columns (the last 16-column chunk is ON % 16 = 8 wide)
template <int DP, int C0 = 0, int C1 = DP / 16, int ON = DP>
__device__ __forceinline__ void rescale_o(uint32_t o_addr, float alpha) {
#pragma unroll
  for (int c = C0; c < C1; ++c) {
    uint32_t r[16];
    if (c * 16 + 16 <= ON) ptx::tmem_ld16(o_addr + c * 16, r);
    else ptx::tmem_ld8p(o_addr + c * 16, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
    if (c * 16 + 16 <= ON) ptx::tmem_st16(o_addr + c * 16, r);
    else ptx::tmem_st8p(o_addr + c * 16, r);
  }
  ptx::tmem_st_wait();
}

// P row -> bf16 -> smem tile [128 rows][128 keys] as two SW128 K-major chunks
// of 64 keys (row pitch 128 B; 16-byte unit u of row r at u ^ (r & 7)).
__device__ __forceinline__ void store_p(uint32_t p_tile, int row, const float (&v)[BKV]) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint32_t rowp = p_tile + c * (BQ * 128) + row * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float* pv = v + c * 64 + u * 8;
      ptx::sts128(rowp + ((u ^ (row & 7)) << 4), ptx::bf16x2(pv[0], pv[1]), ptx::bf16x2(pv[2], pv[3]),
                  ptx::bf16x2(pv[4], pv[5]), ptx::bf16x2(pv[6], pv[7]));
    }
  }
  ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
}

// O / l -> bf16 -> output row of query qi of sequence seq, head h (plain
// [row][ld_out] at col_off, or the sequence-parallel a2a #2 send layout).
// C0..C1: the 16-column chunks of O this thread writes (all by default).
// Output row of query qi (sequence seq, head h): plain [seq * out_seq_rows + qi]
// rows, or the sequence-parallel branch-major send blocks (spo).
__device__ __forceinline__ __nv_bfloat16* out_row(const AttnTcParams& p, int qi, int seq, int h) {
  if (p.spo.P == 0)
    return p.out + (int64_t)(seq * p.out_seq_rows + qi) * p.ld_out + p.col_off +
           (int64_t)h * (p.head_slot ? p.head_slot : p.dh);
  const int f = p.spo.branch == 0 ? seq : qi / p.spo.Lv;
  const int lpos = p.spo.branch == 0 ? qi : qi - f * p.spo.Lv;
  const int r = sp_owner(p.spo.vb, p.spo.P, lpos);
  if (r + 1 == p.spo.self_r1)
    return p.spo.self_out + sp_token_to_row(p.spo.vb, r, f, lpos) * p.spo.self_ld +
           (int64_t)h * (p.head_slot ? p.head_slot : p.dh);
  // base[r] already points at this branch's block for rank r
  return p.out + p.spo.base[r] + sp_token_to_row(p.spo.vb, r, f, lpos) * p.spo.Dg +
         (int64_t)h * (p.head_slot ? p.head_slot : p.dh);
}

template <int DP, int C0 = 0, int C1 = DP / 16, int ON = DP>
__device__ __forceinline__ void store_out(const AttnTcParams& p, uint32_t o_addr, float l, int qi, int seq,
                                          int h) {
  const float inv = 1.f / l;
  __nv_bfloat16* orow = qi < p.Lq ? out_row(p, qi, seq, h) : nullptr;
  if (p.head_slot) {  // whole 16-column chunks (zeros past dh): full-sector 16-byte stores
#pragma unroll
    for (int c = C0; c < C1; ++c) {
      uint32_t r[16];
      if (c * 16 + 16 <= ON) {
        ptx::tmem_ld16(o_addr + c * 16, r);
      } else {  // O holds ON = 16c + 8 columns: the rest are past dh (zero in the slot)
        ptx::tmem_ld8p(o_addr + c * 16, r);
#pragma unroll
        for (int i = 8; i < 16; ++i) r[i] = 0u;
      }
      ptx::tmem_ld_wait();
      if (orow) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float a = (c * 16 + 2 * i < p.dh) ? __uint_as_float(r[2 * i]) * inv : 0.f;
          const float b = (c * 16 + 2 * i + 1 < p.dh) ? __uint_as_float(r[2 * i + 1]) * inv : 0.f;
          __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
          w[i] = *reinterpret_cast<uint32_t*>(&t);
        }
        uint4* o = reinterpret_cast<uint4*>(orow + c * 16);
        o[0] = make_uint4(w[0], w[1], w[2], w[3]);
        o[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    return;
  }
#ifdef VC_ATTN_TRACE
  if (!p.out) orow = nullptr;  // trace builds: time the kernel without its output stores
#endif
#pragma unroll
  for (int c = C0; c < C1; ++c) {
    uint32_t r[16];
    if (c * 16 + 16 <= ON) {
      ptx::tmem_ld16(o_addr + c * 16, r);
    } else {
      ptx::tmem_ld8p(o_addr + c * 16, r);
#pragma unroll
      for (int i = 8; i < 16; ++i) r[i] = 0u;
    }
    ptx::tmem_ld_wait();
    if (orow) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const int d = c * 16 + i;
        if (d + 1 < p.dh) {
          __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r[i]) * inv, __uint_as_float(r[i + 1]) * inv);
          if ((((uintptr_t)(orow + d)) & 3) == 0)
            *reinterpret_cast<__nv_bfloat162*>(orow + d) = b;
          else { orow[d] = b.x; orow[d + 1] = b.y; }
        } else if (d < p.dh) {
          orow[d] = __float2bfloat16_rn(__uint_as_float(r[i]) * inv);
        }
      }
    }
  }
}

// TMA descriptors shared by the kernels (Q box rows = BQ, K box rows = KROWS,
// V^T box = 64 keys x DP).
struct AttnMaps {
  CUtensorMap q64, q16, k64, k16, v;
};
template <int DP, int KROWS = BKV>
inline int make_attn_maps(AttnMaps& m, const AttnTcParams& p, const void* q, const void* k, const void* vt,
                          int nseq, int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key) {
  constexpr bool TAIL = (DP % 64) != 0;
  const uint64_t eb = 2;
  {
    const uint64_t dims[4] = {(uint64_t)DP, (uint64_t)p.H, (uint64_t)p.Lq, (uint64_t)nseq};
    const uint64_t str[3] = {DP * eb, (uint64_t)p.H * DP * eb, (uint64_t)q_rows_per_seq * p.H * DP * eb};
    const uint32_t box64[4] = {64, 1, BQ, 1}, box16[4] = {16, 1, BQ, 1};
    VC_TRY(make_tmap_4d_bf16(&m.q64, q, dims, str, box64, CU_TENSOR_MAP_SWIZZLE_128B));
    if (TAIL) VC_TRY(make_tmap_4d_bf16(&m.q16, q, dims, str, box16, CU_TENSOR_MAP_SWIZZLE_32B));
    else m.q16 = m.q64;
  }
  {
    const uint64_t dims[4] = {(uint64_t)DP, (uint64_t)p.H, (uint64_t)p.Lk, (uint64_t)nseq};
    const uint64_t str[3] = {DP * eb, (uint64_t)p.H * DP * eb, (uint64_t)k_rows_per_seq * p.H * DP * eb};
    const uint32_t box64[4] = {64, 1, KROWS, 1}, box16[4] = {16, 1, KROWS, 1};
    VC_TRY(make_tmap_4d_bf16(&m.k64, k, dims, str, box64, CU_TENSOR_MAP_SWIZZLE_128B));
    if (TAIL) VC_TRY(make_tmap_4d_bf16(&m.k16, k, dims, str, box16, CU_TENSOR_MAP_SWIZZLE_32B));
    else m.k16 = m.k64;
  }
  {
    const uint64_t dims[4] = {(uint64_t)p.Lk, (uint64_t)DP, (uint64_t)p.H, (uint64_t)nseq};
    const uint64_t str[3] = {(uint64_t)ld_key * eb, (uint64_t)DP * ld_key * eb, (uint64_t)p.H * DP * ld_key * eb};
    const uint32_t box[4] = {64, DP, 1, 1};
    VC_TRY(make_tmap_4d_bf16(&m.v, vt, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  return VC_OK;
}

}  // namespace attn
}  // namespace vc
