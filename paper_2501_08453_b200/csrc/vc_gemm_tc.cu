// bf16 GEMM on the 5th-generation tensor cores (tcgen05) for sm_100a.
//
//   C[M][N] = A[M][K] . B[N][K]^T     (bf16 operands, fp32 accumulation)
//
// Both operands K-major (row pitch = K), fed by TMA (cp.async.bulk.tensor,
// 128B swizzle) into a 4-stage shared-memory ring; one elected thread issues
// tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM accumulator so
// the epilogue of tile i overlaps the MMAs of tile i+1. Persistent: one CTA
// per SM walking a static tile schedule.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w3 idle, w4..w7 epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
//
// Epilogues (the fused work of the block forward, model.py:181-190,:324):
//   EPI_F32      out fp32 = acc (+ bias[n]) (+ R[m][n])   O-projection+residual
//   EPI_BF16     out bf16 = acc + bias[n]                   plain projection
//   EPI_QKV      acc + bias scattered into the attention layouts: Q/K
//                [row][H][DP] (head dim zero-padded to DP), V transposed per
//                sequence [seq][H][DP][keys] (the K-major B operand of P.V),
//                temporal branch plain [row][3D].
#include "vc_gemm_tc.h"
#include "vc_tuning.h"
#include "vc_ptx.cuh"

namespace vc {

namespace {
constexpr int BM = 128, BK = 64;
// as many smem stages as fit next to the barriers / bias staging (4..6)
template <int BN>
constexpr int stages_for() {
  return (216 * 1024) / (BM * BK * 2 + BN * BK * 2) > 8 ? 8 : (216 * 1024) / (BM * BK * 2 + BN * BK * 2);
}
constexpr int kThreads = 256;

template <int BN>
constexpr size_t smem_bytes() {
  return (size_t)stages_for<BN>() * (BM * BK * 2 + BN * BK * 2) + 256 /*barriers*/ + 4 * 256 * 4 /*bias*/ +
         1024 /*align*/;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- QKV scatter (EPI_QKV) ----
// GEMM row m -> Q row / K row / (sequence, key) of the attention layouts.
__device__ __forceinline__ int qkv_frame(const QkvScatter& s, int64_t m) { return (int)m / (s.Lf ? s.Lf : (int)s.Lv); }
// sp_f: frame of row m (qkv_frame), hoisted out of the chunk loop by the caller
__device__ __forceinline__ void qkv_rows(const QkvScatter& s, int b, int64_t m, int sp_f, int64_t& qrow,
                                         int64_t& krow, int64_t& seq, int64_t& key) {
  // 32-bit index math (rows < 2^31): a 64-bit division is a long software
  // sequence and the epilogue runs it per chunk
  const int mi = (int)m, Lv = (int)s.Lv, Lt = (int)s.Lt;
  if (s.text_rows) {            // prompt rows: full-sequence keys [0, Lt), no queries
    qrow = -1; krow = mi; seq = 0; key = mi;
  } else if (b == 0) {          // spatial: one sequence per frame
    qrow = mi; krow = mi; seq = sp_f; key = mi - sp_f * Lv;
  } else {                      // full sequence: text keys first, then visual
    qrow = mi; krow = mi + Lt; seq = 0; key = mi + Lt;
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmTcParams& p, int64_t m, int n0,
                                               const uint32_t (&r)[16], const float* sbias,
                                               const float* sgate = nullptr, int sp_f = -1) {
  if (m >= p.M) return;
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) + (sbias ? sbias[j] : 0.f);  // smem broadcast
  if constexpr (EPI == EPI_F32G) {  // R + gate * (acc + bias); gate staged in smem per tile
    float* o = p.out_f32 + m * p.ldo + n0;
    const float* R = p.R + m * p.ldr + n0;
    if (n0 + 16 <= p.N && (p.ldo % 4) == 0 && (p.ldr % 4) == 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 rr = *reinterpret_cast<const float4*>(R + j);
        float4 w;
        w.x = fmaf(sgate[j], v[j], rr.x); w.y = fmaf(sgate[j + 1], v[j + 1], rr.y);
        w.z = fmaf(sgate[j + 2], v[j + 2], rr.z); w.w = fmaf(sgate[j + 3], v[j + 3], rr.w);
        *reinterpret_cast<float4*>(o + j) = w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (n0 + j < p.N) o[j] = fmaf(sgate[j], v[j], R[j]);
    }
  } else if constexpr (EPI == EPI_GELU) {
    __nv_bfloat16* o = p.out_bf16 + m * p.ldo + n0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
      const float u = 0.7978845608028654f * fmaf(0.044715f * v[j], v[j] * v[j], v[j]);
      float th;
      asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(u));
      v[j] = 0.5f * v[j] * (1.f + th);
    }
    if (n0 + 16 <= p.N && (p.ldo % 8) == 0) {
      uint4 a, b;
      a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]);
      a.z = pack_bf16x2(v[4], v[5]); a.w = pack_bf16x2(v[6], v[7]);
      b.x = pack_bf16x2(v[8], v[9]); b.y = pack_bf16x2(v[10], v[11]);
      b.z = pack_bf16x2(v[12], v[13]); b.w = pack_bf16x2(v[14], v[15]);
      reinterpret_cast<uint4*>(o)[0] = a;
      reinterpret_cast<uint4*>(o)[1] = b;
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (n0 + j < p.N) o[j] = __float2bfloat16_rn(v[j]);
    }
  } else if constexpr (EPI == EPI_F32) {
    float* o = p.out_f32 + m * p.ldo + n0;
    const float* R = p.R ? p.R + m * p.ldr + n0 : nullptr;
    if (n0 + 16 <= p.N && (p.ldo % 4) == 0 && (!R || (p.ldr % 4) == 0)) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        float4 w = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (R) {
          float4 rr = *reinterpret_cast<const float4*>(R + j);
          w.x += rr.x; w.y += rr.y; w.z += rr.z; w.w += rr.w;
        }
        *reinterpret_cast<float4*>(o + j) = w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (n0 + j < p.N) o[j] = v[j] + (R ? R[j] : 0.f);
    }
  } else if constexpr (EPI == EPI_BF16) {
    __nv_bfloat16* o = p.out_bf16 + m * p.ldo + n0;
    if (n0 + 16 <= p.N && (p.ldo % 8) == 0) {
      uint4 a, b;
      a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]);
      a.z = pack_bf16x2(v[4], v[5]); a.w = pack_bf16x2(v[6], v[7]);
      b.x = pack_bf16x2(v[8], v[9]); b.y = pack_bf16x2(v[10], v[11]);
      b.z = pack_bf16x2(v[12], v[13]); b.w = pack_bf16x2(v[14], v[15]);
      reinterpret_cast<uint4*>(o)[0] = a;
      reinterpret_cast<uint4*>(o)[1] = b;
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (n0 + j < p.N) o[j] = __float2bfloat16_rn(v[j]);
    }
  } else {  // EPI_QKV: 16 columns of the head-padded space (vc_kernels.h QkvPad)
    const QkvScatter& s = p.qkv;
    const QkvPad& q = s.pad;
    const int64_t n = n0 + s.n_base;
    if (n >= 3 * q.SEG && n < q.fs_base()) {  // temporal: plain [row][3D]
      const int64_t j = n - 3 * q.SEG;
      int64_t row = m;
      if (s.tm_F) {  // position-major: row l*F + f
        const int fr = sp_f >= 0 ? sp_f : qkv_frame(s, m);
        row = (m - (int64_t)fr * (s.Lf ? s.Lf : s.Lv)) * s.tm_F + fr;
      }
      __nv_bfloat16* o = s.tm + row * 3 * s.D + j;
      if (j + 16 <= 3 * s.D && n0 + 16 <= p.N) {
        uint4 a, b;
        a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]);
        a.z = pack_bf16x2(v[4], v[5]); a.w = pack_bf16x2(v[6], v[7]);
        b.x = pack_bf16x2(v[8], v[9]); b.y = pack_bf16x2(v[10], v[11]);
        b.z = pack_bf16x2(v[12], v[13]); b.w = pack_bf16x2(v[14], v[15]);
        reinterpret_cast<uint4*>(o)[0] = a;
        reinterpret_cast<uint4*>(o)[1] = b;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (j + i < 3 * s.D && n0 + i < p.N) o[i] = __float2bfloat16_rn(v[i]);
      }
      return;
    }
    const int b = n < 3 * q.SEG ? 0 : 2;
    const int r = (int)(b == 0 ? n : n - q.fs_base());  // 32-bit: column indices are small
    const int seg = (int)q.SEG;
    const int which = r / seg;
    const int jj = r - which * seg;
    if (q.compact && jj >= q.MAIN) {  // compact tail chunk: (h, 64), (h, 65) pairs of 8 heads (mode 0)
      const BranchOut& bo = b == 0 ? s.sp : s.fs;
      int64_t qrow, krow, seq, key;
      qkv_rows(s, b, m, sp_f >= 0 ? sp_f : qkv_frame(s, m), qrow, krow, seq, key);
      const int h0 = (jj - (int)q.MAIN) >> 1;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int h = h0 + i - s.head_base;
        if (h >= s.H) break;
        if (which < 2) {  // d 64, 65 and the zero padding 66..79 of the head slot
          const int64_t row = which == 0 ? qrow : krow;
          if (row < 0) continue;
          uint4* o = reinterpret_cast<uint4*>((which == 0 ? bo.q : bo.k) + (row * s.H + h) * q.DP + 64);
          o[0] = make_uint4(pack_bf16x2(v[2 * i], v[2 * i + 1]), 0u, 0u, 0u);
          o[1] = make_uint4(0u, 0u, 0u, 0u);
        } else {  // V^T rows 64, 65 (rows 66..79: fill_vt_pad_kernel)
          __nv_bfloat16* o = bo.vt + ((seq * s.H + h) * q.DP + 64) * bo.ld_key + key;
          o[0] = __float2bfloat16_rn(v[2 * i]);
          o[bo.ld_key] = __float2bfloat16_rn(v[2 * i + 1]);
        }
      }
      return;
    }
    const int hg = jj / q.HW, d0 = jj - hg * q.HW;  // 16 | HW: the chunk is inside head hg
    if (s.mode == 1) {  // sequence-parallel send layout, branch-major: [b'][g][which][m][Hg][DP]
      const int g = hg / s.Hg, hl = hg - g * s.Hg;
      const int P = s.H / s.Hg;
      if (g + 1 == s.self_g) {  // own head group: straight into this rank's attention layouts
        const BranchOut& bo = b == 0 ? s.sp : s.fs;
        const int f = sp_f >= 0 ? sp_f : qkv_frame(s, m);
        const int l = (int)m - f * s.Lf + s.self_v0;  // position in the frame
        const int tok = f * (int)s.Lv + l;
        __nv_bfloat16* o;
        if (which < 2) {
          const int64_t row = (which == 1 && b != 0) ? tok + s.Lt : tok;
          o = (which == 0 ? bo.q : bo.k) + (row * s.Hg + hl) * q.DP + d0;
        } else {  // V^T: 16 head dims of one key; lanes are consecutive keys (coalesced)
          const int64_t seq = b == 0 ? f : 0, key = b == 0 ? l : tok + s.Lt;
          __nv_bfloat16* vo = bo.vt + ((seq * s.Hg + hl) * q.DP + d0) * bo.ld_key + key;
#pragma unroll
          for (int i = 0; i < 16; ++i, vo += bo.ld_key) *vo = __float2bfloat16_rn(v[i]);
          return;
        }
        uint4 a, c;
        a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]);
        a.z = pack_bf16x2(v[4], v[5]); a.w = pack_bf16x2(v[6], v[7]);
        c.x = pack_bf16x2(v[8], v[9]); c.y = pack_bf16x2(v[10], v[11]);
        c.z = pack_bf16x2(v[12], v[13]); c.w = pack_bf16x2(v[14], v[15]);
        reinterpret_cast<uint4*>(o)[0] = a;
        reinterpret_cast<uint4*>(o)[1] = c;
        return;
      }
      const int gs = (s.self_g && g >= s.self_g) ? g - 1 : g;  // slot among the sent groups
      const int Ps = s.self_g ? P - 1 : P;
      const int64_t rowlen = (int64_t)s.Hg * q.DP;
      __nv_bfloat16* o = s.send + ((int64_t)(b == 0 ? 0 : 1) * Ps + gs) * 3 * s.send_rows * rowlen +
                         (which * s.send_rows + m) * rowlen + hl * q.DP + d0;
      uint4 a, c;
      a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]);
      a.z = pack_bf16x2(v[4], v[5]); a.w = pack_bf16x2(v[6], v[7]);
      c.x = pack_bf16x2(v[8], v[9]); c.y = pack_bf16x2(v[10], v[11]);
      c.z = pack_bf16x2(v[12], v[13]); c.w = pack_bf16x2(v[14], v[15]);
      reinterpret_cast<uint4*>(o)[0] = a;
      reinterpret_cast<uint4*>(o)[1] = c;
      return;
    }
    const int h = hg - s.head_base;
    const BranchOut& bo = b == 0 ? s.sp : s.fs;
    int64_t qrow, krow, seq, key;
    qkv_rows(s, b, m, sp_f >= 0 ? sp_f : qkv_frame(s, m), qrow, krow, seq, key);
    if (which < 2) {
      const int64_t row = which == 0 ? qrow : krow;
      if (row < 0) return;
      __nv_bfloat16* o = (which == 0 ? bo.q : bo.k) + (row * s.H + h) * q.DP + d0;
      uint4 a, c;
      a.x = pack_bf16x2(v[0], v[1]); a.y = pack_bf16x2(v[2], v[3]);
      a.z = pack_bf16x2(v[4], v[5]); a.w = pack_bf16x2(v[6], v[7]);
      c.x = pack_bf16x2(v[8], v[9]); c.y = pack_bf16x2(v[10], v[11]);
      c.z = pack_bf16x2(v[12], v[13]); c.w = pack_bf16x2(v[14], v[15]);
      reinterpret_cast<uint4*>(o)[0] = a;
      reinterpret_cast<uint4*>(o)[1] = c;
    } else {  // V^T: 16 head dims of one key; lanes are consecutive keys (coalesced)
      __nv_bfloat16* o = bo.vt + ((seq * s.H + h) * q.DP + d0) * bo.ld_key + key;
      const int64_t ld = bo.ld_key;
#pragma unroll
      for (int i = 0; i < 16; ++i, o += ld) *o = __float2bfloat16_rn(v[i]);
    }
  }
}

// ---- EPI_QKVN: one head (DP columns) of one row, QK-RMSNorm + 3D RoPE ----
// The tile is head aligned (BN % DP == 0, the launch starts at a segment
// base), so the thread owning row m holds every column of head hg: it loads
// the DP accumulator columns from TMEM, adds the bias, and for Q / K of the
// spatial and full-sequence branches normalises over the dh real dims
// (rms(u) * w, eps 1e-6), rotates the dh/2 pairs by the token's (frame, row,
// column) angles and stores the DP-wide head row.  V and the temporal
// columns take the plain EPI_QKV chunk path.  (oracle/vchitect_ext_oracle.py)
// DH: the real head dim when known at compile time (0: runtime s.dh), which
// turns the dh guards and the RoPE axis selection into constants.
template <int DP, int DH = 0>
__device__ __forceinline__ void qkvn_head(const GemmTcParams& p, int64_t m, int n0, uint32_t taddr,
                                          const float* sbias) {
  const QkvScatter& s = p.qkv;
  const QkvPad& q = s.pad;
  const int64_t n = n0 + s.n_base;
  const bool tmseg = n >= 3 * q.SEG && n < q.fs_base();
  int b = 0, which = 2, hg = 0;
  if (!tmseg) {
    b = n < 3 * q.SEG ? 0 : 2;
    const int64_t r = b == 0 ? n : n - q.fs_base();
    which = (int)(r / q.SEG);
    hg = (int)((r - which * q.SEG) / DP);
  }
  uint32_t u[DP];
#pragma unroll
  for (int c = 0; c < DP / 16; ++c) ptx::tmem_ld16p(taddr + c * 16, u + c * 16);
  ptx::tmem_ld_wait();
  if (tmseg || which == 2) {  // warp-uniform: V^T / temporal columns, plain scatter
#pragma unroll
    for (int c = 0; c < DP / 16; ++c) {
      if (n0 + c * 16 >= p.N) break;
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = u[c * 16 + j];
      epilogue_chunk<EPI_QKV>(p, m, n0 + c * 16, r, sbias ? sbias + c * 16 : nullptr);
    }
    return;
  }
  if (m >= p.M) return;
  float v[DP];
  float ss4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 partial sums: short dependency chains
#pragma unroll
  for (int d = 0; d < DP; d += 4) {
    // bias: one 16-byte smem broadcast per 4 columns (the head block is 16-byte aligned)
    const float4 bb = sbias ? *reinterpret_cast<const float4*>(sbias + d) : make_float4(0.f, 0.f, 0.f, 0.f);
    v[d] = __uint_as_float(u[d]) + bb.x; v[d + 1] = __uint_as_float(u[d + 1]) + bb.y;
    v[d + 2] = __uint_as_float(u[d + 2]) + bb.z; v[d + 3] = __uint_as_float(u[d + 3]) + bb.w;
#pragma unroll
    for (int j = 0; j < 4; ++j) ss4[j] = fmaf(v[d + j], v[d + j], ss4[j]);  // padding columns are exact zeros
  }
  const float ss = (ss4[0] + ss4[1]) + (ss4[2] + ss4[3]);
  const int bi = b == 0 ? 0 : 1;
  const float2* w2 = reinterpret_cast<const float2*>(which == 0 ? s.qn[bi] : s.kn[bi]);  // dh even: 8-byte aligned
  const int dh = DH ? DH : s.dh;
  const float rs = rsqrtf(ss / (float)dh + 1e-6f);
#pragma unroll
  for (int i = 0; i < DP / 2; ++i)
    if (2 * i < dh) {
      const float2 w = __ldg(w2 + i);
      v[2 * i] *= rs * w.x;
      v[2 * i + 1] *= rs * w.y;
    }
  int64_t qrow, krow, seq, key;
  qkv_rows(s, b, m, qkv_frame(s, m), qrow, krow, seq, key);
  if (!s.text_rows) {  // visual token: (frame, row, column) rotation
    const int64_t f = m / s.Lv, l = m - f * s.Lv;
    const int y = (int)(l / s.gw), x = (int)(l - (int64_t)(l / s.gw) * s.gw);
    // compile-time split when DH is known (vc_ext.cu rope_split: ny = nx = P/3)
    const int nt = DH ? DH / 2 - 2 * (DH / 6) : s.rope_nt;
    const int nty = DH ? DH / 2 - DH / 6 : s.rope_nt + s.rope_ny;
    const float2* pt = s.rope + f * nt;
    const float2* py = s.rope + s.rope_off_y + (int64_t)y * s.rope_ny - nt;
    const float2* px = s.rope + s.rope_off_x + (int64_t)x * s.rope_nx - nty;
#pragma unroll
    for (int i = 0; i < DP / 2; ++i) {
      if (2 * i < dh) {
        const float2 cs = __ldg(i < nt ? pt + i : i < nty ? py + i : px + i);
        const float a = v[2 * i], c = v[2 * i + 1];
        v[2 * i] = a * cs.x - c * cs.y;
        v[2 * i + 1] = fmaf(a, cs.y, c * cs.x);
      }
    }
  }
  const int h = hg - s.head_base;
  const BranchOut& bo = b == 0 ? s.sp : s.fs;
  const int64_t row = which == 0 ? qrow : krow;
  if (row < 0) return;
  uint4* o = reinterpret_cast<uint4*>((which == 0 ? bo.q : bo.k) + (row * s.H + h) * DP);
#pragma unroll
  for (int c = 0; c < DP / 8; ++c) {
    uint4 a;
    a.x = pack_bf16x2(v[8 * c], v[8 * c + 1]); a.y = pack_bf16x2(v[8 * c + 2], v[8 * c + 3]);
    a.z = pack_bf16x2(v[8 * c + 4], v[8 * c + 5]); a.w = pack_bf16x2(v[8 * c + 6], v[8 * c + 7]);
    o[c] = a;
  }
}

// Rasterised tile order: cluster tiles are walked in groups of kGroupM rows
// (M) sweeping all N tiles, so the ~148 tiles in flight touch only a few A
// row-panels and B column-panels and both stay resident in L2.
constexpr int kGroupM = 4;
__device__ __forceinline__ void tile_coords(int ct, int num_mc, int num_n, int& mc, int& nt, int group_m = 0) {
  const int gm = group_m > 0 ? group_m : kGroupM;
  const int per_group = gm * num_n;
  const int g = ct / per_group, r = ct - g * per_group;
  const int first = g * gm;
  const int gsize = min(num_mc - first, gm);
  mc = first + r % gsize;
  nt = r / gsize;
}

// CM = CTAs per cluster along M. The CM CTAs of a cluster work on CM
// consecutive M tiles of the SAME N tile: each loads its own A tile and 1/CM
// of the B tile, multicast (TMA .multicast::cluster) into every CTA of the
// cluster, so B crosses L2 once per cluster instead of once per CTA. A stage
// is refilled only after all CM CTAs' MMAs released it (each MMA commit
// arrives on the empty barrier of every CTA in the cluster).
template <int BN, int EPI, int CM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int STAGES = stages_for<BN>();
  constexpr uint32_t kABytes = BM * BK * 2, kBBytes = BN * BK * 2;
  constexpr int kBSlice = BN / CM;  // B rows each CTA loads and multicasts
  static_assert(kBSlice % 8 == 0, "B slice must keep 8-row swizzle atoms");
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * kBBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int rank = CM > 1 ? (int)ptx::cluster_ctarank() : 0;
  const int cluster = blockIdx.x / CM, nclusters = gridDim.x / CM;
  const int num_m = (int)cdiv(p.M, BM), num_n = (int)cdiv(p.N, BN);
  const int num_mc = (num_m + CM - 1) / CM;  // cluster tiles along M
  const int ctiles = num_mc * num_n;
  const int kblocks = (int)cdiv(p.K, BK);

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], CM); }
    for (int a = 0; a < 2; ++a) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 128); }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  if constexpr (CM > 1) ptx::cluster_sync();  // peers' barriers exist before any multicast
  ptx::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (ptx::elect_one()) {
      int s = 0; uint32_t ph = 0;
      for (int ct = cluster; ct < ctiles; ct += nclusters) {
        int mc, nt;
        tile_coords(ct, num_mc, num_n, mc, nt, p.group_m);
        const int mt = mc * CM + rank;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&empty[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], kABytes + kBBytes);
          ptx::tma_load_2d(sA + s * kABytes, &tmA, &full[s], kb * BK, mt * BM);
          if constexpr (CM == 1) {
            ptx::tma_load_2d(sB + s * kBBytes, &tmB, &full[s], kb * BK, nt * BN);
          } else {
            ptx::tma_load_2d_mc(sB + s * kBBytes + rank * kBSlice * 128, &tmB, &full[s], kb * BK,
                                nt * BN + rank * kBSlice, (uint16_t)((1u << CM) - 1));
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
    int s = 0; uint32_t ph = 0; int local = 0;
    for (int ct = cluster; ct < ctiles; ct += nclusters, ++local) {
      const int acc = local & 1;
      ptx::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
      ptx::fence_after_sync();
      const uint32_t dtmem = tmem_base + acc * 256;
      for (int kb = 0; kb < kblocks; ++kb) {
        ptx::mbar_wait(&full[s], ph);
        ptx::fence_after_sync();
        if (ptx::elect_one()) {
          const uint32_t a0 = ptx::smem_u32(sA + s * kABytes);
          const uint32_t b0 = ptx::smem_u32(sB + s * kBBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = ptx::smem_desc(a0 + kk * 32, 0, 1024, ptx::kLayoutSW128);
            const uint64_t bd = ptx::smem_desc(b0 + kk * 32, 0, 1024, ptx::kLayoutSW128);
            ptx::mma_bf16_ss(dtmem, ad, bd, idesc, (kb | kk) != 0);
          }
          if constexpr (CM == 1) ptx::mma_commit(&empty[s]);
          else ptx::mma_commit_mc(&empty[s], (uint16_t)((1u << CM) - 1));
          if (kb == kblocks - 1) ptx::mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int lane = threadIdx.x & 31;
    float* sbias = reinterpret_cast<float*>(bars + 2 * STAGES + 8) + q * 256;
    int local = 0;
    for (int ct = cluster; ct < ctiles; ct += nclusters, ++local) {
      const int acc = local & 1;
      int mc, nt;
        tile_coords(ct, num_mc, num_n, mc, nt, p.group_m);
        const int mt = mc * CM + rank;
      // this tile's bias columns -> a per-warp smem copy (read back as broadcasts)
      if (p.bias) {
        __syncwarp();
        for (int c = lane; c < BN; c += 32) {
          const int n = nt * BN + c;
          sbias[c] = n < p.N ? __ldg(p.bias + n) : 0.f;
        }
        __syncwarp();
      }
      ptx::mbar_wait(&tfull[acc], (local >> 1) & 1);
      ptx::fence_after_sync();
      const int64_t m = (int64_t)mt * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256;
#pragma unroll 1
      for (int c = 0; c < BN / 16; ++c) {
        const int n0 = nt * BN + c * 16;
        if (n0 >= p.N || (int64_t)mt * BM >= p.M) break;
        uint32_t r[16];
        ptx::tmem_ld16(tbase + c * 16, r);
        ptx::tmem_ld_wait();
        epilogue_chunk<EPI>(p, m, n0, r, p.bias ? sbias + c * 16 : nullptr);
      }
      ptx::fence_before_sync();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  if constexpr (CM > 1) ptx::cluster_sync();  // no CTA leaves while peers may still signal it
  if (warp == 2) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

// ---- CTA-pair GEMM (tcgen05 cta_group::2) ------------------------------------------
// A cluster of 2 CTAs on one TPC computes a 256 x BN tile: each CTA TMAs its
// 128 A rows and BN/2 B rows; the leader issues M=256 MMAs that read both
// CTAs' shared memory and write each CTA's TMEM (its 128 rows x BN columns).
// Per SM the operand bytes per MMA cycle drop by a third against the
// single-CTA tile (B is split across the pair instead of replicated), which is
// what limits the single-CTA kernel (L2 -> SMEM feed, ~96 B/clk needed).
template <int BN>
constexpr int stages2_for() {
  return (216 * 1024) / (BM * BK * 2 + (BN / 2) * BK * 2) > 8 ? 8 : (216 * 1024) / (BM * BK * 2 + (BN / 2) * BK * 2);
}
template <int BN, int EPI, int EW = 4>
constexpr size_t smem2_bytes() {  // stages + barriers + bias staging per epilogue warp (+ gate, EPI_F32G) + align
  return (size_t)stages2_for<BN>() * (BM * BK * 2 + (BN / 2) * BK * 2) + 256 + EW * 256 * 4 +
         (EPI == EPI_F32G ? EW * 256 * 4 : 0) + 1024;
}

// NP = CTA pairs per cluster.  NP = 2: the two pairs of a 4-CTA cluster
// compute neighbouring N tiles of the same 256-row M tile and SHARE A: pair p
// loads 64-row slice p of each CTA's 128-row A half and multicasts it to the
// same-rank CTA of the other pair, halving the A bytes each SM pulls from L2
// (the pair kernel was L2 -> SMEM bound: 9.3 GB of L2 reads for the QKV GEMM).
//
// EW = epilogue warps (4 or 8).  The QKV scatter epilogue (V^T transposed
// stores, per-chunk layout math) is slower than the 25 k-block main loop of
// a K = D tile: with 4 warps the MMA warp waits on tempty (ncu: the QKV GEMM
// was epilogue-bound).  EW = 8 puts two warps on each TMEM lane quarter
// (warp w reads lanes 32 * (w % 4)), splitting the tile's 16-column chunks.
template <int BN, int EPI, int NP, int EW = 4>
__global__ void __launch_bounds__(128 + 32 * EW, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int STAGES = stages2_for<BN>();
  constexpr int BNH = BN / 2;
  static_assert(BNH % 8 == 0, "half tile must keep 8-row swizzle atoms");
  constexpr uint32_t kABytes = BM * BK * 2, kBBytes = BNH * BK * 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * kBBytes);
  uint64_t* full = bars;                // leader's: both CTAs' bytes
  uint64_t* empty = bars + STAGES;      // each CTA's: leader MMA commit multicast
  uint64_t* tfull = bars + 2 * STAGES;  // each CTA's
  uint64_t* tempty = tfull + 2;         // leader's: both CTAs' epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias_all = reinterpret_cast<float*>(bars + 2 * STAGES + 8);

  const int warp = threadIdx.x >> 5;
  const uint32_t crank = ptx::cluster_ctarank();
  const uint32_t rank = crank & 1;          // rank inside the CTA pair
  const int pair = (int)(crank >> 1);       // pair inside the cluster
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / (2 * NP), nclusters = gridDim.x / (2 * NP);
  const int num_m = (int)cdiv(p.M, 2 * BM), num_n = (int)cdiv(p.N, BN);
  const int num_nc = (int)cdiv(num_n, NP);  // N tiles per cluster step
  const int tiles = num_m * num_nc;
  const int kblocks = (int)cdiv(p.K, BK);

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    // full[s] (leader): one arrival, the leader's expect_tx of BOTH CTAs' bytes
    // (the peer's TMA may land first: the tx count just dips below zero)
    // empty[s]: one commit from every pair leader that reads this CTA's stage
    // (NP = 2: the A slice this CTA loads also lands in the other pair)
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], NP); }
    // tempty (leader): one arrival per epilogue warp of both CTAs
    for (int a = 0; a < 2; ++a) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 2 * EW); }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::cluster_sync();
  ptx::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (ptx::elect_one()) {
      int s = 0; uint32_t ph = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        int mt, ntc;
        tile_coords(t, num_m, num_nc, mt, ntc, p.group_m);
        const int nt = ntc * NP + pair;  // may be >= num_n (odd count): B is OOB, no output
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&empty[s], ph ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * (kABytes + kBBytes));
          if (NP == 1) {
            ptx::tma_load_2d_2sm(sA + s * kABytes, &tmA, &full[s], kb * BK, mt * 2 * BM + rank * BM);
          } else {  // slice `pair` (64 rows) of this rank's A half -> both pairs' same-rank CTAs
            ptx::tma_load_2d_2sm_mc(sA + s * kABytes + pair * (BM / 2) * 128, &tmA, &full[s], kb * BK,
                                    mt * 2 * BM + rank * BM + pair * (BM / 2), (uint16_t)((1u << rank) | (1u << (rank + 2))));
          }
          ptx::tma_load_2d_2sm(sB + s * kBBytes, &tmB, &full[s], kb * BK, nt * BN + rank * BNH);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * BM, BN);
      int s = 0; uint32_t ph = 0; int local = 0;
      for (int t = cluster; t < tiles; t += nclusters, ++local) {
        const int acc = local & 1;
        ptx::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        ptx::fence_after_sync();
        const uint32_t dtmem = tmem_base + acc * 256;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&full[s], ph);
          ptx::fence_after_sync();
          if (ptx::elect_one()) {
            const uint32_t a0 = ptx::smem_u32(sA + s * kABytes);
            const uint32_t b0 = ptx::smem_u32(sB + s * kBBytes);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = ptx::smem_desc(a0 + kk * 32, 0, 1024, ptx::kLayoutSW128);
              const uint64_t bd = ptx::smem_desc(b0 + kk * 32, 0, 1024, ptx::kLayoutSW128);
              ptx::mma_bf16_ss_2sm(dtmem, ad, bd, idesc, (kb | kk) != 0);
            }
            ptx::mma_commit_2sm_mc(&empty[s], (uint16_t)((1u << (2 * NP)) - 1));  // every CTA that fed it
            if (kb == kblocks - 1) ptx::mma_commit_2sm_mc(&tfull[acc], (uint16_t)(0x3u << (2 * pair)));
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;           // TMEM lane quarter
    const int ew = warp - 4;          // epilogue warp index
    const int sub = ew >> 2;          // which of the EW / 4 warps on this quarter
    const int lane = threadIdx.x & 31;
    float* sbias = sbias_all + ew * 256;
    float* sgate = sbias_all + EW * 256 + ew * 256;  // EPI_F32G only (smem2_bytes)
    const uint32_t tempty_leader = ptx::mapa_shared(ptx::smem_u32(tempty), (uint32_t)(2 * pair));
    int local = 0;
    for (int t = cluster; t < tiles; t += nclusters, ++local) {
      const int acc = local & 1;
      int mt, ntc;
      tile_coords(t, num_m, num_nc, mt, ntc, p.group_m);
      const int nt = ntc * NP + pair;
      if (p.bias) {
        __syncwarp();
        for (int c = lane; c < BN; c += 32) {
          const int n = nt * BN + c;
          sbias[c] = n < p.N ? __ldg(p.bias + n) : 0.f;
        }
        __syncwarp();
      }
      const int64_t mrow0 = (int64_t)mt * 2 * BM + rank * BM;
      const int64_t m = mrow0 + q * 32 + lane;
      if constexpr (EPI == EPI_F32G) {
        __syncwarp();
        for (int c = lane; c < BN; c += 32) {
          const int n = nt * BN + c;
          sgate[c] = n < p.N ? __ldg(p.gate + n) : 0.f;
        }
        __syncwarp();
      }
      if constexpr (EPI == EPI_F32 || EPI == EPI_F32G) {
        // the residual rows do not depend on the accumulator: pull this
        // thread's R segment into L2 while the tile's MMAs run, so the
        // epilogue's loads hit L2 instead of paying HBM latency per chunk
        if (p.R && m < p.M) {
          const char* rp = reinterpret_cast<const char*>(p.R + m * p.ldr + (int64_t)nt * BN);
          const int nb = min(BN, p.N - nt * BN) * 4;
          for (int b = 0; b < nb; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + b));
        }
      }
      ptx::mbar_wait(&tfull[acc], (local >> 1) & 1);
      ptx::fence_after_sync();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256;
      if constexpr ((EPI & 255) == EPI_QKVN) {  // EPI = EPI_QKVN | DP << 8: head by head
        constexpr int EDP = (EPI >> 8) & 255, EDH = EPI >> 16;
#pragma unroll 1
        for (int hb = 0; hb < BN / EDP; ++hb) {
          const int n0 = nt * BN + hb * EDP;
          if (n0 >= p.N || mrow0 >= p.M) break;
          qkvn_head<EDP, EDH>(p, m, n0, tbase + hb * EDP, p.bias ? sbias + hb * EDP : nullptr);
        }
      } else {
        const int sp_f = EPI == EPI_QKV && m < p.M ? qkv_frame(p.qkv, m) : 0;
#pragma unroll 1
        for (int c = sub; c < BN / 16; c += EW / 4) {
          const int n0 = nt * BN + c * 16;
          if (n0 >= p.N || mrow0 >= p.M) break;
          uint32_t r[16];
          ptx::tmem_ld16(tbase + c * 16, r);
          ptx::tmem_ld_wait();
          epilogue_chunk<EPI>(p, m, n0, r, p.bias ? sbias + c * 16 : nullptr, sgate + c * 16, sp_f);
        }
      }
      ptx::fence_before_sync();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + acc * 8);
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc_2sm(tmem_base, 512);
  }
}

// ---- host side -------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int EPI, int CM>
int launch_impl(const CUtensorMap& ta, const CUtensorMap& tb, const GemmTcParams& p,
                cudaStream_t st) {
  static bool attr_set = false;
  constexpr size_t smem = smem_bytes<BN>();
  if (!attr_set) {
    VC_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI, CM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int64_t ctiles = cdiv(cdiv(p.M, BM), CM) * cdiv(p.N, BN);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CM;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid = the clusters that can be resident at once (GPC packing
  // limits clusters of 4 well below num_SMs / 4)
  static int resident = 0;
  if (!resident) {
    cfg.gridDim = dim3((unsigned)(num_sms() / CM * CM));
    if (cudaOccupancyMaxActiveClusters(&resident, gemm_tc_kernel<BN, EPI, CM>, &cfg) != cudaSuccess || resident <= 0)
      resident = num_sms() / CM;
    if (tuning_debug()) fprintf(stderr, "gemm_tc CM=%d: %d resident clusters\n", CM, resident);
  }
  const int clusters = (int)std::min<int64_t>(ctiles, resident);
  cfg.gridDim = dim3((unsigned)(clusters * CM));
  VC_CHECK_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, EPI, CM>, ta, tb, p));
  VC_CHECK_LAUNCH();
  return VC_OK;
}

template <int BN, int EPI, int NP, int EW = 4>
int launch_impl2(const CUtensorMap& ta, const CUtensorMap& tb, const GemmTcParams& p, cudaStream_t st) {
  static bool attr_set = false;
  constexpr size_t smem = smem2_bytes<BN, EPI, EW>();
  if (!attr_set) {
    VC_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<BN, EPI, NP, EW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    attr_set = true;
  }
  const int64_t ctiles = cdiv(p.M, 2 * BM) * cdiv(cdiv(p.N, BN), NP);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(128 + 32 * EW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * NP;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int resident = 0;  // co-resident clusters (see launch_impl)
  if (!resident) {
    cfg.gridDim = dim3((unsigned)(num_sms() / (2 * NP) * 2 * NP));
    if (cudaOccupancyMaxActiveClusters(&resident, gemm_tc2_kernel<BN, EPI, NP, EW>, &cfg) != cudaSuccess ||
        resident <= 0)
      resident = num_sms() / (2 * NP);
    if (tuning_debug()) fprintf(stderr, "gemm_tc2 NP=%d: %d resident clusters\n", NP, resident);
  }
  const int clusters = (int)std::min<int64_t>(ctiles, resident);
  cfg.gridDim = dim3((unsigned)(clusters * 2 * NP));
  VC_CHECK_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<BN, EPI, NP, EW>, ta, tb, p));
  VC_CHECK_LAUNCH();
  return VC_OK;
}
}  // namespace

int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                      CUtensorMapSwizzle swz) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable (driver too old?)"); return VC_ECUDA; }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(2d) failed: %d (inner %llu outer %llu pitch %llu)", (int)r,
              (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_pitch_bytes);
    return VC_ECUDA;
  }
  return VC_OK;
}

int make_tmap_4d_bf16(CUtensorMap* map, const void* base, const uint64_t dims_[4],
                      const uint64_t strides_bytes[3], const uint32_t box_[4],
                      CUtensorMapSwizzle swz) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return VC_ECUDA; }
  cuuint64_t dims[4] = {dims_[0], dims_[1], dims_[2], dims_[3]};
  cuuint64_t strides[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  cuuint32_t box[4] = {box_[0], box_[1], box_[2], box_[3]};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(4d) failed: %d", (int)r);
    return VC_ECUDA;
  }
  return VC_OK;
}

int gemm_tc_pick_bn(int N, int np) {
  // smallest padded width among the instantiated tile widths, counting the
  // idle tile of an odd N-tile count when pairs share A (np = 2); ties go to
  // the wider tile (fewer A re-reads)
  const int cands[6] = {256, 240, 208, 176, 160, 128};
  int best = 256;
  int64_t best_pad = INT64_MAX;
  for (int bn : cands) {
    const int64_t pad = cdiv(cdiv(N, bn), np) * np * bn - N;
    if (pad < best_pad) { best_pad = pad; best = bn; }
  }
  return best;
}

// The north-star extension epilogues (EPI_QKVN / EPI_GELU / EPI_F32G) run on
// the CTA-pair kernel only (one pair per cluster, any M: rows past M are TMA
// zero fill).  EPI_QKVN needs head-aligned tiles: BN a multiple of the padded
// head dim and the launch's first column on a head boundary (the caller
// starts each launch at a segment base).
static int launch_gemm_tc_ext(const void* A, int64_t lda, const void* B, int64_t ldb,
                              const GemmTcParams& p, int epi, cudaStream_t st) {
  if (epi == EPI_F32G && p.M > BM) {
    // gated residual (long-K GEMMs: O projection, FFN down): two CTA pairs per
    // cluster sharing A, like the O GEMM of the reference-semantics block
    const int bn2 = gemm_tc_pick_bn(p.N, 2);
    if (cdiv(p.N, bn2) >= 2) {
      CUtensorMap ta, tb;
      VC_TRY(make_tmap_2d_bf16(&ta, A, p.K, p.M, lda * 2, BK, BM / 2, CU_TENSOR_MAP_SWIZZLE_128B));
      VC_TRY(make_tmap_2d_bf16(&tb, B, p.K, p.N, ldb * 2, BK, bn2 / 2, CU_TENSOR_MAP_SWIZZLE_128B));
      switch (bn2) {
        case 256: return launch_impl2<256, EPI_F32G, 2>(ta, tb, p, st);
        case 240: return launch_impl2<240, EPI_F32G, 2>(ta, tb, p, st);
        case 208: return launch_impl2<208, EPI_F32G, 2>(ta, tb, p, st);
        case 176: return launch_impl2<176, EPI_F32G, 2>(ta, tb, p, st);
        case 160: return launch_impl2<160, EPI_F32G, 2>(ta, tb, p, st);
        default: return launch_impl2<128, EPI_F32G, 2>(ta, tb, p, st);
      }
    }
  }
  const int dp = epi == EPI_QKVN ? p.qkv.pad.DP : 16;
  int bn = 0;
  int64_t best = INT64_MAX;
  for (int c : {256, 240, 160, 128}) {
    if (c % dp) continue;
    const int64_t pad = cdiv(p.N, c) * c - p.N;
    if (pad < best) { best = pad; bn = c; }
  }
  if (!bn) { set_error("no head-aligned GEMM tile for padded head dim %d", dp); return VC_ENOTSUP; }
  CUtensorMap ta, tb;
  VC_TRY(make_tmap_2d_bf16(&ta, A, p.K, p.M, lda * 2, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B));
  VC_TRY(make_tmap_2d_bf16(&tb, B, p.K, p.N, ldb * 2, BK, bn / 2, CU_TENSOR_MAP_SWIZZLE_128B));
  if (epi == EPI_QKVN) {
    if (dp == 64 && bn == 256) return launch_impl2<256, EPI_QKVN | (64 << 8), 1>(ta, tb, p, st);
    if (dp == 64 && bn == 128) return launch_impl2<128, EPI_QKVN | (64 << 8), 1>(ta, tb, p, st);
    // the 2B head dim (66) specialised; other dims take the runtime-dh epilogue
    if (dp == 80 && bn == 240 && p.qkv.dh == 66) return launch_impl2<240, EPI_QKVN | (80 << 8) | (66 << 16), 1>(ta, tb, p, st);
    if (dp == 80 && bn == 160 && p.qkv.dh == 66) return launch_impl2<160, EPI_QKVN | (80 << 8) | (66 << 16), 1>(ta, tb, p, st);
    if (dp == 80 && bn == 240) return launch_impl2<240, EPI_QKVN | (80 << 8), 1>(ta, tb, p, st);
    if (dp == 80 && bn == 160) return launch_impl2<160, EPI_QKVN | (80 << 8), 1>(ta, tb, p, st);
    if (dp == 128 && bn == 256) return launch_impl2<256, EPI_QKVN | (128 << 8), 1>(ta, tb, p, st);
    if (dp == 128 && bn == 128) return launch_impl2<128, EPI_QKVN | (128 << 8), 1>(ta, tb, p, st);
  }
#define VC_GEMM_EXT(BNV)                                                             \
  if (bn == BNV) return epi == EPI_GELU ? launch_impl2<BNV, EPI_GELU, 1>(ta, tb, p, st) \
                                        : launch_impl2<BNV, EPI_F32G, 1>(ta, tb, p, st);
  VC_GEMM_EXT(256)
  VC_GEMM_EXT(240)
  VC_GEMM_EXT(160)
  VC_GEMM_EXT(128)
#undef VC_GEMM_EXT
  set_error("internal: no extension GEMM for epilogue %d tile %d", epi, bn);
  return VC_ENOTSUP;
}

int launch_gemm_tc(const void* A, int64_t lda, const void* B, int64_t ldb, const GemmTcParams& p_in,
                   int epi, cudaStream_t st, int bn) {
  if (p_in.M <= 0 || p_in.N <= 0) return VC_OK;
  GemmTcParams p = p_in;
  // M tiles per rasterization group: 32 for the QKV GEMM (N = 9D wide: fewer
  // re-reads of the weight panels, 0.771 vs 0.816 ms at kGroupM = 4), the
  // default 4 elsewhere (the O GEMM: 0.251 vs 0.292 at 32); tools/ab_bench.sh
  static const int group_env = tuning_int("VC_GEMM_GROUPM", 0);
  if (!p.group_m) p.group_m = group_env ? group_env : (epi == EPI_QKV ? 32 : 0);
  if (epi >= EPI_QKVN) {
    if (p.K <= 0 || (lda * 2) % 16 || (ldb * 2) % 16 || ((uintptr_t)A % 16) || ((uintptr_t)B % 16)) {
      set_error("tcgen05 GEMM needs 16-byte aligned operands and row pitches");
      return VC_EINVAL;
    }
    return launch_gemm_tc_ext(A, lda, B, ldb, p, epi, st);
  }
  if (p.K <= 0 || (lda * 2) % 16 || (ldb * 2) % 16 || ((uintptr_t)A % 16) || ((uintptr_t)B % 16)) {
    set_error("tcgen05 GEMM needs 16-byte aligned operands and row pitches (lda %lld ldb %lld)",
              (long long)lda, (long long)ldb);
    return VC_EINVAL;
  }
  static const int bn_env = tuning_int("VC_GEMM_BN", 0);  // tuning switch
  // pairs per cluster: 2 sharing A by multicast for the O GEMM (EPI_F32:
  // 0.245 vs 0.264 ms), 1 for the QKV GEMM (0.94 vs 0.98: only 33 clusters of
  // 4 fit at once, 132 of 148 SMs, which eats the L2 saving); VC_GEMM_NP
  // overrides.  (Before the grid was sized with cudaOccupancyMaxActiveClusters
  // the 4-CTA clusters ran in two waves and looked 1.7x slower.)
  static const int np_env = tuning_int("VC_GEMM_NP", 0);
  // epilogue warps of the QKV scatter (8 default; VC_GEMM_EW=4 is the A/B switch)
  static const int ew = tuning_int("VC_GEMM_EW", 8);
  // 2-CTA clusters along M multicast the B tile (halves its L2 traffic);
  // VC_GEMM_NO_MC=1 forces the single-CTA kernel (A/B switch for profiling).
  static const bool no_mc = tuning_int("VC_GEMM_NO_MC", 0) != 0;
  // default: CTA-pair kernel (cta_group::2, 256-row tiles); VC_GEMM_1SM=1
  // selects the single-CTA kernel with B multicast (A/B switch for profiling)
  static const bool one_sm = tuning_int("VC_GEMM_1SM", 0) != 0;
  const bool pair = !one_sm && epi != EPI_BF16 && cdiv(p.M, BM) >= 2;
  static const int cm_env = tuning_int("VC_GEMM_CM", 2);  // 1-CTA kernel cluster
  const int cm = (!no_mc && epi != EPI_BF16 && cdiv(p.M, BM) >= 2) ? (cm_env == 4 && cdiv(p.M, BM) >= 4 ? 4 : 2) : 1;
  const int np_want = np_env ? np_env : (epi == EPI_F32 ? 2 : 1);
  if (bn == 0) bn = bn_env ? bn_env : gemm_tc_pick_bn(p.N, pair && np_want == 2 ? 2 : 1);
  const int np = pair && np_want == 2 && cdiv(p.N, bn) >= 2 ? 2 : 1;
  CUtensorMap ta, tb;
  VC_TRY(make_tmap_2d_bf16(&ta, A, p.K, p.M, lda * 2, BK, np == 2 ? BM / 2 : BM, CU_TENSOR_MAP_SWIZZLE_128B));
  const int cm_eff = cm == 4 && (bn / 4) % 8 != 0 ? 2 : cm;
  VC_TRY(make_tmap_2d_bf16(&tb, B, p.K, p.N, ldb * 2, BK, bn / (pair ? 2 : cm_eff), CU_TENSOR_MAP_SWIZZLE_128B));
#define VC_GEMM_CASE(BNV)                                                                    \
  if (bn == BNV) {                                                                           \
    if (pair && np == 2) return epi == EPI_F32 ? launch_impl2<BNV, EPI_F32, 2>(ta, tb, p, st)  \
                                               : launch_impl2<BNV, EPI_QKV, 2>(ta, tb, p, st); \
    if (pair) return epi == EPI_F32 ? launch_impl2<BNV, EPI_F32, 1>(ta, tb, p, st)           \
                                    : (ew == 8 ? launch_impl2<BNV, EPI_QKV, 1, 8>(ta, tb, p, st) \
                                               : launch_impl2<BNV, EPI_QKV, 1>(ta, tb, p, st)); \
    if (epi == EPI_BF16) return launch_impl<BNV, EPI_BF16, 1>(ta, tb, p, st);                \
    if (cm == 4 && (BNV / 4) % 8 == 0)                                                       \
      return epi == EPI_F32 ? launch_impl<BNV, EPI_F32, ((BNV / 4) % 8 == 0 ? 4 : 2)>(ta, tb, p, st) \
                            : launch_impl<BNV, EPI_QKV, ((BNV / 4) % 8 == 0 ? 4 : 2)>(ta, tb, p, st); \
    if (epi == EPI_F32)                                                                      \
      return cm >= 2 ? launch_impl<BNV, EPI_F32, 2>(ta, tb, p, st)                           \
                     : launch_impl<BNV, EPI_F32, 1>(ta, tb, p, st);                          \
    return cm >= 2 ? launch_impl<BNV, EPI_QKV, 2>(ta, tb, p, st)                             \
                   : launch_impl<BNV, EPI_QKV, 1>(ta, tb, p, st);                            \
  }
  VC_GEMM_CASE(256)
  VC_GEMM_CASE(240)
  VC_GEMM_CASE(208)
  VC_GEMM_CASE(176)
  VC_GEMM_CASE(160)
  VC_GEMM_CASE(128)
#undef VC_GEMM_CASE
  set_error("internal: no GEMM tile of width %d", bn);
  return VC_ENOTSUP;
}

}  // namespace vc
