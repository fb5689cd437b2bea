// Sequence-parallel block forward: the three rank-local stages around the two
// all-to-alls of the paper's memory-efficient hybrid-parallel scheme
// (executor.py:561-626, spatial shard axis, head-parallel attention,
// "separate" text placement).  The collectives themselves are NCCL
// all_to_all_single calls issued by the host (paper_2501_08453_b200/sp.py);
// this file owns every byte layout on either side of them.
//
// Rank r holds visual rows [vb[r], vb[r+1]) of every frame (vb =
// contiguous_bounds(Lv, P), executor.py:187-191) and the whole prompt
// (text is static, anchored context any rank can regenerate; executor.py
// docstring).  Head group g = heads [g*H/P, (g+1)*H/P) is owned by rank g.
//
//   stage 1 (rank r): LN + QKV GEMM of the local rows; the epilogue writes the
//       spatial / full-seq q, k, v of the peers' head groups straight into the
//       a2a #1 send layout send1[b'][g][which][m][Hg][DP] and those of the own
//       head group straight into the attention layouts (they never travel);
//       temporal q/k/v position-major, the temporal branch is rank-local.
//   a2a #1 (NCCL)
//   stage 2 (rank g): unpack the peers' rows into the attention layouts for
//       the Hg heads of the group, text K/V of the group's heads from the
//       local prompt copy, tcgen05 attention whose epilogue writes the a2a #2
//       send layout send2[b'][r][m][Dg] (executor.py:395-412) for the peers'
//       rows and the O GEMM input for the own rows.
//   a2a #2 (NCCL)
//   stage 3 (rank r): gather the peers' head-group column blocks into [A_sp|
//       A_tm|A_fs] and run the O GEMM + residual for the local rows.
// At one rank nothing is exchanged or unpacked: the stages are the
// single-GPU block's kernels.
#include <math.h>

#include "vc_attn_tc.h"
#include "vc_gemm_tc.h"
#include "vc_kernels.h"
#include "vc_sp_maps.cuh"

namespace vc {

namespace {

inline size_t aup(size_t v) { return (v + 1023) / 1024 * 1024; }

struct Sp {
  int64_t F, Lv, Lt, D, H, dh, Nv, P, rank, Hg, Dg, DP, Lv_ld, Lk_ld;
  // head-parallel, dh 66: attention outputs in 80-column head slots (S = DP)
  // through send2 / recv2 and acat [m][3][H][S] (whole-sector stores, the
  // single-GPU block's layout); BW = acat columns per branch (H*S or D)
  int64_t S, BW;
  int32_t vb[17];
  int64_t M[16];       // local rows F*vc_r per rank
  // exchange buffers are branch-major: [b'][peer][...]; offsets of the
  // per-peer blocks inside one branch half, and the half sizes. The own
  // block never enters the buffers (size 0 here): stage 1 writes the own
  // head group's q, k, V^T straight into the attention layouts and stage 2
  // the own rows' outputs straight into the O GEMM's input.
  int64_t s1_off[17];  // recv1 (by source rank): 3 * M_r * Hg * DP each
  int64_t s2_off[17];  // send2 (by destination rank): M_r * Dg each
  int64_t half1, half2;
  QkvPad pad;
};

// counts_only: the exchange sizes are integer formulas; they are also asked
// for shapes the bf16 kernels do not take (the reference's D = 12 toy plans)
int sp_make(const vc_sp_plan* pl, Sp* o, bool gather = false, bool counts_only = false) {
  if (!pl) { set_error("null plan"); return VC_EINVAL; }
  const vc_block_shape& s = pl->shape;
  if (!counts_only) VC_TRY(vc_block_shape_check(&s));
  else if (s.frames <= 0 || s.visual_len <= 0 || s.dim <= 0 || s.heads <= 0 || s.dim % s.heads) {
    set_error("bad block shape");
    return VC_EINVAL;
  }
  if (s.dtype != VC_DTYPE_BF16) { set_error("sequence parallelism runs the bf16 path"); return VC_ENOTSUP; }
  const int P = pl->nranks;
  if (P < 1 || P > 16 || pl->rank < 0 || pl->rank >= P) {
    set_error("bad rank %d of %d (1..16 ranks)", pl->rank, P);
    return VC_EINVAL;
  }
  if (P > s.visual_len) {  // executor.py:521-524
    set_error("cannot spread %d visual tokens per frame over %d devices", s.visual_len, P);
    return VC_EINVAL;
  }
  if (!gather && P > 1 && s.heads % P != 0) {  // executor.py:525-529
    set_error("head-parallel attention needs sp_size to divide %d heads, got %d", s.heads, P);
    return VC_EINVAL;
  }
  Sp& x = *o;
  x.F = s.frames; x.Lv = s.visual_len; x.Lt = s.text_len; x.D = s.dim; x.H = s.heads;
  x.dh = x.D / x.H; x.Nv = x.F * x.Lv; x.P = P; x.rank = pl->rank;
  x.Hg = gather ? x.H : x.H / P;
  x.pad = qkv_pad_layout(x.D, x.H);
  x.DP = x.pad.DP;
  x.S = (!gather && qkv_compact_ok(x.D, x.H)) ? x.DP : 0;
  x.Dg = x.Hg * (x.S ? x.S : x.dh);
  x.BW = x.S ? x.H * x.S : x.D;
  x.Lv_ld = round_up(x.Lv, 8);
  x.Lk_ld = round_up(x.Lt + x.Nv, 8);
  for (int r = 0; r <= P; ++r) x.vb[r] = (int32_t)((int64_t)r * x.Lv / P);  // contiguous_bounds
  x.s1_off[0] = 0; x.s2_off[0] = 0;
  for (int r = 0; r < P; ++r) {
    x.M[r] = x.F * (x.vb[r + 1] - x.vb[r]);
    const int64_t remote = r != x.rank;
    x.s1_off[r + 1] = x.s1_off[r] + remote * 3 * x.M[r] * x.Hg * x.DP;
    x.s2_off[r + 1] = x.s2_off[r] + remote * x.M[r] * x.Dg;
  }
  x.half1 = x.s1_off[P];
  x.half2 = x.s2_off[P];
  return VC_OK;
}

struct SpWs {
  size_t xhat, tm, qsp, ksp, vtsp, qfs, kfs, vtfs, acat, total;
};
SpWs sp_ws(const Sp& x) {
  SpWs w;
  const int64_t Mr = x.M[x.rank];
  const size_t qk = (size_t)x.Hg * x.DP * 2;
  size_t o = 0;
  w.xhat = o; o = aup(o + (size_t)(Mr + x.Lt) * x.D * 2);
  w.tm = o; o = aup(o + (size_t)Mr * 3 * x.D * 2);
  w.qsp = o; o = aup(o + (size_t)x.Nv * qk);
  w.ksp = o; o = aup(o + (size_t)x.Nv * qk);
  w.vtsp = o; o = aup(o + (size_t)x.F * x.Hg * x.DP * x.Lv_ld * 2);
  w.qfs = o; o = aup(o + (size_t)x.Nv * qk);
  w.kfs = o; o = aup(o + (size_t)(x.Lt + x.Nv) * qk);
  w.vtfs = o; o = aup(o + (size_t)x.Hg * x.DP * x.Lk_ld * 2);
  w.acat = o; o = aup(o + (size_t)Mr * 3 * x.BW * 2);
  w.total = o;
  return w;
}

struct PackedPtrs {
  const __nv_bfloat16* wqkv;
  const float* bias;
  const __nv_bfloat16* wo;    // [D][3D]
  const __nv_bfloat16* wo_s;  // [D][3*H*S] head-slot Wo (== wo when the shape has none)
};
PackedPtrs packed_ptrs(const Sp& x, const void* packed) {
  size_t wqkv, bias, wo, total, wqkv_c, bias_c, wo_s;
  packed_offsets(x.D, x.H, true, &wqkv, &bias, &wo, &total, &wqkv_c, &bias_c, &wo_s);
  const char* p = (const char*)packed;
  return PackedPtrs{(const __nv_bfloat16*)(p + wqkv), (const float*)(p + bias), (const __nv_bfloat16*)(p + wo),
                    (const __nv_bfloat16*)(p + wo_s)};
}

struct UnpackArgs {
  const __nv_bfloat16* recv;  // this branch's half of recv1: [r][which][M_r][Hg][DP]
  int32_t P, F, Lv, Lt, Hg, DP;
  int32_t branch;  // 0 spatial, 1 full sequence
  int32_t vb[17];
  int64_t off[17];  // block offsets by source rank inside the half
  int64_t groups[17];  // prefix count of 32-row groups by source rank
  __nv_bfloat16 *qsp, *ksp, *vtsp, *qfs, *kfs, *vtfs;
  int64_t Lv_ld, Lk_ld;
};

// recv1[b'][r][which][m][Hg][DP] (one branch half) -> attention layouts of this
// head group.  One warp per 32 consecutive local rows of one (source, which) block;
// lane = row. Q/K rows are copied whole (16-byte vectors); V is transposed
// (lanes write consecutive keys of one head dim: coalesced).
__global__ void __launch_bounds__(256) sp_unpack1_kernel(UnpackArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int rowlen = a.Hg * a.DP;
  for (int64_t w = gw; w < a.groups[a.P]; w += nw) {
    int r = 0;
    while (w >= a.groups[r + 1]) ++r;
    const int vc = a.vb[r + 1] - a.vb[r];
    const int64_t Mr = (int64_t)a.F * vc;
    const int64_t gpb = (Mr + 31) / 32;  // row groups per which-block
    const int64_t wl = w - a.groups[r];
    const int which = (int)(wl / gpb);
    const int bp = a.branch, blk = which;
    if (which < 2) {  // Q / K rows: the warp copies one row at a time, lanes across it (coalesced)
      const int64_t m0 = (wl - which * gpb) * 32;
      for (int rr = 0; rr < 32; ++rr) {
        const int64_t m = m0 + rr;
        if (m >= Mr) break;
        int f, l;
        sp_row_to_token(a.vb, r, m, f, l);
        const int64_t tok = (int64_t)f * a.Lv + l;
        const uint4* s4 = reinterpret_cast<const uint4*>(a.recv + a.off[r] + ((int64_t)blk * Mr + m) * rowlen);
        __nv_bfloat16* dst;
        if (bp == 0) dst = (which == 0 ? a.qsp : a.ksp) + tok * rowlen;
        else dst = which == 0 ? a.qfs + tok * rowlen : a.kfs + (a.Lt + tok) * rowlen;
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        // all of the row's loads first (up to 8 x 16 bytes per lane in flight), then the stores
        const int n = rowlen / 8;
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (lane + 32 * u < n) v[u] = s4[lane + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (lane + 32 * u < n) d4[lane + 32 * u] = v[u];
        for (int i = lane + 256; i < n; i += 32) d4[i] = s4[i];  // rows longer than 256 x 16 bytes
      }
      continue;
    }
    const int64_t m = (wl - which * gpb) * 32 + lane;
    if (m >= Mr) continue;
    int f, l;
    sp_row_to_token(a.vb, r, m, f, l);
    const __nv_bfloat16* src = a.recv + a.off[r] + ((int64_t)blk * Mr + m) * rowlen;
    const int64_t tok = (int64_t)f * a.Lv + l;  // visual token index
    if (which < 2) {
      __nv_bfloat16* dst;
      if (bp == 0) dst = (which == 0 ? a.qsp : a.ksp) + tok * rowlen;
      else dst = which == 0 ? a.qfs + tok * rowlen : a.kfs + (a.Lt + tok) * rowlen;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      for (int i = 0; i < rowlen / 8; ++i) d4[i] = s4[i];
    } else {
      __nv_bfloat16* base;
      int64_t ld, key;
      if (bp == 0) { base = a.vtsp + (int64_t)f * a.Hg * a.DP * a.Lv_ld; ld = a.Lv_ld; key = l; }
      else { base = a.vtfs; ld = a.Lk_ld; key = a.Lt + tok; }
      const int n = rowlen / 8;  // DP is a multiple of 16: n is even
      for (int i = 0; i < n; i += 2) {  // two 16-byte loads in flight before the 16 stores
        const uint4 v0 = reinterpret_cast<const uint4*>(src)[i];
        const uint4 v1 = reinterpret_cast<const uint4*>(src)[i + 1];
        const __nv_bfloat16* e0 = reinterpret_cast<const __nv_bfloat16*>(&v0);
        const __nv_bfloat16* e1 = reinterpret_cast<const __nv_bfloat16*>(&v1);
#pragma unroll
        for (int k = 0; k < 8; ++k) base[(int64_t)(i * 8 + k) * ld + key] = e0[k];  // row hl*DP+d of Vt
#pragma unroll
        for (int k = 0; k < 8; ++k) base[(int64_t)(i * 8 + 8 + k) * ld + key] = e1[k];
      }
    }
  }
}

// recv2[b'][g][m][Dg] (g over the peers) -> acat[m][b'*2BW + g*Dg + c]  (b'=0 spatial cols [0,BW), b'=1 full-seq [2BW,3BW);
// BW = D, or H*S with head slots)
// One warp per (b', g, m) row, lanes across the row: 16-byte words when Dg and
// D are multiples of 8 (every row then starts 16-byte aligned), else 4-byte.
__global__ void __launch_bounds__(256) sp_unpack2_kernel(const __nv_bfloat16* __restrict__ recv,
                                                         __nv_bfloat16* __restrict__ acat, int P, int self,
                                                         int64_t Mr, int64_t Dg, int64_t D) {  // D: branch width BW
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)P * 2 * Mr;  // P: the peers in recv2 (own group not in it)
  const bool v16 = (Dg % 8) == 0 && (D % 8) == 0;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t m = row % Mr;
    const int64_t gb = row / Mr;  // b'*P + g' (g' skips the own group)
    const int bp = (int)(gb / P), gs = (int)(gb % P), g = gs + (gs >= self);
    const __nv_bfloat16* src = recv + row * Dg;
    __nv_bfloat16* dst = acat + m * 3 * D + bp * 2 * D + (int64_t)g * Dg;
    if (v16) {
      for (int64_t i = lane; i < Dg / 8; i += 32)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {  // Dg even (dh even): 4-byte words
      for (int64_t i = lane; i < Dg / 2; i += 32)
        reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[i];
    }
  }
}

// ---- gather mode (executor.py:416-459) ----
// One rank's slot of the gather buffer (identical size on every rank, local
// row counts padded to vcmax = max_r vc_r):
//   A  spatial K   [F][vcmax][H][DP]   (local row m = f*vc_r + l)
//   B  spatial V^T [F][H][DP][vcl_ld]  (local key l)
//   C  full-seq K  [F*vcmax][H][DP]    (local row m)
//   Dv full-seq V^T [H][DP][fsl_ld]    (local key m)
struct SpgSlot {
  int64_t vcmax, vcl_ld, fsl_ld, A, B, C, Dv, total;  // offsets in bf16 elements
};
SpgSlot spg_slot(const Sp& x) {
  SpgSlot g;
  int vmax = 0;
  for (int r = 0; r < x.P; ++r) vmax = std::max(vmax, x.vb[r + 1] - x.vb[r]);
  g.vcmax = vmax;
  g.vcl_ld = round_up(g.vcmax, 8);
  g.fsl_ld = round_up(x.F * g.vcmax, 8);
  const int64_t row = x.H * x.DP;
  g.A = 0;
  g.B = g.A + x.F * g.vcmax * row;
  g.C = g.B + x.F * row * g.vcl_ld;
  g.Dv = g.C + x.F * g.vcmax * row;
  g.total = round_up(g.Dv + row * g.fsl_ld, 512);  // keep every slot 1 KB aligned
  return g;
}

struct SpgWs {
  size_t xhat, tm, qsp, qfs, ksp, vtsp, kfs, vtfs, acat, total;
};
SpgWs spg_ws(const Sp& x) {
  SpgWs w;
  const int64_t Mr = x.M[x.rank];
  const size_t qk = (size_t)x.H * x.DP * 2;
  size_t o = 0;
  w.xhat = o; o = aup(o + (size_t)(Mr + x.Lt) * x.D * 2);
  w.tm = o; o = aup(o + (size_t)Mr * 3 * x.D * 2);
  w.qsp = o; o = aup(o + (size_t)Mr * qk);                       // local queries
  w.qfs = o; o = aup(o + (size_t)Mr * qk);
  w.ksp = o; o = aup(o + (size_t)x.Nv * qk);                     // global keys / values
  w.vtsp = o; o = aup(o + (size_t)x.F * x.H * x.DP * x.Lv_ld * 2);
  w.kfs = o; o = aup(o + (size_t)(x.Lt + x.Nv) * qk);
  w.vtfs = o; o = aup(o + (size_t)x.H * x.DP * x.Lk_ld * 2);
  w.acat = o; o = aup(o + (size_t)Mr * 3 * x.D * 2);
  w.total = o;
  return w;
}

struct SpgUnpack {
  const __nv_bfloat16* gather;
  int32_t P, F, Lv, Lt, H, DP;
  int32_t vb[17];
  int64_t slot, vcl_ld, fsl_ld, offA, offB, offC, offD, Lv_ld, Lk_ld;
  __nv_bfloat16 *ksp, *vtsp, *kfs, *vtfs;
};

// K rows of every rank's slot -> global spatial K [F][Lv][H][DP] and full-seq
// K [Lt + Nv][H][DP] (text rows untouched).  One warp per (rank, branch, row):
// a row is H*DP bf16, copied as 16-byte vectors.
__global__ void __launch_bounds__(256) spg_unpack_k_kernel(SpgUnpack a) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t vec = (int64_t)a.H * a.DP / 8;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < 2LL * a.F * a.Lv; w += nw) {
    const int b = (int)(w / ((int64_t)a.F * a.Lv));   // 0 spatial, 1 full sequence
    const int64_t tok = w - (int64_t)b * a.F * a.Lv;   // global visual token f*Lv + l
    const int f = (int)(tok / a.Lv), l = (int)(tok - (int64_t)f * a.Lv);
    const int r = sp_owner(a.vb, a.P, l);
    const int64_t m = sp_token_to_row(a.vb, r, f, l);
    const uint4* src = reinterpret_cast<const uint4*>(a.gather + r * a.slot + (b == 0 ? a.offA : a.offC) +
                                                      m * a.H * a.DP);
    uint4* dst = reinterpret_cast<uint4*>(b == 0 ? a.ksp + tok * a.H * a.DP : a.kfs + (a.Lt + tok) * a.H * a.DP);
    for (int64_t i = lane; i < vec; i += 32) dst[i] = src[i];
  }
}

// V^T rows of every rank's slot -> global V^T.  Spatial: row (f, h, d) of rank
// r holds keys [0, vc_r) -> keys [vb[r], vb[r+1]) of row (f, h, d) of
// [F][H][DP][Lv_ld].  Full-seq: row (h, d) holds keys m = f*vc_r + l -> key
// Lt + f*Lv + vb[r] + l of [H][DP][Lk_ld].  One block per (rank, branch, row),
// threads over keys.
__global__ void __launch_bounds__(256) spg_unpack_vt_kernel(SpgUnpack a) {
  const int64_t hd = (int64_t)a.H * a.DP;
  const int64_t per_rank = (int64_t)a.F * hd + hd;  // spatial rows + full-seq rows
  for (int64_t job = blockIdx.x; job < a.P * per_rank; job += gridDim.x) {
    const int r = (int)(job / per_rank);
    const int64_t j = job - r * per_rank;
    const int vc = a.vb[r + 1] - a.vb[r];
    const __nv_bfloat16* base = a.gather + r * a.slot;
    if (j < (int64_t)a.F * hd) {  // spatial row j = (f*H + h)*DP + d
      const __nv_bfloat16* src = base + a.offB + j * a.vcl_ld;
      __nv_bfloat16* dst = a.vtsp + j * a.Lv_ld + a.vb[r];
      for (int l = threadIdx.x; l < vc; l += blockDim.x) dst[l] = src[l];
    } else {  // full-sequence row (h, d)
      const int64_t row = j - (int64_t)a.F * hd;
      const __nv_bfloat16* src = base + a.offD + row * a.fsl_ld;
      __nv_bfloat16* dst = a.vtfs + row * a.Lk_ld + a.Lt + a.vb[r];
      const int64_t n = (int64_t)a.F * vc;
      for (int64_t m = threadIdx.x; m < n; m += blockDim.x) {
        const int f = (int)(m / vc);
        dst[(int64_t)f * a.Lv + (m - (int64_t)f * vc)] = src[m];
      }
    }
  }
}

// Frame-wise -> spatial reshard (executor.py:252-287, spatial axis): rank d
// embeds the frames f = d, d + P, ... (round_robin_frames, executor.py:194-196);
// every peer r receives rows [vb[r], vb[r+1]) of each of them.  One warp per
// row, 16-byte copies (D % 4 == 0).
struct ReshardArgs {
  int32_t P, rank, F, Lv, D;
  int32_t vb[17];
  int64_t off[17];  // per-peer block offsets (elements) in the send / recv buffer
};
__device__ __forceinline__ int frames_of(int F, int P, int d) { return d < F ? (F - d + P - 1) / P : 0; }

__global__ void __launch_bounds__(256) reshard_pack_kernel(const float* __restrict__ local, float* __restrict__ send,
                                                           ReshardArgs a) {
  const int lane = threadIdx.x & 31;
  const int nf = frames_of(a.F, a.P, a.rank);
  const int64_t rows = (int64_t)nf * a.Lv;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rows;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int i = (int)(w / a.Lv), l = (int)(w - (int64_t)i * a.Lv);  // my i-th frame, position l
    const int r = sp_owner(a.vb, a.P, l);
    const int vc = a.vb[r + 1] - a.vb[r];
    const float4* src = reinterpret_cast<const float4*>(local + w * a.D);
    float4* dst = reinterpret_cast<float4*>(send + a.off[r] + ((int64_t)i * vc + (l - a.vb[r])) * a.D);
    for (int c = lane; c < a.D / 4; c += 32) dst[c] = src[c];
  }
}

__global__ void __launch_bounds__(256) reshard_unpack_kernel(const float* __restrict__ recv, float* __restrict__ resident,
                                                             ReshardArgs a) {
  const int lane = threadIdx.x & 31;
  const int vc = a.vb[a.rank + 1] - a.vb[a.rank];
  const int64_t rows = (int64_t)a.F * vc;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rows;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int f = (int)(w / vc), lp = (int)(w - (int64_t)f * vc);  // resident row (frame f, local position lp)
    const int s = f % a.P, i = f / a.P;                            // source rank, its i-th frame
    const float4* src = reinterpret_cast<const float4*>(recv + a.off[s] + ((int64_t)i * vc + lp) * a.D);
    float4* dst = reinterpret_cast<float4*>(resident + w * a.D);
    for (int c = lane; c < a.D / 4; c += 32) dst[c] = src[c];
  }
}

int reshard_args(const Sp& x, int which, ReshardArgs* a) {
  if (x.D % 4) { set_error("reshard needs dim %% 4 == 0"); return VC_EINVAL; }
  a->P = (int)x.P; a->rank = (int)x.rank; a->F = (int)x.F; a->Lv = (int)x.Lv; a->D = (int)x.D;
  for (int r = 0; r <= x.P; ++r) a->vb[r] = x.vb[r];
  int64_t o = 0;
  for (int r = 0; r < x.P; ++r) {
    a->off[r] = o;
    const int nf = which == 0 ? (x.rank < x.F ? (int)((x.F - x.rank + x.P - 1) / x.P) : 0)
                              : (r < x.F ? (int)((x.F - r + x.P - 1) / x.P) : 0);
    const int vc = which == 0 ? x.vb[r + 1] - x.vb[r] : x.vb[x.rank + 1] - x.vb[x.rank];
    o += (int64_t)nf * vc * x.D;
  }
  a->off[x.P] = o;
  return VC_OK;
}

}  // namespace

}  // namespace vc

using namespace vc;

extern "C" {

int vc_sp_check(const vc_sp_plan* plan) {
  Sp x;
  return sp_make(plan, &x);
}

int vc_sp_bounds(const vc_sp_plan* plan, int32_t* vbounds) {
  Sp x;
  VC_TRY(sp_make(plan, &x));
  for (int r = 0; r <= x.P; ++r) vbounds[r] = x.vb[r];
  return VC_OK;
}

size_t vc_sp_workspace_bytes(const vc_sp_plan* plan) {
  Sp x;
  if (sp_make(plan, &x) != VC_OK) return 0;
  return sp_ws(x).total;
}

int64_t vc_sp_exchange_elems(const vc_sp_plan* plan, int32_t which, int32_t peer) {
  Sp x;
  if (sp_make(plan, &x, false, which >= 4) != VC_OK || peer < 0 || peer >= x.P) return -1;
  const int64_t me = x.M[x.rank];
  if (which < 4 && peer == x.rank) return 0;  // the own block stays on the rank (sp_make)
  switch (which) {
    case 0: return 6 * me * x.Hg * x.DP;           // send1 to peer (my rows, peer's heads)
    case 1: return 6 * x.M[peer] * x.Hg * x.DP;    // recv1 from peer (peer's rows, my heads)
    case 2: return 2 * x.M[peer] * x.Dg;           // send2 to peer (peer's rows, my heads)
    case 3: return 2 * me * x.Dg;                  // recv2 from peer (my rows, peer's heads)
    // the same exchanges without the layout padding (head dim dh, not DP;
    // head-group width Hg*dh, not the head slots): the reference's payload
    // (executor.py:344-347, :395-412), for the byte accounting
    case 4: return 6 * me * x.Hg * x.dh;
    case 5: return 6 * x.M[peer] * x.Hg * x.dh;
    case 6: return 2 * x.M[peer] * x.Hg * x.dh;
    case 7: return 2 * me * x.Hg * x.dh;
  }
  return -1;
}

int64_t vc_sp_reshard_elems(const vc_sp_plan* plan, int32_t which, int32_t peer) {
  Sp x;
  if (sp_make(plan, &x, true, true) != VC_OK || peer < 0 || peer >= x.P || which < 0 || which > 1) return -1;
  ReshardArgs a;
  if (reshard_args(x, which, &a) != VC_OK) return -1;
  return a.off[peer + 1] - a.off[peer];
}

int vc_sp_reshard_pack(const vc_sp_plan* plan, const float* local_frames, float* send, void* stream) {
  Sp x;
  VC_TRY(sp_make(plan, &x, true, true));  // any P <= Lv (no head-group condition), fp32 rows
  ReshardArgs a;
  VC_TRY(reshard_args(x, 0, &a));
  const int64_t rows = (int64_t)(x.rank < x.F ? (x.F - x.rank + x.P - 1) / x.P : 0) * x.Lv;
  if (rows == 0) return VC_OK;
  const int blocks = (int)std::min<int64_t>(cdiv(rows, 8), 148 * 16);
  reshard_pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(local_frames, send, a);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

int vc_sp_reshard_unpack(const vc_sp_plan* plan, const float* recv, float* resident, void* stream) {
  Sp x;
  VC_TRY(sp_make(plan, &x, true, true));
  ReshardArgs a;
  VC_TRY(reshard_args(x, 1, &a));
  const int64_t rows = x.F * (int64_t)(x.vb[x.rank + 1] - x.vb[x.rank]);
  if (rows == 0) return VC_OK;
  const int blocks = (int)std::min<int64_t>(cdiv(rows, 8), 148 * 16);
  reshard_unpack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(recv, resident, a);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

int vc_sp_row_map(const vc_sp_plan* plan, int32_t which, int64_t* out) {
  Sp x;
  VC_TRY(sp_make(plan, &x, false, true));
  if (!out || which < 0 || which > 1) { set_error("vc_sp_row_map: which must be 0 or 1"); return VC_EINVAL; }
  if (which == 0) {  // recv rows (source rank, local row) -> visual token, as sp_unpack1 places them
    int64_t i = 0;
    for (int r = 0; r < x.P; ++r)
      for (int64_t m = 0; m < x.M[r]; ++m) {
        int f, l;
        sp_row_to_token(x.vb, r, m, f, l);
        out[i++] = (int64_t)f * x.Lv + l;
      }
  } else {  // visual token -> (owner rank, local row) as one index into the rank-ordered row list (out_row)
    int64_t first[17];
    first[0] = 0;
    for (int r = 0; r < x.P; ++r) first[r + 1] = first[r] + x.M[r];
    for (int f = 0; f < x.F; ++f)
      for (int l = 0; l < x.Lv; ++l) {
        const int r = sp_owner(x.vb, (int)x.P, l);
        out[(int64_t)f * x.Lv + l] = first[r] + sp_token_to_row(x.vb, r, f, l);
      }
  }
  return VC_OK;
}

int vc_sp_stage1(const vc_sp_plan* plan, const void* packed, const float* x_local, const float* prompt,
                 void* send1, void* ws, size_t ws_bytes, void* stream) {
  return vc_sp_stage1_part(plan, packed, x_local, prompt, send1, 2, ws, ws_bytes, stream);
}

int vc_sp_stage1_part(const vc_sp_plan* plan, const void* packed, const float* x_local, const float* prompt,
                      void* send1, int32_t part, void* ws, size_t ws_bytes, void* stream) {
  if (part < 0 || part > 2) { set_error("stage-1 part must be 0 (LN + QKV GEMM), 1 (temporal) or 2 (both)"); return VC_EINVAL; }
  Sp x;
  VC_TRY(sp_make(plan, &x));
  const SpWs w = sp_ws(x);
  if (ws_bytes < w.total) { set_error("SP workspace too small"); return VC_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  profile_begin(st);
  char* W = (char*)ws;
  typedef __nv_bfloat16 bf;
  const PackedPtrs pp = packed_ptrs(x, packed);
  const int64_t Mr = x.M[x.rank];
  const int vc = x.vb[x.rank + 1] - x.vb[x.rank];
  bf* xhat = (bf*)(W + w.xhat);
  bf* tm = (bf*)(W + w.tm);
  bf* acat = (bf*)(W + w.acat);
  if (part != 1) {
    VC_TRY(launch_ln_rows<bf>(x_local, Mr, prompt, x.Lt, (int)x.D, xhat, st));
    profile_mark(st, "sp_ln");
  }
  if (Mr > 0 && part != 1) {
    GemmTcParams g{};
    g.M = Mr; g.N = (int)x.pad.Npad; g.K = (int)x.D; g.bias = pp.bias;
    QkvScatter& s = g.qkv;
    s.pad = x.pad; s.D = x.D; s.Lv = x.Lv; s.Lt = x.Lt; s.H = (int)x.H; s.tm = tm;
    s.mode = 1; s.Hg = (int)x.Hg; s.send_rows = Mr; s.send = (bf*)send1;
    s.Lf = vc; s.tm_F = (int)x.F;  // temporal q/k/v position-major over the local positions
    s.self_g = (int)x.rank + 1; s.self_v0 = x.vb[x.rank];
    s.sp = BranchOut{(bf*)(W + w.qsp), (bf*)(W + w.ksp), (bf*)(W + w.vtsp), x.Lv_ld};
    s.fs = BranchOut{(bf*)(W + w.qfs), (bf*)(W + w.kfs), (bf*)(W + w.vtfs), x.Lk_ld};
    VC_TRY(launch_gemm_tc(xhat, x.D, pp.wqkv, x.D, g, EPI_QKV, st));
    profile_mark(st, "sp_qkv_gemm");
  }
  if (Mr > 0 && part != 0) {
    // temporal branch is rank-local: sequence = local position, tokens = frames (stride vc)
    VC_TRY(launch_temporal_bf16(tm, 3 * x.D, x.D, acat + x.BW, 3 * x.BW, (int)x.F, vc, (int)x.H, (int)x.dh, st,
                               (int)x.S, 1));
    profile_mark(st, "sp_attn_temporal");
  }
  profile_end();
  return VC_OK;
}

int vc_sp_stage2_branch(const vc_sp_plan* plan, const void* packed, const void* recv1, void* send2, int branch,
                        void* ws, size_t ws_bytes, void* stream) {
  Sp x;
  VC_TRY(sp_make(plan, &x));
  const SpWs w = sp_ws(x);
  if (ws_bytes < w.total) { set_error("SP workspace too small"); return VC_EINVAL; }
  if (branch < 0 || branch > 1) { set_error("branch must be 0 (spatial) or 1 (full sequence)"); return VC_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  profile_begin(st);
  char* W = (char*)ws;
  typedef __nv_bfloat16 bf;
  const PackedPtrs pp = packed_ptrs(x, packed);
  const int64_t Mr = x.M[x.rank];
  bf* xhat = (bf*)(W + w.xhat);
  BranchOut sp{(bf*)(W + w.qsp), (bf*)(W + w.ksp), (bf*)(W + w.vtsp), x.Lv_ld};
  BranchOut fs{(bf*)(W + w.qfs), (bf*)(W + w.kfs), (bf*)(W + w.vtfs), x.Lk_ld};
  {
    UnpackArgs a{};
    a.recv = (const bf*)recv1 + branch * x.half1;
    a.P = (int)x.P; a.F = (int)x.F; a.Lv = (int)x.Lv; a.Lt = (int)x.Lt;
    a.Hg = (int)x.Hg; a.DP = (int)x.DP; a.branch = branch;
    a.groups[0] = 0;
    for (int r = 0; r <= x.P; ++r) { a.vb[r] = x.vb[r]; a.off[r] = x.s1_off[r]; }
    for (int r = 0; r < x.P; ++r) a.groups[r + 1] = a.groups[r] + (r == x.rank ? 0 : 3 * cdiv(x.M[r], 32));
    a.qsp = sp.q; a.ksp = sp.k; a.vtsp = sp.vt; a.qfs = fs.q; a.kfs = fs.k; a.vtfs = fs.vt;
    a.Lv_ld = x.Lv_ld; a.Lk_ld = x.Lk_ld;
    const int64_t warps = a.groups[x.P];
    const int blocks = (int)std::min<int64_t>(cdiv(warps, 8), 148 * 8);
    if (blocks > 0) {  // the peers' rows (the own ones were written by stage 1)
      sp_unpack1_kernel<<<blocks, 256, 0, st>>>(a);
      VC_CHECK_LAUNCH();
      profile_mark(st, branch == 0 ? "sp_unpack1_spatial" : "sp_unpack1_fullseq");
    }
  }
  const int g = (int)x.rank;
  if (branch == 1 && x.Lt > 0) {  // text K, V of this head group from the local prompt copy
    for (int part = 0; part < 2; ++part) {
      const int64_t n0 = x.pad.fs_base() + (1 + part) * x.pad.SEG + (int64_t)g * x.Hg * x.DP;
      GemmTcParams gp{};
      gp.M = x.Lt; gp.N = (int)(x.Hg * x.DP); gp.K = (int)x.D; gp.bias = pp.bias + n0;
      QkvScatter& s = gp.qkv;
      s.pad = x.pad; s.D = x.D; s.Lv = x.Lv; s.Lt = x.Lt; s.H = (int)x.Hg; s.head_base = g * (int)x.Hg;
      s.n_base = n0; s.text_rows = 1; s.sp = sp; s.fs = fs; s.mode = 0;
      VC_TRY(launch_gemm_tc(xhat + Mr * x.D, x.D, pp.wqkv + n0 * x.D, x.D, gp, EPI_QKV, st));
    }
    profile_mark(st, "sp_text_kv_gemm");
  }
  const float scale_log2 = (float)(1.4426950408889634 / sqrt((double)x.dh));
  AttnTcParams a{};
  a.H = (int)x.Hg; a.dh = (int)x.dh; a.scale_log2 = scale_log2;
  a.out = (bf*)send2; a.ld_out = 0; a.col_off = 0; a.out_seq_rows = 0;
  a.spo.P = (int)x.P; a.spo.branch = branch; a.spo.F = (int)x.F; a.spo.Lv = (int)x.Lv; a.spo.Dg = x.Dg;
  a.head_slot = (int)x.S;
  for (int r = 0; r <= x.P; ++r) { a.spo.vb[r] = x.vb[r]; a.spo.base[r] = branch * x.half2 + x.s2_off[r]; }
  a.spo.self_r1 = (int)x.rank + 1;  // own rows: straight into acat (branch b' columns b'*2BW + g*Dg)
  a.spo.self_out = (bf*)(W + w.acat) + branch * 2 * x.BW + g * x.Dg;
  a.spo.self_ld = 3 * x.BW;
  if (branch == 0) {
    a.Lq = (int)x.Lv; a.Lk = (int)x.Lv; a.n_bias = 0; a.bias_log2 = 0.f;
    VC_TRY(launch_attn_tc(a, sp.q, sp.k, sp.vt, (int)x.F, x.Lv, x.Lv, x.Lv_ld, (int)x.DP, st));
    profile_mark(st, "sp_attn_spatial");
  } else {
    a.Lq = (int)x.Nv; a.Lk = (int)(x.Lt + x.Nv); a.n_bias = (int)x.Lt; a.bias_log2 = (float)log2((double)x.F);
    VC_TRY(launch_attn_tc(a, fs.q, fs.k, fs.vt, 1, x.Nv, x.Lt + x.Nv, x.Lk_ld, (int)x.DP, st));
    profile_mark(st, "sp_attn_fullseq");
  }
  profile_end();
  return VC_OK;
}

int vc_sp_stage2(const vc_sp_plan* plan, const void* packed, const void* recv1, void* send2, void* ws,
                 size_t ws_bytes, void* stream) {
  VC_TRY(vc_sp_stage2_branch(plan, packed, recv1, send2, 0, ws, ws_bytes, stream));
  return vc_sp_stage2_branch(plan, packed, recv1, send2, 1, ws, ws_bytes, stream);
}

int vc_sp_stage3(const vc_sp_plan* plan, const void* packed, const void* recv2, const float* x_local,
                 float* out_local, int add_residual, void* ws, size_t ws_bytes, void* stream) {
  Sp x;
  VC_TRY(sp_make(plan, &x));
  const SpWs w = sp_ws(x);
  if (ws_bytes < w.total) { set_error("SP workspace too small"); return VC_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  profile_begin(st);
  typedef __nv_bfloat16 bf;
  const PackedPtrs pp = packed_ptrs(x, packed);
  const int64_t Mr = x.M[x.rank];
  if (Mr == 0) return VC_OK;
  bf* acat = (bf*)((char*)ws + w.acat);
  if (x.P > 1) {  // the peers' head groups (the own one was written by stage 2)
    const int64_t rows = (x.P - 1) * 2 * Mr;  // one warp per row
    const int blocks = (int)std::min<int64_t>(cdiv(rows, 8), 148 * 16);
    sp_unpack2_kernel<<<blocks, 256, 0, st>>>((const bf*)recv2, acat, (int)x.P - 1, (int)x.rank, Mr, x.Dg, x.BW);
    VC_CHECK_LAUNCH();
    profile_mark(st, "sp_unpack2");
  }
  GemmTcParams g{};
  g.M = Mr; g.N = (int)x.D; g.K = (int)(3 * x.BW);
  g.out_f32 = out_local; g.ldo = x.D; g.R = add_residual ? x_local : nullptr; g.ldr = x.D;
  VC_TRY(launch_gemm_tc(acat, 3 * x.BW, x.S ? pp.wo_s : pp.wo, 3 * x.BW, g, EPI_F32, st));
  profile_mark(st, "sp_oproj_gemm");
  profile_end();
  return VC_OK;
}

// ---- gather mode ----

int vc_spg_check(const vc_sp_plan* plan) {
  Sp x;
  return sp_make(plan, &x, true);
}

size_t vc_spg_workspace_bytes(const vc_sp_plan* plan) {
  Sp x;
  if (sp_make(plan, &x, true) != VC_OK) return 0;
  return spg_ws(x).total;
}

int64_t vc_spg_slot_elems(const vc_sp_plan* plan) {
  Sp x;
  if (sp_make(plan, &x, true) != VC_OK) return -1;
  return spg_slot(x).total;
}

int vc_spg_stage1(const vc_sp_plan* plan, const void* packed, const float* x_local, const float* prompt,
                  void* gather, void* ws, size_t ws_bytes, void* stream) {
  Sp x;
  VC_TRY(sp_make(plan, &x, true));
  const SpgWs w = spg_ws(x);
  const SpgSlot gs = spg_slot(x);
  if (ws_bytes < w.total) { set_error("SP workspace too small"); return VC_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  profile_begin(st);
  char* W = (char*)ws;
  typedef __nv_bfloat16 bf;
  const PackedPtrs pp = packed_ptrs(x, packed);
  const int64_t Mr = x.M[x.rank];
  const int vc = x.vb[x.rank + 1] - x.vb[x.rank];
  bf* xhat = (bf*)(W + w.xhat);
  bf* tm = (bf*)(W + w.tm);
  bf* acat = (bf*)(W + w.acat);
  bf* slot = (bf*)gather + x.rank * gs.total;
  VC_TRY(launch_ln_rows<bf>(x_local, Mr, prompt, x.Lt, (int)x.D, xhat, st));
  profile_mark(st, "spg_ln");
  if (Mr > 0) {
    // the block's QKV GEMM over the local rows with the local geometry (Lv :=
    // vc_r, no text): Q stays here, K and V^T land in this rank's slot
    GemmTcParams g{};
    g.M = Mr; g.N = (int)x.pad.Npad; g.K = (int)x.D; g.bias = pp.bias;
    QkvScatter& s = g.qkv;
    s.pad = x.pad; s.D = x.D; s.Lv = vc; s.Lt = 0; s.H = (int)x.H; s.tm = tm;
    s.sp = BranchOut{(bf*)(W + w.qsp), slot + gs.A, slot + gs.B, gs.vcl_ld};
    s.fs = BranchOut{(bf*)(W + w.qfs), slot + gs.C, slot + gs.Dv, gs.fsl_ld};
    VC_TRY(launch_gemm_tc(xhat, x.D, pp.wqkv, x.D, g, EPI_QKV, st));
    profile_mark(st, "spg_qkv_gemm");
    VC_TRY(launch_temporal_bf16(tm, 3 * x.D, x.D, acat + x.D, 3 * x.D, (int)x.F, vc, (int)x.H, (int)x.dh, st));
    profile_mark(st, "spg_attn_temporal");
  }
  if (x.Lt > 0) {  // text K, V of all heads from the local prompt copy -> global full-seq keys [0, Lt)
    const int64_t n0 = x.pad.fs_base() + x.pad.SEG;
    GemmTcParams g{};
    g.M = x.Lt; g.N = (int)(2 * x.pad.SEG); g.K = (int)x.D; g.bias = pp.bias + n0;
    QkvScatter& s = g.qkv;
    s.pad = x.pad; s.D = x.D; s.Lv = x.Lv; s.Lt = x.Lt; s.H = (int)x.H;
    s.n_base = n0; s.text_rows = 1;
    s.sp = BranchOut{nullptr, (bf*)(W + w.ksp), (bf*)(W + w.vtsp), x.Lv_ld};
    s.fs = BranchOut{(bf*)(W + w.qfs), (bf*)(W + w.kfs), (bf*)(W + w.vtfs), x.Lk_ld};
    VC_TRY(launch_gemm_tc(xhat + Mr * x.D, x.D, pp.wqkv + n0 * x.D, x.D, g, EPI_QKV, st));
    profile_mark(st, "spg_text_kv_gemm");
  }
  profile_end();
  return VC_OK;
}

int vc_spg_stage2(const vc_sp_plan* plan, const void* packed, const void* gather, const float* x_local,
                  float* out_local, int add_residual, void* ws, size_t ws_bytes, void* stream) {
  Sp x;
  VC_TRY(sp_make(plan, &x, true));
  const SpgWs w = spg_ws(x);
  const SpgSlot gs = spg_slot(x);
  if (ws_bytes < w.total) { set_error("SP workspace too small"); return VC_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  profile_begin(st);
  char* W = (char*)ws;
  typedef __nv_bfloat16 bf;
  const PackedPtrs pp = packed_ptrs(x, packed);
  const int64_t Mr = x.M[x.rank];
  const int vc = x.vb[x.rank + 1] - x.vb[x.rank];
  {
    SpgUnpack a{};
    a.gather = (const bf*)gather; a.P = (int)x.P; a.F = (int)x.F; a.Lv = (int)x.Lv; a.Lt = (int)x.Lt;
    a.H = (int)x.H; a.DP = (int)x.DP;
    for (int r = 0; r <= x.P; ++r) a.vb[r] = x.vb[r];
    a.slot = gs.total; a.vcl_ld = gs.vcl_ld; a.fsl_ld = gs.fsl_ld;
    a.offA = gs.A; a.offB = gs.B; a.offC = gs.C; a.offD = gs.Dv; a.Lv_ld = x.Lv_ld; a.Lk_ld = x.Lk_ld;
    a.ksp = (bf*)(W + w.ksp); a.vtsp = (bf*)(W + w.vtsp); a.kfs = (bf*)(W + w.kfs); a.vtfs = (bf*)(W + w.vtfs);
    const int64_t kwarps = 2 * x.F * x.Lv;
    spg_unpack_k_kernel<<<(int)std::min<int64_t>(cdiv(kwarps, 8), 148 * 16), 256, 0, st>>>(a);
    VC_CHECK_LAUNCH();
    const int64_t vjobs = x.P * (x.F + 1) * x.H * x.DP;
    spg_unpack_vt_kernel<<<(int)std::min<int64_t>(vjobs, 148 * 32), 256, 0, st>>>(a);
    VC_CHECK_LAUNCH();
    profile_mark(st, "spg_unpack");
  }
  if (Mr == 0) return VC_OK;
  bf* acat = (bf*)(W + w.acat);
  const float scale_log2 = (float)(1.4426950408889634 / sqrt((double)x.dh));
  {  // spatial: the local rows of every frame against all Lv keys of that frame
    AttnTcParams a{};
    a.Lq = vc; a.Lk = (int)x.Lv; a.H = (int)x.H; a.dh = (int)x.dh;
    a.n_bias = 0; a.bias_log2 = 0.f; a.scale_log2 = scale_log2;
    a.out = acat; a.ld_out = 3 * x.D; a.col_off = 0; a.out_seq_rows = vc;
    VC_TRY(launch_attn_tc(a, W + w.qsp, W + w.ksp, W + w.vtsp, (int)x.F, vc, x.Lv, x.Lv_ld, (int)x.DP, st));
    profile_mark(st, "spg_attn_spatial");
  }
  {  // full sequence: the local rows against the deduplicated text + all visual keys
    AttnTcParams a{};
    a.Lq = (int)Mr; a.Lk = (int)(x.Lt + x.Nv); a.H = (int)x.H; a.dh = (int)x.dh;
    a.n_bias = (int)x.Lt; a.bias_log2 = (float)log2((double)x.F); a.scale_log2 = scale_log2;
    a.out = acat; a.ld_out = 3 * x.D; a.col_off = 2 * x.D; a.out_seq_rows = 0;
    VC_TRY(launch_attn_tc(a, W + w.qfs, W + w.kfs, W + w.vtfs, 1, Mr, x.Lt + x.Nv, x.Lk_ld, (int)x.DP, st));
    profile_mark(st, "spg_attn_fullseq");
  }
  GemmTcParams g{};
  g.M = Mr; g.N = (int)x.D; g.K = (int)(3 * x.D);
  g.out_f32 = out_local; g.ldo = x.D; g.R = add_residual ? x_local : nullptr; g.ldr = x.D;
  VC_TRY(launch_gemm_tc(acat, 3 * x.D, pp.wo, 3 * x.D, g, EPI_F32, st));
  profile_mark(st, "spg_oproj_gemm");
  profile_end();
  return VC_OK;
}

}  // extern "C"
