// Flash attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Semantics: numerics.py:87-107 per (sequence, head), non-causal, applied to
// the spatial branch (one sequence per frame, model.py:230-235) and the
// anchored full sequence (model.py:247-260) with its F identical text copies
// collapsed into ONE key segment whose logits carry + log2(F) (exact: a key
// repeated F times has F times the softmax weight; reference key/value
// permutation invariance, tests/test_numerics.py:131-140).
//
// Layouts (written by the QKV GEMM epilogue, vc_gemm_tc.cu EPI_QKV):
//   Q  [seq][Lq][H][DP]  bf16, head dim zero-padded dh -> DP (64/80/128)
//   K  [seq][Lk][H][DP]  (full sequence: keys 0..Lt-1 are the text keys)
//   Vt [seq][H][DP][Lk_ld] V transposed: the K-major B operand of P.V
// DP = 64*n64 (+16): the 64-wide part is TMA'd with 128B swizzle, a 16-wide
// tail with 32B swizzle; each tcgen05.mma (K = 16) picks its descriptor.
//
// One CTA = 128 queries of one (sequence, head); 256 threads:
//   w0 TMA producer (Q once, then K/Vt tiles of 128 keys, 2-stage ring)
//   w1 MMA issuer: S(j+1) = Q K^T issued ahead of O += P(j) V(j)
//   w2 TMEM owner (512 columns: S double buffer 2x128, O at 256)
//   w4..w7 softmax: thread = query row = TMEM lane; online softmax in the
//         log2 domain with lazy rescale (O in TMEM is rescaled only when the
//         running max grows by > 8, so P <= 2^8), P -> bf16 -> smem (SW128
//         K-major, double buffered) for the SS MMA.
#include <math.h>

#include "vc_attn_tc_common.cuh"
#include "vc_tuning.h"

namespace vc {

namespace {

using namespace attn;  // BQ, BKV, kRescaleThreshold, qk_desc, store_out (vc_attn_tc_common.cuh)
constexpr int kThreads = 256;

template <int DP>
struct Cfg {
  static constexpr int N64 = DP / 64;                  // SW128 64-wide chunks of the head dim
  static constexpr int TAIL = DP % 64;                 // 0 or 16 (SW32 chunk)
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int QK_BYTES = BQ * DP * 2;         // one Q (or K) tile
  static constexpr int V_BYTES = DP * BKV * 2;         // one Vt tile (2 chunks of 64 keys)
  static constexpr int P_BYTES = BQ * BKV * 2;         // one P tile
  static constexpr int KS = DP <= 80 ? 3 : 2;          // K and V ring depth
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + QK_BYTES;       // KS stages
  static constexpr int OFF_V = OFF_K + KS * QK_BYTES;  // KS stages
  static constexpr int OFF_P = OFF_V + KS * V_BYTES;   // 2 buffers
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;               // MMA K steps of S = Q K^T
  static_assert(SMEM <= 232448, "shared memory budget");
};

// POLY: exp pairs on the FMA-pipe polynomial (0 none; 207: degree 2 on 2
// pairs in 7, as attn_tp_kernel; 103: degree 2 on 1 pair in 3)
template <int DP, bool FIXM, int POLY = 0>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmQ16,
                   const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                   const __grid_constant__ CUtensorMap tmV, const AttnTcParams p) {
  using CF = Cfg<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [KS]  K tile landed
  uint64_t* k_empty = k_full + KS;        // [KS]  S MMA done reading it
  uint64_t* v_full = k_empty + KS;        // [KS]
  uint64_t* v_empty = v_full + KS;        // [KS]  PV MMA done reading it
  uint64_t* s_full = v_empty + KS;        // [2]   S in TMEM
  uint64_t* s_empty = s_full + 2;         // [2]   softmax has read S
  uint64_t* p_full = s_empty + 2;         // [2]   P in smem
  uint64_t* pv_done = p_full + 2;         // [2]   PV MMA complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * BQ;
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_tiles = (p.Lk + BKV - 1) / BKV;

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmQ64); ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmV);
    if (CF::TAIL) { ptx::prefetch_tmap(&tmQ16); ptx::prefetch_tmap(&tmK16); }
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_empty[i], 128);
      ptx::mbar_init(&p_full[i], 128);
      ptx::mbar_init(&pv_done[i], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;          // S buffers at columns 0 and 128
  const uint32_t tO = tmem + 256;    // O accumulator, DP columns

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (ptx::elect_one()) {
      uint8_t* sQ = smem + CF::OFF_Q;
      ptx::mbar_arrive_expect_tx(q_full, CF::QK_BYTES);
      for (int c = 0; c < CF::N64; ++c)
        ptx::tma_load_4d(sQ + c * BQ * 128, &tmQ64, q_full, c * 64, h, q0, seq);
      if (CF::TAIL) ptx::tma_load_4d(sQ + CF::N64 * BQ * 128, &tmQ16, q_full, CF::N64 * 64, h, q0, seq);
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % KS;
        const uint32_t ph = ((j / KS) & 1) ^ 1;
        const int k0 = j * BKV;
        ptx::mbar_wait(&k_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&k_full[s], CF::QK_BYTES);
        uint8_t* sK = smem + CF::OFF_K + s * CF::QK_BYTES;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d(sK + c * BKV * 128, &tmK64, &k_full[s], c * 64, h, k0, seq);
        if (CF::TAIL) ptx::tma_load_4d(sK + CF::N64 * BKV * 128, &tmK16, &k_full[s], CF::N64 * 64, h, k0, seq);
        ptx::mbar_wait(&v_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&v_full[s], CF::V_BYTES);
        uint8_t* sV = smem + CF::OFF_V + s * CF::V_BYTES;
        ptx::tma_load_4d(sV, &tmV, &v_full[s], k0, 0, h, seq);
        ptx::tma_load_4d(sV + DP * 128, &tmV, &v_full[s], k0 + 64, 0, h, seq);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BKV);
    constexpr uint32_t idO = ptx::idesc_bf16_f32(BQ, DP);
    const uint32_t aQ = ptx::smem_u32(smem + CF::OFF_Q);
    ptx::mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int s = j & 1, ks = j % KS;
      ptx::mbar_wait(&k_full[ks], (j / KS) & 1);
      ptx::mbar_wait(&s_empty[s], ((j >> 1) & 1) ^ 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::QK_BYTES);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c)
          ptx::mma_bf16_ss(tS + s * BKV, qk_desc<DP>(aQ, c), qk_desc<DP>(aK, c), idS, c > 0);
        ptx::mma_commit(&s_full[s]);
        ptx::mma_commit(&k_empty[ks]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < n_tiles; ++j) {
      if (j + 1 < n_tiles) issue_s(j + 1);
      const int s = j & 1, ks = j % KS;
      ptx::mbar_wait(&v_full[ks], (j / KS) & 1);
      ptx::mbar_wait(&p_full[s], (j >> 1) & 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aP = ptx::smem_u32(smem + CF::OFF_P + s * CF::P_BYTES);
        const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::V_BYTES);
#pragma unroll
        for (int c = 0; c < BKV / 16; ++c) {
          const uint64_t ad = ptx::smem_desc(aP + (c >> 2) * (BQ * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
          const uint64_t bd = ptx::smem_desc(aV + (c >> 2) * (DP * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
          ptx::mma_bf16_ss(tO, ad, bd, idO, (j > 0 || c > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&v_empty[ks]);
        ptx::mma_commit(&pv_done[s]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== softmax / correction / epilogue =====================
    const int qw = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row = qw * 32 + lane;                 // query row in the tile = TMEM lane
    const uint32_t lane_off = (uint32_t)(qw * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int s = j & 1;
      const int k0 = j * BKV;
      ptx::mbar_wait(&s_full[s], (j >> 1) & 1);
      ptx::fence_after_sync();
      float v[BKV];
      {
        uint32_t r[BKV];
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c)
          ptx::tmem_ld32(tS + s * BKV + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < BKV; ++i) v[i] = __uint_as_float(r[i]);
      }
      ptx::fence_before_sync();
      ptx::mbar_arrive(&s_empty[s]);
      // logits in the log2 domain: s * log2(e)/sqrt(dh) (+ log2 F on text keys).
      // Interior tiles keep raw scores and fold the scale into one FFMA below;
      // text-key and tail tiles (warp-uniform) are converted explicitly.
      float scale = p.scale_log2;
      if (k0 < p.n_bias || k0 + BKV > p.Lk) {
#pragma unroll
        for (int i = 0; i < BKV; ++i) {
          float t = v[i] * p.scale_log2;
          if (k0 + i < p.n_bias) t += p.bias_log2;
          if (k0 + i >= p.Lk) t = -INFINITY;
          v[i] = t;
        }
        scale = 1.f;
      }
      float alpha = 1.f;
      if (!FIXM || j == 0) {  // FIXM: the offset is fixed after the first tile (kFixedMaxMargin)
        float m8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m8[i] = v[i];
#pragma unroll
        for (int i = 8; i < BKV; ++i) m8[i & 7] = fmaxf(m8[i & 7], v[i]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * scale;
        if (FIXM) {
          m_used = mx + kFixedMaxMargin;
        } else if (mx > m_used + kRescaleThreshold) {
          alpha = ptx::ex2(m_used - mx);  // 0 on the first tile
          m_used = mx;
        }
      }
      // p = 2^(s*scale - m): FFMA2 (two logits per instruction) + MUFU.EX2;
      // row sum in four FADD2 partials
      const float2 sc2 = make_float2(scale, scale), nm2 = make_float2(-m_used, -m_used);
      float2 s4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) s4[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < BKV; i += 2) {
        float2 t = ptx::ffma2(make_float2(v[i], v[i + 1]), sc2, nm2);
        constexpr int PG = POLY % 100 > 0 ? POLY % 100 : 1;
        const bool off = POLY >= 200 ? (((i >> 1) % PG) == 1 || ((i >> 1) % PG) == 3)
                                     : (POLY > 0 && ((i >> 1) % PG) == PG - 1);
        if (off) {
          t = ptx::ex2_poly2_d2(t);
        } else {
          t.x = ptx::ex2(t.x);
          t.y = ptx::ex2(t.y);
        }
        v[i] = t.x;
        v[i + 1] = t.y;
        s4[(i >> 1) & 3] = ptx::fadd2(s4[(i >> 1) & 3], t);
      }
      const float2 s2 = ptx::fadd2(ptx::fadd2(s4[0], s4[1]), ptx::fadd2(s4[2], s4[3]));
      const float sum = s2.x + s2.y;
      l = l * alpha + sum;
      // PV(i) arrives on pv_done[i & 1] (its completion #(i >> 1) there). The
      // P buffer s was last read by PV(j-2); O holds P(j-1) V(j-1) only once
      // PV(j-1) completes, which matters only if O must be rescaled -- so the
      // common case lets PV(j-1) run under this tile's softmax.
      if (j >= 2) ptx::mbar_wait(&pv_done[s], ((j - 2) >> 1) & 1);
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        ptx::mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        ptx::fence_after_sync();
        {
#pragma unroll
          for (int c = 0; c < DP / 16; ++c) {
            uint32_t r[16];
            ptx::tmem_ld16(tO + lane_off + c * 16, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            ptx::tmem_st16(tO + lane_off + c * 16, r);
          }
          ptx::tmem_st_wait();
        }
      }
      // P -> bf16 -> smem, SW128 K-major: chunk of 64 keys, row pitch 128 B,
      // 16-byte unit u of row r stored at u ^ (r & 7).
      const uint32_t sP = ptx::smem_u32(smem + CF::OFF_P + s * CF::P_BYTES);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t rowp = sP + c * (BQ * 128) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float* pv = v + c * 64 + u * 8;
          ptx::sts128(rowp + ((u ^ (row & 7)) << 4), ptx::bf16x2(pv[0], pv[1]), ptx::bf16x2(pv[2], pv[3]),
                      ptx::bf16x2(pv[4], pv[5]), ptx::bf16x2(pv[6], pv[7]));
        }
      }
      ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      ptx::fence_before_sync();
      ptx::mbar_arrive(&p_full[s]);
    }
    // ---- epilogue: O / l -> bf16 -> out[row][col_off + h*dh + d], d < dh ----
    ptx::mbar_wait(&pv_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
    ptx::fence_after_sync();
    // shared epilogue: plain rows, head slots or the SP send layout (out_row)
    store_out<DP>(p, tO + lane_off, l, q0 + row, seq, h);
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 2) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int DP>
int launch_dp(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
              int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg<DP>;
  CUtensorMap mq64, mq16, mk64, mk16, mv;
  const uint64_t eb = 2;
  {
    const uint64_t dims[4] = {(uint64_t)DP, (uint64_t)p.H, (uint64_t)p.Lq, (uint64_t)nseq};
    const uint64_t str[3] = {DP * eb, (uint64_t)p.H * DP * eb, (uint64_t)q_rows_per_seq * p.H * DP * eb};
    const uint32_t box64[4] = {64, 1, BQ, 1}, box16[4] = {16, 1, BQ, 1};
    VC_TRY(make_tmap_4d_bf16(&mq64, q, dims, str, box64, CU_TENSOR_MAP_SWIZZLE_128B));
    if (CF::TAIL) VC_TRY(make_tmap_4d_bf16(&mq16, q, dims, str, box16, CU_TENSOR_MAP_SWIZZLE_32B));
    else mq16 = mq64;
  }
  {
    const uint64_t dims[4] = {(uint64_t)DP, (uint64_t)p.H, (uint64_t)p.Lk, (uint64_t)nseq};
    const uint64_t str[3] = {DP * eb, (uint64_t)p.H * DP * eb, (uint64_t)k_rows_per_seq * p.H * DP * eb};
    const uint32_t box64[4] = {64, 1, BKV, 1}, box16[4] = {16, 1, BKV, 1};
    VC_TRY(make_tmap_4d_bf16(&mk64, k, dims, str, box64, CU_TENSOR_MAP_SWIZZLE_128B));
    if (CF::TAIL) VC_TRY(make_tmap_4d_bf16(&mk16, k, dims, str, box16, CU_TENSOR_MAP_SWIZZLE_32B));
    else mk16 = mk64;
  }
  {
    const uint64_t dims[4] = {(uint64_t)p.Lk, (uint64_t)DP, (uint64_t)p.H, (uint64_t)nseq};
    const uint64_t str[3] = {(uint64_t)ld_key * eb, (uint64_t)DP * ld_key * eb, (uint64_t)p.H * DP * ld_key * eb};
    const uint32_t box[4] = {64, DP, 1, 1};
    VC_TRY(make_tmap_4d_bf16(&mv, vt, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  // fixed-offset softmax after the first key tile (vc_attn_tc_common.cuh
  // kFixedMaxMargin); VC_ATTN_FIXM=0: lazy rescale
  static const int fixm = tuning_int("VC_ATTN_FIXM", 1);
  // exp offload onto the FMA pipe (this kernel has one softmax warp per SM
  // sub-partition, 128 exponentials per row per block: MUFU-bound): degree-2
  // polynomial on 2 pairs in 5 (config 5 full sequence 3.03 ms vs 3.11 for 2
  // in 7, 3.09 for 1 in 2, 3.37 without offload; 3 rounds, tools/ab_bench.sh)
  static const int poly = tuning_int("VC_ATTN128_POLY", 205);
  auto kern = !fixm ? attn_tc_kernel<DP, false> : poly == 205 ? attn_tc_kernel<DP, true, 205>
#ifdef VC_TUNING
            : poly == 207 ? attn_tc_kernel<DP, true, 207> : poly == 102 ? attn_tc_kernel<DP, true, 102>
            : poly == 103 ? attn_tc_kernel<DP, true, 103>
#endif
            : attn_tc_kernel<DP, true, 0>;
  static bool attr[6] = {false, false, false, false, false, false};
  const int ai = !fixm ? 0 : poly == 205 ? 1 : poly == 207 ? 2 : poly == 102 ? 4 : poly == 103 ? 5 : 3;
  if (!attr[ai]) {
    VC_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr[ai] = true;
  }
  dim3 grid((unsigned)cdiv(p.Lq, BQ), (unsigned)p.H, (unsigned)nseq);
  kern<<<grid, kThreads, CF::SMEM, st>>>(mq64, mq16, mk64, mk16, mv, p);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

}  // namespace

int attn_tc_head_pad(int dh) {
  if (dh <= 64) return 64;
  if (dh <= 80) return 80;
  if (dh <= 128) return 128;
  return 0;
}

int launch_attn_tc(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                   int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, int DP,
                   cudaStream_t st) {
  if (p.Lq <= 0 || nseq <= 0) return VC_OK;
  if (p.Lk <= 0) { set_error("attention needs at least one key"); return VC_EINVAL; }
  if (nseq > 65535 || p.H > 65535) { set_error("attention grid too large"); return VC_ENOTSUP; }
  // DP <= 80 (the 2B head dim 66 -> 80, dh 64): attn_tp_kernel (P in TMEM,
  // split-row fixed-offset softmax, vc_attn_tp.cu); DP = 128: the one-tile
  // kernel above.  Variants measured slower are in git history or tuning
  // builds (profiles/r01/attn_study, profiles/r02/attn).
  // VC_ATTN_IMPL (tuning builds): 3 = the round-1 split-row kernel with half
  // of P in shared memory; default 4 = P entirely in TMEM (vc_attn_tp.cu)
  static const int impl = tuning_int("VC_ATTN_IMPL", 4);
  switch (DP) {
    case 64:
#ifdef VC_TUNING
      if (impl == 3) return launch_attn_tc3<64>(p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key, st);
#endif
      return launch_attn_tp<64>(p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key, st);
    case 80:
#ifdef VC_TUNING
      if (impl == 3) return launch_attn_tc3<80>(p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key, st);
#endif
      return launch_attn_tp<80>(p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key, st);
    case 128: return launch_dp<128>(p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key, st);
  }
  set_error("tcgen05 attention: unsupported padded head dim %d", DP);
  return VC_ENOTSUP;
}

}  // namespace vc
