// Flash attention, two query tiles per CTA ping-ponging on one tensor core
// (the FA4 schedule) for padded head dims DP <= 80 (the 2B shape: dh 66 -> 80).
//
// Same semantics and layouts as vc_attn_tc.cu (see there).  One CTA = 256
// queries (tiles A, B) of one (sequence, head); every K/V tile TMA'd into
// smem serves both query tiles.  384 threads:
//   w0 TMA producer (Q_A, Q_B once; K and V rings of 3 stages each)
//   w1 MMA issuer:  S_A(j+1) | PV_A(j) | S_B(j+1) | PV_B(j) per key tile
//   w2 TMEM owner (512 cols: S_A 0, O_A 128, S_B 256, O_B 384)
//   w4..w7  softmax of tile A, w8..w11 softmax of tile B (thread = row)
// While one tile's softmax runs (MUFU / FMA bound) the tensor core works on
// the other tile, and two softmax warps per SM sub-partition hide each
// other's latencies.
#include "vc_attn_tc_common.cuh"

namespace vc {

namespace {

using namespace attn;

constexpr int kThreads2 = 384;
// Fraction of exponentials computed by the FMA-pipe polynomial instead of
// MUFU.EX2: one pair in kPolyEvery (MUFU is the softmax limiter on B200).
#ifndef VC_POLY_EVERY
#define VC_POLY_EVERY 4
#endif
constexpr int kPolyEvery = VC_POLY_EVERY;

template <int DP>
struct Cfg2 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int QK_BYTES = BQ * DP * 2;
  static constexpr int V_BYTES = DP * BKV * 2;
  static constexpr int P_BYTES = BQ * BKV * 2;
  static constexpr int KS = 3;
  static constexpr int OFF_Q = 0;                          // 2 tiles
  static constexpr int OFF_K = OFF_Q + 2 * QK_BYTES;       // KS stages
  static constexpr int OFF_V = OFF_K + KS * QK_BYTES;      // KS stages
  static constexpr int OFF_P = OFF_V + KS * V_BYTES;       // 1 buffer per tile
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// ONES: V's first padding column (d == dh) holds 1.0 (vc_rowops.cu pack), so
// O[:, dh] accumulates the softmax row sum on the tensor core and the softmax
// warps skip the sum entirely.
template <int DP, int POLY, bool ONES>
__global__ void __launch_bounds__(kThreads2, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmQ16,
                    const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmV, const AttnTcParams p) {
  using CF = Cfg2<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;      // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]  both tiles' S MMAs done with it
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]  both tiles' PV MMAs done with it
  uint64_t* s_full = v_empty + KS;  // [2 tiles]
  uint64_t* s_empty = s_full + 2;   // [2 tiles] softmax has read S
  uint64_t* p_full = s_empty + 2;   // [2 tiles]
  uint64_t* pv_done = p_full + 2;   // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * (2 * BQ);
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
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&s_empty[t], 128);
      ptx::mbar_init(&p_full[t], 128);
      ptx::mbar_init(&pv_done[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (ptx::elect_one()) {
      ptx::mbar_arrive_expect_tx(q_full, 2 * CF::QK_BYTES);
      for (int t = 0; t < 2; ++t) {
        uint8_t* sQ = smem + CF::OFF_Q + t * CF::QK_BYTES;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d(sQ + c * BQ * 128, &tmQ64, q_full, c * 64, h, q0 + t * BQ, seq);
        if (CF::TAIL) ptx::tma_load_4d(sQ + CF::N64 * BQ * 128, &tmQ16, q_full, CF::N64 * 64, h, q0 + t * BQ, seq);
      }
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
    ptx::mbar_wait(q_full, 0);
    // S_t(j) = Q_t K(j)^T into the tile's S columns
    auto issue_s = [&](int t, int j) {
      const int ks = j % KS;
      if (j > 0) ptx::mbar_wait(&s_empty[t], (j - 1) & 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aQ = ptx::smem_u32(smem + CF::OFF_Q + t * CF::QK_BYTES);
        const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::QK_BYTES);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c)
          ptx::mma_bf16_ss(tmem + t * 256, qk_desc<DP>(aQ, c), qk_desc<DP>(aK, c), idS, c > 0);
        ptx::mma_commit(&s_full[t]);
        if (t == 1) ptx::mma_commit(&k_empty[ks]);  // covers both tiles' S MMAs
      }
      __syncwarp();
    };
    // O_t += P_t(j) V(j)
    auto issue_pv = [&](int t, int j) {
      const int ks = j % KS;
      ptx::mbar_wait(&p_full[t], j & 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aP = ptx::smem_u32(smem + CF::OFF_P + t * CF::P_BYTES);
        const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::V_BYTES);
#pragma unroll
        for (int c = 0; c < BKV / 16; ++c) {
          const uint64_t ad = ptx::smem_desc(aP + (c >> 2) * (BQ * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
          const uint64_t bd = ptx::smem_desc(aV + (c >> 2) * (DP * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
          ptx::mma_bf16_ss(tmem + t * 256 + 128, ad, bd, idO, (j > 0 || c > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&pv_done[t]);
        if (t == 1) ptx::mma_commit(&v_empty[ks]);  // covers both tiles' PV MMAs
      }
      __syncwarp();
    };
    ptx::mbar_wait(&k_full[0], 0);
    issue_s(0, 0);
    issue_s(1, 0);
    for (int j = 0; j < n_tiles; ++j) {
      const bool more = j + 1 < n_tiles;
      if (more) ptx::mbar_wait(&k_full[(j + 1) % KS], ((j + 1) / KS) & 1);
      ptx::mbar_wait(&v_full[j % KS], (j / KS) & 1);
      if (more) issue_s(0, j + 1);
      issue_pv(0, j);
      if (more) issue_s(1, j + 1);
      issue_pv(1, j);
    }
  } else if (warp >= 4) {
    // ===================== softmax (tile t), correction, epilogue =====================
    const int t = (warp - 4) >> 2;
    const int qw = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row = qw * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qw * 32) << 16;
    const uint32_t tS = tmem + t * 256 + lane_off;
    const uint32_t tO = tS + 128;
    const uint32_t sP = ptx::smem_u32(smem + CF::OFF_P + t * CF::P_BYTES);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int k0 = j * BKV;
      const bool slow = k0 < p.n_bias || k0 + BKV > p.Lk;  // warp-uniform: text keys / tail mask
      ptx::mbar_wait(&s_full[t], j & 1);
      ptx::fence_after_sync();
      // pass 1 (TMEM -> registers, 64 logits at a time): row max
      float mx = -INFINITY;
#pragma unroll
      for (int h64 = 0; h64 < 2; ++h64) {
        uint32_t r[64];
        ptx::tmem_ld32(tS + h64 * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tS + h64 * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_ld_wait();
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          float x = __uint_as_float(r[i]);
          if (slow) {
            const int key = k0 + h64 * 64 + i;
            x *= p.scale_log2;
            if (key < p.n_bias) x += p.bias_log2;
            if (key >= p.Lk) x = -INFINITY;
          }
          m4[i & 3] = fmaxf(m4[i & 3], x);
        }
        mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
      }
      if (!slow) mx *= p.scale_log2;
      float alpha = 1.f;
      if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
        alpha = ptx::ex2(m_used - mx);         // 0 on the first tile
        m_used = mx;
      }
      // single P buffer per tile: PV_t(j-1) must be done reading it (and O
      // must hold P(j-1)V(j-1) before a rescale)
      if (j > 0) {
        ptx::mbar_wait(&pv_done[t], (j - 1) & 1);
        ptx::fence_after_sync();
      }
      // pass 2: p = 2^(s*scale - m) (FFMA2 + MUFU), row sum, bf16 P -> smem
      const float sc = slow ? 1.f : p.scale_log2;
      const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m_used, -m_used);
      float2 s2 = make_float2(0.f, 0.f), s2b = make_float2(0.f, 0.f);
#pragma unroll
      for (int h64 = 0; h64 < 2; ++h64) {
        uint32_t r[64];
        ptx::tmem_ld32(tS + h64 * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tS + h64 * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_ld_wait();
        if (h64 == 1) {  // S fully consumed: the MMA warp may overwrite it
          ptx::fence_before_sync();
          ptx::mbar_arrive(&s_empty[t]);
        }
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float x0 = __uint_as_float(r[i]), x1 = __uint_as_float(r[i + 1]);
          if (slow) {
            const int key = k0 + h64 * 64 + i;
            x0 *= p.scale_log2; x1 *= p.scale_log2;
            if (key < p.n_bias) x0 += p.bias_log2;
            if (key + 1 < p.n_bias) x1 += p.bias_log2;
            if (key >= p.Lk) x0 = -INFINITY;
            if (key + 1 >= p.Lk) x1 = -INFINITY;
          }
          float2 e = ptx::ffma2(make_float2(x0, x1), sc2, nm2);
          if (POLY > 0 && ((i >> 1) % POLY) == POLY - 1) {
            e = ptx::ex2_poly2(e);  // every POLY-th pair on the FMA pipe
          } else {
            e.x = ptx::ex2(e.x);
            e.y = ptx::ex2(e.y);
          }
          if (!ONES) {
            if (i & 2) s2b = ptx::fadd2(s2b, e); else s2 = ptx::fadd2(s2, e);
          }
          pk[i >> 1] = ptx::bf16x2(e.x, e.y);
        }
        const uint32_t rowp = sP + h64 * (BQ * 128) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          ptx::sts128(rowp + ((u ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      if (!ONES) {
        s2 = ptx::fadd2(s2, s2b);
        l = l * alpha + (s2.x + s2.y);
      }
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) rescale_o<DP>(tO, alpha);
      ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
      ptx::fence_before_sync();
      ptx::mbar_arrive(&p_full[t]);
    }
    ptx::mbar_wait(&pv_done[t], (n_tiles - 1) & 1);
    ptx::fence_after_sync();
    if (ONES) {  // row sum accumulated by the tensor core in the ones column
      uint32_t r1;
      ptx::tmem_ld1(tO + p.dh, r1);
      ptx::tmem_ld_wait();
      l = __uint_as_float(r1);
    }
    store_out<DP>(p, tO, l, q0 + t * BQ + row, seq, h);
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 2) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

template <int DP>
int launch_attn_tc2(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg2<DP>;
  AttnMaps m;
  VC_TRY(make_attn_maps<DP>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key));
  static const int poly = getenv("VC_POLY_EVERY") ? atoi(getenv("VC_POLY_EVERY")) : kPolyEvery;
  // the ones column exists iff the head dim is padded (V pad column dh = 1.0)
  static const bool no_ones = getenv("VC_NO_ONES_COLUMN") != nullptr;
  const bool ones = !no_ones && p.dh < DP;
  dim3 grid((unsigned)cdiv(p.Lq, 2 * BQ), (unsigned)p.H, (unsigned)nseq);
#define VC_ATTN2_CASE(PV, ON)                                                                              \
  if (poly == PV && ones == ON) {                                                                          \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc2_kernel<DP, PV, ON>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));          \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc2_kernel<DP, PV, ON><<<grid, kThreads2, CF::SMEM, st>>>(m.q64, m.q16, m.k64, m.k16, m.v, p);   \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN2_CASE(0, false)
  VC_ATTN2_CASE(0, true)
  VC_ATTN2_CASE(4, false)
  VC_ATTN2_CASE(4, true)
  VC_ATTN2_CASE(2, true)
  VC_ATTN2_CASE(3, true)
#undef VC_ATTN2_CASE
  set_error("VC_POLY_EVERY must be 0 or 4 (2, 3 with the ones column)");
  return VC_EINVAL;
}

template int launch_attn_tc2<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc2<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
