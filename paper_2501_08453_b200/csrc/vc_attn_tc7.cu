// Flash attention on CTA PAIRS (cta_group::2), DP <= 80 (the 2B shape).
//
// vc_attn_tc3.cu's schedule (two 128-query tiles, split-row softmax, the P
// of keys 0..63 in TMEM) with every MMA issued as M = 256 across a cluster of
// two CTAs on two SMs: each CTA keeps its own 128 query rows per tile (A
// operand, its TMEM accumulators, its softmax), while the B operand — K for
// S = QK^T, V^T for O += PV — is split by N across the pair: CTA r loads and
// holds keys [64r, 64r+64) of every K block and head dims [r*DP/2, (r+1)*DP/2)
// of every V^T block.  Per SM that halves the K/V TMA fills and the tensor
// core's K/V operand reads on the shared-memory port (the port the
// ncu capture of tc3 shows ~79% busy), and halves the MMA instruction count.
//
// Pair protocol (leader = cluster rank 0 issues all MMAs):
//   q_full / k_full / v_full  leader's barriers; the leader posts expect_tx of
//                             BOTH CTAs' bytes, the peer's TMA (cta_group::2
//                             form) completes on the leader's barrier
//   k_empty / v_empty         each CTA's own, signalled by the leader's commit
//                             multicast -> each producer refills its half
//   s_full / pv_done          each CTA's own, commit multicast
//   s_empty / p_full          leader's, one arrival per softmax warp of both
//                             CTAs (the peer's remote, release.cluster)
// 18 warps per CTA: w0 TMA, w1 MMA issuer (leader) + TMEM owner, w2..w17
// softmax (tile t = sw>>3, key half = (sw>>2)&1, w%4 = TMEM lane quarter).
#include "vc_attn_tc_common.cuh"

namespace vc {

namespace {

using namespace attn;

constexpr int kWarps7 = 18;
constexpr int kThreads7 = kWarps7 * 32;
constexpr int kPolyEvery7 = 4;

template <int DP>
struct Cfg7 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int DPH = DP / 2;                  // V^T rows (head dims) per CTA
  static constexpr int QK_BYTES = BQ * DP * 2;        // one Q tile
  static constexpr int KH_BYTES = 64 * DP * 2;        // half a K block (64 keys)
  static constexpr int VH_BYTES = DPH * BKV * 2;      // half a V^T block (DP/2 dims x 128 keys)
  static constexpr int PH_BYTES = BQ * 64 * 2;        // P of keys 64..127 (SW128 [128][64])
  static constexpr int KS = 6;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QK_BYTES;
  static constexpr int OFF_V = OFF_K + KS * KH_BYTES;
  static constexpr int OFF_P = OFF_V + KS * VH_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * PH_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int NC = DP / 16;
  static constexpr int NC0 = (NC + 1) / 2;
  static constexpr int PCOL = 128 + DP;               // P of keys 0..63: 32 columns
  static constexpr int XCOL = PCOL + 32 + 8;          // row-max exchange cells
  static_assert(XCOL + 4 <= 256, "per-tile TMEM columns");
  static_assert(DPH % 8 == 0, "V half must keep 8-row swizzle atoms");
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int DP, int POLY, bool ONES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads7, 1)
    attn_tc7_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmQ16,
                    const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmVh, const AttnTcParams p) {
  using CF = Cfg7<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* q_full = bars + 0;      // leader's
  uint64_t* k_full = bars + 1;      // [KS] leader's
  uint64_t* k_empty = k_full + KS;  // [KS] each CTA's
  uint64_t* v_full = k_empty + KS;  // [KS] leader's
  uint64_t* v_empty = v_full + KS;  // [KS] each CTA's
  uint64_t* s_full = v_empty + KS;  // [2] each CTA's
  uint64_t* s_empty = s_full + 2;   // [2] leader's (16 warp arrivals)
  uint64_t* p_full = s_empty + 2;   // [2] leader's (16 warp arrivals)
  uint64_t* pv_done = p_full + 2;   // [2] each CTA's
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_tiles = (p.Lk + BKV - 1) / BKV;

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmQ64); ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmVh);
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
      ptx::mbar_init(&s_empty[t], 16);
      ptx::mbar_init(&p_full[t], 16);
      ptx::mbar_init(&pv_done[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc_2sm(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::cluster_sync();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (this CTA's halves) =====================
    if (ptx::elect_one()) {
      if (leader) ptx::mbar_arrive_expect_tx(q_full, 2 * 2 * CF::QK_BYTES);
      for (int t = 0; t < 2; ++t) {
        uint8_t* sQ = smem + CF::OFF_Q + t * CF::QK_BYTES;
        const int qrow = pair * 4 * BQ + t * 2 * BQ + (int)rank * BQ;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d_2sm(sQ + c * BQ * 128, &tmQ64, q_full, c * 64, h, qrow, seq);
        if (CF::TAIL) ptx::tma_load_4d_2sm(sQ + CF::N64 * BQ * 128, &tmQ16, q_full, CF::N64 * 64, h, qrow, seq);
      }
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % KS;
        const uint32_t ph = ((j / KS) & 1) ^ 1;
        const int k0 = j * BKV;
        ptx::mbar_wait(&k_empty[s], ph);
        if (leader) ptx::mbar_arrive_expect_tx(&k_full[s], 2 * CF::KH_BYTES);
        uint8_t* sK = smem + CF::OFF_K + s * CF::KH_BYTES;
        const int kr = k0 + (int)rank * 64;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d_2sm(sK + c * 64 * 128, &tmK64, &k_full[s], c * 64, h, kr, seq);
        if (CF::TAIL) ptx::tma_load_4d_2sm(sK + CF::N64 * 64 * 128, &tmK16, &k_full[s], CF::N64 * 64, h, kr, seq);
        ptx::mbar_wait(&v_empty[s], ph);
        if (leader) ptx::mbar_arrive_expect_tx(&v_full[s], 2 * CF::VH_BYTES);
        uint8_t* sV = smem + CF::OFF_V + s * CF::VH_BYTES;
        ptx::tma_load_4d_2sm(sV, &tmVh, &v_full[s], k0, (int)rank * CF::DPH, h, seq);
        ptx::tma_load_4d_2sm(sV + CF::DPH * 128, &tmVh, &v_full[s], k0 + 64, (int)rank * CF::DPH, h, seq);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader) =====================
    if (leader) {
      constexpr uint32_t idS = ptx::idesc_bf16_f32(2 * BQ, BKV);
      constexpr uint32_t idO = ptx::idesc_bf16_f32(2 * BQ, DP);
      ptx::mbar_wait(q_full, 0);
      auto issue_s = [&](int t, int j) {
        const int ks = j % KS;
        if (j > 0) ptx::mbar_wait_cluster(&s_empty[t], (j - 1) & 1);
        ptx::fence_after_sync();
        if (ptx::elect_one()) {
          const uint32_t aQ = ptx::smem_u32(smem + CF::OFF_Q + t * CF::QK_BYTES);
          const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::KH_BYTES);
#pragma unroll
          for (int c = 0; c < CF::KSTEPS; ++c)
            ptx::mma_bf16_ss_2sm(tmem + t * 256, qk_desc<DP>(aQ, c), qk_desc<DP, 64>(aK, c), idS, c > 0);
          ptx::mma_commit_2sm_mc(&s_full[t], 0x3);
          if (t == 1) ptx::mma_commit_2sm_mc(&k_empty[ks], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {
        const int ks = j % KS;
        ptx::mbar_wait_cluster(&p_full[t], j & 1);
        ptx::fence_after_sync();
        if (ptx::elect_one()) {
          const uint32_t aP = ptx::smem_u32(smem + CF::OFF_P + t * CF::PH_BYTES);
          const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::VH_BYTES);
#pragma unroll
          for (int c = 0; c < BKV / 16; ++c) {
            const uint64_t bd =
                ptx::smem_desc(aV + (c >> 2) * (CF::DPH * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
            const uint32_t acc = (j > 0 || c > 0) ? 1u : 0u;
            if (c < 4)
              ptx::mma_bf16_ts_2sm(tmem + t * 256 + 128, tmem + t * 256 + CF::PCOL + 8 * c, bd, idO, acc);
            else
              ptx::mma_bf16_ss_2sm(tmem + t * 256 + 128,
                                   ptx::smem_desc(aP + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128), bd, idO, acc);
          }
          ptx::mma_commit_2sm_mc(&pv_done[t], 0x3);
          if (t == 1) ptx::mma_commit_2sm_mc(&v_empty[ks], 0x3);
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
        if (more) issue_s(1, j + 1);
        issue_pv(0, j);
        issue_pv(1, j);
      }
    }
  } else {
    // ===================== softmax (tile t, key half), correction, epilogue =====================
    const int sw = warp - 2;
    const int t = sw >> 3;
    const int half = (sw >> 2) & 1;
    const int quarter = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + t * 256 + lane_off + half * 64;
    const uint32_t tO = tmem + t * 256 + 128 + lane_off;
    const uint32_t tX = tmem + t * 256 + CF::XCOL + lane_off;
    const uint32_t bar_id = 1 + t * 4 + quarter;
    const uint32_t rowp = ptx::smem_u32(smem + CF::OFF_P + t * CF::PH_BYTES) + row * 128;
    const uint32_t s_empty_l = ptx::mapa_shared(ptx::smem_u32(&s_empty[t]), 0);
    const uint32_t p_full_l = ptx::mapa_shared(ptx::smem_u32(&p_full[t]), 0);
    const int qi = pair * 4 * BQ + t * 2 * BQ + (int)rank * BQ + row;
    // one arrival per warp on the leader's barrier (remote from the peer)
    // (release.cluster on the peer's arrivals: 5.3 ms; plain arrivals: 4.0 ms
    // but without a formal ordering guarantee for the peer's P stores)
    static const bool kRel = true;
    auto warp_arrive = [&](uint64_t* local_bar, uint32_t leader_addr) {
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(local_bar);
        else if (kRel) ptx::mbar_arrive_cluster_release(leader_addr);
        else ptx::mbar_arrive_cluster(leader_addr);
      }
    };
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int kt = j * BKV;
      const int k0 = kt + half * 64;
      const bool slow = kt < p.n_bias || kt + BKV > p.Lk;  // tile-uniform: text keys / tail mask
      ptx::mbar_wait(&s_full[t], j & 1);
      ptx::fence_after_sync();
      uint32_t r[64];
      ptx::tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(r));
      ptx::tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
      ptx::tmem_ld_wait();
      ptx::fence_before_sync();
      warp_arrive(&s_empty[t], s_empty_l);  // S lives in registers now
      if (slow) {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          float x = __uint_as_float(r[i]) * p.scale_log2;
          if (k0 + i < p.n_bias) x += p.bias_log2;
          if (k0 + i >= p.Lk) x = -INFINITY;
          r[i] = __float_as_uint(x);
        }
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 64; ++i) m4[i & 3] = fmaxf(m4[i & 3], __uint_as_float(r[i]));
      float pm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      if (!slow) pm *= p.scale_log2;
      const uint32_t xc = tX + 2 * (j & 1);
      ptx::tmem_st1(xc + half, __float_as_uint(pm));
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::named_bar_sync(bar_id, 64);
      ptx::fence_after_sync();
      uint32_t o;
      ptx::tmem_ld1(xc + (half ^ 1), o);
      ptx::tmem_ld_wait();
      const float mx = fmaxf(pm, __uint_as_float(o));
      float alpha = 1.f;
      if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
        alpha = ptx::ex2(m_used - mx);
        m_used = mx;
      }
      if (j > 0) {  // single P buffer per tile: PV_t(j-1) must be done with it
        ptx::mbar_wait(&pv_done[t], (j - 1) & 1);
        ptx::fence_after_sync();
      }
      const float sc = slow ? 1.f : p.scale_log2;
      const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m_used, -m_used);
      float2 s2 = make_float2(0.f, 0.f), s2b = make_float2(0.f, 0.f);
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        float2 e = ptx::ffma2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sc2, nm2);
        if (POLY > 0 && ((i >> 1) % (POLY > 0 ? POLY : 1)) == POLY - 1) {
          e = ptx::ex2_poly2(e);
        } else {
          e.x = ptx::ex2(e.x);
          e.y = ptx::ex2(e.y);
        }
        if (!ONES) {
          if (i & 2) s2b = ptx::fadd2(s2b, e); else s2 = ptx::fadd2(s2, e);
        }
        pk[i >> 1] = ptx::bf16x2(e.x, e.y);
      }
      if (half == 0) {
        ptx::tmem_st32(tmem + t * 256 + lane_off + CF::PCOL, pk);  // keys [0, 64) -> TMEM
        ptx::tmem_st_wait();
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          ptx::sts128(rowp + ((u ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      if (!ONES) {
        s2 = ptx::fadd2(s2, s2b);
        l = l * alpha + (s2.x + s2.y);
      }
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        if (half == 0) rescale_o<DP, 0, CF::NC0>(tO, alpha);
        else rescale_o<DP, CF::NC0, CF::NC>(tO, alpha);
      }
      ptx::fence_proxy_async_smem();
      ptx::fence_before_sync();
      warp_arrive(&p_full[t], p_full_l);
    }
    ptx::mbar_wait(&pv_done[t], (n_tiles - 1) & 1);
    ptx::fence_after_sync();
    if (ONES) {
      uint32_t r1;
      ptx::tmem_ld1(tO + p.dh, r1);
      ptx::tmem_ld_wait();
      l = __uint_as_float(r1);
    } else {
      ptx::tmem_st1(tX + 4 + half, __float_as_uint(l));
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::named_bar_sync(bar_id, 64);
      ptx::fence_after_sync();
      uint32_t other;
      ptx::tmem_ld1(tX + 4 + (half ^ 1), other);
      ptx::tmem_ld_wait();
      l += __uint_as_float(other);
    }
    if (half == 0) store_out<DP, 0, CF::NC0>(p, tO, l, qi, seq, h);
    else store_out<DP, CF::NC0, CF::NC>(p, tO, l, qi, seq, h);
  }
  ptx::fence_before_sync();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc_2sm(tmem, 512);
  }
}

}  // namespace

template <int DP>
int launch_attn_tc7(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg7<DP>;
  AttnMaps m;
  VC_TRY((make_attn_maps<DP, 64>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key)));
  CUtensorMap vh;  // V^T half box: 64 keys x DP/2 head dims
  {
    const uint64_t eb = 2;
    const uint64_t dims[4] = {(uint64_t)p.Lk, (uint64_t)DP, (uint64_t)p.H, (uint64_t)nseq};
    const uint64_t str[3] = {(uint64_t)ld_key * eb, (uint64_t)DP * ld_key * eb, (uint64_t)p.H * DP * ld_key * eb};
    const uint32_t box[4] = {64, (uint32_t)CF::DPH, 1, 1};
    VC_TRY(make_tmap_4d_bf16(&vh, vt, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  static const bool no_ones = getenv("VC_NO_ONES_COLUMN") != nullptr;
  const bool ones = !no_ones && p.dh < DP;
  dim3 grid((unsigned)(2 * cdiv(p.Lq, 4 * BQ)), (unsigned)p.H, (unsigned)nseq);
#define VC_ATTN7_CASE(ON)                                                                                  \
  if (ones == ON) {                                                                                        \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc7_kernel<DP, kPolyEvery7, ON>,                             \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));          \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc7_kernel<DP, kPolyEvery7, ON><<<grid, kThreads7, CF::SMEM, st>>>(m.q64, m.q16, m.k64, m.k16,    \
                                                                            vh, p);                        \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN7_CASE(true)
  VC_ATTN7_CASE(false)
#undef VC_ATTN7_CASE
  return VC_EINVAL;
}

template int launch_attn_tc7<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc7<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
