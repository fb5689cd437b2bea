// Flash attention with P entirely in TMEM ("tp"): two query tiles per CTA,
// split-row softmax, key blocks of BK = 112 (DP 80) / 128 (DP 64).
//
// Same semantics and layouts as vc_attn_tc3.cu (numerics.py:87-107 per
// (sequence, head); the full-sequence text keys deduplicated with + log2 F;
// the ones column of V^T accumulating the row sum).  What changes is where P
// lives.  In tc3 half of every P tile went through shared memory, and the
// single P buffer made the exponentials of block j+1 wait for P.V of block j
// (profiles/r01/attn_study: MUFU 60% busy, tensor pipe 49%, the period =
// exp phase + P.V + handshakes).  Here, per 128-row tile, TMEM holds
//     S [0, BK)   fp32 logits of the current key block
//     P [BK, BK + BK/2)   bf16x2 probabilities (the A operand of a "ts" P.V)
//     O [BK + BK/2, + DP) fp32 output accumulator (+ ones column)
// which fits the tile's 256 columns because BK = 112: 112 + 56 + 80 = 248
// (BK = 128 would need 272).  Consequences:
//   * no P traffic on the shared-memory port and no generic->async proxy
//     fence per block (tc3: P stores + P operand reads were ~40% of the
//     port's wavefronts);
//   * the softmax loads S(j+1), takes its max and exponentiates while
//     P.V(j) still runs, and waits for P.V(j) only before overwriting P --
//     in steady state P.V(j) finished long before (it is issued at the end
//     of block j's exponentials), so the MUFU work of consecutive blocks is
//     back to back.
// The row max of the two warps sharing a row meets in shared memory.
// 19 warps: w0 TMA, w1 / w2 MMA issuers of tile 0 / 1 (w1 owns TMEM),
// w3..w18 softmax (w = 3 + 8*tile + 4*half + i; w % 4 is the TMEM lane
// quarter).
#include "vc_attn_tc_common.cuh"
#include "vc_tuning.h"

namespace vc {

namespace {

using namespace attn;

#ifdef VC_ATTN_TRACE
// clock64 phase stamps of one CTA (tools/attn_trace.cu): role 0 = MMA issuer,
// 1 + sw = softmax warp sw (lane 0); j = key block (255: prologue/epilogue)
__device__ unsigned long long g_attn_tracep[18][256][8];
#define VC_TRP(cond, role, j, k)                                             \
  do {                                                                       \
    if ((cond) && (j) < 256) g_attn_tracep[role][j][k] = clock64();         \
  } while (0)
// per-CTA timeline: clock64 at entry, first S seen, last P.V done, output
// stored (after the final barrier), then %smid (tools/attn_trace.cu: per-SM gaps)
__device__ unsigned long long g_attn_cta[16384][5];
#define VC_CTA(slot)                                                                                \
  do {                                                                                              \
    const unsigned b_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);          \
    if (b_ < 16384) g_attn_cta[b_][slot] = clock64();                                              \
    if ((slot) == 0 && b_ < 16384) {                                                                \
      unsigned sm_;                                                                                 \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                              \
      g_attn_cta[b_][4] = sm_;                                                                      \
    }                                                                                               \
  } while (0)
#else
#define VC_CTA(slot) \
  do {               \
  } while (0)
#define VC_TRP(cond, role, j, k) \
  do {                           \
  } while (0)
#endif

#ifdef VC_TP_SM_SPIN
#define VC_SM_WAIT ptx::mbar_wait
#else
#define VC_SM_WAIT ptx::mbar_wait_sleep
#endif


// NARROW (DP 80, dh <= 71): 120-key blocks with O in 72 columns (dh + the
// ones column): S 120 + P 64 + O 72 = 256. P.V runs over 128 keys (P zero for
// keys 120..127) with N = 72; M = 128 MMAs with N % 16 == 8 are exact
// (tools/mma_mn_test.cu case 5). 1350 keys take 12 blocks instead of 13.
// FR (full row): one softmax thread per query row (4 warps per tile, 12
// warps: w0 TMA, w1 / w2 MMA issuers, w3 idle, w4..w11 softmax) instead of
// two warps per row meeting in shared memory for the row max.
// NT: query tiles per CTA. NT = 1 (short sequences: the spatial branch):
// 256 TMEM columns and a 2-deep K / V ring, so two CTAs share an SM and one's
// prologue / epilogue runs under the other's main loop.
// NARROW 2 (DP 80, dh <= 71): 112-key blocks with O in 72 columns (P.V N = 72).
template <int DP, int NARROW = 0, bool FR = false, int NT = 2>
struct CfgTp {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static_assert(DP <= 80, "S + P + O must fit 256 TMEM columns per tile");
  static_assert(!NARROW || DP == 80, "the narrow layout is the DP 80 one");
  static constexpr int BK = NARROW == 1 ? 120 : DP == 64 ? 128 : 112;  // keys per block
  static constexpr int HK = FR ? BK : BK / 2;                     // keys per softmax thread
  static constexpr int WARPS = FR ? 4 + 4 * NT : 3 + 8 * NT;
  static constexpr int TMEM_COLS = 256 * NT;
  static constexpr int SM0 = FR ? 4 : 3;                          // first softmax warp
  static constexpr int SM_ARRIVALS = FR ? 128 : 256;              // softmax threads per tile
  static constexpr int PKEYS = NARROW == 1 ? 128 : BK;            // the P.V K extent
  static constexpr int ON = NARROW ? 72 : DP;                     // O columns
  static constexpr int SCOL = 0, PCOL = BK, OCOL = BK + PKEYS / 2;
  static_assert(OCOL + ON <= 256, "per-tile TMEM columns");
  static constexpr int Q_BYTES = BQ * DP * 2;
  static constexpr int K_BYTES = BK * DP * 2;
  static constexpr int K_STAGE = (K_BYTES + 1023) / 1024 * 1024;  // SW128 tiles start 1024-aligned
  static constexpr int V_BYTES = DP * 128 * 2;  // two 64-key TMA boxes (keys past BK unused)
  static constexpr int KS = NT == 1 ? 2 : 3;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NT * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KS * K_STAGE;
  static constexpr int OFF_X = OFF_V + KS * V_BYTES;       // row-max exchange [2][2 tiles][2 halves][128]
  static constexpr int OFF_BAR = OFF_X + 2 * 2 * 2 * BQ * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int NC = (ON + 15) / 16;
  static constexpr int NC0 = (NC + 1) / 2;
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int DP, int POLY, bool ONES, int NARROW, bool FR = false, int NT = 2, bool FIXM = false>
__global__ void __launch_bounds__(CfgTp<DP, NARROW, FR, NT>::WARPS * 32, NT == 1 ? 2 : 1)
    attn_tp_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmQ16,
                   const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                   const __grid_constant__ CUtensorMap tmV, const AttnTcParams p) {
  using CF = CfgTp<DP, NARROW, FR, NT>;
  constexpr int KS = CF::KS, BK = CF::BK, HK = CF::HK;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;      // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]
  uint64_t* s_full = v_empty + KS;  // [2 tiles]
  uint64_t* s_empty = s_full + 2;   // [2 tiles] S read into registers by both halves
  uint64_t* p_full = s_empty + 2;   // [2 tiles] P written to TMEM
  uint64_t* pv_done = p_full + 2;   // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * (NT * BQ);
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_tiles = (p.Lk + BK - 1) / BK;
  const int ntile = NT == 1 ? 1 : q0 + BQ < p.Lq ? 2 : 1;  // the last CTA of a sequence may hold one tile
  [[maybe_unused]] const bool tr = blockIdx.x == min(20u, gridDim.x - 1) && blockIdx.y == 3 && blockIdx.z == 0;
  if (threadIdx.x == 0) VC_CTA(0);

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmQ64); ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmV);
    if (CF::TAIL) { ptx::prefetch_tmap(&tmQ16); ptx::prefetch_tmap(&tmK16); }
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], ntile);  // one commit per tile issuer
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], ntile);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&s_empty[t], CF::SM_ARRIVALS);
      ptx::mbar_init(&p_full[t], CF::SM_ARRIVALS);
      ptx::mbar_init(&pv_done[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, CF::TMEM_COLS);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (ptx::elect_one()) {
      ptx::mbar_arrive_expect_tx(q_full, ntile * CF::Q_BYTES);
      for (int t = 0; t < ntile; ++t) {
        uint8_t* sQ = smem + CF::OFF_Q + t * CF::Q_BYTES;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d(sQ + c * BQ * 128, &tmQ64, q_full, c * 64, h, q0 + t * BQ, seq);
        if (CF::TAIL) ptx::tma_load_4d(sQ + CF::N64 * BQ * 128, &tmQ16, q_full, CF::N64 * 64, h, q0 + t * BQ, seq);
      }
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % KS;
        const uint32_t ph = ((j / KS) & 1) ^ 1;
        const int k0 = j * BK;
        ptx::mbar_wait_sleep(&k_empty[s], ph);
        VC_TRP(tr, 1, j, 5);  // producer: K(j) issued
        ptx::mbar_arrive_expect_tx(&k_full[s], CF::K_BYTES);
        uint8_t* sK = smem + CF::OFF_K + s * CF::K_STAGE;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d(sK + c * BK * 128, &tmK64, &k_full[s], c * 64, h, k0, seq);
        if (CF::TAIL) ptx::tma_load_4d(sK + CF::N64 * BK * 128, &tmK16, &k_full[s], CF::N64 * 64, h, k0, seq);
        ptx::mbar_wait_sleep(&v_empty[s], ph);
        VC_TRP(tr, 1, j, 6);  // producer: V(j) issued
        ptx::mbar_arrive_expect_tx(&v_full[s], CF::V_BYTES);
        uint8_t* sV = smem + CF::OFF_V + s * CF::V_BYTES;
        ptx::tma_load_4d(sV, &tmV, &v_full[s], k0, 0, h, seq);
        ptx::tma_load_4d(sV + DP * 128, &tmV, &v_full[s], k0 + 64, 0, h, seq);
      }
    }
  } else if (warp <= 2) {
    // ===================== MMA issuers: warp 1 -> tile 0, warp 2 -> tile 1 =====================
    // One issuer per query tile, so a tile's S(j+1) goes out the moment its
    // softmax has read S(j) (s_empty) and its P.V(j) the moment P(j) is in
    // TMEM, whatever the other tile is doing (a single in-order issuer tied
    // each tile's next S to the other tile's P: the softmax waited ~500 clk
    // per block for its logits, clock64 trace).  K / V stages are released
    // when both tiles' MMAs have read them (k_empty / v_empty count ntile).
    // Warp-uniform control flow, one elected lane issues; descriptors are
    // bases + constant offsets in the start-address field (16-byte units).
    const int t = warp - 1;
    if (t < ntile) {
      constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BK);
      constexpr uint32_t idO = ptx::idesc_bf16_f32(BQ, CF::ON);
      const uint32_t sQ = ptx::smem_u32(smem + CF::OFF_Q + t * CF::Q_BYTES), sK = ptx::smem_u32(smem + CF::OFF_K),
                     sV = ptx::smem_u32(smem + CF::OFF_V);
      const uint64_t dQ = ptx::smem_desc(sQ, 0, 1024, ptx::kLayoutSW128);
      const uint64_t dQt = ptx::smem_desc(sQ + CF::N64 * BQ * 128, 0, 256, ptx::kLayoutSW32);
      const uint64_t dK = ptx::smem_desc(sK, 0, 1024, ptx::kLayoutSW128);
      const uint64_t dKt = ptx::smem_desc(sK + CF::N64 * BK * 128, 0, 256, ptx::kLayoutSW32);
      const uint64_t dV = ptx::smem_desc(sV, 0, 1024, ptx::kLayoutSW128);
      const uint32_t tSd = tmem + t * 256 + CF::SCOL, tOd = tmem + t * 256 + CF::OCOL, tPa = tmem + t * 256 + CF::PCOL;
      auto mma_s = [&](int ks) {  // S_t = Q_t K(ks)^T
        const uint64_t ko = (uint64_t)((ks * CF::K_STAGE) >> 4);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c) {
          const bool tail = c >= 4 * CF::N64;
          const uint64_t a = tail ? dQt : dQ + (uint64_t)(((c >> 2) * BQ * 128 + (c & 3) * 32) >> 4);
          const uint64_t b = tail ? dKt + ko : dK + ko + (uint64_t)(((c >> 2) * BK * 128 + (c & 3) * 32) >> 4);
          ptx::mma_bf16_ss(tSd, a, b, idS, c > 0);
        }
        ptx::mma_commit(&s_full[t]);
        ptx::mma_commit(&k_empty[ks]);
      };
      auto mma_pv = [&](int ks, int j) {  // O_t += P_t V(ks)
        const uint64_t vo = (uint64_t)((ks * CF::V_BYTES) >> 4);
#pragma unroll
        for (int c = 0; c < CF::PKEYS / 16; ++c)
          ptx::mma_bf16_ts(tOd, tPa + 8 * c, dV + vo + (uint64_t)(((c >> 2) * DP * 128 + (c & 3) * 32) >> 4), idO,
                           (j > 0 || c > 0) ? 1u : 0u);
        ptx::mma_commit(&pv_done[t]);
        ptx::mma_commit(&v_empty[ks]);
      };
      ptx::mbar_wait_sleep(q_full, 0);
      ptx::mbar_wait_sleep(&k_full[0], 0);
      ptx::fence_after_sync();
      if (ptx::elect_one()) mma_s(0);
      __syncwarp();
      for (int j = 0; j < n_tiles; ++j) {
        const int ks = j % KS;
        VC_TRP(tr && (threadIdx.x & 31) == 0, t, j, 0);
        if (j + 1 < n_tiles) {  // S(j+1) as soon as the softmax holds S(j) in registers
          const int ks1 = (j + 1) % KS;
          ptx::mbar_wait_sleep(&k_full[ks1], ((j + 1) / KS) & 1);
          VC_TRP(tr && (threadIdx.x & 31) == 0, t, j, 3);  // K(j+1) landed
          ptx::mbar_wait_sleep(&s_empty[t], j & 1);
          ptx::fence_after_sync();
          if (ptx::elect_one()) mma_s(ks1);
          __syncwarp();
        }
        VC_TRP(tr && (threadIdx.x & 31) == 0, t, j, 1);
        ptx::mbar_wait_sleep(&v_full[ks], (j / KS) & 1);
        ptx::mbar_wait_sleep(&p_full[t], j & 1);
        ptx::fence_after_sync();
        if (ptx::elect_one()) mma_pv(ks, j);
        __syncwarp();
        VC_TRP(tr && (threadIdx.x & 31) == 0, t, j, 2);
      }
    }
  } else if (warp >= CF::SM0) {
    // ===================== softmax (tile t, key half), correction, epilogue =====================
    const int sw = warp - CF::SM0;
    const int t = FR ? sw >> 2 : sw >> 3;
    const int half = FR ? 0 : (sw >> 2) & 1;
    const int quarter = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + t * 256 + lane_off + CF::SCOL + half * HK;
    const uint32_t tP = tmem + t * 256 + lane_off + CF::PCOL + half * (HK / 2);
    const uint32_t tO = tmem + t * 256 + lane_off + CF::OCOL;
    float* xs = reinterpret_cast<float*>(smem + CF::OFF_X);
    const uint32_t bar_id = 1 + t * 4 + quarter;
    const bool trs = tr && lane == 0;
    if (t < ntile) {
      if constexpr (CF::PKEYS > BK) {  // P of keys BK..PKEYS-1 stays zero (written once)
        if (half == (FR ? 0 : 1)) {
          const uint32_t z[(CF::PKEYS - BK) / 2] = {};
          ptx::tmem_st_cols<0, (CF::PKEYS - BK) / 2>(tmem + t * 256 + lane_off + CF::PCOL + BK / 2, z);
          ptx::tmem_st_wait();
        }
      }
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int kt = j * BK;
        const int k0 = kt + half * HK;
        const bool slow = kt < p.n_bias || kt + BK > p.Lk;  // tile-uniform: text keys / tail mask
        VC_SM_WAIT(&s_full[t], j & 1);
        ptx::fence_after_sync();
        VC_TRP(trs, 2 + sw, j, 0);
        if (j == 0 && sw == 0 && lane == 0) VC_CTA(1);
        uint32_t r[HK];
        // 32 / 16 / 8-column pieces (half 1 starts at column 56: the loads
        // need no 32-column alignment; 7 x8 loads measured 2% slower)
        ptx::tmem_ld_cols<0, HK>(tS, r);
        ptx::tmem_ld_wait();
        ptx::fence_before_sync();
        ptx::mbar_arrive(&s_empty[t]);  // S lives in registers now
        if (slow) {
#pragma unroll
          for (int i = 0; i < HK; ++i) {
            float x = __uint_as_float(r[i]) * p.scale_log2;
            if (k0 + i < p.n_bias) x += p.bias_log2;
            if (k0 + i >= p.Lk) x = -INFINITY;
            r[i] = __float_as_uint(x);
          }
        }
        float alpha = 1.f;
        if (!FIXM || j == 0) {
          // row max of this half: four FMNMX3 chains (two logits per instruction)
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < HK; i += 2)
            m4[(i >> 1) & 3] = ptx::fmax3(m4[(i >> 1) & 3], __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
          float pm = ptx::fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
          if (!slow) pm *= p.scale_log2;
          float mx = pm;
          if constexpr (!FR) {  // the two halves' partial maxima meet in shared memory (parity-buffered)
            float* xj = xs + ((j & 1) * 4 + t * 2) * BQ;
            xj[half * BQ + row] = pm;
            ptx::named_bar_sync(bar_id, 64);
            mx = fmaxf(pm, xj[(half ^ 1) * BQ + row]);
          }
          if (FIXM) {
            m_used = mx + kFixedMaxMargin;  // fixed for the whole row from here on
          } else if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
            alpha = ptx::ex2(m_used - mx);                // 0 on the first block
            m_used = mx;
          }
        }
        VC_TRP(trs, 2 + sw, j, 1);
        const float sc = slow ? 1.f : p.scale_log2;
        const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m_used, -m_used);
        float2 s2 = make_float2(0.f, 0.f), s2b = make_float2(0.f, 0.f);
        uint32_t pk[HK / 2];
#pragma unroll
        for (int i = 0; i < HK; i += 2) {
          float2 e = ptx::ffma2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sc2, nm2);
          // POLY >= 100: the degree-2 polynomial on 1 pair in POLY % 100; 2xx: on
          // 2 pairs in POLY % 100 (pair indices 1 and 3 of each group)
          constexpr int PR = POLY % 100;
          constexpr int PG = PR > 0 ? PR : 1;
          const bool off = POLY >= 200 ? (((i >> 1) % PG) == 1 || ((i >> 1) % PG) == 3)
                                       : (PR > 0 && ((i >> 1) % PG) == PR - 1);
          if (off) {
            e = POLY >= 100 ? ptx::ex2_poly2_d2(e) : ptx::ex2_poly2(e);
          } else {
            e.x = ptx::ex2(e.x);
            e.y = ptx::ex2(e.y);
          }
          if (!ONES) {
            if (i & 2) s2b = ptx::fadd2(s2b, e); else s2 = ptx::fadd2(s2, e);
          }
          pk[i >> 1] = ptx::bf16x2(e.x, e.y);
        }
        if (!ONES) {
          s2 = ptx::fadd2(s2, s2b);
          l = l * alpha + (s2.x + s2.y);  // this half's partial row sum
        }
        VC_TRP(trs, 2 + sw, j, 2);
        if (j > 0) {  // P.V(j-1) must be done reading P (and adding into O) before P and O change
          VC_SM_WAIT(&pv_done[t], (j - 1) & 1);
          ptx::fence_after_sync();
        }
        VC_TRP(trs, 2 + sw, j, 3);
        ptx::tmem_st_cols<0, HK / 2>(tP, pk);  // 16 / 8 / 4-column pieces (x4 only: 2% slower)
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          if (FR) rescale_o<DP, 0, CF::NC, CF::ON>(tO, alpha);
          else if (half == 0) rescale_o<DP, 0, CF::NC0, CF::ON>(tO, alpha);
          else rescale_o<DP, CF::NC0, CF::NC, CF::ON>(tO, alpha);
        }
        ptx::tmem_st_wait();
        ptx::fence_before_sync();
        ptx::mbar_arrive(&p_full[t]);
        VC_TRP(trs, 2 + sw, j, 4);
      }
      VC_SM_WAIT(&pv_done[t], (n_tiles - 1) & 1);
      ptx::fence_after_sync();
      if (sw == 0 && lane == 0) VC_CTA(2);
      if (ONES) {  // row sum accumulated by the tensor core in the ones column
        uint32_t r1;
        ptx::tmem_ld1(tO + p.dh, r1);
        ptx::tmem_ld_wait();
        l = __uint_as_float(r1);
      } else if (!FR) {  // the two halves' partial sums (same alpha history) add up
        float* xj = xs + ((n_tiles & 1) * 4 + t * 2) * BQ;
        xj[half * BQ + row] = l;
        ptx::named_bar_sync(bar_id, 64);
        l += xj[(half ^ 1) * BQ + row];
      }
      if (FR) store_out<DP, 0, CF::NC, CF::ON>(p, tO, l, q0 + t * BQ + row, seq, h);
      else if (half == 0) store_out<DP, 0, CF::NC0, CF::ON>(p, tO, l, q0 + t * BQ + row, seq, h);
      else store_out<DP, CF::NC0, CF::NC, CF::ON>(p, tO, l, q0 + t * BQ + row, seq, h);
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (threadIdx.x == 0) VC_CTA(3);
  if (warp == 1) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, CF::TMEM_COLS);
  }
}

}  // namespace

#ifdef VC_ATTN_TRACE
int attn_tracep_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_tracep, sizeof(g_attn_tracep)) == cudaSuccess ? 0 : -1;
}
int attn_cta_read(unsigned long long* host) {  // [16384][5]
  return cudaMemcpyFromSymbol(host, g_attn_cta, sizeof(g_attn_cta)) == cudaSuccess ? 0 : -1;
}
#endif

// One launch of a kernel variant (maps built with its key-block rows).
template <int DP, int POLY, bool ONES, int NARROW, bool FR, int NT, bool FIXM>
int run_tp(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq, int64_t q_rows_per_seq,
           int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = CfgTp<DP, NARROW, FR, NT>;
  AttnMaps m;
  VC_TRY((make_attn_maps<DP, CF::BK>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key)));
  auto kern = attn_tp_kernel<DP, POLY, ONES, NARROW, FR, NT, FIXM>;
  static bool attr = false;
  if (!attr) {
    VC_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr = true;
  }
  dim3 grid((unsigned)cdiv(p.Lq, NT * BQ), (unsigned)p.H, (unsigned)nseq);
  kern<<<grid, CF::WARPS * 32, CF::SMEM, st>>>(m.q64, m.q16, m.k64, m.k16, m.v, p);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

template <int DP>
int launch_attn_tp(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                   int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  const bool ones = p.dh < DP;
#define VC_TP_ARGS p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key, st
  // one query tile per CTA, two CTAs per SM for short key ranges (the spatial
  // branch: 0.318 vs 0.328 ms at config 2, tools/ab_bench.sh; 3.86 vs 3.39 ms
  // on the full sequence, where K / V traffic doubles). VC_ATTN_1T: 0 off, 2 always.
  static const int one_tile = tuning_int("VC_ATTN_1T", 1);
  const bool nt1 = one_tile == 2 || (one_tile == 1 && p.Lk <= 4096);
  // fixed-offset softmax (kFixedMaxMargin: no per-block row max, half-row
  // exchange or rescale after the first key block): full sequence 3.13 ->
  // 2.84 ms, spatial 0.320 -> 0.287 ms at config 2 (tools/ab_bench.sh, 3
  // rounds). VC_ATTN_FIXM=0: the lazy-rescale online softmax.
  static const int fixm = tuning_int("VC_ATTN_FIXM", 1);
  // P.V into a 72-column O when dh + the ones column fit (dh <= 71): 10%
  // less P.V work (full sequence 2.859 vs 2.872 ms, 3 rounds). VC_ATTN_NARROW:
  // 2 this (default), 0 the 80-column O, 1 120-key blocks as well (dropped)
  static const int narrow_on = tuning_int("VC_ATTN_NARROW", 2);
  const bool o72 = DP == 80 && ones && p.dh < 72 && narrow_on == 2 && fixm;
  // exponentials: 2 pairs in 7 on the FMA pipe as a degree-2 polynomial
  // (ex2_poly2_d2, error below a bf16 P's rounding step): full sequence
  // 2.807 ms vs 2.817 for 1 pair in 3, 2.85 for the cubic on 1 in 4, 2.91
  // for 2 in 5 (3 rounds each; no offload 3.16)
#ifdef VC_TUNING
  static const int poly72 = tuning_int("VC_POLY_EVERY", 207);
  if (o72 && poly72 != 207) {  // exp-offload A/B on the default layout
#define VC_TP_POLY(PV) \
    if (poly72 == PV) return nt1 ? run_tp<80, PV, true, 2, false, 1, true>(VC_TP_ARGS) \
                                 : run_tp<80, PV, true, 2, false, 2, true>(VC_TP_ARGS);
    VC_TP_POLY(0) VC_TP_POLY(3) VC_TP_POLY(4) VC_TP_POLY(6) VC_TP_POLY(103) VC_TP_POLY(104) VC_TP_POLY(102) VC_TP_POLY(205)
#undef VC_TP_POLY
  }
#endif
  if (o72) return nt1 ? run_tp<80, 207, true, 2, false, 1, true>(VC_TP_ARGS)
                      : run_tp<80, 207, true, 2, false, 2, true>(VC_TP_ARGS);
#ifdef VC_TUNING
  // measured-and-dropped variants (profiles/r02/attn/README.md): tuning builds only
  static const int poly = tuning_int("VC_POLY_EVERY", 4);
  static const int fr = tuning_int("VC_ATTN_FR", 0);
  if (DP == 80 && ones && p.dh < 72 && narrow_on == 1) return run_tp<80, 4, true, 1, false, 2, true>(VC_TP_ARGS);
  if (fr) return ones ? run_tp<DP, 4, true, false, true, 2, false>(VC_TP_ARGS)
                      : run_tp<DP, 4, false, false, true, 2, false>(VC_TP_ARGS);
  if (poly != 4 && ones) {
    if (poly == 0) return run_tp<DP, 0, true, false, false, 2, true>(VC_TP_ARGS);
    if (poly == 2) return run_tp<DP, 2, true, false, false, 2, true>(VC_TP_ARGS);
    if (poly == 3) return run_tp<DP, 3, true, false, false, 2, true>(VC_TP_ARGS);
    if (poly == 6) return run_tp<DP, 6, true, false, false, 2, true>(VC_TP_ARGS);
    if (poly == 8) return run_tp<DP, 8, true, false, false, 2, true>(VC_TP_ARGS);
  }
#endif
#define VC_TP_PICK(ON)                                                                                   \
  if (nt1) return fixm ? run_tp<DP, 4, ON, false, false, 1, true>(VC_TP_ARGS)                           \
                       : run_tp<DP, 4, ON, false, false, 1, false>(VC_TP_ARGS);                         \
  return fixm ? run_tp<DP, 4, ON, false, false, 2, true>(VC_TP_ARGS)                                    \
              : run_tp<DP, 4, ON, false, false, 2, false>(VC_TP_ARGS);
  if (ones) { VC_TP_PICK(true) }
  VC_TP_PICK(false)
#undef VC_TP_PICK
#undef VC_TP_ARGS
}

template int launch_attn_tp<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t, int64_t,
                                int64_t, cudaStream_t);
template int launch_attn_tp<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t, int64_t,
                                int64_t, cudaStream_t);

}  // namespace vc
