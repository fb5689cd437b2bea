// Flash attention, two query tiles per CTA ping-ponging on one tensor core,
// each tile's softmax split across TWO warpgroups ("split rows").
//
// Same semantics and layouts as vc_attn_tc.cu (DP <= 80: the 2B shape dh
// 66 -> 80), two query tiles per CTA.  What changes is the softmax: in the
// round-1 two-tile kernel with one softmax thread per row (git history) one
// thread owns a query row's 128 logits of a key tile, and the measured
// per-tile chain (TMEM load -> row max -> TMEM reload -> 128 exp2 -> P store,
// tools/attn_trace.cu) ran at ~0.3 instructions/clock per warp, so two
// softmax warps per SM sub-partition left MUFU idle 45% of the time.  Here
// the two threads that own a row (warps w and w+4: same TMEM lane quarter,
// same sub-partition) take 64 logits each:
//   * logits stay in registers (one TMEM load, S released at once),
//   * the two partial row maxima meet through two spare TMEM columns and a
//     64-thread named barrier (both threads then agree bit-exactly on the
//     lazily tracked max, so P, alpha and l match the one-thread kernel),
//   * four softmax warps per sub-partition hide each other's latencies.
// 18 warps: w0 TMA producer, w1 MMA issuer + TMEM owner, w2..w17 softmax
// (w = 2 + 8*tile + 4*half + i; w % 4 is the TMEM lane quarter).
// Tuning builds only (-DVC_TUNING, VC_ATTN_IMPL=3): the round-1 kernel kept
// as the A/B reference of profiles/r02/attn/README.md; the product library
// does not contain it.
#ifdef VC_TUNING
#include "vc_attn_tc_common.cuh"
#include "vc_tuning.h"

namespace vc {

namespace {

using namespace attn;

constexpr int kWarps3 = 18;
constexpr int kThreads3 = kWarps3 * 32;
#ifndef VC_POLY_EVERY
#define VC_POLY_EVERY 4
#endif
constexpr int kPolyEvery3 = VC_POLY_EVERY;

#ifdef VC_ATTN_TRACE
__device__ unsigned long long g_attn_trace3[17][256][8];
#define VC_TR3(cond, role, j, k)                                             \
  do {                                                                       \
    if ((cond) && (j) < 256) g_attn_trace3[role][j][k] = clock64();         \
  } while (0)
#else
#define VC_TR3(cond, role, j, k) \
  do {                           \
  } while (0)
#endif

template <int DP>
struct Cfg3 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static_assert(DP <= 80, "O + exchange columns must fit 256 TMEM columns per tile");
  static constexpr int QK_BYTES = BQ * DP * 2;
  static constexpr int V_BYTES = DP * BKV * 2;
  static constexpr int P_BYTES = BQ * BKV * 2;
  static constexpr int KS = 3;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QK_BYTES;
  static constexpr int OFF_V = OFF_K + KS * QK_BYTES;
  static constexpr int OFF_P = OFF_V + KS * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int NC = DP / 16;       // 16-column chunks of O
  static constexpr int NC0 = (NC + 1) / 2;  // chunks [0, NC0) -> half 0, rest -> half 1
  static constexpr int QCOL = 128 + DP;     // Q in TMEM (QT): DP/2 packed bf16x2 columns
  static constexpr int XCOL = QCOL + DP / 2;  // exchange columns
  static constexpr int QW = DP / 4;           // Q u32 words per half row
  static_assert(XCOL + 6 <= 256, "per-tile TMEM columns");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// QT: Q lives in TMEM (loaded by the softmax threads, S MMA in the "ts" form
// reading only K from shared memory) instead of smem (TMA, "ss" form).
// PH (needs !QT): the P of keys [0, 64) (half 0) goes to TMEM over the idle
// Q columns and the PV MMA reads it from there ("ts" k-steps 0..3); only keys
// [64, 128) go through shared memory — half the P store + P operand traffic
// on the SM's shared-memory port, the kernel's busiest shared resource.
template <int DP, int POLY, bool ONES, bool QT, bool PH = false>
__global__ void __launch_bounds__(kThreads3, 1)
    attn_tc3_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmQ16,
                    const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmV, const __nv_bfloat16* __restrict__ qg,
                    const int64_t q_rows_per_seq, const AttnTcParams p, const bool LOCK) {
  using CF = Cfg3<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;      // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]
  uint64_t* s_full = v_empty + KS;  // [2 tiles]
  uint64_t* s_empty = s_full + 2;   // [2 tiles] both halves hold S in registers
  uint64_t* p_full = s_empty + 2;   // [2 tiles]
  uint64_t* pv_done = p_full + 2;   // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * (2 * BQ);
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_tiles = (p.Lk + BKV - 1) / BKV;
  // the last CTA of a sequence may have no rows in its second query tile
  // (e.g. 1350 = 5 x 256 + 70): then only tile A runs (CTA-uniform)
  const int ntile = q0 + BQ < p.Lq ? 2 : 1;
  [[maybe_unused]] const bool tr = blockIdx.x == min(20u, gridDim.x - 1) && blockIdx.y == 3 && blockIdx.z == 0;
  VC_TR3(tr && threadIdx.x == 32, 0, 255, 0);  // entry (trace builds: CTA fixed-cost marks in j = 255)

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmQ64); ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmV);
    if (CF::TAIL) { ptx::prefetch_tmap(&tmQ16); ptx::prefetch_tmap(&tmK16); }
    ptx::mbar_init(q_full, QT ? 512 : 1);
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&s_empty[t], 256);
      ptx::mbar_init(&p_full[t], 256);
      ptx::mbar_init(&pv_done[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  VC_TR3(tr && threadIdx.x == 32, 0, 255, 1);  // barriers + TMEM ready

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (ptx::elect_one()) {
      if (!QT) ptx::mbar_arrive_expect_tx(q_full, 2 * CF::QK_BYTES);
      for (int t = 0; t < 2 && !QT; ++t) {
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
      VC_TR3(tr, 0, 254, 0);  // TMA producer issued its last load
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BKV);
    constexpr uint32_t idO = ptx::idesc_bf16_f32(BQ, DP);
    ptx::mbar_wait(q_full, 0);
    auto issue_s = [&](int t, int j) {
      const int ks = j % KS;
      if (j > 0) ptx::mbar_wait(&s_empty[t], (j - 1) & 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aQ = ptx::smem_u32(smem + CF::OFF_Q + t * CF::QK_BYTES);
        const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::QK_BYTES);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c) {
          if (QT)
            ptx::mma_bf16_ts(tmem + t * 256, tmem + t * 256 + CF::QCOL + 8 * c, qk_desc<DP>(aK, c), idS, c > 0);
          else
            ptx::mma_bf16_ss(tmem + t * 256, qk_desc<DP>(aQ, c), qk_desc<DP>(aK, c), idS, c > 0);
        }
        ptx::mma_commit(&s_full[t]);
        if (t == ntile - 1) ptx::mma_commit(&k_empty[ks]);
      }
      __syncwarp();
    };
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
          if (PH && c < 4)
            ptx::mma_bf16_ts(tmem + t * 256 + 128, tmem + t * 256 + CF::QCOL + 8 * c, bd, idO, (j > 0 || c > 0) ? 1u : 0u);
          else
            ptx::mma_bf16_ss(tmem + t * 256 + 128, ad, bd, idO, (j > 0 || c > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&pv_done[t]);
        if (t == ntile - 1) ptx::mma_commit(&v_empty[ks]);
      }
      __syncwarp();
    };
    const bool trm = tr && (threadIdx.x & 31) == 0;
    VC_TR3(trm, 0, 255, 2);  // Q landed
    ptx::mbar_wait(&k_full[0], 0);
    VC_TR3(trm, 0, 255, 3);  // first K block landed
    issue_s(0, 0);
    if (ntile == 2) issue_s(1, 0);
    for (int j = 0; j < n_tiles; ++j) {
      const bool more = j + 1 < n_tiles;
      if (more) ptx::mbar_wait(&k_full[(j + 1) % KS], ((j + 1) / KS) & 1);
      VC_TR3(trm, 0, j, 0);
      ptx::mbar_wait(&v_full[j % KS], (j / KS) & 1);
      VC_TR3(trm, 0, j, 1);
      if (LOCK) {
        // lock-step: both tiles' S(j+1) first, then both PV(j); the two
        // softmax groups then run their exp phases at the same time (4 warps
        // per SM sub-partition in MUFU/FMA work instead of 2)
        if (more) issue_s(0, j + 1);
        VC_TR3(trm, 0, j, 2);
        if (more && ntile == 2) issue_s(1, j + 1);
        VC_TR3(trm, 0, j, 3);
        issue_pv(0, j);
        VC_TR3(trm, 0, j, 4);
        if (ntile == 2) issue_pv(1, j);
        VC_TR3(trm, 0, j, 5);
      } else {
        if (more) issue_s(0, j + 1);
        VC_TR3(trm, 0, j, 2);
        issue_pv(0, j);
        VC_TR3(trm, 0, j, 3);
        if (more && ntile == 2) issue_s(1, j + 1);
        VC_TR3(trm, 0, j, 4);
        if (ntile == 2) issue_pv(1, j);
        VC_TR3(trm, 0, j, 5);
      }
    }
    VC_TR3(trm, 0, 254, 1);  // MMA issuer done
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
    if (QT) {  // this thread's half of its Q row -> TMEM (A operand of the S MMA)
      const int qi = q0 + t * BQ + row;
      uint32_t qv[CF::QW];
      if (qi < p.Lq) {
        const uint4* src = reinterpret_cast<const uint4*>(
            qg + ((int64_t)seq * q_rows_per_seq + qi) * ((int64_t)p.H * DP) + (int64_t)h * DP + half * (DP / 2));
#pragma unroll
        for (int u = 0; u < CF::QW / 4; ++u) {
          const uint4 w = __ldg(src + u);
          qv[4 * u] = w.x; qv[4 * u + 1] = w.y; qv[4 * u + 2] = w.z; qv[4 * u + 3] = w.w;
        }
      } else {
#pragma unroll
        for (int u = 0; u < CF::QW; ++u) qv[u] = 0u;
      }
      const uint32_t tQ = tmem + t * 256 + lane_off + CF::QCOL + half * CF::QW;
      ptx::tmem_st16(tQ, *reinterpret_cast<uint32_t(*)[16]>(qv));
      if (CF::QW == 20) ptx::tmem_st4(tQ + 16, *reinterpret_cast<uint32_t(*)[4]>(qv + 16));
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(q_full);
    }
    const uint32_t bar_id = 1 + t * 4 + quarter;
    const uint32_t rowp = ptx::smem_u32(smem + CF::OFF_P + t * CF::P_BYTES) + half * (BQ * 128) + row * 128;
    const bool trs = tr && lane == 0;
    if (t < ntile) {  // a tile with no query rows has nothing to compute
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int kt = j * BKV;
        const int k0 = kt + half * 64;
        const bool slow = kt < p.n_bias || kt + BKV > p.Lk;  // tile-uniform: text keys / tail mask
        ptx::mbar_wait(&s_full[t], j & 1);
        ptx::fence_after_sync();
        VC_TR3(trs, 1 + sw, j, 0);
        uint32_t r[64];
        ptx::tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_ld_wait();
        ptx::fence_before_sync();
        ptx::mbar_arrive(&s_empty[t]);  // S lives in registers now
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
        // partial maxima of the row's two halves meet (parity-buffered) in the
        // idle Q smem region when Q lives in TMEM, else in spare TMEM columns
        float other;
        if (QT) {
          float* xs = reinterpret_cast<float*>(smem + CF::OFF_Q) + ((j & 1) * 2 * 2 + t * 2) * BQ;
          xs[half * BQ + row] = pm;
          ptx::named_bar_sync(bar_id, 64);
          other = xs[(half ^ 1) * BQ + row];
        } else {
          const uint32_t xc = tX + 2 * (j & 1);
          ptx::tmem_st1(xc + half, __float_as_uint(pm));
          ptx::tmem_st_wait();
          ptx::fence_before_sync();
          ptx::named_bar_sync(bar_id, 64);
          ptx::fence_after_sync();
          uint32_t o;
          ptx::tmem_ld1(xc + (half ^ 1), o);
          ptx::tmem_ld_wait();
          other = __uint_as_float(o);
        }
        const float mx = fmaxf(pm, other);
        VC_TR3(trs, 1 + sw, j, 1);
        float alpha = 1.f;
        if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
          alpha = ptx::ex2(m_used - mx);         // 0 on the first tile
          m_used = mx;
        }
        if (j > 0) {  // single P buffer per tile: PV_t(j-1) must be done with it
          ptx::mbar_wait(&pv_done[t], (j - 1) & 1);
          ptx::fence_after_sync();
        }
        VC_TR3(trs, 1 + sw, j, 2);
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
        if (PH && half == 0) {
          ptx::tmem_st32(tmem + t * 256 + lane_off + CF::QCOL, pk);  // keys [0, 64) -> 32 TMEM columns
          ptx::tmem_st_wait();
        } else {
  #pragma unroll
          for (int u = 0; u < 8; ++u)
            ptx::sts128(rowp + ((u ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        VC_TR3(trs, 1 + sw, j, 3);
        if (!ONES) {
          s2 = ptx::fadd2(s2, s2b);
          l = l * alpha + (s2.x + s2.y);  // this half's partial row sum
        }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          if (half == 0) rescale_o<DP, 0, CF::NC0>(tO, alpha);
          else rescale_o<DP, CF::NC0, CF::NC>(tO, alpha);
        }
        ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
        ptx::fence_before_sync();
        ptx::mbar_arrive(&p_full[t]);
        VC_TR3(trs, 1 + sw, j, 4);
      }
      ptx::mbar_wait(&pv_done[t], (n_tiles - 1) & 1);
      ptx::fence_after_sync();
      VC_TR3(trs, 1 + sw, 255, 0);  // last P.V done
      if (ONES) {  // row sum accumulated by the tensor core in the ones column
        uint32_t r1;
        ptx::tmem_ld1(tO + p.dh, r1);
        ptx::tmem_ld_wait();
        l = __uint_as_float(r1);
      } else {  // the two halves' partial sums (same alpha history) add up
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
      VC_TR3(trs, 1 + sw, 255, 2);  // row sum read
      if (half == 0) store_out<DP, 0, CF::NC0>(p, tO, l, q0 + t * BQ + row, seq, h);
      else store_out<DP, CF::NC0, CF::NC>(p, tO, l, q0 + t * BQ + row, seq, h);
      VC_TR3(trs, 1 + sw, 255, 1);  // output stored
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  VC_TR3(tr && threadIdx.x == 32, 0, 255, 4);  // all warps done
  if (warp == 1) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

#ifdef VC_ATTN_TRACE
int attn_trace3_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_trace3, sizeof(g_attn_trace3)) == cudaSuccess ? 0 : -1;
}
#endif

template <int DP>
int launch_attn_tc3(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg3<DP>;
  AttnMaps m;
  VC_TRY(make_attn_maps<DP>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key));
  // defaults: 1 exp pair in 4 on the FMA polynomial, the ones column whenever
  // dh < DP, P half in TMEM (so Q stays in smem), lock-step MMA issue
  static const int poly = tuning_int("VC_POLY_EVERY", kPolyEvery3);
  const bool ones = tuning_int("VC_NO_ONES_COLUMN", 0) == 0 && p.dh < DP;
  static const bool ph = tuning_int("VC_ATTN_PHALF", 1) != 0;
  // Q in TMEM (only without the P half; needs 16-byte aligned Q rows)
  const bool qt = !ph && tuning_int("VC_ATTN_QSMEM", 0) == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0;
  const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q);
  // MMA issue order: lock-step (S_A S_B PV_A PV_B, default) or ping-pong (S_A PV_A S_B PV_B)
  static const bool lock = tuning_int("VC_ATTN_PINGPONG", 0) == 0;
  dim3 grid((unsigned)cdiv(p.Lq, 2 * BQ), (unsigned)p.H, (unsigned)nseq);
#define VC_ATTN3_CASE(PV, ON, Q, PHV)                                                                      \
  if (poly == PV && ones == ON && qt == Q && ph == PHV) {                                                  \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc3_kernel<DP, PV, ON, Q, PHV>,                              \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));          \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc3_kernel<DP, PV, ON, Q, PHV><<<grid, kThreads3, CF::SMEM, st>>>(m.q64, m.q16, m.k64, m.k16, m.v, \
                                                                           qb, q_rows_per_seq, p, lock);   \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN3_CASE(4, true, false, true)
  VC_ATTN3_CASE(4, false, false, true)
#ifdef VC_TUNING
  VC_ATTN3_CASE(0, false, false, false)
  VC_ATTN3_CASE(0, true, false, false)
  VC_ATTN3_CASE(4, false, false, false)
  VC_ATTN3_CASE(4, true, false, false)
  VC_ATTN3_CASE(2, true, false, false)
  VC_ATTN3_CASE(3, true, false, false)
  VC_ATTN3_CASE(0, false, true, false)
  VC_ATTN3_CASE(0, true, true, false)
  VC_ATTN3_CASE(4, false, true, false)
  VC_ATTN3_CASE(4, true, true, false)
  VC_ATTN3_CASE(2, true, true, false)
  VC_ATTN3_CASE(3, true, true, false)
  VC_ATTN3_CASE(3, true, false, true)
#endif
#undef VC_ATTN3_CASE
  set_error("attention variant not built (tuning builds: VC_POLY_EVERY 0, 2, 3, 4)");
  return VC_EINVAL;
}

template int launch_attn_tc3<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc3<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
#endif  // VC_TUNING
