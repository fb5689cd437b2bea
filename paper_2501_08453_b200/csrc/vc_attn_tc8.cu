// Persistent flash attention for DP <= 80 (the 2B shape dh 66 -> 80): the
// default kernel.
//
// Per work item (one sequence, one head, 256 queries = two 128-row tiles) the
// schedule is vc_attn_tc3.cu's (split-row softmax, P of keys 0..63 in TMEM,
// S_A S_B PV_A PV_B issue order).  What is new: one CTA per SM loops over
// items, keeping the TMEM allocation, the barriers and the K/V ring alive
// across items, and overlapping item i's tail (last PV, O epilogue) with item
// i+1's head (Q load, K/V prefetch, first S).  For the 1350-token spatial
// sequences (11 key blocks per item) the per-CTA launch / prologue /
// epilogue was ~35% of the kernel (profiles/r01/attn_study).
//
// Items are dealt round-robin (item = blockIdx.x + k * gridDim.x) in
// (sequence, head, query pair) order, so the ~148 items in flight share a few
// (sequence, head) K/V streams in L2, as the non-persistent grid did.
//
// Barrier phases run on per-role counters across items:
//   K/V ring   g   = key blocks produced / consumed so far (all items)
//   Q          c   = items started (q_full / q_empty phase c & 1)
//   S, P, PV   n_t = blocks issued on tile t so far (tile B is skipped on
//                    items whose second query tile is empty)
//   O          o_free[t] (softmax finished reading O_t) before the first PV_t
//              of the tile's next item overwrites it (phase = items the tile
//              was active in).
// 18 warps: w0 TMA, w1 MMA issuer + TMEM owner, w2..w17 softmax (tile t =
// sw>>3, key half = (sw>>2)&1, w%4 = TMEM lane quarter).
#include "vc_attn_tc_common.cuh"

namespace vc {

namespace {

using namespace attn;

constexpr int kWarps8 = 18;
constexpr int kThreads8 = kWarps8 * 32;
constexpr int kPoly8 = 4;  // one exp2 pair in 4 on the FMA-pipe polynomial

template <int DP>
struct Cfg8 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static_assert(DP <= 80, "O + P half + exchange must fit 256 TMEM columns per tile");
  static constexpr int QK_BYTES = BQ * DP * 2;
  static constexpr int V_BYTES = DP * BKV * 2;
  static constexpr int PH_BYTES = BQ * 64 * 2;  // P of keys 64..127, SW128 [128][64]
  static constexpr int KS = 3;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * QK_BYTES;
  static constexpr int OFF_V = OFF_K + KS * QK_BYTES;
  static constexpr int OFF_P = OFF_V + KS * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * PH_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int NC = DP / 16;
  static constexpr int NC0 = (NC + 1) / 2;
  static constexpr int PCOL = 128 + DP;        // P of keys 0..63: 32 columns
  static constexpr int XCOL = PCOL + 32 + 8;   // row-max / row-sum exchange cells
  static_assert(XCOL + 6 <= 256, "per-tile TMEM columns");
  static_assert(SMEM <= 232448, "shared memory budget");
};

struct Item {
  int seq, h, q0, ntile;
};

__device__ __forceinline__ Item item_of(int it, int nqp, int H, int Lq) {
  Item r;
  r.q0 = (it % nqp) * 2 * BQ;
  r.h = (it / nqp) % H;
  r.seq = it / (nqp * H);
  r.ntile = r.q0 + BQ < Lq ? 2 : 1;  // e.g. 1350 = 5 x 256 + 70: last item has one tile
  return r;
}

template <int DP, bool ONES>
__global__ void __launch_bounds__(kThreads8, 1)
    attn_tc8_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmQ16,
                    const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmV, const AttnTcParams p, const int nseq) {
  using CF = Cfg8<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;     // both tiles' last S MMA of the item done
  uint64_t* k_full = bars + 2;      // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]
  uint64_t* s_full = v_empty + KS;  // [2]
  uint64_t* s_empty = s_full + 2;   // [2] both halves hold S in registers (256)
  uint64_t* p_full = s_empty + 2;   // [2] P in TMEM/smem, O rescaled (256)
  uint64_t* pv_done = p_full + 2;   // [2]
  uint64_t* o_free = pv_done + 2;   // [2] epilogue read O (256)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = threadIdx.x >> 5;
  const int n_kb = (p.Lk + BKV - 1) / BKV;  // key blocks per item
  const int nqp = (p.Lq + 2 * BQ - 1) / (2 * BQ);
  const int n_items = nqp * p.H * nseq;

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmQ64); ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmV);
    if (CF::TAIL) { ptx::prefetch_tmap(&tmQ16); ptx::prefetch_tmap(&tmK16); }
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
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
      ptx::mbar_init(&o_free[t], 256);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer: Q per item, K/V ring across items =====================
    if (ptx::elect_one()) {
      int g = 0, c = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++c) {
        const Item I = item_of(it, nqp, p.H, p.Lq);
        ptx::mbar_wait(q_empty, (c & 1) ^ 1);  // previous item's S MMAs are done with Q
        ptx::mbar_arrive_expect_tx(q_full, 2 * CF::QK_BYTES);
        for (int t = 0; t < 2; ++t) {
          uint8_t* sQ = smem + CF::OFF_Q + t * CF::QK_BYTES;
          for (int cc = 0; cc < CF::N64; ++cc)
            ptx::tma_load_4d(sQ + cc * BQ * 128, &tmQ64, q_full, cc * 64, I.h, I.q0 + t * BQ, I.seq);
          if (CF::TAIL)
            ptx::tma_load_4d(sQ + CF::N64 * BQ * 128, &tmQ16, q_full, CF::N64 * 64, I.h, I.q0 + t * BQ, I.seq);
        }
        for (int j = 0; j < n_kb; ++j, ++g) {
          const int s = g % KS;
          const uint32_t ph = ((g / KS) & 1) ^ 1;
          const int k0 = j * BKV;
          ptx::mbar_wait(&k_empty[s], ph);
          ptx::mbar_arrive_expect_tx(&k_full[s], CF::QK_BYTES);
          uint8_t* sK = smem + CF::OFF_K + s * CF::QK_BYTES;
          for (int cc = 0; cc < CF::N64; ++cc)
            ptx::tma_load_4d(sK + cc * BKV * 128, &tmK64, &k_full[s], cc * 64, I.h, k0, I.seq);
          if (CF::TAIL) ptx::tma_load_4d(sK + CF::N64 * BKV * 128, &tmK16, &k_full[s], CF::N64 * 64, I.h, k0, I.seq);
          ptx::mbar_wait(&v_empty[s], ph);
          ptx::mbar_arrive_expect_tx(&v_full[s], CF::V_BYTES);
          uint8_t* sV = smem + CF::OFF_V + s * CF::V_BYTES;
          ptx::tma_load_4d(sV, &tmV, &v_full[s], k0, 0, I.h, I.seq);
          ptx::tma_load_4d(sV + DP * 128, &tmV, &v_full[s], k0 + 64, 0, I.h, I.seq);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BKV);
    constexpr uint32_t idO = ptx::idesc_bf16_f32(BQ, DP);
    int g = 0, c = 0;
    int nS[2] = {0, 0}, nP[2] = {0, 0};  // S / PV blocks issued per tile so far
    int nI[2] = {0, 0};                  // items each tile has been active in (o_free phases)
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++c) {
      const Item I = item_of(it, nqp, p.H, p.Lq);
      const int g0 = g;  // K/V block index of this item's key block 0
      ptx::mbar_wait(q_full, c & 1);
      // S_t(j) = Q_t K(j)^T (A = Q, B = K from smem)
      auto issue_s = [&](int t, int j, bool last_tile, bool last_block) {
        const int ks = (g0 + j) % KS;
        if (nS[t] > 0) ptx::mbar_wait(&s_empty[t], (nS[t] - 1) & 1);
        ptx::fence_after_sync();
        if (ptx::elect_one()) {
          const uint32_t aQ = ptx::smem_u32(smem + CF::OFF_Q + t * CF::QK_BYTES);
          const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::QK_BYTES);
#pragma unroll
          for (int cc = 0; cc < CF::KSTEPS; ++cc)
            ptx::mma_bf16_ss(tmem + t * 256, qk_desc<DP>(aQ, cc), qk_desc<DP>(aK, cc), idS, cc > 0);
          ptx::mma_commit(&s_full[t]);
          if (last_tile) ptx::mma_commit(&k_empty[ks]);
          if (last_tile && last_block) ptx::mma_commit(q_empty);  // Q free for the next item
        }
        __syncwarp();
        ++nS[t];
      };
      // O_t (+)= P_t(j) V(j): keys 0..63 of P from TMEM, 64..127 from smem
      auto issue_pv = [&](int t, int j, bool last_tile) {
        const int ks = (g0 + j) % KS;
        if (j == 0 && nI[t] > 0) ptx::mbar_wait(&o_free[t], (nI[t] - 1) & 1);  // previous item's O read
        ptx::mbar_wait(&p_full[t], nP[t] & 1);
        ptx::fence_after_sync();
        if (ptx::elect_one()) {
          const uint32_t aP = ptx::smem_u32(smem + CF::OFF_P + t * CF::PH_BYTES);
          const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::V_BYTES);
#pragma unroll
          for (int cc = 0; cc < BKV / 16; ++cc) {
            const uint64_t bd =
                ptx::smem_desc(aV + (cc >> 2) * (DP * 128) + (cc & 3) * 32, 0, 1024, ptx::kLayoutSW128);
            const uint32_t acc = (j > 0 || cc > 0) ? 1u : 0u;
            if (cc < 4)
              ptx::mma_bf16_ts(tmem + t * 256 + 128, tmem + t * 256 + CF::PCOL + 8 * cc, bd, idO, acc);
            else
              ptx::mma_bf16_ss(tmem + t * 256 + 128, ptx::smem_desc(aP + (cc & 3) * 32, 0, 1024, ptx::kLayoutSW128),
                               bd, idO, acc);
          }
          ptx::mma_commit(&pv_done[t]);
          if (last_tile) ptx::mma_commit(&v_empty[ks]);
        }
        __syncwarp();
        ++nP[t];
      };
      const bool two = I.ntile == 2;
      ptx::mbar_wait(&k_full[g0 % KS], (g0 / KS) & 1);
      issue_s(0, 0, !two, n_kb == 1);
      if (two) issue_s(1, 0, true, n_kb == 1);
      for (int j = 0; j < n_kb; ++j) {
        const bool more = j + 1 < n_kb;
        if (more) ptx::mbar_wait(&k_full[(g0 + j + 1) % KS], ((g0 + j + 1) / KS) & 1);
        ptx::mbar_wait(&v_full[(g0 + j) % KS], ((g0 + j) / KS) & 1);
        if (more) issue_s(0, j + 1, !two, j + 2 == n_kb);
        if (more && two) issue_s(1, j + 1, true, j + 2 == n_kb);
        issue_pv(0, j, !two);
        if (two) issue_pv(1, j, true);
      }
      g += n_kb;
      ++nI[0];
      if (two) ++nI[1];
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
    int n = 0;  // blocks of this tile processed so far (S / PV phase counter)
    int c = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++c) {
      const Item I = item_of(it, nqp, p.H, p.Lq);
      if (t >= I.ntile) continue;  // empty second tile: nothing issued for it this item
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kb; ++j, ++n) {
        const int kt = j * BKV;
        const int k0 = kt + half * 64;
        const bool slow = kt < p.n_bias || kt + BKV > p.Lk;  // block-uniform: text keys / tail mask
        ptx::mbar_wait(&s_full[t], n & 1);
        ptx::fence_after_sync();
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
        // partial maxima of the row's two halves meet in TMEM (parity-buffered)
        const uint32_t xc = tX + 2 * (n & 1);
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
          alpha = ptx::ex2(m_used - mx);         // 0 on the first block
          m_used = mx;
        }
        if (j > 0) {  // single P buffer per tile: PV_t(j-1) must be done with it
          ptx::mbar_wait(&pv_done[t], (n - 1) & 1);
          ptx::fence_after_sync();
        }
        const float sc = slow ? 1.f : p.scale_log2;
        const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m_used, -m_used);
        float2 s2 = make_float2(0.f, 0.f), s2b = make_float2(0.f, 0.f);
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float2 e = ptx::ffma2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sc2, nm2);
          if (((i >> 1) % kPoly8) == kPoly8 - 1) {
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
          ptx::tmem_st32(tmem + t * 256 + lane_off + CF::PCOL, pk);  // keys [0, 64) -> 32 TMEM columns
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
        ptx::mbar_arrive(&p_full[t]);
      }
      // epilogue: the item's last PV, then O / l -> output rows, then O is free
      ptx::mbar_wait(&pv_done[t], (n - 1) & 1);
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
      const int qi = I.q0 + t * BQ + row;
      if (half == 0) store_out<DP, 0, CF::NC0>(p, tO, l, qi, I.seq, I.h);
      else store_out<DP, CF::NC0, CF::NC>(p, tO, l, qi, I.seq, I.h);
      ptx::fence_before_sync();
      ptx::mbar_arrive(&o_free[t]);
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

template <int DP>
int launch_attn_tc8(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg8<DP>;
  AttnMaps m;
  VC_TRY(make_attn_maps<DP>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key));
  static const bool no_ones = getenv("VC_NO_ONES_COLUMN") != nullptr;
  const bool ones = !no_ones && p.dh < DP;
  const int64_t items = cdiv(p.Lq, 2 * BQ) * (int64_t)p.H * nseq;
  if (items > INT32_MAX) { set_error("attention: too many work items"); return VC_ENOTSUP; }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    VC_CHECK_CUDA(cudaGetDevice(&dev));
    VC_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const unsigned grid = (unsigned)std::min<int64_t>(items, sms);
#define VC_ATTN8_CASE(ON)                                                                                  \
  if (ones == ON) {                                                                                        \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc8_kernel<DP, ON>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         CF::SMEM));                                                       \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc8_kernel<DP, ON><<<grid, kThreads8, CF::SMEM, st>>>(m.q64, m.q16, m.k64, m.k16, m.v, p, nseq);  \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN8_CASE(true)
  VC_ATTN8_CASE(false)
#undef VC_ATTN8_CASE
  return VC_EINVAL;
}

template int launch_attn_tc8<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc8<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
