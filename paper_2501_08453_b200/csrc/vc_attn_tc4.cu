// Flash attention with Q and P resident in tensor memory (DP <= 80: the 2B
// shape dh 66 -> 80).  Two query tiles per CTA ping-pong on one tensor core;
// each tile's softmax is split over two warpgroups (64 keys of the row each,
// as in vc_attn_tc3.cu).
//
// Why: in vc_attn_tc2/tc3 every MMA operand came from shared memory and the
// softmax wrote P there, so per key tile the SM's shared-memory port moved
// Q,K (S MMA) + P,V (PV MMA) + the P stores + the K/V TMA fills; measured
// tensor-core smem wavefronts 51% + LSU stores 21% + TMA fills ~12% of one
// 128 B/clk port — the port, not MUFU or the tensor core, set the pace.  Here
//   * Q is loaded once per CTA from global into TMEM (the S MMA's A operand,
//     tcgen05.mma "ts" form), so the S MMA reads only K from smem;
//   * P (bf16) is written by the softmax with tcgen05.st over the S columns it
//     has just consumed and the PV MMA reads it from TMEM, so the only smem
//     traffic left is the K/V TMA fill and the K/V operand reads.
// P aliasing S orders the tensor core: PV_t(j) must precede S_t(j+1) (the
// pipe executes in issue order), so the MMA warp issues PV_A(j), S_A(j+1),
// PV_B(j), S_B(j+1) and one commit per S also certifies the PV before it.
//
// TMEM columns per tile t (base 256 t): S/P [0,128) | O [128,128+DP) |
// Q [QCOL, QCOL+DP/2) | exchange cells [XCOL, XCOL+6).
// 18 warps: w0 TMA (K/V rings), w1 MMA issuer + TMEM owner, w2..w17 softmax
// (w = 2 + 8*tile + 4*half + i; w % 4 is the TMEM lane quarter).
#include "vc_attn_tc_common.cuh"

namespace vc {

namespace {

using namespace attn;

constexpr int kWarps4 = 18;
constexpr int kThreads4 = kWarps4 * 32;
#ifndef VC_POLY_EVERY
#define VC_POLY_EVERY 4
#endif
constexpr int kPolyEvery4 = VC_POLY_EVERY;

#ifdef VC_ATTN_TRACE
__device__ unsigned long long g_attn_trace4[17][256][8];
#define VC_TR4(cond, role, j, k)                                             \
  do {                                                                       \
    if ((cond) && (j) < 256) g_attn_trace4[role][j][k] = clock64();         \
  } while (0)
#else
#define VC_TR4(cond, role, j, k) \
  do {                           \
  } while (0)
#endif

template <int DP>
struct Cfg4 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int K_BYTES = BKV * DP * 2;
  static constexpr int V_BYTES = DP * BKV * 2;
  static constexpr int KS = 4;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KS * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + KS * V_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int NC = DP / 16;        // 16-column chunks of O
  static constexpr int NC0 = (NC + 1) / 2;  // chunks [0, NC0) -> half 0, rest -> half 1
  static constexpr int QCOL = 128 + DP;     // Q: DP/2 packed bf16x2 columns
  static constexpr int XCOL = QCOL + DP / 2;
  static constexpr int QW = DP / 4;         // Q u32 words per half row
  static_assert(XCOL + 6 <= 256, "per-tile TMEM columns");
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int DP, int POLY, bool ONES>
__global__ void __launch_bounds__(kThreads4, 1)
    attn_tc4_kernel(const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmV, const __nv_bfloat16* __restrict__ qg,
                    const int64_t q_rows_per_seq, const AttnTcParams p) {
  using CF = Cfg4<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* k_full = bars;          // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]
  uint64_t* q_full = v_empty + KS;  // [2 tiles] Q rows in TMEM (256 arrivals)
  uint64_t* s_full = q_full + 2;    // [2 tiles] S_t(j) (and PV_t(j-1)) complete
  uint64_t* p_full = s_full + 2;    // [2 tiles] P_t(j) in TMEM, O rescaled (256 arrivals)
  uint64_t* o_done = p_full + 2;    // [2 tiles] last PV complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * (2 * BQ);
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_tiles = (p.Lk + BKV - 1) / BKV;
  [[maybe_unused]] const bool tr = blockIdx.x == 20 && blockIdx.y == 3 && blockIdx.z == 0;

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmV);
    if (CF::TAIL) ptx::prefetch_tmap(&tmK16);
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&q_full[t], 256);
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 256);
      ptx::mbar_init(&o_done[t], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (K, V rings) =====================
    if (ptx::elect_one()) {
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % KS;
        const uint32_t ph = ((j / KS) & 1) ^ 1;
        const int k0 = j * BKV;
        ptx::mbar_wait(&k_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&k_full[s], CF::K_BYTES);
        uint8_t* sK = smem + CF::OFF_K + s * CF::K_BYTES;
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
    const bool trm = tr && (threadIdx.x & 31) == 0;
    // S_t(j) = Q_t K(j)^T: A = Q from TMEM (8 columns per 16-wide k step)
    auto issue_s = [&](int t, int j) {
      const int ks = j % KS;
      if (ptx::elect_one()) {
        const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::K_BYTES);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c)
          ptx::mma_bf16_ts(tmem + t * 256, tmem + t * 256 + CF::QCOL + 8 * c, qk_desc<DP>(aK, c), idS, c > 0);
        ptx::mma_commit(&s_full[t]);
        if (t == 1) ptx::mma_commit(&k_empty[ks]);  // both tiles' S MMAs done with K(j)
      }
      __syncwarp();
    };
    // O_t += P_t(j) V(j): A = P from TMEM (over S_t's first 64 columns)
    auto issue_pv = [&](int t, int j, bool last) {
      const int ks = j % KS;
      ptx::mbar_wait(&p_full[t], j & 1);
      ptx::fence_after_sync();
      VC_TR4(trm, 0, j, 6 + t);
      if (ptx::elect_one()) {
        const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::V_BYTES);
#pragma unroll
        for (int c = 0; c < BKV / 16; ++c) {
          const uint64_t bd = ptx::smem_desc(aV + (c >> 2) * (DP * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
          ptx::mma_bf16_ts(tmem + t * 256 + 128, tmem + t * 256 + 8 * c, bd, idO, (j > 0 || c > 0) ? 1u : 0u);
        }
        if (t == 1) ptx::mma_commit(&v_empty[ks]);  // both tiles' PV MMAs done with V(j)
        if (last) ptx::mma_commit(&o_done[t]);
      }
      __syncwarp();
    };
    ptx::mbar_wait(&k_full[0], 0);
    ptx::mbar_wait(&q_full[0], 0);
    ptx::fence_after_sync();
    issue_s(0, 0);
    ptx::mbar_wait(&q_full[1], 0);
    ptx::fence_after_sync();
    issue_s(1, 0);
    for (int j = 0; j < n_tiles; ++j) {
      const bool more = j + 1 < n_tiles;
      ptx::mbar_wait(&v_full[j % KS], (j / KS) & 1);
      VC_TR4(trm, 0, j, 0);
      issue_pv(0, j, !more);
      VC_TR4(trm, 0, j, 1);
      if (more) {
        ptx::mbar_wait(&k_full[(j + 1) % KS], ((j + 1) / KS) & 1);
        VC_TR4(trm, 0, j, 2);
        issue_s(0, j + 1);
      }
      VC_TR4(trm, 0, j, 3);
      issue_pv(1, j, !more);
      VC_TR4(trm, 0, j, 4);
      if (more) issue_s(1, j + 1);
      VC_TR4(trm, 0, j, 5);
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
    const uint32_t tT = tmem + t * 256 + lane_off;  // tile base (S / P)
    const uint32_t tO = tT + 128;
    const uint32_t tX = tT + CF::XCOL;
    const uint32_t bar_id = 1 + t * 4 + quarter;
    const bool trs = tr && lane == 0;
    // ---- Q row half -> TMEM (A operand of the S MMA) ----
    {
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
      const uint32_t tQ = tT + CF::QCOL + half * CF::QW;
      ptx::tmem_st16(tQ, *reinterpret_cast<uint32_t(*)[16]>(qv));
      if (CF::QW == 20) ptx::tmem_st4(tQ + 16, *reinterpret_cast<uint32_t(*)[4]>(qv + 16));
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(&q_full[t]);
    }
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int kt = j * BKV;
      const int k0 = kt + half * 64;
      const bool slow = kt < p.n_bias || kt + BKV > p.Lk;  // tile-uniform: text keys / tail mask
      ptx::mbar_wait(&s_full[t], j & 1);
      ptx::fence_after_sync();
      VC_TR4(trs, 1 + sw, j, 0);
      uint32_t r[64];
      ptx::tmem_ld32(tT + half * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
      ptx::tmem_ld32(tT + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
      ptx::tmem_ld_wait();
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
      // the row's two partial maxima meet in TMEM; the barrier also certifies
      // that both halves hold their S in registers before P overwrites it
      const uint32_t xc = tX + 2 * (j & 1);
      ptx::tmem_st1(xc + half, __float_as_uint(pm));
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::named_bar_sync(bar_id, 64);
      ptx::fence_after_sync();
      uint32_t other;
      ptx::tmem_ld1(xc + (half ^ 1), other);
      ptx::tmem_ld_wait();
      const float mx = fmaxf(pm, __uint_as_float(other));
      VC_TR4(trs, 1 + sw, j, 1);
      float alpha = 1.f;
      if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
        alpha = ptx::ex2(m_used - mx);         // 0 on the first tile
        m_used = mx;
      }
      // O holds PV(j-1) (complete: S(j) was issued after it)
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        if (half == 0) rescale_o<DP, 0, CF::NC0>(tO, alpha);
        else rescale_o<DP, CF::NC0, CF::NC>(tO, alpha);
      }
      VC_TR4(trs, 1 + sw, j, 2);
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
      ptx::tmem_st32(tT + half * 32, pk);  // P keys [64 half, +64) -> columns [32 half, +32)
      VC_TR4(trs, 1 + sw, j, 3);
      if (!ONES) {
        s2 = ptx::fadd2(s2, s2b);
        l = l * alpha + (s2.x + s2.y);  // this half's partial row sum
      }
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(&p_full[t]);
      VC_TR4(trs, 1 + sw, j, 4);
    }
    ptx::mbar_wait(&o_done[t], 0);
    ptx::fence_after_sync();
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
    if (half == 0) store_out<DP, 0, CF::NC0>(p, tO, l, q0 + t * BQ + row, seq, h);
    else store_out<DP, CF::NC0, CF::NC>(p, tO, l, q0 + t * BQ + row, seq, h);
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

#ifdef VC_ATTN_TRACE
int attn_trace4_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_trace4, sizeof(g_attn_trace4)) == cudaSuccess ? 0 : -1;
}
#endif

template <int DP>
int launch_attn_tc4(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg4<DP>;
  if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) {
    set_error("attention: Q must be 16-byte aligned");
    return VC_EINVAL;
  }
  AttnMaps m;
  VC_TRY(make_attn_maps<DP>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key));
  static const int poly = getenv("VC_POLY_EVERY") ? atoi(getenv("VC_POLY_EVERY")) : kPolyEvery4;
  static const bool no_ones = getenv("VC_NO_ONES_COLUMN") != nullptr;
  const bool ones = !no_ones && p.dh < DP;
  const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q);
  dim3 grid((unsigned)cdiv(p.Lq, 2 * BQ), (unsigned)p.H, (unsigned)nseq);
#define VC_ATTN4_CASE(PV, ON)                                                                              \
  if (poly == PV && ones == ON) {                                                                          \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc4_kernel<DP, PV, ON>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));          \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc4_kernel<DP, PV, ON><<<grid, kThreads4, CF::SMEM, st>>>(m.k64, m.k16, m.v, qb, q_rows_per_seq, p); \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN4_CASE(0, false)
  VC_ATTN4_CASE(0, true)
  VC_ATTN4_CASE(4, false)
  VC_ATTN4_CASE(4, true)
  VC_ATTN4_CASE(2, true)
  VC_ATTN4_CASE(3, true)
#undef VC_ATTN4_CASE
  set_error("VC_POLY_EVERY must be 0 or 4 (2, 3 with the ones column)");
  return VC_EINVAL;
}

template int launch_attn_tc4<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc4<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
