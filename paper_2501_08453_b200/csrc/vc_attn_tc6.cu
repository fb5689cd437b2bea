// Flash attention, one 128-query tile per CTA, 128-key blocks with S
// DOUBLE-BUFFERED in tensor memory, Q and P resident in TMEM, and each query
// row's softmax spread over FOUR warps (32 keys per thread).  DP <= 80 (the
// 2B shape dh 66 -> 80).
//
// Measured (tools/attn_trace.cu, tools/softmax_bench.cu): the exp phase is the
// limiter — per SM sub-partition it runs ~2x faster with four warps in flight
// than with two, and the ping-pong kernels (tc2/tc3) only ever had two warps
// of a sub-partition in their exp phase.  Here all 16 softmax warps work on
// the same block at once, and the tensor core computes S(j+1) (other buffer)
// while they do, so they never wait for it:
//   MMA order: S(0) S(1) S(2) | PV(0) S(3) | PV(1) S(4) | ...  (in-order
//   pipe: PV(j) has read P(j) before S(j+3) overwrites that buffer)
// TMEM columns: S/P buffers [0,128) [128,256) [256,384) | O [384, 384+DP) |
// Q [384+DP, +DP/2)  (P(j) = bf16 pairs over the first 64 columns of S(j)'s
// buffer; three buffers so S(j+1) is complete before block j's softmax ends
// and its TMEM load overlaps block j's exponentials).
// 18 warps: w0 TMA (K/V rings), w1 MMA issuer + TMEM owner, w2..w17 softmax:
// group g = (w-2)/4 owns keys [32g, 32g+32) of every block, w % 4 = TMEM lane
// quarter; the four partial row maxima meet in shared memory.
#include "vc_attn_tc_common.cuh"

namespace vc {

namespace {

using namespace attn;

constexpr int kWarps6 = 18;
constexpr int kThreads6 = kWarps6 * 32;
#ifndef VC_POLY_EVERY6
#define VC_POLY_EVERY6 3
#endif
constexpr int kPolyEvery6 = VC_POLY_EVERY6;

#ifdef VC_ATTN_TRACE
__device__ unsigned long long g_attn_trace6[17][256][8];
#define VC_TR6(cond, role, j, k)                                             \
  do {                                                                       \
    if ((cond) && (j) < 256) g_attn_trace6[role][j][k] = clock64();         \
  } while (0)
#else
#define VC_TR6(cond, role, j, k) \
  do {                           \
  } while (0)
#endif

template <int DP>
struct Cfg6 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int K_BYTES = BKV * DP * 2;
  static constexpr int V_BYTES = DP * BKV * 2;
  static constexpr int KS = 4;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KS * K_BYTES;
  static constexpr int OFF_X = OFF_V + KS * V_BYTES;  // row-max exchange [2 parity][4 groups][128 rows] f32
  static constexpr int OFF_BAR = OFF_X + 2 * 4 * 128 * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int NBUF = 3;      // S/P buffers
  static constexpr int OCOL = NBUF * 128;
  static constexpr int QCOL = OCOL + DP;
  static constexpr int QW = DP / 2;  // Q u32 words (bf16 pairs) per row
  static constexpr int NC = DP / 16;  // 16-column chunks of O
  static_assert(QCOL + QW <= 512, "TMEM columns");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// O chunk range [c0, c1) of softmax group g (NC chunks over 4 groups)
template <int NC>
__device__ __forceinline__ void o_chunks(int g, int& c0, int& c1) {
  c0 = (g * NC) / 4;
  c1 = ((g + 1) * NC) / 4;
}

template <int DP>
__device__ __forceinline__ void rescale_o_range(uint32_t o_addr, float alpha, int c0, int c1) {
#pragma unroll
  for (int c = 0; c < DP / 16; ++c) {
    if (c < c0 || c >= c1) continue;
    uint32_t r[16];
    ptx::tmem_ld16(o_addr + c * 16, r);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
    ptx::tmem_st16(o_addr + c * 16, r);
  }
  ptx::tmem_st_wait();
}

template <int DP, int POLY, bool ONES>
__global__ void __launch_bounds__(kThreads6, 1)
    attn_tc6_kernel(const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmV, const __nv_bfloat16* __restrict__ qg,
                    const int64_t q_rows_per_seq, const AttnTcParams p) {
  using CF = Cfg6<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* k_full = bars;          // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]
  uint64_t* q_full = v_empty + KS;  // Q rows in TMEM (512 arrivals)
  uint64_t* s_full = q_full + 1;    // [NBUF buffers]
  uint64_t* p_full = s_full + CF::NBUF;  // P(j) in TMEM, O rescaled (512 arrivals)
  uint64_t* pv_done = p_full + 1;   // [2] PV(j) completes a phase of pv_done[j & 1]
  uint64_t* o_done = pv_done + 2;   // the last PV
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);
  float* xmax = reinterpret_cast<float*>(smem + CF::OFF_X);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * BQ;
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_blk = (p.Lk + BKV - 1) / BKV;
  [[maybe_unused]] const bool tr = blockIdx.x == 40 && blockIdx.y == 3 && blockIdx.z == 0;

  if (warp == 0 && ptx::elect_one()) {
    ptx::prefetch_tmap(&tmK64); ptx::prefetch_tmap(&tmV);
    if (CF::TAIL) ptx::prefetch_tmap(&tmK16);
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    ptx::mbar_init(q_full, 512);
    for (int i = 0; i < CF::NBUF; ++i) ptx::mbar_init(&s_full[i], 1);
    ptx::mbar_init(p_full, 512);
    ptx::mbar_init(&pv_done[0], 1);
    ptx::mbar_init(&pv_done[1], 1);
    ptx::mbar_init(o_done, 1);
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
      for (int j = 0; j < n_blk; ++j) {
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
    auto issue_s = [&](int j) {  // S(j) = Q K(j)^T into buffer j % NBUF
      const int ks = j % KS;
      ptx::mbar_wait(&k_full[ks], (j / KS) & 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::K_BYTES);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c)
          ptx::mma_bf16_ts(tmem + (j % CF::NBUF) * 128, tmem + CF::QCOL + 8 * c, qk_desc<DP>(aK, c), idS, c > 0);
        ptx::mma_commit(&s_full[j % CF::NBUF]);
        ptx::mma_commit(&k_empty[ks]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int j) {  // O += P(j) V(j), P over buffer j % NBUF
      const int ks = j % KS;
      ptx::mbar_wait(&v_full[ks], (j / KS) & 1);
      ptx::mbar_wait(p_full, j & 1);
      ptx::fence_after_sync();
      if (ptx::elect_one()) {
        const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::V_BYTES);
#pragma unroll
        for (int c = 0; c < BKV / 16; ++c) {
          const uint64_t bd = ptx::smem_desc(aV + (c >> 2) * (DP * 128) + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
          ptx::mma_bf16_ts(tmem + CF::OCOL, tmem + (j % CF::NBUF) * 128 + 8 * c, bd, idO, (j > 0 || c > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&pv_done[j & 1]);
        if (j + 1 == n_blk) ptx::mma_commit(o_done);
        ptx::mma_commit(&v_empty[ks]);
      }
      __syncwarp();
    };
    ptx::mbar_wait(q_full, 0);
    ptx::fence_after_sync();
    for (int j = 0; j < CF::NBUF && j < n_blk; ++j) issue_s(j);
    for (int j = 0; j < n_blk; ++j) {
      VC_TR6(trm, 0, j, 0);
      issue_pv(j);
      VC_TR6(trm, 0, j, 1);
      if (j + CF::NBUF < n_blk) issue_s(j + CF::NBUF);
      VC_TR6(trm, 0, j, 2);
    }
  } else {
    // ===================== softmax (key group g), correction, epilogue =====================
    const int g = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tT = tmem + lane_off;
    const uint32_t tO = tT + CF::OCOL;
    const uint32_t bar_id = 1 + quarter;  // the 4 warps (128 threads) of this lane quarter
    const bool trs = tr && lane == 0;
    const int role = 1 + (warp - 2);
    int oc0, oc1;
    o_chunks<CF::NC>(g, oc0, oc1);
    // ---- Q row (this group's quarter of it) -> TMEM ----
    {
      const int qi = q0 + row;
      constexpr int QG = CF::QW / 4;  // u32 words per group: 10 (DP 80) or 8 (DP 64)
      uint32_t qv[QG];
      if (qi < p.Lq) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(
            qg + ((int64_t)seq * q_rows_per_seq + qi) * ((int64_t)p.H * DP) + (int64_t)h * DP) + g * QG;
#pragma unroll
        for (int u = 0; u < QG / 2; ++u) {
          const uint2 w = __ldg(reinterpret_cast<const uint2*>(src) + u);
          qv[2 * u] = w.x; qv[2 * u + 1] = w.y;
        }
      } else {
#pragma unroll
        for (int u = 0; u < QG; ++u) qv[u] = 0u;
      }
      const uint32_t tQ = tT + CF::QCOL + g * QG;
      ptx::tmem_st8(tQ, *reinterpret_cast<uint32_t(*)[8]>(qv));
      if (QG == 10) {
        ptx::tmem_st1(tQ + 8, qv[8]);
        ptx::tmem_st1(tQ + 9, qv[QG - 1]);
      }
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(q_full);
    }
    // Software pipeline: the logits of block j+1 are loaded from TMEM (and
    // their partial row max published) while block j's exponentials run, so
    // the next step starts with the 128-thread exchange barrier only.
    auto load_block = [&](int j, uint32_t (&r)[32]) {
      ptx::mbar_wait(&s_full[j % CF::NBUF], (j / CF::NBUF) & 1);
      ptx::fence_after_sync();
      ptx::tmem_ld32(tT + (j % CF::NBUF) * 128 + g * 32, r);
    };
    auto publish_max = [&](int j, uint32_t (&r)[32]) {  // after the load completed
      const int k0 = j * BKV + g * 32;
      const bool slow = j * BKV < p.n_bias || j * BKV + BKV > p.Lk;  // block-uniform
      if (slow) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = __uint_as_float(r[i]) * p.scale_log2;
          if (k0 + i < p.n_bias) x += p.bias_log2;
          if (k0 + i >= p.Lk) x = -INFINITY;
          r[i] = __float_as_uint(x);
        }
      }
      float m4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) m4[i] = __uint_as_float(r[i]);
#pragma unroll
      for (int i = 4; i < 32; ++i) m4[i & 3] = fmaxf(m4[i & 3], __uint_as_float(r[i]));
      float pm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      if (!slow) pm *= p.scale_log2;
      // parity-buffered: buffer (j & 1) was last read before barrier j-1,
      // which every thread of the quarter has passed
      xmax[(j & 1) * 512 + g * 128 + row] = pm;
    };
    float m_used = -INFINITY, l = 0.f;
    uint32_t r[32];
    load_block(0, r);
    ptx::tmem_ld_wait_dep32(r);
    publish_max(0, r);
    for (int j = 0; j < n_blk; ++j) {
      const int b = j % CF::NBUF;
      const bool slow = j * BKV < p.n_bias || j * BKV + BKV > p.Lk;
      VC_TR6(trs, role, j, 0);
      // the row's four partial maxima (smem); the barrier also certifies every
      // group holds its S(j) in registers before P(j) overwrites the buffer
      ptx::named_bar_sync(bar_id, 128);
      const float* xm = xmax + (j & 1) * 512;
      const float mx = fmaxf(fmaxf(xm[row], xm[128 + row]), fmaxf(xm[256 + row], xm[384 + row]));
      const bool more = j + 1 < n_blk;
      uint32_t rn[32];
      if (more) load_block(j + 1, rn);  // completes under the exponentials below
      VC_TR6(trs, role, j, 1);
      float alpha = 1.f;
      if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
        alpha = ptx::ex2(m_used - mx);         // 0 on the first block
        m_used = mx;
      }
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        // O must hold PV(j-1).  pv_done[(j-1) & 1] carries PV(j-1), PV(j-3), ..;
        // S(j) certifies PV(j-3) and PV(j+1) is not issued yet, so the parity
        // wait below is exact without tracking phases.
        ptx::mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        ptx::fence_after_sync();
        rescale_o_range<DP>(tO, alpha, oc0, oc1);
      }
      VC_TR6(trs, role, j, 2);
      const float sc = slow ? 1.f : p.scale_log2;
      const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m_used, -m_used);
      float2 s2 = make_float2(0.f, 0.f);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float2 e = ptx::ffma2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sc2, nm2);
        if (POLY > 0 && ((i >> 1) % (POLY > 0 ? POLY : 1)) == POLY - 1) {
          e = ptx::ex2_poly2(e);
        } else {
          e.x = ptx::ex2(e.x);
          e.y = ptx::ex2(e.y);
        }
        if (!ONES) s2 = ptx::fadd2(s2, e);
        pk[i >> 1] = ptx::bf16x2(e.x, e.y);
      }
      ptx::tmem_st16(tT + b * 128 + g * 16, pk);  // P keys [32g, 32g+32) -> columns [16g, 16g+16)
      if (!ONES) l = l * alpha + (s2.x + s2.y);
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(p_full);
      VC_TR6(trs, role, j, 3);
      if (more) {
        ptx::tmem_ld_wait_dep32(rn);
        publish_max(j + 1, rn);
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = rn[i];
      }
    }
    ptx::mbar_wait(o_done, 0);
    ptx::fence_after_sync();
    if (ONES) {  // row sum accumulated by the tensor core in the ones column
      uint32_t r1;
      ptx::tmem_ld1(tO + p.dh, r1);
      ptx::tmem_ld_wait();
      l = __uint_as_float(r1);
    } else {  // the four groups' partial sums (same alpha history) add up
      float* xl = xmax;  // free again: every group is past its last max exchange
      ptx::named_bar_sync(bar_id, 128);
      xl[g * 128 + row] = l;
      ptx::named_bar_sync(bar_id, 128);
      l = (xl[row] + xl[128 + row]) + (xl[256 + row] + xl[384 + row]);
    }
    const int qi = q0 + row;
    if (g == 0) store_out<DP, 0, CF::NC / 4>(p, tO, l, qi, seq, h);
    else if (g == 1) store_out<DP, CF::NC / 4, 2 * CF::NC / 4>(p, tO, l, qi, seq, h);
    else if (g == 2) store_out<DP, 2 * CF::NC / 4, 3 * CF::NC / 4>(p, tO, l, qi, seq, h);
    else store_out<DP, 3 * CF::NC / 4, CF::NC>(p, tO, l, qi, seq, h);
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
int attn_trace6_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_trace6, sizeof(g_attn_trace6)) == cudaSuccess ? 0 : -1;
}
#endif

template <int DP>
int launch_attn_tc6(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg6<DP>;
  if ((reinterpret_cast<uintptr_t>(q) & 7) != 0) {
    set_error("attention: Q must be 8-byte aligned");
    return VC_EINVAL;
  }
  AttnMaps m;
  VC_TRY(make_attn_maps<DP>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key));
  static const int poly = getenv("VC_POLY_EVERY") ? atoi(getenv("VC_POLY_EVERY")) : kPolyEvery6;
  static const bool no_ones = getenv("VC_NO_ONES_COLUMN") != nullptr;
  const bool ones = !no_ones && p.dh < DP;
  const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q);
  dim3 grid((unsigned)cdiv(p.Lq, BQ), (unsigned)p.H, (unsigned)nseq);
#define VC_ATTN6_CASE(PV, ON)                                                                              \
  if (poly == PV && ones == ON) {                                                                          \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc6_kernel<DP, PV, ON>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));          \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc6_kernel<DP, PV, ON><<<grid, kThreads6, CF::SMEM, st>>>(m.k64, m.k16, m.v, qb, q_rows_per_seq, p); \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN6_CASE(0, false)
  VC_ATTN6_CASE(0, true)
  VC_ATTN6_CASE(3, false)
  VC_ATTN6_CASE(3, true)
  VC_ATTN6_CASE(2, true)
  VC_ATTN6_CASE(4, true)
#undef VC_ATTN6_CASE
  set_error("VC_POLY_EVERY must be 0 or 3 (2, 4 with the ones column)");
  return VC_EINVAL;
}

template int launch_attn_tc6<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc6<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
