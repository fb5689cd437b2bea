// Flash attention, two query tiles per CTA, 64-key blocks with a
// DOUBLE-BUFFERED S in tensor memory, Q and P resident in TMEM (DP <= 80: the
// 2B shape dh 66 -> 80).  The default kernel for padded head dims 64 / 80.
//
// Measured history (tools/attn_trace.cu, per 128x128 score block):
//   tc2 (1 thread/row, P in smem)          1289 clk  - smem port + softmax latency
//   tc4 (split rows, Q/P in TMEM, BKV 128) 1426 clk  - S(j+1) waits PV(j): the
//        tensor-core latency sat inside every softmax step
// The exp phase alone (tools/softmax_bench.cu) needs ~900 clk per block with
// two warps per SM sub-partition, so the softmax warps must never wait.  With
// 64-key blocks a tile needs S0/S1 (2 x 64 columns) + O (DP) + Q (DP/2) <= 248
// TMEM columns, so two tiles fit in 512 with S double-buffered: while the
// softmax turns S(j) into P(j) (written over S(j) with tcgen05.st), the tensor
// core already computes S(j+1) into the other buffer, and S(j+2) is issued
// right behind PV(j) (in-order pipe: PV(j) has read P(j) before S(j+2)
// overwrites that buffer).  One thread owns a query row (64 logits per block,
// no cross-thread max exchange); the two tiles' softmax warps share each
// sub-partition.
//
// TMEM columns per tile t (base 256 t): S/P buffers [0,64) [64,128) |
// O [128,128+DP) | Q [128+DP, 128+DP+DP/2).
// 10 warps: w0 TMA (K/V rings), w1 MMA issuer + TMEM owner, w2..w5 softmax of
// tile 0, w6..w9 tile 1 (w % 4 = TMEM lane quarter).
#include "vc_attn_tc_common.cuh"

namespace vc {

namespace {

using namespace attn;

constexpr int kBK = 64;  // keys per block
constexpr int kWarps5 = 10;
constexpr int kThreads5 = kWarps5 * 32;
#ifndef VC_POLY_EVERY5
#define VC_POLY_EVERY5 3
#endif
constexpr int kPolyEvery5 = VC_POLY_EVERY5;

#ifdef VC_ATTN_TRACE
__device__ unsigned long long g_attn_trace5[9][512][8];
#define VC_TR5(cond, role, j, k)                                             \
  do {                                                                       \
    if ((cond) && (j) < 512) g_attn_trace5[role][j][k] = clock64();         \
  } while (0)
#else
#define VC_TR5(cond, role, j, k) \
  do {                           \
  } while (0)
#endif

template <int DP>
struct Cfg5 {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int K_BYTES = kBK * DP * 2;
  static constexpr int V_BYTES = DP * kBK * 2;
  static constexpr int KS = 8;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KS * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + KS * V_BYTES;
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
  static constexpr int KSTEPS = DP / 16;
  static constexpr int QCOL = 128 + DP;
  static constexpr int QW = DP / 2;  // Q u32 words (bf16 pairs) per row
  static_assert(QCOL + QW <= 256, "per-tile TMEM columns");
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int DP, int POLY, bool ONES>
__global__ void __launch_bounds__(kThreads5, 1)
    attn_tc5_kernel(const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmK16,
                    const __grid_constant__ CUtensorMap tmV, const __nv_bfloat16* __restrict__ qg,
                    const int64_t q_rows_per_seq, const AttnTcParams p) {
  using CF = Cfg5<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* k_full = bars;          // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* v_full = k_empty + KS;  // [KS]
  uint64_t* v_empty = v_full + KS;  // [KS]
  uint64_t* q_full = v_empty + KS;  // [2 tiles] Q rows in TMEM (128 arrivals)
  uint64_t* s_full = q_full + 2;    // [2 tiles][2 buffers]
  uint64_t* p_full = s_full + 4;    // [2 tiles] P(j) in TMEM, O rescaled (128 arrivals)
  uint64_t* pv_done = p_full + 2;   // [2 tiles] one phase per PV (waited at most one behind)
  uint64_t* o_done = pv_done + 2;   // [2 tiles] the last PV
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5;
  const int q0 = blockIdx.x * (2 * BQ);
  const int h = blockIdx.y;
  const int seq = blockIdx.z;
  const int n_blk = (p.Lk + kBK - 1) / kBK;
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
      ptx::mbar_init(&q_full[t], 128);
      ptx::mbar_init(&s_full[2 * t], 1);
      ptx::mbar_init(&s_full[2 * t + 1], 1);
      ptx::mbar_init(&p_full[t], 128);
      ptx::mbar_init(&pv_done[t], 1);
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
      for (int j = 0; j < n_blk; ++j) {
        const int s = j % KS;
        const uint32_t ph = ((j / KS) & 1) ^ 1;
        const int k0 = j * kBK;
        ptx::mbar_wait(&k_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&k_full[s], CF::K_BYTES);
        uint8_t* sK = smem + CF::OFF_K + s * CF::K_BYTES;
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d(sK + c * kBK * 128, &tmK64, &k_full[s], c * 64, h, k0, seq);
        if (CF::TAIL) ptx::tma_load_4d(sK + CF::N64 * kBK * 128, &tmK16, &k_full[s], CF::N64 * 64, h, k0, seq);
        ptx::mbar_wait(&v_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&v_full[s], CF::V_BYTES);
        ptx::tma_load_4d(smem + CF::OFF_V + s * CF::V_BYTES, &tmV, &v_full[s], k0, 0, h, seq);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, kBK);
    constexpr uint32_t idO = ptx::idesc_bf16_f32(BQ, DP);
    const bool trm = tr && (threadIdx.x & 31) == 0;
    // S_t(j) = Q_t K(j)^T into buffer j & 1 (A = Q from TMEM)
    auto issue_s = [&](int t, int j) {
      const int ks = j % KS;
      if (ptx::elect_one()) {
        const uint32_t aK = ptx::smem_u32(smem + CF::OFF_K + ks * CF::K_BYTES);
#pragma unroll
        for (int c = 0; c < CF::KSTEPS; ++c)
          ptx::mma_bf16_ts(tmem + t * 256 + (j & 1) * 64, tmem + t * 256 + CF::QCOL + 8 * c,
                           qk_desc<DP, kBK>(aK, c), idS, c > 0);
        ptx::mma_commit(&s_full[2 * t + (j & 1)]);
        if (t == 1) ptx::mma_commit(&k_empty[ks]);  // both tiles' S MMAs done with K(j)
      }
      __syncwarp();
    };
    // O_t += P_t(j) V(j) (A = P from TMEM over buffer j & 1)
    auto issue_pv = [&](int t, int j) {
      const int ks = j % KS;
      ptx::mbar_wait(&p_full[t], j & 1);
      ptx::fence_after_sync();
      VC_TR5(trm, 0, j, 5 + t);
      if (ptx::elect_one()) {
        const uint32_t aV = ptx::smem_u32(smem + CF::OFF_V + ks * CF::V_BYTES);
#pragma unroll
        for (int c = 0; c < kBK / 16; ++c)
          ptx::mma_bf16_ts(tmem + t * 256 + 128, tmem + t * 256 + (j & 1) * 64 + 8 * c,
                           ptx::smem_desc(aV + c * 32, 0, 1024, ptx::kLayoutSW128), idO, (j > 0 || c > 0) ? 1u : 0u);
        ptx::mma_commit(&pv_done[t]);
        if (j + 1 == n_blk) ptx::mma_commit(&o_done[t]);
        if (t == 1) ptx::mma_commit(&v_empty[ks]);  // both tiles' PV MMAs done with V(j)
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
    if (n_blk > 1) {
      ptx::mbar_wait(&k_full[1 % KS], 0);
      issue_s(0, 1);
      issue_s(1, 1);
    }
    for (int j = 0; j < n_blk; ++j) {
      const bool more = j + 2 < n_blk;
      ptx::mbar_wait(&v_full[j % KS], (j / KS) & 1);
      VC_TR5(trm, 0, j, 0);
      issue_pv(0, j);
      VC_TR5(trm, 0, j, 1);
      if (more) {
        ptx::mbar_wait(&k_full[(j + 2) % KS], ((j + 2) / KS) & 1);
        VC_TR5(trm, 0, j, 7);
        issue_s(0, j + 2);
      }
      VC_TR5(trm, 0, j, 2);
      issue_pv(1, j);
      VC_TR5(trm, 0, j, 3);
      if (more) issue_s(1, j + 2);
      VC_TR5(trm, 0, j, 4);
    }
  } else {
    // ===================== softmax (tile t), correction, epilogue =====================
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tT = tmem + t * 256 + lane_off;
    const uint32_t tO = tT + 128;
    const bool trs = tr && lane == 0;
    const int role = 1 + (warp - 2);
    // ---- Q row -> TMEM (A operand of the S MMA) ----
    {
      const int qi = q0 + t * BQ + row;
      uint32_t qv[CF::QW];
      if (qi < p.Lq) {
        const uint4* src = reinterpret_cast<const uint4*>(
            qg + ((int64_t)seq * q_rows_per_seq + qi) * ((int64_t)p.H * DP) + (int64_t)h * DP);
#pragma unroll
        for (int u = 0; u < CF::QW / 4; ++u) {
          const uint4 w = __ldg(src + u);
          qv[4 * u] = w.x; qv[4 * u + 1] = w.y; qv[4 * u + 2] = w.z; qv[4 * u + 3] = w.w;
        }
      } else {
#pragma unroll
        for (int u = 0; u < CF::QW; ++u) qv[u] = 0u;
      }
      const uint32_t tQ = tT + CF::QCOL;
      ptx::tmem_st32(tQ, *reinterpret_cast<uint32_t(*)[32]>(qv));
      if (CF::QW == 40) ptx::tmem_st8(tQ + 32, *reinterpret_cast<uint32_t(*)[8]>(qv + 32));
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(&q_full[t]);
    }
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_blk; ++j) {
      const int k0 = j * kBK;
      const int b = j & 1;
      const bool slow = k0 < p.n_bias || k0 + kBK > p.Lk;  // block-uniform: text keys / tail mask
      ptx::mbar_wait(&s_full[2 * t + b], (j >> 1) & 1);
      ptx::fence_after_sync();
      VC_TR5(trs, role, j, 0);
      uint32_t r[64];
      ptx::tmem_ld32(tT + b * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
      ptx::tmem_ld32(tT + b * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
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
      float m8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) m8[i] = __uint_as_float(r[i]);
#pragma unroll
      for (int i = 8; i < 64; ++i) m8[i & 7] = fmaxf(m8[i & 7], __uint_as_float(r[i]));
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      if (!slow) mx *= p.scale_log2;
      VC_TR5(trs, role, j, 1);
      float alpha = 1.f;
      if (mx > m_used + kRescaleThreshold) {  // lazy rescale: P stays <= 2^8
        alpha = ptx::ex2(m_used - mx);         // 0 on the first block
        m_used = mx;
      }
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        // O must hold PV(j-1) before it is rescaled (S(j) only certifies PV(j-2),
        // so pv_done has completed j-1 or j phases: the parity wait is exact)
        ptx::mbar_wait(&pv_done[t], (j - 1) & 1);
        ptx::fence_after_sync();
        rescale_o<DP>(tO, alpha);
      }
      VC_TR5(trs, role, j, 2);
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
      ptx::tmem_st32(tT + b * 64, pk);  // P(j) over the first 32 columns of S(j)'s buffer
      if (!ONES) {
        s2 = ptx::fadd2(s2, s2b);
        l = l * alpha + (s2.x + s2.y);
      }
      ptx::tmem_st_wait();
      ptx::fence_before_sync();
      ptx::mbar_arrive(&p_full[t]);
      VC_TR5(trs, role, j, 3);
    }
    ptx::mbar_wait(&o_done[t], 0);
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
  if (warp == 1) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

#ifdef VC_ATTN_TRACE
int attn_trace5_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_trace5, sizeof(g_attn_trace5)) == cudaSuccess ? 0 : -1;
}
#endif

template <int DP>
int launch_attn_tc5(const AttnTcParams& p, const void* q, const void* k, const void* vt, int nseq,
                    int64_t q_rows_per_seq, int64_t k_rows_per_seq, int64_t ld_key, cudaStream_t st) {
  using CF = Cfg5<DP>;
  if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) {
    set_error("attention: Q must be 16-byte aligned");
    return VC_EINVAL;
  }
  AttnMaps m;
  VC_TRY((make_attn_maps<DP, kBK>(m, p, q, k, vt, nseq, q_rows_per_seq, k_rows_per_seq, ld_key)));
  static const int poly = getenv("VC_POLY_EVERY") ? atoi(getenv("VC_POLY_EVERY")) : kPolyEvery5;
  static const bool no_ones = getenv("VC_NO_ONES_COLUMN") != nullptr;
  const bool ones = !no_ones && p.dh < DP;
  const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q);
  dim3 grid((unsigned)cdiv(p.Lq, 2 * BQ), (unsigned)p.H, (unsigned)nseq);
#define VC_ATTN5_CASE(PV, ON)                                                                              \
  if (poly == PV && ones == ON) {                                                                          \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      VC_CHECK_CUDA(cudaFuncSetAttribute(attn_tc5_kernel<DP, PV, ON>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));          \
      attr = true;                                                                                         \
    }                                                                                                      \
    attn_tc5_kernel<DP, PV, ON><<<grid, kThreads5, CF::SMEM, st>>>(m.k64, m.k16, m.v, qb, q_rows_per_seq, p); \
    VC_CHECK_LAUNCH();                                                                                     \
    return VC_OK;                                                                                          \
  }
  VC_ATTN5_CASE(0, false)
  VC_ATTN5_CASE(0, true)
  VC_ATTN5_CASE(3, false)
  VC_ATTN5_CASE(3, true)
  VC_ATTN5_CASE(2, true)
  VC_ATTN5_CASE(4, true)
#undef VC_ATTN5_CASE
  set_error("VC_POLY_EVERY must be 0 or 3 (2, 4 with the ones column)");
  return VC_EINVAL;
}

template int launch_attn_tc5<64>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);
template int launch_attn_tc5<80>(const AttnTcParams&, const void*, const void*, const void*, int, int64_t,
                                 int64_t, int64_t, cudaStream_t);

}  // namespace vc
