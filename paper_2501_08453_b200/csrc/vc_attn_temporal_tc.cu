// Temporal-branch attention on the 5th-generation tensor cores (tcgen05 +
// TMEM, operands by TMA), model.py:238-244: one sequence per spatial
// position l made of the F tokens {f*Lv + l}, numerics.py:87-107 per head.
//
// The sequences are short (F = 16..160) and there are Lv*H of them: the
// branch is HBM-bound (~F/2 flop per byte), so the design goal is to stream
// q, k, v once at full bandwidth, not tensor-core efficiency. One CTA takes
// one head of a group of npos = 128 / F consecutive positions (F <= 128) or
// of one position (128 < F <= 176, two 128-row query tiles):
//   * the QKV GEMM epilogue writes the temporal q, k, v rows position-major
//     ([Lv*F][3D], row l*F + f; GemmTcParams.qkv.tm_F), so a group's rows are
//     consecutive and TMA copies them as whole boxes; its NK = npos*F keys
//     form npos diagonal blocks of F;
//   * S = Q K^T (M 128, N NK, K = dh padded to 80 / 128; Q's padding columns,
//     which the plain layout fills with the next head, are zeroed in shared
//     memory) and O = P V with V read in place as an MN-major B operand (no
//     transposed copy anywhere);
//   * the softmax reads only each row's own diagonal block and writes P
//     (zeros off the block) over S in TMEM; the row sum is summed on the
//     CUDA cores (V has no ones column here).
// The block-diagonal MMA does npos times the useful MMA work, which is free
// at this arithmetic intensity. Two CTAs per SM (<= 256 TMEM columns each)
// keep one group's loads in flight under the other's math.
//
// In : qkv bf16 [Lv*F][ld] position-major, q at column 0, k at +D, v at +2D
// Out: o bf16 [F*Lv][ldo], head h at h*hs (hs = dh, or a head slot whose
//      columns past dh are written as zeros)
#include <math.h>

#include "vc_gemm_tc.h"
#include "vc_kernels.h"
#include "vc_ptx.cuh"
#include "vc_tuning.h"

namespace vc {

namespace {

// w0..w3 softmax / epilogue (row = TMEM lane), w4 TMA producer, w5 MMA issuer
constexpr int kTmThreads = 192;

template <int DP>
struct CfgTm {
  static constexpr int N64 = DP / 64;
  static constexpr int TAIL = DP % 64;  // 0 or 16: SW32 part of Q / K (and V's 16-column chunk)
  static_assert(TAIL == 0 || TAIL == 16, "DP must be 64*n or 64*n+16");
  static constexpr int SHIFT = DP == 80 ? 8 : 0;  // room for the <= 6-column head offset (dh % 8 != 0)
  static constexpr int NKMAX = (256 - DP - SHIFT) / 16 * 16;  // S + O in one TMEM set of 256 columns
  static constexpr int Q_BYTES = 128 * DP * 2;
  static constexpr int K_BYTES = (NKMAX * DP * 2 + 1023) / 1024 * 1024;
  static constexpr int STAGE = Q_BYTES + 2 * K_BYTES;  // Q, K, V of one work item
  static constexpr int KS = (220 * 1024) / STAGE >= 3 ? 3 : 2;
  static constexpr int OFF_BAR = KS * STAGE;
  static constexpr int SMEM = OFF_BAR + 128 + 1024;
  static_assert(STAGE % 1024 == 0, "1024-aligned tiles");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// B operand in MN-major layout (V: rows = keys = K, columns = dh = N)
__host__ __device__ constexpr uint32_t idesc_bf16_f32_bmn(int M, int N) {
  return ptx::idesc_bf16_f32(M, N) | (1u << 16);
}

// Persistent: CTA b takes work items b, b + gridDim.x, ...; item = (position
// group, head), heads fastest (the CTAs working at one time read the same
// rows). Q, K, V of an item go through a KS-deep shared-memory ring (TMA two
// items ahead of the math), S / O through two TMEM sets (the epilogue of one
// item overlaps the next item's S).
template <int DP>
__global__ void __launch_bounds__(kTmThreads, 1)
    temporal_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQt,
                       const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKt,
                       const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmVt,
                       __nv_bfloat16* __restrict__ o, int64_t ldo, int F, int Lv, int H, int dh, int hs, int npos,
                       int NK, int n_items, float scale_log2) {
  using CF = CfgTm<DP>;
  constexpr int KS = CF::KS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* full = bars;            // [KS] Q, K, V of the stage's item landed
  uint64_t* empty = full + KS;      // [KS] the stage's MMAs are done with it
  uint64_t* s_full = empty + KS;    // [2 TMEM sets]
  uint64_t* p_full = s_full + 2;    // [2] P written (128 arrivals)
  uint64_t* o_full = p_full + 2;    // [2]
  uint64_t* o_free = o_full + 2;    // [2] S / O read out (128 arrivals)
  uint64_t* q2_full = o_free + 2;   // a second query tile's Q landed (F > 128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q2_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows_kv = npos * F;            // rows a K / V box writes (NK rounds it up to 16)
  const int rows_q = npos * min(F, 128);   // rows a Q box writes (out-of-range frames / positions as zeros)
  const int nq = (npos * F + 127) / 128;   // query tiles per item (2 only when F > 128)
  const int q_bytes = rows_q * DP * 2, kv_bytes = rows_kv * DP * 2;
  const int k_off = CF::Q_BYTES, v_off = CF::Q_BYTES + CF::K_BYTES;

  if (warp == 4 && ptx::elect_one()) {
    for (int i = 0; i < KS; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::mbar_init(q2_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 128);
      ptx::mbar_init(&o_full[i], 1);
      ptx::mbar_init(&o_free[i], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 5) ptx::tmem_alloc(tmem_slot, 512);
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  // work unit u = (item, query tile): S / O set u & 1, stage of the item it % KS
  if (warp == 4) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int h = item % H, l0 = (item / H) * npos;
        const int kcol = (h * dh) & ~7;  // 16-byte aligned box start (see the MMA issuer)
        const int st = it % KS;
        uint8_t* sb = smem + st * CF::STAGE;
        ptx::mbar_wait(&empty[st], ((it / KS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[st], q_bytes + 2 * kv_bytes);
        for (int c = 0; c < CF::N64; ++c) {
          ptx::tma_load_4d(sb + k_off + c * NK * 128, &tmK, &full[st], kcol + 64 * c, l0 * F, 0, 0);
          ptx::tma_load_4d(sb + v_off + c * NK * 128, &tmV, &full[st], kcol + 64 * c, l0 * F, 0, 0);
        }
        if (CF::TAIL) {
          ptx::tma_load_4d(sb + k_off + CF::N64 * NK * 128, &tmKt, &full[st], kcol + 64 * CF::N64, l0 * F, 0, 0);
          ptx::tma_load_4d(sb + v_off + CF::N64 * NK * 128, &tmVt, &full[st], kcol + 64 * CF::N64, l0 * F, 0, 0);
        }
        // Q of the item's first query tile (a second tile, F > 128, reuses the
        // buffer after the first tile's S MMA: loaded by the MMA issuer)
        for (int c = 0; c < CF::N64; ++c)
          ptx::tma_load_4d(sb + c * 128 * 128, &tmQ, &full[st], kcol + 64 * c, l0 * F, 0, 0);
        if (CF::TAIL) ptx::tma_load_4d(sb + CF::N64 * 128 * 128, &tmQt, &full[st], kcol + 64 * CF::N64, l0 * F, 0, 0);
      }
    }
  } else if (warp == 5) {
    // ===================== MMA issuer (lane 0; the warp zeroes padding) =====================
    int it = 0, u = 0, n_reload = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int h = item % H;
      // TMA boxes start on a 16-byte column boundary: the head's columns
      // [h*dh, h*dh + dh) sit at offset sh (0..6) of the tile, the same in Q,
      // K and V, so Q K^T is unchanged once Q is zero outside [sh, sh + dh),
      // and O's head columns are O[sh .. sh + dh)
      const int sh = h * dh - ((h * dh) & ~7);
      const int st = it % KS;
      uint8_t* sb = smem + st * CF::STAGE;
      const uint32_t sQ = ptx::smem_u32(sb), sK = sQ + k_off, sV = sQ + v_off;
      const uint64_t dK = ptx::smem_desc(sK, 0, 1024, ptx::kLayoutSW128);
      const uint64_t dKt = ptx::smem_desc(sK + CF::N64 * NK * 128, 0, 256, ptx::kLayoutSW32);
      const uint64_t dQ = ptx::smem_desc(sQ, 0, 1024, ptx::kLayoutSW128);
      const uint64_t dQt = ptx::smem_desc(sQ + CF::N64 * 128 * 128, 0, 256, ptx::kLayoutSW32);
      // MN-major V: 64-column chunks NK*128 bytes apart (LBO), 8-key groups 1024 apart (SBO)
      const uint64_t dV = ptx::smem_desc(sV, NK * 128, 1024, ptx::kLayoutSW128);
      const uint64_t dVt = ptx::smem_desc(sV + CF::N64 * NK * 128, 0, 256, ptx::kLayoutSW32);
      const uint32_t idS = ptx::idesc_bf16_f32(128, NK);
      const uint32_t idO = idesc_bf16_f32_bmn(128, 64 * CF::N64), idOt = idesc_bf16_f32_bmn(128, 16);
      ptx::mbar_wait(&full[st], (it / KS) & 1);
      if (rows_kv < NK) {  // K / V rows rows_kv..NK-1 are never written: zero them (0 * stale NaN != 0)
        for (int c = 0; c < CF::N64; ++c)
          for (int i = lane; i < (NK - rows_kv) * 8; i += 32) {
            const int off = c * NK * 128 + (rows_kv + i / 8) * 128 + (i % 8) * 16;
            *reinterpret_cast<uint4*>(sb + k_off + off) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(sb + v_off + off) = make_uint4(0, 0, 0, 0);
          }
        if (CF::TAIL)
          for (int i = lane; i < (NK - rows_kv) * 2; i += 32) {
            const int off = CF::N64 * NK * 128 + (rows_kv + i / 2) * 32 + (i % 2) * 16;
            *reinterpret_cast<uint4*>(sb + k_off + off) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(sb + v_off + off) = make_uint4(0, 0, 0, 0);
          }
      }
      for (int q = 0; q < nq; ++q, ++u) {
        const int ts = u & 1;
        const uint32_t tS = tmem + ts * 256, tO = tS + NK;
        if (q > 0) {  // the second query tile's Q over the first's (its S MMA has completed)
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(q2_full, q_bytes);
            for (int c = 0; c < CF::N64; ++c)
              ptx::tma_load_4d(sb + c * 128 * 128, &tmQ, q2_full, ((h * dh) & ~7) + 64 * c,
                               item / H * npos * F + 128 * q, 0, 0);
            if (CF::TAIL)
              ptx::tma_load_4d(sb + CF::N64 * 128 * 128, &tmQt, q2_full, ((h * dh) & ~7) + 64 * CF::N64,
                               item / H * npos * F + 128 * q, 0, 0);
          }
          ptx::mbar_wait(q2_full, n_reload & 1);
          ++n_reload;
        }
        if (dh + sh < DP || sh > 0 || rows_q < 128) {
          // zero Q outside its head's columns [sh, sh + dh) (the plain layout
          // holds the neighbouring heads there; zeros in Q drop them out of
          // Q K^T) and the rows a short box left unwritten, 16 bytes at a time.
          // 64-column chunks: [128 rows][128 B] SW128 (16-byte unit ^= row & 7);
          // the tail: [128 rows][32 B] SW32 (16-byte unit ^= row bit 2)
          constexpr int UNITS = DP / 8;
          for (int e = lane; e < 128 * UNITS; e += 32) {
            const int r = e / UNITS, un = e - r * UNITS;  // logical unit un = columns 8un .. 8un+7
            const int lo = max(sh - 8 * un, 0), hi = min(sh + dh - 8 * un, 8);  // real columns inside it
            if (r < rows_q && lo == 0 && hi == 8) continue;
            const int ch = un >> 3, w = un & 7;
            uint8_t* addr = ch < CF::N64 ? sb + ch * 128 * 128 + r * 128 + ((w ^ (r & 7)) << 4)
                                         : sb + CF::N64 * 128 * 128 + r * 32 + (((un - 8 * CF::N64) ^ ((r >> 2) & 1)) << 4);
            uint4 v = *reinterpret_cast<uint4*>(addr);
            uint16_t* hv = reinterpret_cast<uint16_t*>(&v);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (r >= rows_q || i < lo || i >= hi) hv[i] = 0;
            *reinterpret_cast<uint4*>(addr) = v;
          }
        }
        ptx::fence_proxy_async_smem();
        if (u >= 2) ptx::mbar_wait(&o_free[ts], ((u - 2) >> 1) & 1);  // TMEM set read out by the epilogue
        __syncwarp();
        ptx::fence_after_sync();
        if (lane == 0) {
#pragma unroll
          for (int c = 0; c < DP / 16; ++c) {
            const bool tail = c >= 4 * CF::N64;
            const uint64_t a = tail ? dQt : dQ + (uint64_t)((((c >> 2) * 128 * 128) + (c & 3) * 32) >> 4);
            const uint64_t b = tail ? dKt : dK + (uint64_t)((((c >> 2) * NK * 128) + (c & 3) * 32) >> 4);
            ptx::mma_bf16_ss(tS, a, b, idS, c > 0);
          }
          ptx::mma_commit(&s_full[ts]);
        }
        __syncwarp();
        ptx::mbar_wait(&p_full[ts], (u >> 1) & 1);
        ptx::fence_after_sync();
        if (lane == 0) {
          for (int c = 0; c < NK / 16; ++c) {  // O = P V, 16 keys per step (P over S: 8 columns per step)
            ptx::mma_bf16_ts(tO, tS + 8 * c, dV + (uint64_t)((c * 16 * 128) >> 4), idO, c > 0);
            if (CF::TAIL)
              ptx::mma_bf16_ts(tO + 64 * CF::N64, tS + 8 * c, dVt + (uint64_t)((c * 16 * 32) >> 4), idOt, c > 0);
          }
          ptx::mma_commit(&o_full[ts]);
          if (q + 1 == nq) ptx::mma_commit(&empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== softmax + epilogue: thread = query row = TMEM lane =====================
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int u = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int h = item % H, l0 = (item / H) * npos;
      const int sh = h * dh - ((h * dh) & ~7);
      for (int q = 0; q < nq; ++q, ++u) {
        const int ts = u & 1;
        const uint32_t tS = tmem + ts * 256, tO = tS + NK;
        const int r = warp * 32 + lane;             // row in the tile
        const int uu = q * 128 + r;                 // row in the group (position-major)
        const int p = uu / F, f = uu - p * F;
        const bool valid = p < npos && l0 + p < Lv && f < F;
        // the warp's key columns: the diagonal blocks of its rows' positions
        const int u_lo = q * 128 + warp * 32, u_hi = min(u_lo + 31, npos * F - 1);
        const int c_lo = u_lo < npos * F ? (u_lo / F) * F : 0;
        const int c_hi = u_lo < npos * F ? min(NK, (u_hi / F + 1) * F) : 0;
        const int k_lo = c_lo & ~15, k_hi = (c_hi + 15) & ~15;  // 16-column chunks covering them
        const int my_lo = p * F, my_hi = p * F + F;           // this row's keys
        ptx::mbar_wait(&s_full[ts], (u >> 1) & 1);
        ptx::fence_after_sync();
        // pass 1: row max over the row's own keys
        float mx = -INFINITY;
        for (int c0 = k_lo; c0 < k_hi; c0 += 16) {
          uint32_t v[16];
          ptx::tmem_ld16(tS + lane_off + c0, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i >= my_lo && c0 + i < my_hi) mx = fmaxf(mx, __uint_as_float(v[i]));
        }
        mx *= scale_log2;
        if (!valid) mx = 0.f;
        // pass 2: P = 2^(s*scale - max), bf16, over S (P chunk c0 -> columns
        // c0/2 .. c0/2 + 7, already read); row sum on the CUDA cores
        float lsum = 0.f;
        for (int c0 = k_lo; c0 < k_hi; c0 += 16) {
          uint32_t v[16], pk[8];
          ptx::tmem_ld16(tS + lane_off + c0, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const bool a = valid && c0 + i >= my_lo && c0 + i < my_hi;
            const bool b = valid && c0 + i + 1 >= my_lo && c0 + i + 1 < my_hi;
            const float ea = a ? ptx::ex2(__uint_as_float(v[i]) * scale_log2 - mx) : 0.f;
            const float eb = b ? ptx::ex2(__uint_as_float(v[i + 1]) * scale_log2 - mx) : 0.f;
            lsum += ea + eb;
            pk[i >> 1] = ptx::bf16x2(ea, eb);
          }
          ptx::tmem_st8p(tS + lane_off + c0 / 2, pk);
        }
        {  // zeros for the P columns outside the warp's chunks (after every S read)
          const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          for (int c = 0; c < k_lo / 2; c += 8) ptx::tmem_st8p(tS + lane_off + c, z);
          for (int c = k_hi / 2; c < NK / 2; c += 8) ptx::tmem_st8p(tS + lane_off + c, z);
        }
        ptx::tmem_st_wait();
        ptx::fence_before_sync();
        ptx::mbar_arrive(&p_full[ts]);
        ptx::mbar_wait(&o_full[ts], (u >> 1) & 1);
        ptx::fence_after_sync();
        // epilogue: O / l -> bf16 -> out row (f, l0 + p), head slot h*hs
        const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
        __nv_bfloat16* orow = valid ? o + ((int64_t)f * Lv + l0 + p) * ldo + (int64_t)h * hs : nullptr;
#pragma unroll
        for (int c = 0; c < DP / 16; ++c) {
          uint32_t v[16];
          ptx::tmem_ld16(tO + lane_off + sh + c * 16, v);  // head column c*16 + i = O column sh + c*16 + i
          ptx::tmem_ld_wait();
          if (orow && c * 16 < hs) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float a = (c * 16 + 2 * i < dh) ? __uint_as_float(v[2 * i]) * inv : 0.f;
              const float b = (c * 16 + 2 * i + 1 < dh) ? __uint_as_float(v[2 * i + 1]) * inv : 0.f;
              w[i] = ptx::bf16x2(a, b);
            }
            if (hs % 8 == 0 && c * 16 + 16 <= hs) {
              uint4* d = reinterpret_cast<uint4*>(orow + c * 16);
              d[0] = make_uint4(w[0], w[1], w[2], w[3]);
              d[1] = make_uint4(w[4], w[5], w[6], w[7]);
            } else {
              for (int i = 0; i < 8; ++i)
                if (c * 16 + 2 * i < hs) *reinterpret_cast<uint32_t*>(orow + c * 16 + 2 * i) = w[i];
            }
          }
        }
        ptx::fence_before_sync();
        ptx::mbar_arrive(&o_free[ts]);
      }
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 5) {
    ptx::fence_after_sync();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Map over one column block (q, k or v) of the position-major rows
// [Lv*F][ld] (row l*F + f): a box of R rows is R consecutive (position,
// frame) rows
int make_tm_map(CUtensorMap* m, const __nv_bfloat16* base, int64_t ld, int64_t cols, int64_t rows, int box_cols,
                int box_rows, CUtensorMapSwizzle swz) {
  const uint64_t dims[4] = {(uint64_t)cols, (uint64_t)rows, 1, 1};
  const uint64_t str[3] = {(uint64_t)ld * 2, (uint64_t)rows * ld * 2, (uint64_t)rows * ld * 2};
  const uint32_t box[4] = {(uint32_t)box_cols, (uint32_t)box_rows, 1, 1};
  return make_tmap_4d_bf16(m, base, dims, str, box, swz);
}

template <int DP>
int launch_dp(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F, int Lv, int H,
              int dh, cudaStream_t st, int hs) {
  using CF = CfgTm<DP>;
  const int npos = F <= 128 ? 128 / F : 1;
  const int NK = (npos * F + 15) / 16 * 16;
  const int rq = npos * std::min(F, 128), rkv = npos * F;  // rows per Q / K,V box
  const int64_t rows = (int64_t)Lv * F;
  CUtensorMap mq, mqt, mk, mkt, mv, mvt;
  const auto W128 = CU_TENSOR_MAP_SWIZZLE_128B, W32 = CU_TENSOR_MAP_SWIZZLE_32B;
  // q, k, v maps see D columns each (a box running past column D reads zeros)
  VC_TRY(make_tm_map(&mq, qkv, ld, D, rows, 64, rq, W128));
  VC_TRY(make_tm_map(&mk, qkv + D, ld, D, rows, 64, rkv, W128));
  VC_TRY(make_tm_map(&mv, qkv + 2 * D, ld, D, rows, 64, rkv, W128));
  mqt = mq; mkt = mk; mvt = mv;
  if (CF::TAIL) {
    VC_TRY(make_tm_map(&mqt, qkv, ld, D, rows, 16, rq, W32));
    VC_TRY(make_tm_map(&mkt, qkv + D, ld, D, rows, 16, rkv, W32));
    VC_TRY(make_tm_map(&mvt, qkv + 2 * D, ld, D, rows, 16, rkv, W32));
  }
  static bool attr = false;
  if (!attr) {
    VC_CHECK_CUDA(cudaFuncSetAttribute(temporal_tc_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr = true;
  }
  const int n_items = (int)cdiv(Lv, npos) * H;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int grid = std::min(n_items, sms);
  const float sl2 = (float)(1.4426950408889634 / sqrt((double)dh));
  temporal_tc_kernel<DP><<<grid, kTmThreads, CF::SMEM, st>>>(mq, mqt, mk, mkt, mv, mvt, o, ldo, F, Lv, H, dh, hs, npos,
                                                            NK, n_items, sl2);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

}  // namespace

bool temporal_tc_supported(int64_t ld, int64_t D, int F, int dh, const void* qkv) {
  const int DP = dh <= 64 ? 64 : dh <= 80 ? 80 : dh <= 128 ? 128 : 0;
  if (!DP || F <= 0 || F > 176) return false;
  if (dh % 8 != 0 && dh + 6 > DP) return false;  // head offset inside 16-byte TMA box starts
  const int npos = F <= 128 ? 128 / F : 1;
  const int NK = (npos * F + 15) / 16 * 16;
  const int nkmax = DP == 64 ? CfgTm<64>::NKMAX : DP == 80 ? CfgTm<80>::NKMAX : CfgTm<128>::NKMAX;
  if (NK > nkmax) return false;
  return (ld * 2) % 16 == 0 && ((uintptr_t)qkv % 16) == 0 && ((uintptr_t)((const __nv_bfloat16*)qkv + D) % 16) == 0;
}

int launch_temporal_tc(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F,
                       int Lv, int H, int dh, cudaStream_t st, int head_slot, int pos_major) {
  if (F <= 0 || Lv <= 0) return VC_OK;
  if (!pos_major) {
    set_error("tcgen05 temporal attention reads position-major q/k/v rows");
    return VC_EINVAL;
  }
  const int hs = head_slot ? head_slot : dh;
  if (!temporal_tc_supported(ld, D, F, dh, qkv)) {
    set_error("tcgen05 temporal attention: unsupported shape (F %d, dh %d)", F, dh);
    return VC_ENOTSUP;
  }
  if (dh <= 64) return launch_dp<64>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs);
  if (dh <= 80) return launch_dp<80>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs);
  return launch_dp<128>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs);
}

namespace {
int g_temporal_impl = 0;  // vc_set_temporal_impl (tests: force one kernel)
}

int launch_temporal_bf16(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F,
                         int Lv, int H, int dh, cudaStream_t st, int head_slot, int pos_major) {
  // Which kernel (measured, config 2 / 4 / 5 block, bench.py --config N):
  // the tcgen05 kernel matches the mma.sync one on 64-frame, dh-128
  // sequences (config 5: 0.151 vs 0.152 ms) but its per-item chain (TMA ->
  // S MMA -> TMEM softmax -> P.V MMA -> TMEM epilogue) leaves it slower on
  // short or narrow-head sequences (config 2, F 16: 0.24 vs 0.085 ms; config
  // 4, F 160: 5.5 vs 5.2 ms). VC_TEMPORAL_IMPL (tuning builds): 1 mma.sync
  // everywhere, 2 tcgen05 wherever supported, 0 (default) the measured rule.
  static const int env_impl = tuning_int("VC_TEMPORAL_IMPL", 0);
  const int impl = g_temporal_impl ? g_temporal_impl : env_impl;
  const bool tc = impl == 2 || (impl == 0 && F >= 64 && F <= 128 && dh >= 128);
  if (tc && pos_major && temporal_tc_supported(ld, D, F, dh, qkv))
    return launch_temporal_tc(qkv, ld, D, o, ldo, F, Lv, H, dh, st, head_slot, pos_major);
  return launch_temporal_mma(qkv, ld, D, o, ldo, F, Lv, H, dh, st, head_slot, pos_major);
}

}  // namespace vc

using namespace vc;

extern "C" int vc_set_temporal_impl(int32_t impl) {
  if (impl < 0 || impl > 2) { set_error("temporal impl must be 0 (measured rule), 1 (mma.sync) or 2 (tcgen05)"); return VC_EINVAL; }
  g_temporal_impl = impl;
  return VC_OK;
}
