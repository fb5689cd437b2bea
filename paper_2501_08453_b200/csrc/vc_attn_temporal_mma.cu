// Temporal-branch attention on tensor cores (bf16 path), model.py:238-244:
// one sequence per spatial position l made of the F tokens {f*Lv + l},
// numerics.py:87-107 per head.
//
// The sequences are short (F = 16..160) and there are Lv*H of them, so the
// right tile is the warp-level m16n8k16 MMA: one warp owns (position, head,
// 16-frame query tile), keeps Q in registers, streams 16-key blocks of K and V
// through a warp-private smem tile (ldmatrix / ldmatrix.trans feed the B
// operands) and runs a flash-style online softmax in registers. tcgen05's
// smallest tile (M = 64) would waste >= 75% of the MMA on 16-frame sequences;
// the kernel is bound by reading q, k, v once from HBM (~F/2 flop per byte).
//
// In : qkv bf16 [rows][ld], q at col 0 (pointer pre-offset), k at +D, v at +2D
// Out: o bf16 [rows][ldo] at head columns h*dh (pointer pre-offset)
#include "vc_kernels.h"
#include "vc_ptx.cuh"
#include "vc_tuning.h"

namespace vc {

namespace {

constexpr int kWarps = 4;
constexpr float kFixedMargin = 60.0f;  // = attn::kFixedMaxMargin (vc_attn_tc_common.cuh)

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}

// global -> smem async copies; src_size 0 zero-fills (padding / frames past F)
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

// Long sequences (SHARED): one CTA per (position, head) stages the whole
// sequence's K and V in shared memory ONCE (every warp of the CTA reads them;
// per-warp staging re-reads them F/16 times and waits for each 16-key block),
// then its warps take the 16-frame query tiles in turn (<= 8 warps, as many
// as balance the tiles: 10 tiles -> 5 warps x 2).
constexpr int kWarpsShared = 8;

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// KS: head-dim k-steps of 16 (dh <= 16*KS); NT: output n-tiles of 8 (dh <= 8*NT);
// VEC16: the head slice of every row is 16-byte aligned (16-byte copies)
template <int KS, int NT, bool VEC16, bool SHARED>
__global__ void __launch_bounds__(SHARED ? kWarpsShared * 32 : kWarps * 32, SHARED ? 2 : KS <= 6 ? 4 : 1)
    temporal_mma_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, int64_t D,
                        __nv_bfloat16* __restrict__ o, int64_t ldo, int F, int Lv, int H, int dh,
                        float scale_log2, int hs, int pos_major) {
  constexpr int KPAD = 16 * KS + 8;  // smem row pitch (elements): conflict-free ldmatrix
  const int NW = SHARED ? (int)(blockDim.x >> 5) : kWarps;
  __shared__ __align__(16) __nv_bfloat16 sKw[SHARED ? 1 : kWarps][16][KPAD];
  __shared__ __align__(16) __nv_bfloat16 sVw[SHARED ? 1 : kWarps][16][KPAD];
  extern __shared__ __align__(16) __nv_bfloat16 sKV[];  // SHARED: K [Fpad][KPAD], then V
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int QT = (F + 15) / 16;
  int qt0, h, l;
  if constexpr (SHARED) {
    h = (int)(blockIdx.x % (unsigned)H);  // heads fastest: concurrent CTAs read the same rows
    l = (int)(blockIdx.x / (unsigned)H);
    qt0 = warp;
  } else {
    const int64_t item = (int64_t)blockIdx.x * kWarps + warp;
    if (item >= (int64_t)Lv * H * QT) return;
    qt0 = (int)(item % QT);
    h = (int)((item / QT) % H);
    l = (int)(item / ((int64_t)QT * H));
  }
  const int64_t col0 = (int64_t)h * dh;
  const int words = 8 * KS;  // 32-bit words per padded row (16*KS bf16)
  const int Fpad = QT * 16;
  if constexpr (SHARED) {
    // ---- the sequence's K and V rows (zero padded to Fpad x 16KS) into shared memory ----
    __nv_bfloat16* sK = sKV;
    __nv_bfloat16* sV = sKV + (size_t)Fpad * KPAD;
    if (VEC16) {
      constexpr int CH = 2 * KS;
      for (int e = threadIdx.x; e < Fpad * CH; e += NW * 32) {
        const int r = e / CH, c = (e - r * CH) * 8;
        const bool ok = r < F && c < dh;
        const int64_t rr0 = pos_major ? (int64_t)l * F + (ok ? r : 0) : (int64_t)(ok ? r : 0) * Lv + l;
        const __nv_bfloat16* row = qkv + rr0 * ld + col0 + (ok ? c : 0);
        cp_async16(ptx::smem_u32(sK + r * KPAD + c), row + D, ok);
        cp_async16(ptx::smem_u32(sV + r * KPAD + c), row + 2 * D, ok);
      }
    } else {
      for (int e = threadIdx.x; e < Fpad * words; e += NW * 32) {
        const int r = e / words, c = 2 * (e - r * words);
        const bool ok = r < F && c < dh;
        const int64_t rr0 = pos_major ? (int64_t)l * F + (ok ? r : 0) : (int64_t)(ok ? r : 0) * Lv + l;
        const __nv_bfloat16* row = qkv + rr0 * ld + col0 + (ok ? c : 0);
        cp_async4(ptx::smem_u32(sK + r * KPAD + c), row + D, ok);
        cp_async4(ptx::smem_u32(sV + r * KPAD + c), row + 2 * D, ok);
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }
  // one 16-frame query tile (a lambda so the per-warp kernel keeps its
  // straight-line register allocation: no loop-carried state)
  auto attend_tile = [&](const int qt) {
  const int f0 = qt * 16;

  // ---- Q fragments (A operand, row-major 16 x 16 per k-step), zero padded ----
  uint32_t qa[KS][4];
  {
    const int fr0 = f0 + g, fr1 = f0 + g + 8;
    const __nv_bfloat16* r0 = qkv + (pos_major ? (int64_t)l * F + fr0 : (int64_t)fr0 * Lv + l) * ld + col0;
    const __nv_bfloat16* r1 = qkv + (pos_major ? (int64_t)l * F + fr1 : (int64_t)fr1 * Lv + l) * ld + col0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int c0 = ks * 16 + 2 * t, c1 = c0 + 8;
      qa[ks][0] = (fr0 < F && c0 < dh) ? *reinterpret_cast<const uint32_t*>(r0 + c0) : 0u;
      qa[ks][1] = (fr1 < F && c0 < dh) ? *reinterpret_cast<const uint32_t*>(r1 + c0) : 0u;
      qa[ks][2] = (fr0 < F && c1 < dh) ? *reinterpret_cast<const uint32_t*>(r0 + c1) : 0u;
      qa[ks][3] = (fr1 < F && c1 < dh) ? *reinterpret_cast<const uint32_t*>(r1 + c1) : 0u;
    }
  }

  float oacc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t kbase = SHARED ? ptx::smem_u32(sKV) : ptx::smem_u32(&sKw[SHARED ? 0 : warp][0][0]);
  uint32_t vbase = SHARED ? ptx::smem_u32(sKV + (size_t)Fpad * KPAD) : ptx::smem_u32(&sVw[SHARED ? 0 : warp][0][0]);

  for (int k0 = 0; k0 < F; k0 += 16) {
    if constexpr (SHARED) {
      if (k0 > 0) { kbase += 16 * KPAD * 2; vbase += 16 * KPAD * 2; }
    } else {
    // ---- stage K and V rows of this 16-key block (zero padded) with async
    //      copies: all loads in flight at once, no register round trip ----
    __syncwarp();
    if (VEC16) {  // 16-byte copies (head slice 16-byte aligned)
      constexpr int CH = 2 * KS;  // 16-byte chunks per padded row
      for (int e = lane; e < 16 * CH; e += 32) {
        const int r = e / CH, c = (e - r * CH) * 8;
        const int fr = k0 + r;
        const bool ok = fr < F && c < dh;
        const int64_t rr0 = pos_major ? (int64_t)l * F + (ok ? fr : 0) : (int64_t)(ok ? fr : 0) * Lv + l;
        const __nv_bfloat16* row = qkv + rr0 * ld + col0 + (ok ? c : 0);
        cp_async16(ptx::smem_u32(&sKw[SHARED ? 0 : warp][r][c]), row + D, ok);
        cp_async16(ptx::smem_u32(&sVw[SHARED ? 0 : warp][r][c]), row + 2 * D, ok);
      }
    } else {
      for (int e = lane; e < 16 * words; e += 32) {
        const int r = e / words, c = 2 * (e - r * words);
        const int fr = k0 + r;
        const bool ok = fr < F && c < dh;
        const int64_t rr0 = pos_major ? (int64_t)l * F + (ok ? fr : 0) : (int64_t)(ok ? fr : 0) * Lv + l;
        const __nv_bfloat16* row = qkv + rr0 * ld + col0 + (ok ? c : 0);
        cp_async4(ptx::smem_u32(&sKw[SHARED ? 0 : warp][r][c]), row + D, ok);
        cp_async4(ptx::smem_u32(&sVw[SHARED ? 0 : warp][r][c]), row + 2 * D, ok);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    }

    // ---- S = Q K^T for keys k0..k0+15 (two n-tiles of 8 keys) ----
    float s[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        // lanes 0-7: rows (keys) 8nt..8nt+7 at cols 16ks; lanes 8-15: cols 16ks+8
        const int rr = 8 * nt + (lane & 7), cc = 16 * ks + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1;
        ldsm_x2(kbase + (rr * KPAD + cc) * 2, b0, b1);
        mma_bf16_16816(s[nt], qa[ks], b0, b1);
      }
    }
    // ---- softmax (rows g and g+8 of the tile; keys past F masked) with the
    //      fixed offset of the tc kernels (vc_attn_tc_common.cuh
    //      kFixedMaxMargin): the first key block's exact row max + 60, then
    //      no per-block max, shuffles or O rescale ----
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const bool ok = k0 + 8 * nt + 2 * t + i < F;
        s[nt][i] = ok ? s[nt][i] * scale_log2 : -INFINITY;
        s[nt][2 + i] = ok ? s[nt][2 + i] * scale_log2 : -INFINITY;
      }
    }
    if (k0 == 0) {
      float bm0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
      float bm1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 1));
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 1));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
      m0 = bm0 + kFixedMargin;
      m1 = bm1 + kFixedMargin;
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        s[nt][i] = ptx::ex2(s[nt][i] - m0);
        s[nt][2 + i] = ptx::ex2(s[nt][2 + i] - m1);
        l0 += s[nt][i];  // per-thread partial sums; reduced over the quad at the end
        l1 += s[nt][2 + i];
      }
    }
    // ---- O += P V (P from the S accumulators, bf16 A fragment) ----
    uint32_t pa[4];
    pa[0] = ptx::bf16x2(s[0][0], s[0][1]);
    pa[1] = ptx::bf16x2(s[0][2], s[0][3]);
    pa[2] = ptx::bf16x2(s[1][0], s[1][1]);
    pa[3] = ptx::bf16x2(s[1][2], s[1][3]);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      // lanes 0-7: keys 0-7 at cols 8j; lanes 8-15: keys 8-15 (transposed load)
      const int rr = (lane & 7) + ((lane >> 3) & 1) * 8;
      uint32_t b0, b1;
      ldsm_x2_t(vbase + (rr * KPAD + 8 * j) * 2, b0, b1);
      mma_bf16_16816(oacc[j], pa, b0, b1);
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const int fr0 = f0 + g, fr1 = f0 + g + 8;
  // hs: output head stride (dh, or a padded slot whose columns past dh get
  // the zeros oacc holds there: V's padding is zero-filled in smem)
  __nv_bfloat16* o0 = o + ((int64_t)fr0 * Lv + l) * ldo + (int64_t)h * hs;
  __nv_bfloat16* o1 = o + ((int64_t)fr1 * Lv + l) * ldo + (int64_t)h * hs;
  int j0 = 0;
  if (hs == 8 * NT) {
    // full-width head slot (16-byte aligned rows): a 4x4 word transpose inside
    // each quad gives thread t the 8 columns of n-tile 4*jg + t, stored as one
    // 16-byte vector per row instead of four 4-byte ones
    const int lb = lane & ~3;
#pragma unroll
    for (int jg = 0; jg + 4 <= NT; jg += 4) {
      uint32_t a[4], b[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a[k] = ptx::bf16x2(oacc[jg + k][0] * i0, oacc[jg + k][1] * i0);
        b[k] = ptx::bf16x2(oacc[jg + k][2] * i1, oacc[jg + k][3] * i1);
      }
      uint32_t oa[4] = {0u, 0u, 0u, 0u}, ob[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int want = (t + r) & 3;  // the n-tile whose words this lane hands to lane (t + r) & 3
        const uint32_t sa = want == 0 ? a[0] : want == 1 ? a[1] : want == 2 ? a[2] : a[3];
        const uint32_t sb = want == 0 ? b[0] : want == 1 ? b[1] : want == 2 ? b[2] : b[3];
        const int src = lb | ((t - r) & 3);
        const uint32_t ra = __shfl_sync(0xffffffffu, sa, src), rb = __shfl_sync(0xffffffffu, sb, src);
        const int pos = (t - r) & 3;  // the source lane's column pair inside n-tile jg + t
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          oa[q] = pos == q ? ra : oa[q];
          ob[q] = pos == q ? rb : ob[q];
        }
      }
      const int c = 8 * (jg + t);
      if (fr0 < F) *reinterpret_cast<uint4*>(o0 + c) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
      if (fr1 < F) *reinterpret_cast<uint4*>(o1 + c) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
    }
    j0 = NT / 4 * 4;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < j0) continue;
    const int c = 8 * j + 2 * t;
    if (c < hs) {
      if (fr0 < F) *reinterpret_cast<__nv_bfloat162*>(o0 + c) = __floats2bfloat162_rn(oacc[j][0] * i0, oacc[j][1] * i0);
      if (fr1 < F) *reinterpret_cast<__nv_bfloat162*>(o1 + c) = __floats2bfloat162_rn(oacc[j][2] * i1, oacc[j][3] * i1);
    }
  }
  };
  if constexpr (SHARED) {
    for (int qt = qt0; qt < QT; qt += NW) attend_tile(qt);
  } else {
    attend_tile(qt0);
  }
}

template <int KS, int NT>
int launch_ks(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F, int Lv,
              int H, int dh, cudaStream_t st, int hs, int pm) {
  const float sl2 = (float)(1.4426950408889634 / sqrt((double)dh));
  const bool vec16 = dh % 8 == 0 && ld % 8 == 0 && D % 8 == 0 && ((uintptr_t)qkv % 16) == 0;
  // long sequences: K / V staged once per (position, head) CTA (measured rule, profiles/r02/temporal)
  static const int min_shared = tuning_int("VC_TEMPORAL_SHARED_MIN_F", 48);
  const int Fpad = (F + 15) / 16 * 16;
  const size_t smem = (size_t)2 * Fpad * (16 * KS + 8) * 2;
  if (F >= min_shared && smem <= 110 * 1024) {
    const int64_t blocks = (int64_t)Lv * H;
    if (blocks > 2147483647) { set_error("temporal grid too large"); return VC_ENOTSUP; }
    auto kern = vec16 ? temporal_mma_kernel<KS, NT, true, true> : temporal_mma_kernel<KS, NT, false, true>;
    static bool attr[2] = {false, false};
    if (!attr[vec16]) {
      VC_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
      attr[vec16] = true;
    }
    const int QT = Fpad / 16, rounds = (QT + kWarpsShared - 1) / kWarpsShared;
    const int nw = (QT + rounds - 1) / rounds;  // warps that balance the query tiles
    kern<<<(unsigned)blocks, nw * 32, smem, st>>>(qkv, ld, D, o, ldo, F, Lv, H, dh, sl2, hs, pm);
    VC_CHECK_LAUNCH();
    return VC_OK;
  }
  const int64_t items = (int64_t)Lv * H * ((F + 15) / 16);
  const int64_t blocks = cdiv(items, kWarps);
  if (blocks > 2147483647) { set_error("temporal grid too large"); return VC_ENOTSUP; }
  if (vec16)
    temporal_mma_kernel<KS, NT, true, false><<<(unsigned)blocks, kWarps * 32, 0, st>>>(qkv, ld, D, o, ldo, F, Lv, H, dh, sl2, hs, pm);
  else
    temporal_mma_kernel<KS, NT, false, false><<<(unsigned)blocks, kWarps * 32, 0, st>>>(qkv, ld, D, o, ldo, F, Lv, H, dh, sl2, hs, pm);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

}  // namespace

int launch_temporal_mma(const __nv_bfloat16* qkv, int64_t ld, int64_t D, __nv_bfloat16* o, int64_t ldo, int F,
                        int Lv, int H, int dh, cudaStream_t st, int head_slot, int pos_major) {
  if (F <= 0 || Lv <= 0) return VC_OK;
  const int hs = head_slot ? head_slot : dh;
  if (hs < dh || (head_slot && head_slot > 16 * ((dh + 15) / 16))) {
    set_error("temporal attention head slot %d does not fit dh %d", head_slot, dh);
    return VC_EINVAL;
  }
  if (dh % 2 != 0 || dh > 128 || (ld % 2) || (D % 2) || (ldo % 2)) {
    set_error("tensor-core temporal attention needs an even head dim <= 128 (dh %d)", dh);
    return VC_ENOTSUP;
  }
  const int ks = (dh + 15) / 16;
  switch (ks) {
    case 1: return launch_ks<1, 2>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    case 2: return launch_ks<2, 4>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    case 3: return launch_ks<3, 6>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    case 4: return launch_ks<4, 8>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    case 5: return launch_ks<5, 10>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    case 6: return launch_ks<6, 12>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    case 7: return launch_ks<7, 14>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
    default: return launch_ks<8, 16>(qkv, ld, D, o, ldo, F, Lv, H, dh, st, hs, pos_major);
  }
}

}  // namespace vc
