// SIMT (FFMA) flash attention over strided sequences.
//
// Semantics: numerics.py:87-107 (per-head softmax(q k^T / sqrt(dh)) v,
// non-causal) applied to every sequence of a branch: spatial (model.py:230-235,
// one sequence per frame), temporal (model.py:238-244, one sequence per
// spatial position: token stride Lv) and the anchored full sequence
// (model.py:247-260) whose F identical text copies are collapsed into one
// shared key segment with logit bias log(F) (exact by the key/value
// permutation invariance, reference tests/test_numerics.py:131-140).
//
// Used for the fp32 parity path (all three branches) and for the temporal
// branch of the bf16 path, whose sequences are F (16..160) tokens long: there
// the work is ~F/2 flop per byte and the kernel is judged against HBM.
//
// CTA = 4 warps x 4 query rows = 16 queries of one (sequence, head); keys are
// staged 32 at a time in shared memory, lane j owns key j of the tile for
// the logits and head dims {lane, lane+32, ...} for the output.
#include "vc_kernels.h"

namespace vc {

constexpr int kAttnRowsPerWarp = 4;
constexpr int kAttnWarps = 4;
constexpr int kAttnRows = kAttnRowsPerWarp * kAttnWarps;
constexpr int kAttnKeys = 32;

template <typename T, typename OutT, int DH_MAX>
__global__ void __launch_bounds__(128) attn_simt_kernel(AttnArgs<T, OutT> a) {
  constexpr int DPL = DH_MAX / 32;  // head dims per lane
  __shared__ float Ks[kAttnKeys][DH_MAX + 1];
  __shared__ float Vs[kAttnKeys][DH_MAX];
  __shared__ float Qs[kAttnRows][DH_MAX];
  __shared__ float Kbias[kAttnKeys];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = blockIdx.y, s = blockIdx.z;
  const int q0 = blockIdx.x * kAttnRows;
  const int dh = a.dh;
  const int64_t col = (int64_t)h * dh;

  // Q rows of this CTA (zero for rows past the sequence end).
  for (int e = tid; e < kAttnRows * dh; e += blockDim.x) {
    int r = e / dh, d = e - r * dh;
    int t = q0 + r;
    float v = 0.f;
    if (t < a.len_q) v = to_f32(a.q[(s * a.q_seq_stride + t * a.q_tok_stride) * a.ldq + col + d]);
    Qs[r][d] = v;
  }

  float m[kAttnRowsPerWarp], l[kAttnRowsPerWarp], o[kAttnRowsPerWarp][DPL];
#pragma unroll
  for (int r = 0; r < kAttnRowsPerWarp; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int i = 0; i < DPL; ++i) o[r][i] = 0.f;
  }

  const int total = a.na + a.len_k;
  for (int k0 = 0; k0 < total; k0 += kAttnKeys) {
    __syncthreads();
    for (int e = tid; e < kAttnKeys * dh; e += blockDim.x) {
      int j = e / dh, d = e - j * dh;
      int key = k0 + j;
      float kv = 0.f, vv = 0.f;
      if (key < a.na) {
        kv = to_f32(a.ka[(int64_t)key * a.lda + col + d]);
        vv = to_f32(a.va[(int64_t)key * a.lda + col + d]);
      } else if (key < total) {
        int64_t row = s * a.k_seq_stride + (int64_t)(key - a.na) * a.k_tok_stride;
        kv = to_f32(a.k[row * a.ldk + col + d]);
        vv = to_f32(a.v[row * a.ldk + col + d]);
      }
      Ks[j][d] = kv;
      Vs[j][d] = vv;
    }
    if (tid < kAttnKeys) {
      int key = k0 + tid;
      Kbias[tid] = key < a.na ? a.log2_weight_a : (key < total ? 0.f : -INFINITY);
    }
    __syncthreads();

#pragma unroll
    for (int r = 0; r < kAttnRowsPerWarp; ++r) {
      const int row = warp * kAttnRowsPerWarp + r;
      float sc = 0.f;
      for (int d = 0; d < dh; ++d) sc = fmaf(Qs[row][d], Ks[lane][d], sc);
      sc = sc * a.scale_log2 + Kbias[lane];  // -inf for keys past the end
      const float m_new = fmaxf(m[r], warp_max(sc));
      const float p = exp2f(sc - m_new);
      const float corr = exp2f(m[r] - m_new);
      l[r] = l[r] * corr + warp_sum(p);
      m[r] = m_new;
#pragma unroll
      for (int i = 0; i < DPL; ++i) o[r][i] *= corr;
#pragma unroll 8
      for (int j = 0; j < kAttnKeys; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          const int d = lane + 32 * i;
          if (d < DH_MAX) o[r][i] = fmaf(pj, Vs[j][d], o[r][i]);
        }
      }
    }
  }

#pragma unroll
  for (int r = 0; r < kAttnRowsPerWarp; ++r) {
    const int t = q0 + warp * kAttnRowsPerWarp + r;
    if (t >= a.len_q) continue;
    const float inv = 1.f / l[r];
    OutT* orow = a.o + (s * a.o_seq_stride + t * a.o_tok_stride) * a.ldo + col;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int d = lane + 32 * i;
      if (d < dh) orow[d] = from_f32<OutT>(o[r][i] * inv);
    }
  }
}

template <typename T, typename OutT>
int launch_attn_simt(const AttnArgs<T, OutT>& a, cudaStream_t st) {
  if (a.dh > 128) {
    set_error("SIMT attention supports head dim <= 128, got %d", a.dh);
    return VC_ENOTSUP;
  }
  if (a.len_q <= 0 || a.n_seq <= 0) return VC_OK;
  if (a.na + a.len_k <= 0) {
    set_error("attention needs at least one key");
    return VC_EINVAL;
  }
  if (a.n_seq > 65535 || a.heads > 65535) {
    set_error("attention grid too large (n_seq %d heads %d)", a.n_seq, a.heads);
    return VC_ENOTSUP;
  }
  dim3 grid((unsigned)cdiv(a.len_q, kAttnRows), a.heads, a.n_seq);
  if (a.dh <= 64)
    attn_simt_kernel<T, OutT, 64><<<grid, 128, 0, st>>>(a);
  else
    attn_simt_kernel<T, OutT, 128><<<grid, 128, 0, st>>>(a);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

template int launch_attn_simt<float, float>(const AttnArgs<float, float>&, cudaStream_t);
template int launch_attn_simt<__nv_bfloat16, __nv_bfloat16>(const AttnArgs<__nv_bfloat16, __nv_bfloat16>&, cudaStream_t);

}  // namespace vc
