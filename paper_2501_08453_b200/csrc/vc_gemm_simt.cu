// fp32 SIMT GEMM for the fp32 parity path:
//   out[m][n] = sum_k A[m][k] * B[k][n] + bias[n] + R[m][n]
// A row-major [M][K] (lda), B row-major [K][N] (ldb) -- the reference's
// `x @ W` orientation (model.py:184, :190) with gamma folded into B.
// 64x64x16 tiles, 256 threads, 4x4 outputs per thread, fp32 FFMA.
// (The bf16 path uses the tcgen05 GEMM in vc_gemm_tc.cu.)
#include "vc_kernels.h"

namespace vc {

__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmF32Args g) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
    // A tile: 64 rows x 16 k; thread loads 4 consecutive k of one row.
    {
      int r = tid >> 2, kk = (tid & 3) * 4;
      int64_t m = m0 + r;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int k = k0 + kk + i;
        As[kk + i][r] = (m < g.M && k < g.K) ? g.A[m * g.lda + k] : 0.f;
      }
    }
    // B tile: 16 k x 64 n; thread loads 4 consecutive n of one k.
    {
      int kk = tid >> 4, c = (tid & 15) * 4;
      int k = k0 + kk;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int n = n0 + c + i;
        Bs[kk][c + i] = (k < g.K && n < g.N) ? g.B[(int64_t)k * g.ldb + n] : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = acc[i][j];
      if (g.bias) v += g.bias[n];
      if (g.R) v += g.R[m * g.ldr + n];
      g.out[m * g.ldo + n] = v;
    }
  }
}

int launch_gemm_f32(const GemmF32Args& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return VC_OK;
  dim3 grid((unsigned)cdiv(g.N, 64), (unsigned)cdiv(g.M, 64));
  if (grid.y > 65535u) {
    set_error("fp32 GEMM: M=%lld too large for the SIMT path", (long long)g.M);
    return VC_ENOTSUP;
  }
  gemm_f32_kernel<<<grid, 256, 0, st>>>(g);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

}  // namespace vc
