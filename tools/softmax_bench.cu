// Micro-benchmark of the attention softmax exp phase in isolation: W warps per
// SM, each thread turning 64 fp32 logits into 32 packed bf16x2 (FFMA2 + MUFU
// ex2, every POLY-th pair on the FMA-pipe polynomial), repeated.  Reports
// clocks per 64-element row step per warp, to compare with the in-kernel
// trace (tools/attn_trace.cu).
#include <cstdint>
#include <cstdio>

#include "../paper_2501_08453_b200/csrc/vc_ptx.cuh"

using namespace vc;

template <int POLY, int N>
__global__ void k(uint32_t* out, int iters, long long* clk, float m) {
  float r[N];
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = -0.01f * ((threadIdx.x * 7 + i * 13) & 255);
  __shared__ __align__(16) uint32_t sink[128 * 32];
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  const float2 sc2 = make_float2(1.4427f, 1.4427f);
  for (int it = 0; it < iters; ++it) {
    const float mm = -m - 1e-7f * it;  // loop-variant: nothing hoists
    const float2 nm2 = make_float2(mm, mm);
    uint32_t pk[N / 2];
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      float2 e = ptx::ffma2(make_float2(r[i], r[i + 1]), sc2, nm2);
      if (POLY == -1 || POLY == -2) {  // f16x2 MUFU: one instruction per pair
        uint32_t hx, hy;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hx) : "f"(e.y), "f"(e.x));
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(hy) : "r"(hx));
        if (POLY == -1) { pk[i >> 1] = hy; continue; }
        // f16x2 -> bf16x2
        float lo, hi;
        asm("{.reg .f16 a, b; mov.b32 {a, b}, %2; cvt.f32.f16 %0, a; cvt.f32.f16 %1, b;}" : "=f"(lo), "=f"(hi) : "r"(hy));
        e = make_float2(lo, hi);
      } else if (POLY > 0 && ((i >> 1) % (POLY > 0 ? POLY : 1)) == POLY - 1) {
        e = ptx::ex2_poly2(e);
      } else {
        e.x = ptx::ex2(e.x);
        e.y = ptx::ex2(e.y);
      }
      pk[i >> 1] = ptx::bf16x2(e.x, e.y);
    }
    // the P store of the real kernel: 16-byte smem stores
    const uint32_t rowp = ptx::smem_u32(sink) + (threadIdx.x & 127) * 128;
#pragma unroll
    for (int u = 0; u < N / 8; ++u)
      ptx::sts128(rowp + ((u ^ (threadIdx.x & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
  }
  acc = sink[threadIdx.x];
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int POLY, int N>
void run(int warps) {
  uint32_t* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 1000;
  k<POLY, N><<<148, warps * 32>>>(out, iters, clk, 0.5f);
  k<POLY, N><<<148, warps * 32>>>(out, iters, clk, 0.5f);
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters;
  const int mufu_pairs = POLY < 0 ? N / 4 : POLY ? (N / 2) - (N / 2) / POLY : N / 2;
  printf("POLY %d N %3d warps/SM %2d: %.0f clk per step (MUFU bound %.0f)\n", POLY, N, warps, per,
         2.0 * mufu_pairs * 8 * (warps / 4));
  cudaFree(out); cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0, 64>(w);
    run<4, 64>(w);
    run<3, 64>(w);
    run<2, 64>(w);
    run<-1, 64>(w);
    run<-2, 64>(w);
  }
  return 0;
}
