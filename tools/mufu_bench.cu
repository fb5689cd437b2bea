// Micro-benchmark: MUFU.EX2 / FFMA2 / F2FP throughput per SM on this GPU
// (one CTA per SM, W warps).  Prints warp-instructions per clock per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a[i]));
      } else if (MODE == 2) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 15]));
        acc += r;
      } else {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  k<MODE><<<148, warps * 32>>>(out, iters, clk);
  k<MODE><<<148, warps * 32>>>(out, iters, clk);
  long long c[148];
  cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  double ops = (double)iters * 16 * warps;
  printf("%-22s warps/SM %2d: %.3f warp-inst/clk/SM (= %.1f lanes/clk/SM)\n", name, warps, ops / c[0],
         32 * ops / c[0]);
  cudaFree(out); cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2.approx.ftz", w);
    run<1>("ex2.approx", w);
    run<2>("cvt.rn.bf16x2.f32", w);
    run<3>("fma (dependent x16)", w);
  }
  return 0;
}
