// Micro-benchmark: tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) issue /
// execution rate per SM for small N, with A from shared memory ("ss") or from
// tensor memory ("ts"), and the cost of a commit after every g MMAs.
// Operands are garbage (uninitialised smem / TMEM): only timing matters.
#include <cstdint>
#include <cstdio>

#include "../paper_2501_08453_b200/csrc/vc_ptx.cuh"

using namespace vc;

template <int N, bool TS, int G>
__global__ void k(long long* clk, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, dummy;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) { ptx::mbar_init(&bar, 1); ptx::mbar_init(&dummy, 1); ptx::fence_barrier_init(); }
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, N);
    const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
    long long t0 = 0;
    uint32_t phase = 0;
    for (int it = 0; it < iters + 1; ++it) {
      if (it == 1) t0 = clock64();
      if (ptx::elect_one()) {
        for (int g = 0; g < 64 / G; ++g) {
#pragma unroll
          for (int c = 0; c < G; ++c) {
            const uint64_t bd = ptx::smem_desc(b + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128);
            if (TS)
              ptx::mma_bf16_ts(tmem + 256, tmem + 8 * (c & 7), bd, id, 1u);
            else
              ptx::mma_bf16_ss(tmem + 256, ptx::smem_desc(a + (c & 3) * 32, 0, 1024, ptx::kLayoutSW128), bd, id, 1u);
          }
          ptx::mma_commit(g + 1 == 64 / G ? &bar : &dummy);
        }
      }
      __syncwarp();
      // wait for the last commit of this iteration (64/G phases completed)
      ptx::mbar_wait(&bar, phase);
      phase ^= 1;
    }
    if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 0) { ptx::fence_after_sync(); ptx::tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, int G>
void run() {
  long long* clk;
  cudaMalloc(&clk, 148 * 8);
  const int iters = 200;
  cudaFuncSetAttribute(k<N, TS, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<N, TS, G><<<148, 64, 64 * 1024>>>(clk, iters);
  k<N, TS, G><<<148, 64, 64 * 1024>>>(clk, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (iters * 64.0);
  printf("N %3d %s commit/%2d MMAs: %.1f clk per MMA (ideal %.0f)  %s\n", N, TS ? "ts" : "ss", G, per,
         128.0 * N * 16 * 2 / 8192, cudaGetErrorString(e));
  cudaFree(clk);
}

int main() {
  run<64, false, 4>(); run<64, true, 4>();
  run<80, false, 4>(); run<80, true, 4>();
  run<128, false, 4>(); run<128, true, 4>();
  run<256, false, 4>(); run<256, true, 4>();
  run<64, true, 16>(); run<80, true, 16>(); run<128, true, 16>();
  run<64, true, 1>(); run<128, true, 1>();
  return 0;
}
