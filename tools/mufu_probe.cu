// Probe: MUFU exp2 throughput for f32 vs packed f16x2 / bf16x2 operands
// (results per SM per clock), one launch per form, 148 x 4 CTAs of 512 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/mufu_probe tools/mufu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

constexpr int ITERS = 4096;

template <int FORM>
__global__ void k(uint32_t* out, float seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = __float_as_uint(seed * (threadIdx.x + i) * 1e-3f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (FORM == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
      if (FORM == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      if (FORM == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345678u) out[0] = s;
}

template <int FORM>
void run(const char* name, int per_op) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, threads = 512;
  k<FORM><<<blocks, threads>>>(out, 1.f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<FORM><<<blocks, threads>>>(out, 1.f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 5.0 * blocks * threads * (double)ITERS * 8;
  const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("%-10s %8.3f ms  %6.2f instr/clk/SM  %6.2f results/clk/SM (at the %d MHz rated clock)\n", name, ms, per_clk_sm,
         per_clk_sm * per_op, clk / 1000);
  cudaFree(out);
}

// warp-level mma.sync m16n8k16 bf16 -> f32: 8 independent accumulators per warp
__global__ void kmma(float* out) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  float d[8][4] = {};
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  {
    float* out;
    cudaMalloc(&out, 4);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int warps : {4, 8, 16, 32}) {
      const int blocks = sms * 2, threads = warps * 16;
      kmma<<<blocks, threads>>>(out);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) kmma<<<blocks, threads>>>(out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double flop = 5.0 * blocks * (threads / 32) * (double)(ITERS / 4) * 8 * 2 * 16 * 8 * 16;
      printf("mma.sync m16n8k16 bf16, %2d warps/SM: %.3f ms  %.1f TFLOP/s  (%.0f MAC/clk/SM at %d MHz)\n", warps, ms,
             flop / (ms * 1e-3) / 1e12, flop / 2 / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
    }
  }
  run<0>("f32", 1);
  run<1>("f16x2", 2);
  run<2>("bf16x2", 2);
  return 0;
}
