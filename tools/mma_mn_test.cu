// Correctness probe for tcgen05.mma with an MN-major B operand (B = V rows:
// K = keys, N = head dims contiguous), the form the temporal kernel uses:
// one M128 x N x K16 MMA, A from shared memory ("ss") or TMEM ("ts"), B in
// the SW128 (N = 64) or SW32 (N = 16) MN-major layout, compared with a CPU
// product of small integers (exact in fp32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tools/_bin/mma_mn_test tools/mma_mn_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_bf16.h>

#include "../paper_2501_08453_b200/csrc/vc_ptx.cuh"

using namespace vc;

// A [128][16], B [16][N] (row k = key), D [128][N]
template <int N, bool TS, int SWB>
__global__ void k(const float* A, const float* B, float* D, int mode_b_major) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[16 * 128];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4) ptx::tmem_alloc(&slot, 256);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  // A: K-major SW128, row m at m*128, 16-byte chunk i at (i ^ (m & 7))
  for (int i = threadIdx.x; i < 128 * 128 / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(sA)[i] = 0;
  for (int i = threadIdx.x; i < 16 * 128 / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(sB)[i] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int m = e / 16, kk = e % 16, ch = kk / 8;
    reinterpret_cast<__nv_bfloat16*>(sA + m * 128 + ((ch ^ (m & 7)) << 4))[kk % 8] = __float2bfloat16(A[e]);
  }
  for (int e = threadIdx.x; e < 16 * N; e += blockDim.x) {
    const int kk = e / N, n = e % N, ch = n / 8;
    if (SWB == 128)  // row kk at kk*128, chunk ch at ch ^ (kk & 7)
      reinterpret_cast<__nv_bfloat16*>(sB + kk * 128 + ((ch ^ (kk & 7)) << 4))[n % 8] = __float2bfloat16(B[e]);
    else  // SW32: row kk at kk*32, chunk ch at ch ^ ((kk >> 2) & 1)
      reinterpret_cast<__nv_bfloat16*>(sB + kk * 32 + ((ch ^ ((kk >> 2) & 1)) << 4))[n % 8] = __float2bfloat16(B[e]);
  }
  ptx::fence_proxy_async_smem();
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = slot;
  if (TS && warp < 4) {  // A into TMEM columns 128..135 (bf16x2 per column)
    const int m = warp * 32 + lane;
    uint32_t r[8];
    for (int c = 0; c < 8; ++c) r[c] = ptx::bf16x2(A[m * 16 + 2 * c], A[m * 16 + 2 * c + 1]);
    ptx::tmem_st8p(tmem + ((uint32_t)(warp * 32) << 16) + 128, r);
    ptx::tmem_st_wait();
  }
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  if (warp == 4 && lane == 0) {
    const uint32_t id = ptx::idesc_bf16_f32(128, N) | (mode_b_major ? (1u << 16) : 0u);
    const uint64_t bd = SWB == 128 ? ptx::smem_desc(ptx::smem_u32(sB), 16 * 128, 1024, ptx::kLayoutSW128)
                                   : ptx::smem_desc(ptx::smem_u32(sB), 0, 256, ptx::kLayoutSW32);
    if (TS) ptx::mma_bf16_ts(tmem, tmem + 128, bd, id, 0u);
    else ptx::mma_bf16_ss(tmem, ptx::smem_desc(ptx::smem_u32(sA), 0, 1024, ptx::kLayoutSW128), bd, id, 0u);
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::fence_after_sync();
  if (warp < 4) {
    const int m = warp * 32 + lane;
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
      ptx::tmem_ld_wait();
      for (int i = 0; i < 16 && c + i < N; ++i) D[m * N + c + i] = __uint_as_float(r[i]);
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 4) { ptx::fence_after_sync(); ptx::tmem_dealloc(tmem, 256); }
}

// K-major B (B stored [N][16] like K rows), SW128, SBO 1024: the shape probe
// for N not a multiple of 16 (M = 128, cta_group::1)
template <int N>
__global__ void kk(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[208 * 128];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4) ptx::tmem_alloc(&slot, 256);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  for (int i = threadIdx.x; i < 128 * 128 / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(sA)[i] = 0;
  for (int i = threadIdx.x; i < 208 * 128 / 2; i += blockDim.x) reinterpret_cast<uint16_t*>(sB)[i] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int m = e / 16, kq = e % 16, ch = kq / 8;
    reinterpret_cast<__nv_bfloat16*>(sA + m * 128 + ((ch ^ (m & 7)) << 4))[kq % 8] = __float2bfloat16(A[e]);
  }
  for (int e = threadIdx.x; e < N * 16; e += blockDim.x) {  // B[k][n] -> row n, element k
    const int kq = e / N, n = e % N, ch = kq / 8;
    reinterpret_cast<__nv_bfloat16*>(sB + n * 128 + ((ch ^ (n & 7)) << 4))[kq % 8] = __float2bfloat16(B[e]);
  }
  ptx::fence_proxy_async_smem();
  ptx::fence_before_sync();
  __syncthreads();
  ptx::fence_after_sync();
  const uint32_t tmem = slot;
  if (warp == 4 && lane == 0) {
    const uint32_t id = ptx::idesc_bf16_f32(128, N);
    ptx::mma_bf16_ss(tmem, ptx::smem_desc(ptx::smem_u32(sA), 0, 1024, ptx::kLayoutSW128),
                     ptx::smem_desc(ptx::smem_u32(sB), 0, 1024, ptx::kLayoutSW128), id, 0u);
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::fence_after_sync();
  if (warp < 4) {
    const int m = warp * 32 + lane;
    for (int c = 0; c < N; c += 8) {
      uint32_t r[8];
      ptx::tmem_ld8p(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
      ptx::tmem_ld_wait();
      for (int i = 0; i < 8 && c + i < N; ++i) D[m * N + c + i] = __uint_as_float(r[i]);
    }
  }
  ptx::fence_before_sync();
  __syncthreads();
  if (warp == 4) { ptx::fence_after_sync(); ptx::tmem_dealloc(tmem, 256); }
}

template <int N>
void run_k(const char* name) {
  std::vector<float> A(128 * 16), B(16 * N), D(128 * N), R(128 * N, 0.f);
  for (auto& v : A) v = (float)(rand() % 7 - 3);
  for (auto& v : B) v = (float)(rand() % 7 - 3);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n)
      for (int q = 0; q < 16; ++q) R[m * N + n] += A[m * 16 + q] * B[q * N + n];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, D.size() * 4);
  kk<N><<<1, 160>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: CUDA error %s\n", name, cudaGetErrorString(e)); exit(1); }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (size_t i = 0; i < D.size(); ++i) err = std::max(err, (double)fabs(D[i] - R[i]));
  printf("%s: max |err| %g\n", name, err);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

template <int N, bool TS, int SWB>
void run(const char* name) {
  std::vector<float> A(128 * 16), B(16 * N), D(128 * N), R(128 * N, 0.f);
  for (auto& v : A) v = (float)(rand() % 7 - 3);
  for (auto& v : B) v = (float)(rand() % 7 - 3);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n)
      for (int kk = 0; kk < 16; ++kk) R[m * N + n] += A[m * 16 + kk] * B[kk * N + n];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  k<N, TS, SWB><<<1, 160>>>(dA, dB, dD, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: CUDA error %s\n", name, cudaGetErrorString(e)); exit(1); }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (size_t i = 0; i < D.size(); ++i) err = std::max(err, (double)fabs(D[i] - R[i]));
  printf("%s: max |err| %g  (D[0..3] %g %g %g %g ref %g %g %g %g)\n", name, err, D[0], D[1], D[2], D[3], R[0], R[1],
         R[2], R[3]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0 || which == 1) run<64, false, 128>("ss  MN-major B SW128 N64");
  if (which == 0 || which == 2) run<64, true, 128>("ts  MN-major B SW128 N64");
  if (which == 0 || which == 3) run<16, false, 32>("ss  MN-major B SW32 N16");
  if (which == 0 || which == 4) run<16, true, 32>("ts  MN-major B SW32 N16");
  if (which == 0 || which == 5) {  // M = 128 shapes with N % 16 == 8
    run_k<112>("ss  K-major B M128 N112");
    run_k<120>("ss  K-major B M128 N120");
    run_k<72>("ss  K-major B M128 N72");
    run_k<200>("ss  K-major B M128 N200");
  }
  return 0;
}
