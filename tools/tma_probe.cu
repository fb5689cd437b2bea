// Probe: which 4-D TMA box / stride / base-offset combinations the temporal
// kernel's maps can use (one CTA, one cp.async.bulk.tensor per case).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tools/_bin/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>

#include "../paper_2501_08453_b200/csrc/vc_ptx.cuh"

using namespace vc;

__global__ void k(const __grid_constant__ CUtensorMap m, int x, int y, int z, uint32_t bytes, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, bytes);
    ptx::tma_load_4d(smem, &m, &bar, x, y, z, 0);
  }
  ptx::mbar_wait(&bar, 0);
  if (threadIdx.x == 0) out[0] = __bfloat162float(reinterpret_cast<__nv_bfloat16*>(smem)[0]);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int which = atoi(argv[1]);
  const int F = 16, Lv = 200, D = 1584, ld = 3 * D;
  __nv_bfloat16* buf;
  cudaMalloc(&buf, (size_t)F * Lv * ld * 2 + 4096);
  cudaMemset(buf, 0, (size_t)F * Lv * ld * 2 + 4096);
  float* out;
  cudaMalloc(&out, 16);
  CUtensorMap m;
  cuuint64_t dims[4], str[3];
  cuuint32_t box[4], es[4] = {1, 1, 1, 1};
  void* base = buf;
  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
  switch (which) {
    case 0:  // plain: cols x frames-major rows, box 64 x 128 rows
      dims[0] = D; dims[1] = (cuuint64_t)F * Lv; dims[2] = 1; dims[3] = 1;
      str[0] = ld * 2; str[1] = (cuuint64_t)F * Lv * ld * 2; str[2] = str[1];
      box[0] = 64; box[1] = 128; box[2] = 1; box[3] = 1;
      break;
    case 1:  // monotonic (cols, Lv, F), box 64 x 8 pos x 16 frames
      dims[0] = D; dims[1] = Lv; dims[2] = F; dims[3] = 1;
      str[0] = ld * 2; str[1] = (cuuint64_t)Lv * ld * 2; str[2] = (cuuint64_t)F * Lv * ld * 2;
      box[0] = 64; box[1] = 8; box[2] = 16; box[3] = 1;
      break;
    case 2:  // permuted (cols, F, Lv), box 64 x 16 frames x 8 pos
      dims[0] = D; dims[1] = F; dims[2] = Lv; dims[3] = 1;
      str[0] = (cuuint64_t)Lv * ld * 2; str[1] = ld * 2; str[2] = (cuuint64_t)F * Lv * ld * 2;
      box[0] = 64; box[1] = 16; box[2] = 8; box[3] = 1;
      break;
    case 3:  // as 1, base + D (k block, 3168 B offset)
      dims[0] = D; dims[1] = Lv; dims[2] = F; dims[3] = 1;
      str[0] = ld * 2; str[1] = (cuuint64_t)Lv * ld * 2; str[2] = (cuuint64_t)F * Lv * ld * 2;
      box[0] = 64; box[1] = 8; box[2] = 16; box[3] = 1;
      base = buf + D;
      break;
    case 4:  // as 1, box 64 x 1 x 128 (one position, 128 frames)... F = 16 so box 16
      dims[0] = D; dims[1] = Lv; dims[2] = F; dims[3] = 1;
      str[0] = ld * 2; str[1] = (cuuint64_t)Lv * ld * 2; str[2] = (cuuint64_t)F * Lv * ld * 2;
      box[0] = 64; box[1] = 1; box[2] = 16; box[3] = 1;
      break;
    case 5:  // as 1 with a 4th dim of 1 and stride 0? (last stride = str[1] * F)
      dims[0] = D; dims[1] = Lv; dims[2] = F; dims[3] = 1;
      str[0] = ld * 2; str[1] = (cuuint64_t)Lv * ld * 2; str[2] = (cuuint64_t)F * Lv * ld * 2;
      box[0] = 64; box[1] = 8; box[2] = 16; box[3] = 1;
      sw = CU_TENSOR_MAP_SWIZZLE_NONE;
      break;
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUresult r = ((EncFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, str, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("case %d encode %d\n", which, (int)r);
  const uint32_t bytes = box[0] * box[1] * box[2] * box[3] * 2;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 32, 64 * 1024>>>(m, 0, 0, 0, bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("case %d: %s\n", which, cudaGetErrorString(e));
  return 0;
}
