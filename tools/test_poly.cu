// Standalone check of the FMA-pipe exp2 polynomials the attention kernels
// offload exponentials to (ptx::ex2_poly2: cubic; ptx::ex2_poly2_d2: degree 2)
// against exp2 in double precision over [-140, 10] (tools/, not the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/_bin/test_poly tools/test_poly.cu
#include <cstdio>
#include <cmath>
#include "../paper_2501_08453_b200/csrc/vc_ptx.cuh"
template <int D2>
__global__ void k(const float* x, float* y, int n) {
  int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < n) {
    float2 r = D2 ? vc::ptx::ex2_poly2_d2(make_float2(x[i], x[i + 1])) : vc::ptx::ex2_poly2(make_float2(x[i], x[i + 1]));
    y[i] = r.x; y[i + 1] = r.y;
  }
}
template <int D2>
void run(const char* name, float* x, float* y, int n) {
  k<D2><<<n / 256, 128>>>(x, y, n);
  cudaDeviceSynchronize();
  double worst = 0; int nan = 0;
  for (int i = 0; i < n; ++i) {
    double ref = exp2((double)x[i]);
    if (std::isnan(y[i])) { if (nan < 5) printf("nan at x=%g\n", x[i]); ++nan; continue; }
    if (ref > 1e-30) worst = fmax(worst, fabs(y[i] - ref) / ref);
  }
  printf("%s: nan %d, worst relative error %.3g (x >= -99); y(-inf)=%g y(0)=%g y(8)=%g y(-150)=%g\n", name, nan, worst,
         y[0], y[2], y[3], y[4]);
}
int main() {
  const int n = 1 << 16;
  float *x, *y;
  cudaMallocManaged(&x, n * 4); cudaMallocManaged(&y, n * 4);
  for (int i = 0; i < n; ++i) x[i] = -140.f + 150.f * i / n;
  x[0] = -INFINITY; x[1] = -0.0f; x[2] = 0.f; x[3] = 8.f; x[4] = -150.f;
  run<0>("cubic   ", x, y, n);
  run<1>("degree 2", x, y, n);
  return 0;
}
