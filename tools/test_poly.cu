// standalone check of ptx::ex2_poly2 (tools/, not part of the library)
#include <cstdio>
#include <cmath>
#include "../paper_2501_08453_b200/csrc/vc_ptx.cuh"
__global__ void k(const float* x, float* y, int n) {
  int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < n) {
    float2 r = vc::ptx::ex2_poly2(make_float2(x[i], x[i + 1]));
    y[i] = r.x; y[i + 1] = r.y;
  }
}
int main() {
  const int n = 1 << 16;
  float *x, *y;
  cudaMallocManaged(&x, n * 4); cudaMallocManaged(&y, n * 4);
  for (int i = 0; i < n; ++i) x[i] = -140.f + 150.f * i / n;
  x[0] = -INFINITY; x[1] = -0.0f; x[2] = 0.f; x[3] = 8.f;
  k<<<n / 256, 128>>>(x, y, n);
  cudaDeviceSynchronize();
  double worst = 0; int nan = 0;
  for (int i = 0; i < n; ++i) {
    double ref = exp2((double)x[i]);
    if (std::isnan(y[i])) { if (nan < 5) printf("nan at x=%g\n", x[i]); ++nan; continue; }
    if (ref > 1e-30) worst = fmax(worst, fabs(y[i] - ref) / ref);
  }
  printf("nan %d worst rel %g  y(-inf)=%g y(0)=%g y(8)=%g y(-1.5)=%g\n", nan, worst, y[0], y[2], y[3], y[n/2]);
  return 0;
}
