// The reference's frame encoder and forward noising, fused: toy_vae_encode
// (model.py:381-403: zero-pad to a multiple of d, d x d block average, fixed
// 3 -> C cosine channel mix) followed by q_sample (diffusion.py:77-84:
// sqrt(abar_t) x0 + sqrt(1 - abar_t) noise) -- the first thing each rank
// does with its round-robin frames in run_sp_iteration (executor.py:535-546).
// HBM-bound: one thread per latent pixel reads its d x d x 3 block.
#include <math.h>

#include "vc_kernels.h"

namespace vc {

namespace {

struct VaeArgs {
  int32_t F, H, W, d, C, gh, gw;
  float mix[3][16];  // [3][C] channel mix, C <= 16
  float sab, somab;  // sqrt(abar_t), sqrt(1 - abar_t); (1, 0) = plain encode
};

__global__ void __launch_bounds__(256) vae_encode_kernel(const float* __restrict__ px, const float* __restrict__ noise,
                                                         float* __restrict__ out, VaeArgs a) {
  const int64_t n = (int64_t)a.F * a.gh * a.gw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / ((int64_t)a.gh * a.gw));
    const int rem = (int)(i - (int64_t)f * a.gh * a.gw);
    const int y = rem / a.gw, x = rem - y * a.gw;
    double s0 = 0, s1 = 0, s2 = 0;  // the block sum in fp64 (the reference pools in float64)
    for (int dy = 0; dy < a.d; ++dy) {
      const int yy = y * a.d + dy;
      if (yy >= a.H) break;  // zero padding
      const float* row = px + (((int64_t)f * a.H + yy) * a.W) * 3;
      for (int dx = 0; dx < a.d; ++dx) {
        const int xx = x * a.d + dx;
        if (xx >= a.W) break;
        s0 += row[xx * 3 + 0];
        s1 += row[xx * 3 + 1];
        s2 += row[xx * 3 + 2];
      }
    }
    const double inv = 1.0 / ((double)a.d * a.d);
    const float p0 = (float)(s0 * inv), p1 = (float)(s1 * inv), p2 = (float)(s2 * inv);
    float* o = out + i * a.C;
    const float* nz = noise ? noise + i * a.C : nullptr;
    for (int c = 0; c < a.C; ++c) {
      const float lat = p0 * a.mix[0][c] + p1 * a.mix[1][c] + p2 * a.mix[2][c];
      o[c] = nz ? a.sab * lat + a.somab * nz[c] : lat;
    }
  }
}

}  // namespace

}  // namespace vc

using namespace vc;

extern "C" int vc_vae_encode_frames(const float* pixels, const float* noise, float* latents, int32_t F, int32_t H,
                                    int32_t W, int32_t downsample, int32_t channels, double sqrt_alpha_bar,
                                    double sqrt_one_minus_alpha_bar, void* stream) {
  if (F <= 0 || H <= 0 || W <= 0) return VC_OK;
  if (downsample < 1 || channels < 1 || channels > 16) {
    set_error("toy VAE: downsample must be >= 1 and 1..16 latent channels, got %d / %d", downsample, channels);
    return VC_EINVAL;
  }
  VaeArgs a;
  a.F = F; a.H = H; a.W = W; a.d = downsample; a.C = channels;
  a.gh = (H + downsample - 1) / downsample;
  a.gw = (W + downsample - 1) / downsample;
  for (int j = 0; j < 3; ++j)  // model.py:399-403: sqrt(2/3) cos(pi (2j+1) i / 6)
    for (int i = 0; i < 16; ++i)
      a.mix[j][i] = i < channels ? (float)(sqrt(2.0 / 3.0) * cos(M_PI * (2 * j + 1) * i / 6.0)) : 0.f;
  a.sab = (float)sqrt_alpha_bar;
  a.somab = (float)sqrt_one_minus_alpha_bar;
  const int64_t n = (int64_t)F * a.gh * a.gw;
  const int blocks = (int)std::min<int64_t>(cdiv(n, 256), 148 * 32);
  vae_encode_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(pixels, noise, latents, a);
  VC_CHECK_LAUNCH();
  return VC_OK;
}
