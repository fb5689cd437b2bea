// Standalone timing + per-phase trace of the tcgen05 attention kernel
// (vc_attn_tc3.cu) on the config-2 full-sequence shape.  Built by
// tools/build_attn_trace.sh with -DVC_ATTN_TRACE (the trace writes clock64()
// stamps of one CTA into a __device__ array; the library build has none).
//
//   attn_trace [Lq Lk H dh n_bias reps]   -> kernel ms, TFLOP/s, trace CSV on stdout
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../paper_2501_08453_b200/csrc/vc_attn_tc.h"

namespace vc {
int attn_trace3_read(unsigned long long* host);
int attn_tracep_read(unsigned long long* host);
int attn_cta_read(unsigned long long* host);
}

__global__ void fill_kernel(__nv_bfloat16* x, size_t n, uint32_t seed, float amp) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    x[i] = __float2bfloat16_rn(amp * (((h & 0xffff) / 32768.f) - 1.f));
  }
}

int main(int argc, char** argv) {
  const int Lq = argc > 1 ? atoi(argv[1]) : 21600;
  const int Lk = argc > 2 ? atoi(argv[2]) : 21856;
  const int H = argc > 3 ? atoi(argv[3]) : 24;
  const int dh = argc > 4 ? atoi(argv[4]) : 66;
  const int n_bias = argc > 5 ? atoi(argv[5]) : 256;
  const int reps = argc > 6 ? atoi(argv[6]) : 10;
  const int DP = vc::attn_tc_head_pad(dh);
  const int ld_key = (Lk + 127) / 128 * 128;
  __nv_bfloat16 *q, *k, *vt, *out;
  const size_t nq = (size_t)Lq * H * DP, nk = (size_t)Lk * H * DP, nv = (size_t)H * DP * ld_key;
  cudaMalloc(&q, nq * 2); cudaMalloc(&k, nk * 2); cudaMalloc(&vt, nv * 2);
  cudaMalloc(&out, (size_t)Lq * H * 80 * 2 + 4096);
  fill_kernel<<<1024, 256>>>(q, nq, 1, 2.f);
  fill_kernel<<<1024, 256>>>(k, nk, 2, 2.f);
  fill_kernel<<<1024, 256>>>(vt, nv, 3, 1.f);
  vc::AttnTcParams p{};
  p.Lq = Lq; p.Lk = Lk; p.H = H; p.dh = dh; p.n_bias = n_bias;
  p.bias_log2 = 2.f; p.scale_log2 = 1.4426950408889634f / sqrtf((float)dh);
  p.out = getenv("VC_TRACE_NO_OUT") ? nullptr : out; p.ld_out = getenv("VC_TRACE_LD80") ? (int64_t)H * 80 : (int64_t)H * dh; p.col_off = 0; p.out_seq_rows = Lq;
  if (getenv("VC_TRACE_SLOT")) { p.head_slot = 80; p.ld_out = (int64_t)H * 80; }  // the block's layout: 80-column head slots
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int rc = vc::launch_attn_tc(p, q, k, vt, 1, Lq, Lk, ld_key, DP, 0);
  if (rc) { fprintf(stderr, "launch rc %d\n", rc); return 1; }
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) vc::launch_attn_tc(p, q, k, vt, 1, Lq, Lk, ld_key, DP, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { fprintf(stderr, "cuda: %s\n", cudaGetErrorString(err)); return 1; }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double flop = 4.0 * Lq * (double)Lk * H * dh;
  printf("# Lq %d Lk %d H %d dh %d DP %d: %.4f ms  %.1f TFLOP/s (algorithmic dh)\n", Lq, Lk, H, dh, DP, ms,
         flop / ms / 1e9);
  if (getenv("VC_TRACE_CTA")) {  // per-CTA phases of the LAST launch, per-SM gaps between CTAs
    std::vector<unsigned long long> c(16384 * 5);
    vc::attn_cta_read(c.data());
    const int nb = 16384;  // every CTA that stamped (one or two tiles per CTA)
    double pro = 0, main_ = 0, epi = 0, gap = 0;
    int ng = 0, n = 0;
    std::vector<std::vector<std::pair<unsigned long long, unsigned long long>>> sm(256);
    for (int b = 0; b < nb && b < 16384; ++b) {
      const unsigned long long* e = &c[b * 5];
      if (!e[0] || !e[1] || !e[2] || !e[3]) continue;
      pro += (double)(e[1] - e[0]); main_ += (double)(e[2] - e[1]); epi += (double)(e[3] - e[2]); ++n;
      sm[e[4] & 255].push_back({e[0], e[3]});
    }
    for (auto& v : sm) {
      std::sort(v.begin(), v.end());
      for (size_t i = 1; i < v.size(); ++i) { gap += (double)v[i].first - (double)v[i - 1].second; ++ng; }
    }
    printf("# CTAs %d: clk per CTA prologue (entry -> first S) %.0f, main (-> last P.V) %.0f, epilogue (-> stored) %.0f; "
           "mean gap between CTAs on one SM %.0f clk (%d gaps)\n", n, pro / n, main_ / n, epi / n, ng ? gap / ng : 0.0, ng);
  }
  const int nj = 256;
  std::vector<unsigned long long> tr(18 * 512 * 8);
  const char* impl = getenv("VC_ATTN_IMPL");
  const int nroles = (impl && atoi(impl) == 3) ? 17 : 18;
  const int iv = impl ? atoi(impl) : 4;
  const int trc = iv == 3 ? vc::attn_trace3_read(tr.data()) : vc::attn_tracep_read(tr.data());
  if (trc == 0) {
    unsigned long long t0 = ~0ull;
    for (auto v : tr) if (v && v < t0) t0 = v;
    printf("role,j,s0,s1,s2,s3,s4,s5,s6,s7\n");
    for (int r = 0; r < nroles; ++r)
      for (int j = 0; j < nj; ++j) {
        const unsigned long long* e = &tr[(r * nj + j) * 8];
        if (!e[0]) continue;
        printf("%d,%d", r, j);
        for (int s = 0; s < 8; ++s) printf(",%lld", e[s] ? (long long)(e[s] - t0) : -1ll);
        printf("\n");
      }
  }
  return 0;
}
