// C-ABI entry for the tensor-core attention on plain fp32 [s][D] operands
// (vc_attention_bf16, include/vchitect_b200.h): pack q, k into the padded
// [s][H][DP] bf16 layouts and v into V^T [H][DP][keys] (with the ones column
// the kernel accumulates the row sum in), run launch_attn_tc, widen the bf16
// output to fp32.  The block forward builds the same layouts in its QKV GEMM
// epilogue; this entry exists for the kernel-level contract and its tests.
#include <math.h>

#include "vc_attn_tc.h"
#include "vc_kernels.h"

namespace vc {
namespace {

inline size_t aup(size_t v) { return (v + 1023) / 1024 * 1024; }

struct AttnWs {
  int DP;
  int64_t ld;
  size_t q, k, vt, o, total;
};
AttnWs attn_ws(int32_t sq, int32_t sk, int32_t dim, int32_t heads) {
  AttnWs w{};
  w.DP = attn_tc_head_pad(dim / heads);
  w.ld = round_up((int64_t)sk, 8);
  size_t o = 0;
  w.q = o; o = aup(o + (size_t)sq * heads * w.DP * 2);
  w.k = o; o = aup(o + (size_t)sk * heads * w.DP * 2);
  w.vt = o; o = aup(o + (size_t)heads * w.DP * w.ld * 2);
  w.o = o; o = aup(o + (size_t)sq * dim * 2);
  w.total = o;
  return w;
}

// x [rows][H*dh] fp32 -> [rows][H][DP] bf16, zero head padding
__global__ void pack_rows_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t rows, int H,
                                 int dh, int DP) {
  const int64_t n = rows * H * DP;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % DP);
    const int64_t rh = e / DP;
    const int h = (int)(rh % H);
    const int64_t r = rh / H;
    y[e] = __float2bfloat16_rn(d < dh ? x[r * H * dh + h * dh + d] : 0.f);
  }
}

// v [keys][H*dh] fp32 -> V^T [H][DP][ld] bf16; padding row d == dh holds 1.0
// (the ones column: the P.V MMA then accumulates the softmax row sum)
__global__ void pack_vt_kernel(const float* __restrict__ v, __nv_bfloat16* __restrict__ vt, int64_t keys,
                               int64_t ld, int H, int dh, int DP) {
  const int64_t n = (int64_t)H * DP * ld;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = e % ld;
    const int64_t hd = e / ld;
    const int d = (int)(hd % DP), h = (int)(hd / DP);
    float val = 0.f;
    if (key < keys) val = d < dh ? v[key * H * dh + h * dh + d] : (d == dh ? 1.f : 0.f);
    vt[e] = __float2bfloat16_rn(val);
  }
}

__global__ void widen_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = __bfloat162float(x[e]);
}

inline int blocks_for(int64_t n) { return (int)std::min<int64_t>(cdiv(n, 256), 148 * 8); }

}  // namespace
}  // namespace vc

using namespace vc;

extern "C" {

size_t vc_attention_bf16_workspace_bytes(int32_t sq, int32_t sk, int32_t dim, int32_t heads) {
  if (sq < 0 || sk < 1 || heads < 1 || dim % heads != 0) return 0;
  const AttnWs w = attn_ws(sq, sk, dim, heads);
  return w.DP ? w.total : 0;
}

int vc_attention_bf16(const float* q, const float* k, const float* v, float* out, int32_t sq, int32_t sk,
                      int32_t dim, int32_t heads, int32_t n_weighted, float key_weight, void* ws, size_t ws_bytes,
                      void* stream) {
  if (heads < 1 || dim % heads != 0) {
    set_error("feature dim %d not divisible by %d heads", dim, heads);
    return VC_EINVAL;
  }
  if (sq < 0 || sk < 1) { set_error("bad attention lengths sq=%d sk=%d", sq, sk); return VC_EINVAL; }
  if (n_weighted < 0 || n_weighted > sk || (n_weighted > 0 && !(key_weight > 0.f))) {
    set_error("weighted keys: need 0 <= n_weighted <= sk and key_weight > 0");
    return VC_EINVAL;
  }
  const int dh = dim / heads;
  const AttnWs w = attn_ws(sq, sk, dim, heads);
  if (!w.DP) { set_error("tensor-core attention supports head dims up to 128, got %d", dh); return VC_ENOTSUP; }
  if (ws_bytes < w.total) { set_error("attention workspace too small"); return VC_EINVAL; }
  if (sq == 0) return VC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  char* W = (char*)ws;
  typedef __nv_bfloat16 bf;
  bf *qb = (bf*)(W + w.q), *kb = (bf*)(W + w.k), *vt = (bf*)(W + w.vt), *ob = (bf*)(W + w.o);
  pack_rows_kernel<<<blocks_for((int64_t)sq * heads * w.DP), 256, 0, st>>>(q, qb, sq, heads, dh, w.DP);
  pack_rows_kernel<<<blocks_for((int64_t)sk * heads * w.DP), 256, 0, st>>>(k, kb, sk, heads, dh, w.DP);
  pack_vt_kernel<<<blocks_for((int64_t)heads * w.DP * w.ld), 256, 0, st>>>(v, vt, sk, w.ld, heads, dh, w.DP);
  VC_CHECK_LAUNCH();
  AttnTcParams a{};
  a.Lq = sq; a.Lk = sk; a.H = heads; a.dh = dh;
  a.n_bias = n_weighted; a.bias_log2 = n_weighted > 0 ? (float)log2((double)key_weight) : 0.f;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)dh));
  a.out = ob; a.ld_out = dim; a.col_off = 0; a.out_seq_rows = 0;
  VC_TRY(launch_attn_tc(a, qb, kb, vt, 1, sq, sk, w.ld, w.DP, st));
  widen_kernel<<<blocks_for((int64_t)sq * dim), 256, 0, st>>>(ob, out, (int64_t)sq * dim);
  VC_CHECK_LAUNCH();
  return VC_OK;
}

}  // extern "C"
