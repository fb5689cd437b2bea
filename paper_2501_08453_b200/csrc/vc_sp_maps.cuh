// Sequence-parallel row maps, shared by the host (the vc_sp_row_map export
// the exact-equality tests read) and every kernel that moves rows between a
// rank's local layout and the assembled sequences -- one definition, so the
// tested map IS the one the unpack kernels and the attention epilogue use.
//
// Rank r holds visual positions [vb[r], vb[r+1]) of every frame, frame-major:
// local row m = f * vc_r + (l - vb[r]) (executor.py:571-626 chunks, frame by
// frame in the order the reference builds them).  The reference assembles
// each sequence with a stable argsort of the chunks' global indices
// (executor.py:349-370, :606-617); for visual rows that order is (f, l)
// lexicographic, i.e. token f * Lv + l.
#pragma once
#include <stdint.h>

namespace vc {

// local row m of rank r -> (frame f, position l)
__host__ __device__ __forceinline__ void sp_row_to_token(const int32_t* vb, int r, int64_t m, int& f, int& l) {
  const int vc = vb[r + 1] - vb[r];
  f = (int)(m / vc);
  l = vb[r] + (int)(m - (int64_t)f * vc);
}

// owner rank of position l (vb = contiguous bounds over P ranks)
__host__ __device__ __forceinline__ int sp_owner(const int32_t* vb, int P, int l) {
  int r = 0;
  while (r + 1 < P && vb[r + 1] <= l) ++r;
  return r;
}

// (frame f, position l) owned by rank r -> its local row
__host__ __device__ __forceinline__ int64_t sp_token_to_row(const int32_t* vb, int r, int f, int l) {
  return (int64_t)f * (vb[r + 1] - vb[r]) + (l - vb[r]);
}

}  // namespace vc
