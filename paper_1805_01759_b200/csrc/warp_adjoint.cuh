// Column-lane adjoint of the warp-per-pixel solvers (k_warp_solver.cu, k_warp_c64.cu).
#pragma once

#include "common.cuh"

namespace tb {

// acc[t] += conj(A[i][c + 32 t]) r_y[i] over all n rows for NP column passes (lane = column; only the
// last pass can be partial: `last` = lane + 32 (NP - 1) < width), rows unrolled by 8 (loop and
// address overhead once per 8 rows), fp32 packed FFMA2 sharing each broadcast r_y load.
// Element (row i, pass t) lives at ap[i rs + t ps]: shared memory column-major (rs = 1, so the 8
// unrolled rows are immediate offsets; ps = 32 column strides) or global row-major (rs = m, ps = 32).
template <int NP, bool ASMEM, bool CM>
__device__ __forceinline__ void adjoint_passes(float2* acc, const float2* ap, int stride, int pstride, const float4* ryv, int n, bool last) {
  const int rs = CM ? 1 : stride;
  int i = 0;
#pragma unroll 1
  for (; i + 8 <= n; i += 8, ap += 8 * rs) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 r = ryv[i + u];
#pragma unroll
      for (int t = 0; t < NP; ++t)
        if (t < NP - 1 || last) cfma_conj_x2(acc[t], ASMEM ? ap[u * rs + t * pstride] : __ldg(ap + u * rs + t * pstride), r);
    }
  }
#pragma unroll 1
  for (; i < n; ++i, ap += rs) {
    const float4 r = ryv[i];
#pragma unroll
    for (int t = 0; t < NP; ++t)
      if (t < NP - 1 || last) cfma_conj_x2(acc[t], ASMEM ? ap[t * pstride] : __ldg(ap + t * pstride), r);
  }
}
// runtime pass count -> compile-time unrolled body (no all-idle passes are issued)
template <int NP, int MAXT, bool ASMEM, bool CM>
__device__ __forceinline__ void adjoint_dispatch(int passes, float2* acc, const float2* ap, int stride, int pstride, const float4* ryv, int n, bool last) {
  if constexpr (NP <= MAXT) {
    if (passes == NP) {
      adjoint_passes<NP, ASMEM, CM>(acc, ap, stride, pstride, ryv, n, last);
      return;
    }
    adjoint_dispatch<NP + 1, MAXT, ASMEM, CM>(passes, acc, ap, stride, pstride, ryv, n, last);
  }
}

}  // namespace tb
