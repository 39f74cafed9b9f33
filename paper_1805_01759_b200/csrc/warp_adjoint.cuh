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

// c += (a, a) * r: one packed FFMA2 with a scalar broadcast operand
__device__ __forceinline__ void ffma2_bcast(float2& c, float a, float2 r) {
  asm("{\n\t.reg .b64 cc, aa, rr;\n\t"
      "mov.b64 cc, {%0, %1};\n\t"
      "mov.b64 aa, {%2, %2};\n\t"
      "mov.b64 rr, {%3, %4};\n\t"
      "fma.rn.f32x2 cc, aa, rr, cc;\n\t"
      "mov.b64 {%0, %1}, cc;\n\t}"
      : "+f"(c.x), "+f"(c.y)
      : "f"(a), "f"(r.x), "f"(r.y));
}

// RBPG form of the column-lane adjoint: r_y is stored as plain (r.x, r.y) pairs (one 8-byte
// broadcast per row instead of the 16-byte (r.x, r.y, r.y, -r.x) quad: the quad load costs two
// shared-memory wavefronts, and the r_y broadcasts were 23% of the kernel's shared wavefronts), and
// each pass keeps two independent packed accumulators, p += a.x r and q += a.y r, combined once:
// conj(a) r summed over rows = (p.x + q.y, p.y - q.x).  Rows are still summed in order.
template <int NP, bool ASMEM, bool CM>
__device__ __forceinline__ void adjoint_passes2(float2* acc, const float2* ap, int stride, int pstride, const float2* ry2, int n, bool last) {
  const int rs = CM ? 1 : stride;
  float2 p[NP], q[NP];
#pragma unroll
  for (int t = 0; t < NP; ++t) p[t] = q[t] = make_float2(0.f, 0.f);
  int i = 0;
#pragma unroll 1
  for (; i + 8 <= n; i += 8, ap += 8 * rs) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float2 r = ry2[i + u];
#pragma unroll
      for (int t = 0; t < NP; ++t)
        if (t < NP - 1 || last) {
          const float2 a = ASMEM ? ap[u * rs + t * pstride] : __ldg(ap + u * rs + t * pstride);
          ffma2_bcast(p[t], a.x, r);
          ffma2_bcast(q[t], a.y, r);
        }
    }
  }
#pragma unroll 1
  for (; i < n; ++i, ap += rs) {
    const float2 r = ry2[i];
#pragma unroll
    for (int t = 0; t < NP; ++t)
      if (t < NP - 1 || last) {
        const float2 a = ASMEM ? ap[t * pstride] : __ldg(ap + t * pstride);
        ffma2_bcast(p[t], a.x, r);
        ffma2_bcast(q[t], a.y, r);
      }
  }
#pragma unroll
  for (int t = 0; t < NP; ++t) acc[t] = make_float2(p[t].x + q[t].y, p[t].y - q[t].x);
}
template <int NP, int MAXT, bool ASMEM, bool CM>
__device__ __forceinline__ void adjoint_dispatch2(int passes, float2* acc, const float2* ap, int stride, int pstride, const float2* ry2, int n, bool last) {
  if constexpr (NP <= MAXT) {
    if (passes == NP) {
      adjoint_passes2<NP, ASMEM, CM>(acc, ap, stride, pstride, ry2, n, last);
      return;
    }
    adjoint_dispatch2<NP + 1, MAXT, ASMEM, CM>(passes, acc, ap, stride, pstride, ry2, n, last);
  }
}

// Variant of adjoint_passes2 taking r_y from registers: lane i holds row i + 32 q in ryr[q] (the
// lane = row layout of the residual step), broadcast per row with two shuffles instead of a shared
// load.  Measured: shuffles compete with the shared loads for the same MIO path, so this is slower
// when the SM is full of warps (cfg2 139 vs 127 ms) and faster when few warps share an SM and
// latency dominates (cfg1, 1,024 pixels: 1.08 vs 1.23 ms); the launcher picks it for batches
// smaller than the resident slots.
template <int NP, int MAXQ, bool ASMEM, bool CM>
__device__ __forceinline__ void adjoint_passes_shfl(float2* acc, const float2* ap, int stride, int pstride, const float2* ryr, int n, bool last) {
  const int rs = CM ? 1 : stride;
  float2 p[NP], q[NP];
#pragma unroll
  for (int t = 0; t < NP; ++t) p[t] = q[t] = make_float2(0.f, 0.f);
#pragma unroll
  for (int h = 0; h < MAXQ; ++h) {
    const int i0 = 32 * h, i1 = min(n, 32 * h + 32);
    const float rx = ryr[h].x, ry = ryr[h].y;
    int i = i0;
#pragma unroll 1
    for (; i + 8 <= i1; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float2 r = make_float2(__shfl_sync(TB_FULL_MASK, rx, i + u - i0), __shfl_sync(TB_FULL_MASK, ry, i + u - i0));
#pragma unroll
        for (int t = 0; t < NP; ++t)
          if (t < NP - 1 || last) {
            const float2 a = ASMEM ? ap[(i + u) * rs + t * pstride] : __ldg(ap + (i + u) * rs + t * pstride);
            ffma2_bcast(p[t], a.x, r);
            ffma2_bcast(q[t], a.y, r);
          }
      }
    }
#pragma unroll 1
    for (; i < i1; ++i) {
      const float2 r = make_float2(__shfl_sync(TB_FULL_MASK, rx, i - i0), __shfl_sync(TB_FULL_MASK, ry, i - i0));
#pragma unroll
      for (int t = 0; t < NP; ++t)
        if (t < NP - 1 || last) {
          const float2 a = ASMEM ? ap[i * rs + t * pstride] : __ldg(ap + i * rs + t * pstride);
          ffma2_bcast(p[t], a.x, r);
          ffma2_bcast(q[t], a.y, r);
        }
    }
  }
#pragma unroll
  for (int t = 0; t < NP; ++t) acc[t] = make_float2(p[t].x + q[t].y, p[t].y - q[t].x);
}
template <int NP, int MAXT, int MAXQ, bool ASMEM, bool CM>
__device__ __forceinline__ void adjoint_dispatch_shfl(int passes, float2* acc, const float2* ap, int stride, int pstride, const float2* ryr, int n, bool last) {
  if constexpr (NP <= MAXT) {
    if (passes == NP) {
      adjoint_passes_shfl<NP, MAXQ, ASMEM, CM>(acc, ap, stride, pstride, ryr, n, last);
      return;
    }
    adjoint_dispatch_shfl<NP + 1, MAXT, MAXQ, ASMEM, CM>(passes, acc, ap, stride, pstride, ryr, n, last);
  }
}

}  // namespace tb
