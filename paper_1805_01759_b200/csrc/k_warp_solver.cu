// Warp-per-pixel proximal-gradient solver: RBPG (paper Alg. 1), FISTA and ISTA.
//
// Reference semantics (paths relative to /root/reference/pkg/src/tomobpdn):
//   rbpg_solve      solver.py:250-338   (block draw, extrapolation, backtracking, monotone accept)
//   _full_vector_pg solver.py:341-376   (ISTA/FISTA, per-iteration backtracking from alpha0)
//   soft_threshold  prox.py:82-96, line_search_ok prox.py:107-119, _window_converged solver.py:227-231
//
// Layout: the dictionary A (complex64, n x m) is staged ONCE per CTA into shared memory with an
// odd row stride (conflict-free both for column-lanes in the adjoint and row-lanes in the
// forward product).  Each warp owns one pixel slot at a time: its iterate x, the extrapolation
// memory, residual vectors and the F-history ring live in shared memory; the drawn block's
// y, gradient and candidate live in registers (lanes own columns c = cs + lane + 32 t).
// Pixels are claimed from a global atomic queue, so retirement of converged pixels and refill
// happen per warp with no CTA-wide barrier; a pixel's arithmetic does not depend on which
// warp/CTA/GPU ran it, so results are independent of scheduling and GPU count.
//
// Numerics: vectors in fp32 (complex64), every scalar that decides control flow in fp64
// (objective F, l1 norms, norms in the backtracking test, window stop).  The backtracking test
// is evaluated in its cancellation-free algebraic form ||A d||^2 <= ||d||^2 / (2 alpha), which is
// exactly the reference inequality f(z) <= f(y) + Re<grad, d> + ||d||^2/(2 alpha) for quadratic f.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "solver_params.h"
#include "warp_adjoint.cuh"

#ifndef TB_WS_RSQRT
#define TB_WS_RSQRT 1  // soft threshold from one fp64 rsqrt
#endif
#ifndef TB_WS_COLMAJOR
#define TB_WS_COLMAJOR 1  // RBPG: shared-memory dictionary column-major (odd column stride n | 1)
#endif
#ifndef TB_WS_BLKBUF
#define TB_WS_BLKBUF 1  // block indices for 32 draws computed at the Philox refill (+2% cfg2 RBPG)
#endif
#ifndef TB_WARP_LB_WIDE
#define TB_WARP_LB_WIDE 384
#endif
#ifndef TB_WARP_LB
#define TB_WARP_LB 512
#endif

namespace tb {

// Tensor memory as a lane-private scratchpad (see k_fista_tile.cu): 4 consecutive 32-bit TMEM columns
// = one double2 per lane, warp-uniform address, ~12-cycle LDTM, no shared-memory wavefront.
__device__ __forceinline__ void ws_tmem_st(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(__double2loint(v.x)),
               "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y))
               : "memory");
}
__device__ __forceinline__ double2 ws_tmem_ld(uint32_t taddr) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
}

// XTM (RBPG whose dictionary does NOT fit in shared memory, cfg3): the fp64 iterate x and the per-block
// delta cache live in tensor memory -- lane l keeps column cs_b + l + 32 t of block b at TMEM columns
// 4 (b T + t), T = ceil(max width / 32), and row l + 32 q of delta_b at 4 (J T + b MAXQ + q).  A slot
// shrinks by (m + J n) * 16 bytes (cfg3: 17.9 -> 3.3 KB), so 16 instead of 11 warps are resident AND
// the unified L1/shared array keeps ~190 KB of L1 for the 200 KiB dictionary every iteration streams.
template <bool RB, int MAXT, int MAXQ, bool ASMEM, bool SHFL, bool XTM>
__global__ void __launch_bounds__(MAXT >= 8 ? TB_WARP_LB_WIDE : TB_WARP_LB, 1) warp_solver_kernel(const SolveParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n = P.n, m = P.m, ms = P.ms;
  constexpr bool CM = ASMEM && RB && TB_WS_COLMAJOR;  // measured: +0.6% RBPG, -2% FISTA (cfg2)
  const int ns = n | 1;  // odd column stride of the column-major shared dictionary
  const bool ista = P.mode == SOLVER_ISTA;

  float2* As = reinterpret_cast<float2*>(smem);
  size_t off = ASMEM ? ((((size_t)(CM ? (size_t)m * ns : (size_t)n * ms)) * sizeof(float2) + 15) & ~(size_t)15) : 0;
  if (ASMEM) {
    for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) {
      int i = idx / m, c = idx - i * m;
      if (CM)
        As[(size_t)c * ns + i] = __ldg(&P.A[idx]);
      else
        As[(size_t)i * ms + c] = __ldg(&P.A[idx]);
    }
    __syncthreads();
  }
  // per-CTA block tables (RBPG): choice CDF, alpha0 = scale / L_i (solver.py:295), block starts
  const int J = RB ? P.num_blocks : 1;
  double* s_cdf = reinterpret_cast<double*>(smem + off);
  double* s_alpha0 = s_cdf + J;
  int* s_bstart = reinterpret_cast<int*>(s_alpha0 + J);
  if (RB) {
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
      s_cdf[j] = P.cdf[j];
      s_alpha0[j] = P.alpha_scale / fmax(P.blk_lip[j], 1e-300);
    }
    for (int j = threadIdx.x; j <= J; j += blockDim.x) s_bstart[j] = P.blk_start[j];
  }
  __syncthreads();
  off += block_table_bytes(J);
  const double alpha0_full = P.alpha_scale / fmax(P.lip_full, 1e-300);  // solver.py:345
  // DC (RBPG): the extrapolation memory d = x - prev lives in fp64 in global memory (L2-resident,
  // one m-vector per warp slot) and delta_b = A_b d_b is cached per block in shared memory, so the
  // reference's r_y = r + A_b dy (solver.py:290-291) is r + m_k delta_b (dy = m_k d_b) with no
  // forward product, and delta_b is refreshed on accept from quantities already at hand:
  // A_b (z_b - x_b) = A_b dz + m_k delta_b.
  constexpr bool DC = RB && TB_WS_DCACHE;
  const size_t per_warp = warp_slot_bytes_for(RB, n, m, P.max_width, J) - (XTM ? ((size_t)m + (size_t)J * n) * 16 : 0);
  unsigned char* wb = smem + off + (size_t)warp * per_warp;
  double2* rv = reinterpret_cast<double2*>(wb);  // r (RBPG) / A x (FISTA)
  double2* apv = rv + n;                         // A x_prev (FISTA)
  double2* xs = DC ? rv + n : apv + n;           // x (fp64 iterate)
  double2* zs = xs + (XTM ? 0 : m);              // broadcast buffer for forward products [max_width]
  float4* ryv = reinterpret_cast<float4*>(zs + P.max_width);  // r_y rounded, as (r.x, r.y, r.y, -r.x)
  float2* ry2 = reinterpret_cast<float2*>(ryv);                // DC: r_y rounded, as (r.x, r.y)
  double2* ds = reinterpret_cast<double2*>(ryv + n);  // d = x - prev, fp64 (y = x + m_k d); not DC
  float2* bv = reinterpret_cast<float2*>(ds + m);  // b; not RBPG
  double2* dlt = reinterpret_cast<double2*>(ryv + n);  // DC: delta [J][n]
  double* ring = DC ? reinterpret_cast<double*>(dlt + (XTM ? 0 : (size_t)J * n)) : reinterpret_cast<double*>(bv + n);  // last STOP_WINDOW+1 objective values
  double* l1blk = ring + 16;                     // RBPG: sum |x_b| per block (updated on accept)
  double2* dg = DC ? P.dglob + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * m : nullptr;
  // XTM: all 512 TMEM columns of this SM; warp w owns lanes 32 (w % 4) .. + 31 and 4 J T columns
  __shared__ uint32_t tmem_base_s;
  const int xt_t = (P.max_width + 31) >> 5;  // passes per block
  uint32_t tm_x = 0;
  if (XTM) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_s)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    tm_x = tmem_base_s + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * (uint32_t)(4 * J * (xt_t + MAXQ));
  }
  const uint32_t tm_dl = tm_x + (uint32_t)(4 * J * xt_t);  // XTM: delta_b, lane = row i + 32 q at columns 4 (b MAXQ + q)

  // acc[q] += sum over the nonzero entries of the step (lane = row), fp64 accumulation.  L1 iterates
  // and their steps are sparse: the lanes compact the nonzero entries with __ballot_sync into
  // zs[0..cnt) in ascending column order, their dictionary columns in clist, and only those
  // columns are visited, two per step (warp-uniform loop).
  auto forward_list = [&](const int* cl, int cnt, double2* acc) {
    const float2* arow[MAXQ];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      acc[q] = make_double2(0.0, 0.0);
      const int i = min(lane + 32 * q, n - 1);
      // CM: cl holds column * ns; A not in shared memory: the column-major copy, element (i, c) at c n + i
      arow[q] = CM ? As + i : ASMEM ? As + i * ms : P.AT + i;
    }
    int e = 0;
    for (; e + 2 <= cnt; e += 2) {
      const int2 cc = *reinterpret_cast<const int2*>(cl + e);
      const double2 v0 = zs[e], v1 = zs[e + 1];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const float2 a0 = ASMEM ? arow[q][cc.x] : __ldg(arow[q] + (size_t)cc.x * n);
        const float2 a1 = ASMEM ? arow[q][cc.y] : __ldg(arow[q] + (size_t)cc.y * n);
        acc[q].x = fma((double)a0.x, v0.x, fma(-(double)a0.y, v0.y, acc[q].x));
        acc[q].y = fma((double)a0.x, v0.y, fma((double)a0.y, v0.x, acc[q].y));
        acc[q].x = fma((double)a1.x, v1.x, fma(-(double)a1.y, v1.y, acc[q].x));
        acc[q].y = fma((double)a1.x, v1.y, fma((double)a1.y, v1.x, acc[q].y));
      }
    }
    if (e < cnt) {
      const int c = cl[e];
      const double2 v = zs[e];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const float2 a = ASMEM ? arow[q][c] : __ldg(arow[q] + (size_t)c * n);
        acc[q].x = fma((double)a.x, v.x, fma(-(double)a.y, v.y, acc[q].x));
        acc[q].y = fma((double)a.x, v.y, fma((double)a.y, v.x, acc[q].y));
      }
    }
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
      if (lane + 32 * q >= n) acc[q] = make_double2(0.0, 0.0);
  };
  const unsigned lt_mask = (1u << lane) - 1u;

  for (;;) {
    unsigned long long pq = 0;
    if (lane == 0) pq = atomicAdd(P.queue, 1ull);
    pq = __shfl_sync(TB_FULL_MASK, pq, 0);
    if (pq >= (unsigned long long)P.num_pixels) break;
    const long long p = (long long)pq;
    const double lamd = (double)P.lam[p];

    // ---- initial state: x = 0, prev = 0, r = -b, F0 = ||b||^2 (solver.py:270-276, 349)
    if (XTM) {
      for (int e = 0; e < J * (xt_t + MAXQ); ++e) ws_tmem_st(tm_x + 4u * e, make_double2(0.0, 0.0));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    for (int c = lane; c < m; c += 32) {
      if (!XTM) xs[c] = make_double2(0.0, 0.0);
      if (DC)
        dg[c] = make_double2(0.0, 0.0);
      else
        ds[c] = make_double2(0.0, 0.0);
    }
    if (DC)
      for (int e = lane; e < (XTM ? 0 : J * n); e += 32) dlt[e] = make_double2(0.0, 0.0);
    double fb = 0.0;
    for (int i = lane; i < n; i += 32) {
      float2 b = P.B[(size_t)p * n + i];
      if (!RB) {
        bv[i] = b;
        apv[i] = make_double2(0.0, 0.0);
      }
      rv[i] = RB ? make_double2(-(double)b.x, -(double)b.y) : make_double2(0.0, 0.0);
      fb += (double)b.x * b.x + (double)b.y * b.y;
    }
    double F = warp_sum(fb);
    double l1 = 0.0;
    if (RB)
      for (int j = lane; j < J; j += 32) l1blk[j] = 0.0;
    if (lane == 0) ring[0] = F;
    int ridx = 0;  // k mod (STOP_WINDOW + 1), kept incrementally
    double* const hrow = P.hist ? P.hist + (size_t)p * P.hist_stride : nullptr;  // all lanes store F (same value)
    if (hrow) hrow[0] = F;
    const uint64_t seed = RB ? P.seeds[p] : 0ull;
    uint64_t* rbuf = reinterpret_cast<uint64_t*>(l1blk + J);  // 32 buffered Philox outputs
    int* clist = reinterpret_cast<int*>(rbuf + 32);               // nonzero columns of zs, ascending
    int status = STATUS_MAX_ITERS;
    int iters = 0;
    bool stopped = false;
    __syncwarp();

    // m_k is read one iteration ahead: the table load (L1 or L2) is off the r_y critical path
    double mk_next = (ista || P.total_iters < 1) ? 0.0 : __ldg(P.mk + 1);
    for (int k = 1; k <= P.total_iters; ++k) {
      iters = k;
      ridx = ridx == STOP_WINDOW ? 0 : ridx + 1;
      // ---- block choice (solver.py:283, 217-219): searchsorted(cdf, u, 'right')
      int blk = 0, cs = 0, ce = m;
      if (RB) {
        // raw draw k-1 of Philox(key=[seed, 0]): counter (k-1)/4 + 1, output (k-1) % 4.  Every 32
        // draws, lanes 0..7 evaluate the next 8 counters in parallel into the slot's buffer.
        const int w = (k - 1) & 31;
#if TB_WS_BLKBUF
        // every 32 draws: lanes 0..7 evaluate 8 counters, then lane l turns draw l into its block
        // (searchsorted(cdf, u, 'right') as a linear scan of the monotone CDF) and the 32 block
        // indices replace the raw draws in the slot's buffer
        int* bbuf = reinterpret_cast<int*>(rbuf);
        if (w == 0) {
          uint64_t c4[4] = {(uint64_t)((k - 1) >> 2) + 1ull + (uint64_t)(lane & 7), 0ull, 0ull, 0ull};
          philox4x64_10(c4, seed, 0ull);
          if (lane < 8) {
#pragma unroll
            for (int q = 0; q < 4; ++q) rbuf[4 * lane + q] = c4[q];
          }
          __syncwarp();
          const double u = raw_to_unit(rbuf[lane]);
          int j = 0;
          while (j < J - 1 && s_cdf[j] <= u) ++j;
          __syncwarp();
          bbuf[lane] = j;
          __syncwarp();
        }
        blk = bbuf[w];
#else
        if (w == 0) {
          uint64_t c4[4] = {(uint64_t)((k - 1) >> 2) + 1ull + (uint64_t)(lane & 7), 0ull, 0ull, 0ull};
          philox4x64_10(c4, seed, 0ull);
          if (lane < 8) {
#pragma unroll
            for (int q = 0; q < 4; ++q) rbuf[4 * lane + q] = c4[q];
          }
          __syncwarp();
        }
        const double u = raw_to_unit(rbuf[w]);
        int j = 0;
        if (J <= 32) {
          // searchsorted(cdf, u, 'right') with cdf[J-1] == 1 > u: count of cdf[q] <= u over q < J-1
          const bool le = lane < J - 1 && s_cdf[lane] <= u;
          j = __popc(__ballot_sync(TB_FULL_MASK, le));
        } else {
          while (j < J - 1 && s_cdf[j] <= u) ++j;
        }
        blk = j;
#endif
        cs = s_bstart[blk];
        ce = s_bstart[blk + 1];
      }
      const int width = ce - cs;
      const double mk = mk_next;  // (k-2)/(k+1), host table (solver.py:222-224); 0 for ISTA
      if (!ista && k < P.total_iters) mk_next = __ldg(P.mk + k + 1);

      // ---- extrapolation y = x + m_k (x - prev) (solver.py:288-289, 356)
      float2 g[MAXT];
      double2 z[RB ? MAXT : 1];
      unsigned masks[MAXT];
      bool any_dy = false;
      int cnt = 0;  // RBPG: compacted nonzero count in zs / clist
      // Column passes are branch-free: lanes past the range read a valid column (cs) and their
      // results are masked, so no divergent-branch reconvergence is paid per pass; passes that lie
      // entirely past the range are skipped with a warp-uniform test.
      // DC: the block's d_b is loaded from L2 here and first used in the backtracking loop, so the
      // load latency hides behind the adjoint.
      // XR: the block's x_b also stays in registers for the whole iteration (one shared read instead
      // of one per trial plus one in the update; measured +1.5% on cfg2, but -19% on cfg3 where A is
      // read through L1 and -4% on the latency-bound small batches, so only for a full SM with A in
      // shared memory)
      constexpr bool XR = DC && ASMEM && !SHFL;
      double2 dvb[DC ? MAXT : 1], xr[XR ? MAXT : 1];
#pragma unroll
      for (int t = 0; t < (DC ? MAXT : 1); ++t) {
        dvb[t] = make_double2(0.0, 0.0);
        if (XR) xr[XR ? t : 0] = make_double2(0.0, 0.0);
        if (DC && (t == 0 || 32 * t < width)) {
          dvb[t] = dg[cs + min(lane + 32 * t, width - 1)];
          if (XR) xr[XR ? t : 0] = XTM ? ws_tmem_ld(tm_x + 4u * (blk * xt_t + t)) : xs[cs + min(lane + 32 * t, width - 1)];
        }
      }
#pragma unroll
      for (int t = 0; t < (DC ? 0 : MAXT); ++t) {
        masks[t] = 0u;
        if (t > 0 && 32 * t >= width) continue;
        const int cl = lane + 32 * t;
        const bool act = cl < width;
        const int col = cs + (act ? cl : 0);
        const double2 xv = xs[col];
        double2 yv = xv;
        if (!ista) {
          // y = x + m_k (x - prev) with the extrapolation memory kept as d = x - prev in fp64;
          // d is exactly 0 after a rejected visit, so `np.any(dy)` (solver.py:291) is preserved
          const double2 dv = ds[col];
          yv.x = fma(mk, dv.x, xv.x);
          yv.y = fma(mk, dv.y, xv.y);
        }
        bool nz = false;
        double2 dyv = make_double2(0.0, 0.0);
        if (RB) {
          dyv = make_double2(yv.x - xv.x, yv.y - xv.y);
          nz = act && ((dyv.x != 0.0) || (dyv.y != 0.0));
        }
        masks[t] = __ballot_sync(TB_FULL_MASK, nz);
        if (RB && nz) {
          const int pos = cnt + __popc(masks[t] & lt_mask);
          zs[pos] = dyv;
          clist[pos] = CM ? col * ns : col;
        }
        cnt += __popc(masks[t]);
        any_dy |= masks[t] != 0u;
      }
      __syncwarp();

      // ---- residual at y (lane = row), fp64: RBPG r_y = r + A_b dy (solver.py:290-291);
      //      FISTA/ISTA r_y = A y - b with A y = A x + m_k (A x - A x_prev) by linearity.
      double2 ry[MAXQ], ay[MAXQ];
      if (DC) {
        // r_y = r + m_k delta_b: delta_b = 0 after a rejected (or no) visit gives r exactly, as the
        // reference's `np.any(dy)` test does
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = lane + 32 * q;
          ry[q] = ay[q] = make_double2(0.0, 0.0);
          double2 dlq = make_double2(0.0, 0.0);
          if (XTM) dlq = ws_tmem_ld(tm_dl + 4u * (blk * MAXQ + q));
          if (i < n) {
            const double2 r = rv[i], dl = XTM ? dlq : dlt[blk * n + i];
            ry[q] = make_double2(fma(mk, dl.x, r.x), fma(mk, dl.y, r.y));
            if (!SHFL) ry2[i] = make_float2((float)ry[q].x, (float)ry[q].y);
          }
        }
      } else if (RB) {
        double2 acc[MAXQ];
        if (any_dy) forward_list(clist, cnt, acc);
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = lane + 32 * q;
          ry[q] = ay[q] = make_double2(0.0, 0.0);
          if (i < n) {
            const double2 r = rv[i];
            ry[q] = any_dy ? make_double2(r.x + acc[q].x, r.y + acc[q].y) : r;
            ryv[i] = conj_operand((float)ry[q].x, (float)ry[q].y);
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = lane + 32 * q;
          ry[q] = ay[q] = make_double2(0.0, 0.0);
          if (i < n) {
            const double2 ax = rv[i], axp = apv[i];
            const float2 b = bv[i];
            double2 a = ax;
            if (!ista) {
              a.x = fma(mk, ax.x - axp.x, ax.x);
              a.y = fma(mk, ax.y - axp.y, ax.y);
            }
            ay[q] = a;
            ry[q] = make_double2(a.x - b.x, a.y - b.y);
            ryv[i] = conj_operand((float)ry[q].x, (float)ry[q].y);
          }
        }
      }
      __syncwarp();

      // ---- block gradient g = 2 A_b^H r_y (solver.py:293, prox.py:77-79), fp32 products;
      //      exactly ceil(width / 32) column passes are issued
      {
        float2 acc[MAXT];
#pragma unroll
        for (int t = 0; t < MAXT; ++t) acc[t] = make_float2(0.f, 0.f);
        const int passes = (width + 31) >> 5;
        const float2* ap = CM ? As + (size_t)(cs + lane) * ns : (ASMEM ? As : P.A) + cs + lane;
        if (DC && SHFL) {
          float2 ryr[MAXQ];
#pragma unroll
          for (int q = 0; q < MAXQ; ++q) ryr[q] = make_float2((float)ry[q].x, (float)ry[q].y);
          adjoint_dispatch_shfl<1, MAXT, MAXQ, ASMEM, CM>(passes, acc, ap, ASMEM ? ms : m, CM ? 32 * ns : 32, ryr, n, lane + 32 * (passes - 1) < width);
        } else if (DC)
          adjoint_dispatch2<1, MAXT, ASMEM, CM>(passes, acc, ap, ASMEM ? ms : m, CM ? 32 * ns : 32, ry2, n, lane + 32 * (passes - 1) < width);
        else
          adjoint_dispatch<1, MAXT, ASMEM, CM>(passes, acc, ap, ASMEM ? ms : m, CM ? 32 * ns : 32, ryv, n, lane + 32 * (passes - 1) < width);
#pragma unroll
        for (int t = 0; t < MAXT; ++t) g[t] = make_float2(2.f * acc[t].x, 2.f * acc[t].y);
      }

      // ---- backtracking (solver.py:295-314; prox.py:122-150), prox step in fp64
      double alpha = RB ? s_alpha0[blk] : alpha0_full;
      bool ok = false;
      double2 adz[MAXQ];
      double l1z = 0.0, fzs = 0.0;
      for (int trial = 0; trial <= P.cap; ++trial) {
        const double tau = alpha * lamd;
        const double tau2 = tau * tau;
        double red[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // |d|^2, |z|, ||A d||^2, f(z), scale (FISTA)
        cnt = 0;
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          masks[t] = 0u;
          if (t > 0 && 32 * t >= width) continue;
          const int cl = lane + 32 * t;
          const bool act = cl < width;
          const int col = cs + (act ? cl : 0);
          // y = x + m_k d; FISTA/ISTA recompute it from shared memory (keeps registers for occupancy)
          // XTM: lanes past the block read their own (zero) cell; their results are masked
          const double2 xv = XR ? xr[XR ? t : 0] : XTM ? ws_tmem_ld(tm_x + 4u * (blk * xt_t + t)) : xs[col];
          double2 yv = xv;
          if (DC) {
            yv.x = fma(mk, dvb[t].x, xv.x);
            yv.y = fma(mk, dvb[t].y, xv.y);
          } else if (!ista) {
            const double2 dv = ds[col];
            yv.x = fma(mk, dv.x, xv.x);
            yv.y = fma(mk, dv.y, xv.y);
          }
          const double2 v = make_double2(fma(-alpha, (double)g[t].x, yv.x), fma(-alpha, (double)g[t].y, yv.y));
          const double mag2 = fma(v.x, v.x, v.y * v.y);
          double2 zz = make_double2(0.0, 0.0);
          // soft_threshold: zero iff |v| <= tau (prox.py:82-96); a NaN v stays NaN, as the
          // reference's v * max(0, 1 - tau / max(|v|, tiny)) propagates it
          if (act && !(mag2 <= tau2)) {
            // scale 1 - tau/|v| and |z| = |v| - tau from one fp64 reciprocal square root
#if TB_WS_RSQRT
            const double rs = rsqrt(mag2);
            const double sc = fma(-tau, rs, 1.0);
            zz = make_double2(v.x * sc, v.y * sc);
            red[1] += fma(mag2, rs, -tau);
#else
            const double mag = sqrt(mag2);
            const double sc = 1.0 - tau / mag;
            zz = make_double2(v.x * sc, v.y * sc);
            red[1] += mag * sc;
#endif
          }
          if (RB) z[t] = zz;
          const double2 d = make_double2(zz.x - yv.x, zz.y - yv.y);
          red[0] += act ? fma(d.x, d.x, d.y * d.y) : 0.0;
          const double2 dw = RB ? d : zz;
          const bool nz = act && ((dw.x != 0.0) || (dw.y != 0.0));
          masks[t] = __ballot_sync(TB_FULL_MASK, nz);
          if (nz) {
            const int pos = cnt + __popc(masks[t] & lt_mask);
            zs[pos] = dw;
            clist[pos] = CM ? col * ns : col;
          }
          cnt += __popc(masks[t]);
        }
        __syncwarp();
        forward_list(clist, cnt, adz);  // RBPG: A_b dz; FISTA/ISTA: A z
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = lane + 32 * q;
          if (i < n) {
            // quadratic-bound test in its exact algebraic form ||A d||^2 <= ||d||^2 / (2 alpha)
            if (RB) {
              red[2] += adz[q].x * adz[q].x + adz[q].y * adz[q].y;
              const double rx = ry[q].x + adz[q].x, ryy = ry[q].y + adz[q].y;
              red[3] += rx * rx + ryy * ryy;
            } else {
              const double dx = adz[q].x - ay[q].x, dyy = adz[q].y - ay[q].y;
              red[2] += dx * dx + dyy * dyy;
              const float2 b = bv[i];
              const double fx = adz[q].x - b.x, fy = adz[q].y - b.y;
              red[3] += fx * fx + fy * fy;
              red[4] += fabs(adz[q].x) + fabs(adz[q].y) + fabs(ay[q].x) + fabs(ay[q].y);
            }
          }
        }
        if (RB) {
          warp_sum4(red);
        } else {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int r = 0; r < 5; ++r) red[r] += __shfl_xor_sync(TB_FULL_MASK, red[r], o);
          }
        }
        __syncwarp();
        l1z = red[1];
        fzs = red[3];
        bool pass;
        if (RB) {
          pass = red[2] * (2.0 * alpha) <= red[0] * (1.0 + 1e-9);  // ||A d||^2 <= ||d||^2/(2 alpha)
        } else {
          pass = sqrt(red[2]) <= sqrt(red[0] / (2.0 * alpha)) + 1e-12 * red[4];  // fp64 rounding of A z - A y
        }
        if (pass) {
          ok = true;
          break;
        }
        alpha *= P.c_alpha;
      }
      if (!ok) {
        // RBPG appends F before breaking (solver.py:311-314); ISTA/FISTA do not (solver.py:357-361)
        if (RB) {
          ring[ridx] = F;
          if (hrow) hrow[k] = F;
        }
        status = STATUS_LINE_SEARCH_FAILURE;
        stopped = true;
        break;
      }

      // ---- update
      if (RB) {
        // incremental l1, monotone acceptance (solver.py:316-325)
        const double l1_new = l1 - l1blk[blk] + l1z;
        double2 rz[MAXQ];
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) rz[q] = make_double2(ry[q].x + adz[q].x, ry[q].y + adz[q].y);
        const double cand = fzs + lamd * l1_new;
        const bool accept = cand <= F;
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          if (t > 0 && 32 * t >= width) continue;
          const int cl = lane + 32 * t;
          if (XTM) {
            // warp-collective TMEM access: lanes past the block keep their zero
            const double2 xv = XR ? xr[XR ? t : 0] : ws_tmem_ld(tm_x + 4u * (blk * xt_t + t));
            const double2 zv = (accept && cl < width) ? z[RB ? t : 0] : xv;
            if (accept) ws_tmem_st(tm_x + 4u * (blk * xt_t + t), zv);
            if (cl < width) dg[cs + cl] = make_double2(zv.x - xv.x, zv.y - xv.y);
          } else if (cl < width) {
            // accept: prev_b <- x_b, x_b <- z_b; reject: prev_b <- x_b (solver.py:318-325)
            const double2 xv = XR ? xr[XR ? t : 0] : xs[cs + cl], zv = accept ? z[RB ? t : 0] : xv;
            if (DC)
              dg[cs + cl] = make_double2(zv.x - xv.x, zv.y - xv.y);
            else
              ds[cs + cl] = make_double2(zv.x - xv.x, zv.y - xv.y);
            xs[cs + cl] = zv;
          }
        }
        if (XTM && accept) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (DC) {
          // delta_b <- A_b (z_b - x_b) = A_b dz + A_b (y_b - x_b) = adz + m_k delta_b, or 0 on reject
#pragma unroll
          for (int q = 0; q < MAXQ; ++q) {
            const int i = lane + 32 * q;
            if (XTM) {
              const double2 o = ws_tmem_ld(tm_dl + 4u * (blk * MAXQ + q));
              ws_tmem_st(tm_dl + 4u * (blk * MAXQ + q), (accept && i < n) ? make_double2(fma(mk, o.x, adz[q].x), fma(mk, o.y, adz[q].y)) : make_double2(0.0, 0.0));
            } else if (i < n) {
              double2* dl = dlt + blk * n + i;
              const double2 o = *dl;
              *dl = accept ? make_double2(fma(mk, o.x, adz[q].x), fma(mk, o.y, adz[q].y)) : make_double2(0.0, 0.0);
            }
          }
        }
        if (XTM) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (accept) {
#pragma unroll
          for (int q = 0; q < MAXQ; ++q) {
            const int i = lane + 32 * q;
            if (i < n) rv[i] = rz[q];
          }
          l1 = l1_new;
          F = cand;
          l1blk[blk] = l1z;
        }
      } else {
        // x_prev <- x, x <- z, F = ||A z - b||^2 + lambda ||z||_1 (solver.py:362-364)
        // z is nonzero only on the compacted list: the owner lane finds its entry from the masks
        int base = 0;
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          if (t > 0 && 32 * t >= width) break;
          const int cl = lane + 32 * t;
          if (cl < width) {
            const double2 xv = xs[cl];
            const double2 zv = (masks[t] >> lane) & 1u ? zs[base + __popc(masks[t] & lt_mask)] : make_double2(0.0, 0.0);
            ds[cl] = make_double2(zv.x - xv.x, zv.y - xv.y);
            xs[cl] = zv;
          }
          base += __popc(masks[t]);
        }
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = lane + 32 * q;
          if (i < n) {
            apv[i] = rv[i];
            rv[i] = adz[q];
          }
        }
        F = fzs + lamd * l1z;
      }
      // ---- history, failure and window stop (solver.py:326-336, 366-374)
      ring[ridx] = F;  // every lane stores the same value (no divergent branch)
      if (hrow) hrow[k] = F;
      __syncwarp();
      if (!isfinite(F)) {
        status = STATUS_NUMERICAL_FAILURE;
        stopped = true;
        break;
      }
      if (!P.fixed && k >= STOP_WINDOW) {
        const double ref = ring[ridx == STOP_WINDOW ? 0 : ridx + 1];  // F at k - STOP_WINDOW
        if (fabs(F - ref) <= P.tol * fmax(fabs(ref), 1e-300)) {
          status = STATUS_CONVERGED;
          stopped = true;
          break;
        }
      }
    }
    if (!stopped && iters >= STOP_WINDOW) {  // for-else re-check (solver.py:334-336)
      const double ref = ring[ridx == STOP_WINDOW ? 0 : ridx + 1];
      if (fabs(F - ref) <= P.tol * fmax(fabs(ref), 1e-300)) status = STATUS_CONVERGED;
    }
    __syncwarp();
    if (XTM) {
      for (int j = 0; j < J; ++j) {
        const int c0 = s_bstart[j], w = s_bstart[j + 1] - c0;
        for (int t = 0; 32 * t < w; ++t) {
          const double2 xv = ws_tmem_ld(tm_x + 4u * (j * xt_t + t));
          if (lane + 32 * t < w) P.X[(size_t)p * m + c0 + lane + 32 * t] = make_float2((float)xv.x, (float)xv.y);
        }
      }
    } else
    for (int c = lane; c < m; c += 32) {
      const double2 xv = xs[c];
      P.X[(size_t)p * m + c] = make_float2((float)xv.x, (float)xv.y);
    }
    if (lane == 0) {
      P.f_final[p] = F;
      P.iters[p] = iters;
      P.status[p] = status;
    }
    __syncwarp();
  }
  if (XTM) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_s));
  }
}

template <bool RB, int MAXT, int MAXQ, bool ASMEM>
static cudaError_t launch_t(const SolveParams& P, int warps, size_t smem, int grid, cudaStream_t st, bool shfl, bool xtm) {
  // r_y from shuffles only for RBPG (DC) batches smaller than the resident slots (see warp_adjoint.cuh)
  auto k = (RB && TB_WS_DCACHE && shfl) ? warp_solver_kernel<RB, MAXT, MAXQ, ASMEM, true, false> : warp_solver_kernel<RB, MAXT, MAXQ, ASMEM, false, false>;
  if constexpr (RB && TB_WS_DCACHE && !ASMEM && MAXT <= 4) {
    if (xtm) k = warp_solver_kernel<RB, MAXT, MAXQ, ASMEM, false, true>;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  k<<<grid, warps * 32, smem, st>>>(P);
  return cudaGetLastError();
}

template <bool RB, int MAXT, bool ASMEM>
static cudaError_t launch_q(const SolveParams& P, int maxq, int warps, size_t smem, int grid, cudaStream_t st, bool shfl, bool xtm) {
  switch (maxq) {
    case 1: return launch_t<RB, MAXT, 1, ASMEM>(P, warps, smem, grid, st, shfl, xtm);
    case 2: return launch_t<RB, MAXT, 2, ASMEM>(P, warps, smem, grid, st, shfl, xtm);
    case 4: return launch_t<RB, MAXT, 4, ASMEM>(P, warps, smem, grid, st, shfl, xtm);
    default: return cudaErrorInvalidValue;
  }
}

template <bool RB, bool ASMEM>
static cudaError_t launch_tq(const SolveParams& P, int maxt, int maxq, int warps, size_t smem, int grid, cudaStream_t st, bool shfl, bool xtm) {
  if (maxt <= 2) return launch_q<RB, 2, ASMEM>(P, maxq, warps, smem, grid, st, shfl, xtm);
  if (maxt <= 4) return launch_q<RB, 4, ASMEM>(P, maxq, warps, smem, grid, st, shfl, xtm);
  if (maxt <= 8) return launch_q<RB, 8, ASMEM>(P, maxq, warps, smem, grid, st, shfl, false);
  if (maxt <= 12) return launch_q<RB, 12, ASMEM>(P, maxq, warps, smem, grid, st, shfl, false);
  if (maxt <= 16) return launch_q<RB, 16, ASMEM>(P, maxq, warps, smem, grid, st, shfl, false);
  return cudaErrorInvalidValue;
}

// Chooses the shared-memory plan and launches a persistent grid (<= resident CTAs).
cudaError_t launch_warp_solver(const SolveParams& P, int num_sms, cudaStream_t st, int* used_warps) {
  const int width = P.max_width;
  int maxt = (width + 31) / 32;
  maxt = maxt <= 2 ? 2 : maxt <= 4 ? 4 : maxt <= 8 ? 8 : maxt <= 12 ? 12 : 16;  // template bucket
  int maxq = (P.n + 31) / 32;
  maxq = maxq <= 1 ? 1 : maxq <= 2 ? 2 : 4;
  const int J = P.mode == SOLVER_RBPG ? P.num_blocks : 1;
  const size_t slot = warp_slot_bytes_for(P.mode == SOLVER_RBPG, P.n, P.m, P.max_width, J);
  const size_t tables = block_table_bytes(J);
  const bool cm = TB_WS_COLMAJOR && P.mode == SOLVER_RBPG;
  const size_t a_bytes = ((size_t)(cm ? (size_t)P.m * (P.n | 1) : (size_t)P.n * P.ms) * sizeof(float2) + 15) & ~(size_t)15;
  const size_t cap = 227 * 1024 - 64;  // 16 static bytes (TMEM base address) + margin
  const int max_warps = maxt >= 8 ? TB_WARP_LB_WIDE / 32 : TB_WARP_LB / 32;
  bool asmem = a_bytes + tables + 4 * slot <= cap;
  size_t avail = cap - tables - (asmem ? a_bytes : 0);
  // RBPG whose dictionary is read through L1 (cfg3): x in tensor memory (TB_WS_XTM=0 disables)
  bool xtm = false;
  size_t slot_used = slot;
  if (P.mode == SOLVER_RBPG && TB_WS_DCACHE && !asmem && maxt <= 4) {
    const char* xe = getenv("TB_WS_XTM");
    const int xcols = 4 * J * ((P.max_width + 31) / 32 + maxq);
    const size_t slot_x = slot - ((size_t)P.m + (size_t)J * P.n) * 16;
    int wx = (int)(avail / slot_x);
    if (wx > max_warps) wx = max_warps;
    if (!(xe && atoi(xe) == 0) && ((wx + 3) / 4) * xcols <= 512) {
      xtm = true;
      slot_used = slot_x;
    }
  }
  int warps = (int)(avail / slot_used);
  if (warps > max_warps) warps = max_warps;
  if (!asmem && !xtm) {
    // dictionary read through L1/L2: RBPG leaves one slot's worth of the unified L1/shared array
    // to the L1 cache that serves A (cfg3: 11 instead of 12 warps is +5%; FISTA measured -2%, so
    // it keeps every slot; TB_WARPS_L1 overrides)
    const char* ev = getenv("TB_WARPS_L1");
    const int cap_l1 = ev ? atoi(ev) : (P.mode == SOLVER_RBPG && warps > 2 ? warps - 1 : warps);
    if (cap_l1 >= 1 && cap_l1 < warps) warps = cap_l1;
  }
  if (const char* wc = getenv("TB_WARPS_CAP")) {  // tuning/diagnostics: cap the warps per CTA
    const int cap_w = atoi(wc);
    if (cap_w >= 1 && cap_w < warps) warps = cap_w;
  }
  if (warps < 1) return cudaErrorInvalidValue;
  // a batch smaller than the resident slots (cfg1: 1,024 pixels vs 148 x 16) is spread over every SM
  // with fewer warps each, instead of filling ceil(P / warps) SMs: each pixel's warp then shares its
  // SM's issue slots and shared-memory pipe with fewer others (the batch time is the slowest pixel's)
  const bool spread = P.num_pixels < (long long)num_sms * warps;
  if (spread) warps = (int)((P.num_pixels + num_sms - 1) / num_sms);
  if (warps < 1) warps = 1;
  size_t smem = (asmem ? a_bytes : 0) + tables + (size_t)warps * slot_used;
  long long need = (P.num_pixels + warps - 1) / warps;
  int grid = num_sms;
  if (need < grid) grid = (int)need;
  if (grid < 1) grid = 1;
  if (used_warps) *used_warps = warps;
  const bool rb = P.mode == SOLVER_RBPG;
  if (rb) return asmem ? launch_tq<true, true>(P, maxt, maxq, warps, smem, grid, st, spread, false) : launch_tq<true, false>(P, maxt, maxq, warps, smem, grid, st, spread, xtm);
  return asmem ? launch_tq<false, true>(P, maxt, maxq, warps, smem, grid, st, false, false) : launch_tq<false, false>(P, maxt, maxq, warps, smem, grid, st, false, false);
}

}  // namespace tb
