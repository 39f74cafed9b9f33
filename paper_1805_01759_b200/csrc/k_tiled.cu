// Large-dictionary solver (cfg4/cfg5): RBPG / FISTA / ISTA with the iterate state in HBM.
//
// One solver "round" advances every pending pixel by one backtracking trial:
//   prep     (warp / pixel)  block draw (Philox4x64-10, draw k-1 of substream(seed)), r_y, alpha0
//   schedule (1 CTA)         bucket pending pixels by block -> tiles of TL_PT pixels sharing columns
//   pass     (tiles x splits) fused: g = 2 A^H r_y (fp32 SIMT GEMM over a TL_CT column tile staged in
//                            shared memory) -> extrapolation + complex soft-threshold in fp64 from the
//                            HBM state -> candidate written to HBM -> forward partial A z (or A dz)
//                            accumulated in fp64 over the tile's nonzero columns only
//   reduce   (warp / pixel)  fixed-order sum of the split partials (the NCCL all-reduce target when
//                            the dictionary is column-sharded across GPUs)
//   update   (warp / pixel)  quadratic-bound test, monotone acceptance (RBPG), history, window stop
// Reference semantics: solver.py:250-376, prox.py:82-150 (same as k_warp_solver.cu).
#include <float.h>

#include "common.cuh"
#include "solver_params.h"
#include "tiled.h"

namespace tb {

__device__ __forceinline__ double2* xrow(const TiledParams& T, int buf, int p) {
  return T.X3 + ((size_t)buf * T.P + p) * (size_t)T.m;
}

// ------------------------------------------------------------------ init
__global__ void tiled_init_kernel(const TiledParams T) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= T.P) return;
  const bool rb = T.mode == SOLVER_RBPG;
  double fb = 0.0;
  for (int i = lane; i < T.n; i += 32) {
    const float2 b = T.B[(size_t)p * T.n + i];
    fb += (double)b.x * b.x + (double)b.y * b.y;
    T.r[(size_t)p * T.n + i] = rb ? make_double2(-(double)b.x, -(double)b.y) : make_double2(0.0, 0.0);
    T.axp[(size_t)p * T.n + i] = make_double2(0.0, 0.0);
  }
  if (rb)
    for (int t = lane; t < T.J * T.n; t += 32) T.delta[(size_t)p * T.J * T.n + t] = make_double2(0.0, 0.0);
  for (int j = lane; j < T.J; j += 32) T.l1blk[(size_t)p * T.J + j] = 0.0;
  fb = warp_sum(fb);
  if (lane == 0) {
    T.phase[p] = PH_PREP;
    T.k[p] = 0;
    T.trial[p] = 0;
    T.status[p] = STATUS_MAX_ITERS;
    T.roles[3 * p + 0] = 0;
    T.roles[3 * p + 1] = 1;
    T.roles[3 * p + 2] = 2;
    T.F[p] = fb;
    T.l1[p] = 0.0;
    T.ring[(size_t)p * 16] = fb;
    if (T.hist) T.hist[(size_t)p * T.hist_stride] = fb;
  }
}

// ------------------------------------------------------------------ prep
__global__ void tiled_prep_kernel(const TiledParams T) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= T.P || T.phase[p] != PH_PREP) return;
  const bool rb = T.mode == SOLVER_RBPG;
  const int k = T.k[p] + 1;
  const double mk = T.mode == SOLVER_ISTA ? 0.0 : T.mk[k];
  int b = 0;
  if (rb) {
    // raw draw number k-1 of Philox(key=[seed, 0]): counter (k-1)/4 + 1, lane (k-1) % 4
    const unsigned long long d = (unsigned long long)(k - 1);
    uint64_t c[4] = {d / 4 + 1, 0ull, 0ull, 0ull};
    philox4x64_10(c, T.seeds[p], 0ull);
    const int w = (int)(d & 3ull);
    const uint64_t raw = w == 0 ? c[0] : w == 1 ? c[1] : w == 2 ? c[2] : c[3];
    const double u = raw_to_unit(raw);
    while (b < T.J - 1 && T.cdf[b] <= u) ++b;
  }
  for (int i = lane; i < T.n; i += 32) {
    const size_t o = (size_t)p * T.n + i;
    double2 ry;
    if (rb) {
      // r_y = r + A_b dy with A_b dy = m_k A_b (x_b - prev_b) = m_k delta_b (solver.py:290-291)
      const double2 r = T.r[o];
      const double2 dl = T.delta[((size_t)p * T.J + b) * T.n + i];
      ry = make_double2(fma(mk, dl.x, r.x), fma(mk, dl.y, r.y));
      T.ry[o] = ry;
      T.ry32[o] = make_float2((float)ry.x, (float)ry.y);
    } else {
      // A y = A x + m_k (A x - A x_prev); r_y = A y - b
      const double2 ax = T.r[o], ap = T.axp[o];
      const double2 ay = make_double2(fma(mk, ax.x - ap.x, ax.x), fma(mk, ax.y - ap.y, ax.y));
      const float2 bb = T.B[o];
      T.ry[o] = ay;
      T.ry32[o] = make_float2((float)(ay.x - bb.x), (float)(ay.y - bb.y));
    }
  }
  if (lane == 0) {
    T.k[p] = k;
    T.blk[p] = b;
    T.trial[p] = 0;
    T.alpha[p] = T.alpha0[b];
    T.phase[p] = PH_TRIAL;
  }
}

// ------------------------------------------------------------------ schedule
// Single CTA: pending pixels bucketed by block, tiles of up to TL_PT pixels per block.
__global__ void __launch_bounds__(1024) tiled_schedule_kernel(const TiledParams T) {
  extern __shared__ int sh[];
  int* cnt = sh;          // [J]
  int* base = sh + T.J;   // [J]
  int* fill = sh + 2 * T.J;
  for (int j = threadIdx.x; j < T.J; j += blockDim.x) {
    cnt[j] = 0;
    fill[j] = 0;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < T.P; p += blockDim.x)
    if (T.phase[p] == PH_TRIAL) atomicAdd(&cnt[T.blk[p]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int off = 0, nt = 0;
    for (int j = 0; j < T.J; ++j) {
      base[j] = off;
      for (int s = 0; s < cnt[j]; s += TL_PT) T.tiles[nt++] = make_int4(j, off + s, min(TL_PT, cnt[j] - s), 0);
      off += cnt[j];
    }
    *T.ntiles = nt;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < T.P; p += blockDim.x)
    if (T.phase[p] == PH_TRIAL) {
      const int j = T.blk[p];
      T.perm[base[j] + atomicAdd(&fill[j], 1)] = p;
    }
}

// ------------------------------------------------------------------ fused pass
#ifndef TB_TILED_FFMA2
#define TB_TILED_FFMA2 0  // packed FFMA2 in the adjoint micro-tile: bit-identical, measured 6% SLOWER (cfg4/cfg5
                          // FISTA: the pass is FMA-pipe bound, not issue bound), so scalar FFMA stays
#endif
constexpr int TL_AS = TL_CT + 1;  // odd row stride of the staged A tile
constexpr int TL_ZS = TL_PT + 1;  // padded row stride of the staged candidate tile (conflict-free epilogue stores)

__host__ __device__ inline size_t tiled_pass_smem(int n) {
  size_t b = (size_t)n * TL_PT * 8;               // sRY
  b += (size_t)n * TL_AS * 8;                     // sA
  b = (b + 15) & ~(size_t)15;
  b += (size_t)TL_CT * TL_ZS * 16;                // sZ
  b += TL_PT * 8;                                 // sMask
  b += TL_PT * (4 * 8 + 4 * 4);                   // per-pixel scalars
  return (b + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(TL_THREADS, 2) tiled_pass_kernel(const TiledParams T) {
  const int tile = blockIdx.x, split = blockIdx.y;
  if (tile >= *T.ntiles) return;
  const int4 td = T.tiles[tile];
  const int b = td.x, off = td.y, count = td.z;
  const int c_begin = T.bstart[b], c_end = T.bstart[b + 1];
  const int s0 = c_begin + split * T.split_width;
  if (s0 >= c_end) return;
  const int s1 = min(c_end, s0 + T.split_width);
  const int n = T.n, m = T.m;
  const bool rb = T.mode == SOLVER_RBPG, ista = T.mode == SOLVER_ISTA;

  extern __shared__ __align__(16) unsigned char sm[];
  float2* sRY = reinterpret_cast<float2*>(sm);  // [n][PT]
  float2* sA = sRY + (size_t)n * TL_PT;         // [n][TL_AS]
  size_t o = ((size_t)n * TL_PT * 8 + (size_t)n * TL_AS * 8 + 15) & ~(size_t)15;
  double2* sZ = reinterpret_cast<double2*>(sm + o);  // [CT][ZS]
  unsigned long long* sMask = reinterpret_cast<unsigned long long*>(sZ + TL_CT * TL_ZS);  // [PT] nonzero columns
  double* sAlpha = reinterpret_cast<double*>(sMask + TL_PT);
  double* sTau = sAlpha + TL_PT;
  double* sMk = sTau + TL_PT;
  double* sPad = sMk + TL_PT;
  int* sPid = reinterpret_cast<int*>(sPad + TL_PT);
  int* sRx = sPid + TL_PT;
  int* sRp = sRx + TL_PT;
  int* sRz = sRp + TL_PT;
  (void)sPad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < TL_PT) {
    const int p = tid < count ? T.perm[off + tid] : -1;
    sPid[tid] = p;
    if (p >= 0) {
      const double a = T.alpha[p];
      sAlpha[tid] = a;
      sTau[tid] = a * (double)T.lam[p];
      sMk[tid] = ista ? 0.0 : T.mk[T.k[p]];
      sRx[tid] = T.roles[3 * p + 0];
      sRp[tid] = T.roles[3 * p + 1];
      sRz[tid] = T.roles[3 * p + 2];
    }
  }
  __syncthreads();
  const bool tc = T.G != nullptr;  // adjoint precomputed on the tensor cores (k_tc_tiled.cu)
  if (!tc)
    for (int idx = tid; idx < n * TL_PT; idx += TL_THREADS) {
      const int i = idx / TL_PT, q = idx - i * TL_PT;
      const int p = sPid[q];
      sRY[idx] = p >= 0 ? T.ry32[(size_t)p * n + i] : make_float2(0.f, 0.f);
    }

  // adjoint/epilogue mapping: 16 column groups x 16 pixel pairs
  const int cg = tid & 15, pg = tid >> 4;
  // forward mapping: row = lane + 32 * (warp & 3), pixels (warp >> 2) * 16 + [0, 16)
  const int frow = lane + 32 * (warp & 3);
  const int fph = (warp >> 2) * 16;
  double2 facc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) facc[q] = make_double2(0.0, 0.0);
  double sd2[2] = {0.0, 0.0}, sz1[2] = {0.0, 0.0}, sy2[2] = {0.0, 0.0};

  for (int col0 = s0; col0 < s1; col0 += TL_CT) {
    const int ncols = min(TL_CT, s1 - col0);
    __syncthreads();  // previous tile's sA / sZ fully consumed
    for (int idx = tid; idx < n * TL_CT; idx += TL_THREADS) {
      const int i = idx / TL_CT, c = idx - i * TL_CT;
      sA[i * TL_AS + c] = c < ncols ? __ldg(&T.A[(size_t)i * m + col0 + c]) : make_float2(0.f, 0.f);
    }
    __syncthreads();

    // ---- adjoint: g = 2 A^H r_y for pixels (2pg, 2pg+1), columns cg + 16 j
    float2 acc[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[q][j] = make_float2(0.f, 0.f);
    if (tc) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int p = sPid[2 * pg + q];
        if (p < 0) continue;
        const float2* g = T.G + (size_t)p * m + col0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (cg + 16 * j < ncols) acc[q][j] = g[cg + 16 * j];
      }
    } else if (count <= 8) {
      // few-RHS tiles (cfg5 RBPG: ~8 RHS per block per round): the (column, pixel pair) items are
      // spread over ALL 256 threads -- 64 columns x 4 pairs, one column each -- instead of leaving
      // the 12 pixel-pair rows of the 16 x 16 mapping idle; results go through shared memory (the
      // candidate tile's space, consumed before the epilogue writes it).  Same per-pixel row order
      // and fmaf sequence as below, so bit-identical.
      float2* sG = reinterpret_cast<float2*>(sZ);  // [8][TL_CT]
      const int c = tid & (TL_CT - 1), pp = tid / TL_CT;
      if (2 * pp < count) {
        float2 g0 = make_float2(0.f, 0.f), g1 = make_float2(0.f, 0.f);
        for (int i = 0; i < n; ++i) {
          const float4 r2 = *reinterpret_cast<const float4*>(&sRY[i * TL_PT + 2 * pp]);
          const float2 a = sA[i * TL_AS + c];
          cfma_conj_x2(g0, a, conj_operand(r2.x, r2.y));
          cfma_conj_x2(g1, a, conj_operand(r2.z, r2.w));
        }
        sG[(2 * pp) * TL_CT + c] = g0;
        sG[(2 * pp + 1) * TL_CT + c] = g1;
      }
      __syncthreads();
      if (2 * pg < count) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[q][j] = sG[(2 * pg + q) * TL_CT + cg + 16 * j];
      }
      __syncthreads();
    } else if (2 * pg < count)  // pixel pairs past the tile's count (few-RHS RBPG rounds) skip the GEMM
    for (int i = 0; i < n; ++i) {
      const float4 r2 = *reinterpret_cast<const float4*>(&sRY[i * TL_PT + 2 * pg]);
      // packed FFMA2 (two per complex conj-MAC, the A element as the scalar-broadcast operand): the
      // same per-component rounding sequence as cfma_conj, half the FMA instructions
      const float4 ra = conj_operand(r2.x, r2.y), rbv = conj_operand(r2.z, r2.w);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = sA[i * TL_AS + cg + 16 * j];
#if TB_TILED_FFMA2
        cfma_conj_x2(acc[0][j], a, ra);
        cfma_conj_x2(acc[1][j], a, rbv);
#else
        cfma_conj(acc[0][j], a, make_float2(r2.x, r2.y));
        cfma_conj(acc[1][j], a, make_float2(r2.z, r2.w));
#endif
      }
    }
    // ---- epilogue: extrapolation + soft threshold in fp64 against the HBM state; all-zero state
    //      tiles (occupancy 0) are not read, all-zero candidate tiles are not written
    const int ft = T.ftile[b] + (col0 - c_begin) / TL_CT;
    const size_t PN = (size_t)T.P * T.NT;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int slot = 2 * pg + q;
      const int p = sPid[slot];
      unsigned long long nzm = 0ull;  // this half-warp's pixel: nonzero columns of the tile
      bool ox = false, op = false;
      if (p >= 0) {
        ox = T.occ[sRx[slot] * PN + (size_t)p * T.NT + ft] != 0;
        op = !ista && T.occ[sRp[slot] * PN + (size_t)p * T.NT + ft] != 0;
      }
      double2 zr[4];
      bool zany = false;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = cg + 16 * j;
        double2 w = make_double2(0.0, 0.0);
        zr[j] = make_double2(0.0, 0.0);
        if (p >= 0 && c < ncols) {
          const int gc = col0 + c;
          const double2 xv = ox ? xrow(T, sRx[slot], p)[gc] : make_double2(0.0, 0.0);
          double2 y = xv;
          if (!ista) {
            const double2 pv = op ? xrow(T, sRp[slot], p)[gc] : make_double2(0.0, 0.0);
            const double mk = sMk[slot];
            y = make_double2(fma(mk, xv.x - pv.x, xv.x), fma(mk, xv.y - pv.y, xv.y));
          }
          const double alpha = sAlpha[slot], tau = sTau[slot];
          const double2 v = make_double2(fma(-alpha, 2.0 * (double)acc[q][j].x, y.x), fma(-alpha, 2.0 * (double)acc[q][j].y, y.y));
          const double mag2 = fma(v.x, v.x, v.y * v.y);
          double2 z = make_double2(0.0, 0.0);
          if (!(mag2 <= tau * tau)) {  // zero iff |v| <= tau; NaN propagates (prox.py:82-96)
            const double mag = sqrt(mag2);
            const double sc = 1.0 - tau / mag;
            z = make_double2(v.x * sc, v.y * sc);
            sz1[q] += mag * sc;
          }
          zr[j] = z;
          zany |= (z.x != 0.0) || (z.y != 0.0);
          const double2 d = make_double2(z.x - y.x, z.y - y.y);
          sd2[q] += fma(d.x, d.x, d.y * d.y);
          sy2[q] += fma(y.x, y.x, y.y * y.y);
          w = rb ? d : z;
        }
        sZ[c * TL_ZS + slot] = w;
        // lanes 0-15 hold pixel slot 2*(2*warp)+q, lanes 16-31 slot 2*(2*warp+1)+q, columns cg + 16 j
        const unsigned bits = __ballot_sync(TB_FULL_MASK, w.x != 0.0 || w.y != 0.0);
        nzm |= (unsigned long long)((lane < 16 ? bits : bits >> 16) & 0xFFFFu) << (16 * j);
      }
      if (cg == 0) sMask[slot] = nzm;
      const unsigned zb = __ballot_sync(TB_FULL_MASK, zany);
      const bool tile_nz = ((lane < 16 ? zb : zb >> 16) & 0xFFFFu) != 0u;
      if (p >= 0) {
        if (tile_nz) {
          double2* zrow = xrow(T, sRz[slot], p) + col0;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (cg + 16 * j < ncols) zrow[cg + 16 * j] = zr[j];
        }
        if (cg == 0) T.occ[sRz[slot] * PN + (size_t)p * T.NT + ft] = tile_nz ? 1 : 0;
      }
    }
    __syncthreads();
    // ---- forward partial, fp64 (lane = row, 16 pixels per thread).  Dense over the union of the
    //      16 pixels' nonzero columns (16 independent accumulator chains per column), or, when under
    //      a quarter of that union x 16 block is nonzero (late, sparse iterates), per pixel over its
    //      own nonzero columns.  Either way each pixel accumulates its columns in ascending order.
    {
      unsigned long long uni = 0ull;
      int nnz = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const unsigned long long mq = sMask[fph + q];
        uni |= mq;
        nnz += __popcll(mq);
      }
      if (4 * nnz >= 16 * __popcll(uni)) {
        while (uni) {
          const int c = __ffsll((long long)uni) - 1;
          uni &= uni - 1;
          const float2 af = frow < n ? sA[frow * TL_AS + c] : make_float2(0.f, 0.f);
          const double ax = af.x, ayv = af.y;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const double2 z = sZ[c * TL_ZS + fph + q];
            facc[q].x = fma(ax, z.x, fma(-ayv, z.y, facc[q].x));
            facc[q].y = fma(ax, z.y, fma(ayv, z.x, facc[q].y));
          }
        }
      } else {
        // two pixels' chains interleaved for ILP (warp-uniform branches)
        auto step = [&](unsigned long long& mq, double2& acc, int q) {
          const int c = __ffsll((long long)mq) - 1;
          mq &= mq - 1;
          const float2 af = frow < n ? sA[frow * TL_AS + c] : make_float2(0.f, 0.f);
          const double2 z = sZ[c * TL_ZS + fph + q];
          acc.x = fma((double)af.x, z.x, fma(-(double)af.y, z.y, acc.x));
          acc.y = fma((double)af.x, z.y, fma((double)af.y, z.x, acc.y));
        };
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
          unsigned long long m0 = sMask[fph + q], m1 = sMask[fph + q + 1];
          while (m0 && m1) {
            step(m0, facc[q], q);
            step(m1, facc[q + 1], q + 1);
          }
          while (m0) step(m0, facc[q], q);
          while (m1) step(m1, facc[q + 1], q + 1);
        }
      }
    }
  }
  // ---- write partials
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int o2 = 8; o2 > 0; o2 >>= 1) {
      sd2[q] += __shfl_xor_sync(TB_FULL_MASK, sd2[q], o2);
      sz1[q] += __shfl_xor_sync(TB_FULL_MASK, sz1[q], o2);
      sy2[q] += __shfl_xor_sync(TB_FULL_MASK, sy2[q], o2);
    }
  }
  if (cg == 0) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int p = sPid[2 * pg + q];
      if (p >= 0) {
        double* ps = T.psc + ((size_t)split * T.P + p) * 4;
        ps[0] = sd2[q];
        ps[1] = sz1[q];
        ps[2] = sy2[q];
      }
    }
  }
  if (frow < n) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int p = sPid[fph + q];
      if (p >= 0) T.part[((size_t)split * T.P + p) * n + frow] = facc[q];
    }
  }
}

// ------------------------------------------------------------------ reduce
__global__ void tiled_reduce_kernel(const TiledParams T) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= T.P) return;
  const int n = T.n;
  if (T.phase[p] != PH_TRIAL) {
    for (int i = lane; i < n; i += 32) T.red[(size_t)p * n + i] = make_double2(0.0, 0.0);
    if (lane < 4) T.redsc[(size_t)p * 4 + lane] = 0.0;
    return;
  }
  const int b = T.blk[p];
  const int w = T.bstart[b + 1] - T.bstart[b];
  const int S = w > 0 ? (w + T.split_width - 1) / T.split_width : 0;
  for (int i = lane; i < n; i += 32) {
    double2 s = make_double2(0.0, 0.0);
    for (int sp = 0; sp < S; ++sp) {
      const double2 v = T.part[((size_t)sp * T.P + p) * n + i];
      s.x += v.x;
      s.y += v.y;
    }
    T.red[(size_t)p * n + i] = s;
  }
  if (lane < 4) {
    double s = 0.0;
    if (lane < 3)
      for (int sp = 0; sp < S; ++sp) s += T.psc[((size_t)sp * T.P + p) * 4 + lane];
    T.redsc[(size_t)p * 4 + lane] = s;
  }
}

// ------------------------------------------------------------------ update
__global__ void tiled_update_kernel(const TiledParams T) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= T.P || T.phase[p] != PH_TRIAL) return;
  const int n = T.n;
  const bool rb = T.mode == SOLVER_RBPG;
  const int k = T.k[p];
  const int b = T.blk[p];
  const double alpha = T.alpha[p];
  const double lamd = (double)T.lam[p];
  const double d2 = T.redsc[(size_t)p * 4 + 0], zsum = T.redsc[(size_t)p * 4 + 1];
  double F = T.F[p];
  // quadratic-bound test ||A d||^2 <= ||d||^2/(2 alpha) (solver.py:297-310, prox.py:107-119)
  double l = 0.0, na = 0.0, fz = 0.0;
  for (int i = lane; i < n; i += 32) {
    const size_t o = (size_t)p * n + i;
    const double2 a = T.red[o], ry = T.ry[o];
    if (rb) {
      l += a.x * a.x + a.y * a.y;
      const double rx = ry.x + a.x, ryy = ry.y + a.y;
      fz += rx * rx + ryy * ryy;
    } else {
      const double dx = a.x - ry.x, dy = a.y - ry.y;
      l += dx * dx + dy * dy;
      na += fabs(a.x) + fabs(a.y) + fabs(ry.x) + fabs(ry.y);
      const float2 bb = T.B[o];
      const double fx = a.x - bb.x, fy = a.y - bb.y;
      fz += fx * fx + fy * fy;
    }
  }
  l = warp_sum(l);
  na = warp_sum(na);
  fz = warp_sum(fz);
  const bool pass = rb ? (l * (2.0 * alpha) <= d2 * (1.0 + 1e-9)) : (sqrt(l) <= sqrt(d2 / (2.0 * alpha)) + 1e-12 * na);
  bool done = false;
  int status = T.status[p];
  if (!pass) {
    const int trial = T.trial[p] + 1;
    if (trial > T.cap) {
      if (rb) {  // solver.py:311-314 appends F before the break; ISTA/FISTA do not
        if (lane == 0) T.ring[(size_t)p * 16 + k % (STOP_WINDOW + 1)] = F;
        if (T.hist && lane == 0) T.hist[(size_t)p * T.hist_stride + k] = F;
      }
      status = STATUS_LINE_SEARCH_FAILURE;
      done = true;
    } else if (lane == 0) {
      T.trial[p] = trial;
      T.alpha[p] = alpha * T.c_alpha;
    }
  } else {
    if (rb) {
      const double mk = T.mode == SOLVER_ISTA ? 0.0 : T.mk[k];
      const double l1_new = T.l1[p] - T.l1blk[(size_t)p * T.J + b] + zsum;
      const double cand = fz + lamd * l1_new;
      const bool accept = cand <= F;  // solver.py:317-325
      // block copies prev_b <- x_b (and x_b <- z_b on accept) run in tiled_commit_kernel
      if (lane == 0) T.commit[p] = accept ? 2 : 1;
      for (int i = lane; i < n; i += 32) {
        const size_t o = (size_t)p * n + i;
        double2* dl = T.delta + ((size_t)p * T.J + b) * n + i;
        if (accept) {
          const double2 a = T.red[o], ry = T.ry[o], dv = *dl;
          T.r[o] = make_double2(ry.x + a.x, ry.y + a.y);
          *dl = make_double2(fma(mk, dv.x, a.x), fma(mk, dv.y, a.y));  // A_b(z - x_old) = A_b dz + m_k delta_b
        } else {
          *dl = make_double2(0.0, 0.0);
        }
      }
      if (accept) {
        F = cand;
        if (lane == 0) {
          T.l1[p] = l1_new;
          T.l1blk[(size_t)p * T.J + b] = zsum;
        }
      }
    } else {
      // x_prev <- x, x <- z by buffer role rotation; A x_prev <- A x, A x <- A z
      for (int i = lane; i < n; i += 32) {
        const size_t o = (size_t)p * n + i;
        T.axp[o] = T.r[o];
        T.r[o] = T.red[o];
      }
      if (lane == 0) {
        const int rx = T.roles[3 * p + 0], rp = T.roles[3 * p + 1], rz = T.roles[3 * p + 2];
        T.roles[3 * p + 0] = rz;
        T.roles[3 * p + 1] = rx;
        T.roles[3 * p + 2] = rp;
      }
      F = fz + lamd * zsum;
    }
    double* ring = T.ring + (size_t)p * 16;
    if (lane == 0) {
      ring[k % (STOP_WINDOW + 1)] = F;
      T.F[p] = F;
      if (T.hist) T.hist[(size_t)p * T.hist_stride + k] = F;
    }
    __syncwarp();
    if (!isfinite(F)) {
      status = STATUS_NUMERICAL_FAILURE;
      done = true;
    } else {
      const bool can = k >= STOP_WINDOW;
      const double ref = can ? ring[(k - STOP_WINDOW) % (STOP_WINDOW + 1)] : 0.0;
      const bool conv = can && fabs(F - ref) <= T.tol * fmax(fabs(ref), 1e-300);
      if (!T.fixed && conv) {
        status = STATUS_CONVERGED;
        done = true;
      } else if (k >= T.total_iters) {
        status = conv ? STATUS_CONVERGED : STATUS_MAX_ITERS;  // for-else (solver.py:334-336)
        done = true;
      } else if (lane == 0) {
        T.phase[p] = PH_PREP;
      }
    }
  }
  if (done && lane == 0) {
    T.status[p] = status;
    T.phase[p] = PH_DONE;
    atomicSub(T.remaining, 1);
  }
}

// ------------------------------------------------------------------ commit (RBPG)
// prev_b <- x_b for every pixel that finished a visit this round, x_b <- z_b if it was accepted
// (solver.py:318-325); grid over (pixel, column chunk) so wide blocks copy at HBM bandwidth.
__global__ void tiled_commit_kernel(const TiledParams T) {
  // one warp per occupancy tile of the drawn block; only nonzero tiles move data, the occupancy
  // bits move with them (prev_b <- x_b, then x_b <- z_b on accept)
  const int p = blockIdx.x;
  const int flag = T.commit[p];
  if (flag == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int b = T.blk[p];
  const int c0 = T.bstart[b], c1 = T.bstart[b + 1];
  const int rx = T.roles[3 * p + 0], rp = T.roles[3 * p + 1], rz = T.roles[3 * p + 2];
  double2* xr = xrow(T, rx, p);
  double2* pr = xrow(T, rp, p);
  const double2* zr = xrow(T, rz, p);
  const size_t PN = (size_t)T.P * T.NT;
  unsigned char* ox = T.occ + rx * PN + (size_t)p * T.NT + T.ftile[b];
  unsigned char* op = T.occ + rp * PN + (size_t)p * T.NT + T.ftile[b];
  const unsigned char* oz = T.occ + rz * PN + (size_t)p * T.NT + T.ftile[b];
  const int ntile = (c1 - c0 + TL_CT - 1) / TL_CT;
  for (int t = blockIdx.y * nw + warp; t < ntile; t += gridDim.y * nw) {
    const unsigned char fx = ox[t], fz = oz[t];
#pragma unroll
    for (int h = 0; h < TL_CT / 32; ++h) {
      const int c = c0 + t * TL_CT + lane + 32 * h;
      if (c < c1) {
        if (fx) pr[c] = xr[c];
        if (flag == 2 && fz) xr[c] = zr[c];
      }
    }
    __syncwarp();
    if (lane == 0) {
      op[t] = fx;
      if (flag == 2) ox[t] = fz;
    }
  }
}

__global__ void tiled_commit_clear_kernel(const TiledParams T) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < T.P) T.commit[p] = 0;
}

// ------------------------------------------------------------------ finish
__global__ void tiled_finish_kernel(const TiledParams T) {
  // complex64 x_hat from the fp64 iterate, one warp per occupancy tile (zero tiles not read)
  const int p = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rx = T.roles[3 * p + 0];
  const double2* xr = xrow(T, rx, p);
  const unsigned char* ox = T.occ + rx * (size_t)T.P * T.NT + (size_t)p * T.NT;
  for (int t = blockIdx.y * nw + warp; t < T.NT; t += gridDim.y * nw) {
    int b = 0;
    while (b + 1 < T.J && T.ftile[b + 1] <= t) ++b;
    const int cs = T.bstart[b] + (t - T.ftile[b]) * TL_CT, ce = min(T.bstart[b + 1], cs + TL_CT);
    const bool f = ox[t] != 0;
#pragma unroll
    for (int h = 0; h < TL_CT / 32; ++h) {
      const int c = cs + lane + 32 * h;
      if (c < ce) {
        const double2 v = f ? xr[c] : make_double2(0.0, 0.0);
        T.X[(size_t)p * T.m + c] = make_float2((float)v.x, (float)v.y);
      }
    }
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    T.f_final[p] = T.F[p];
    T.iters[p] = T.k[p];
  }
}

static inline int warp_grid(int P) { return (P + 7) / 8; }

cudaError_t tiled_init(const TiledParams& T, cudaStream_t st) {
  count_launch();
  tiled_init_kernel<<<warp_grid(T.P), 256, 0, st>>>(T);
  return cudaGetLastError();
}

cudaError_t tiled_prep(const TiledParams& T, cudaStream_t st) {
  count_launch();
  tiled_prep_kernel<<<warp_grid(T.P), 256, 0, st>>>(T);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // bucket counters: 3 ints per block in dynamic shared memory (tb_tiled_create bounds J)
  const size_t sched_smem = 3 * (size_t)T.J * sizeof(int);
  if (sched_smem > 48 * 1024) {
    e = cudaFuncSetAttribute(tiled_schedule_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sched_smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  tiled_schedule_kernel<<<1, 1024, sched_smem, st>>>(T);
  return cudaGetLastError();
}

cudaError_t tiled_pass(const TiledParams& T, int num_sms, cudaStream_t st) {
  (void)num_sms;
  const size_t smem = tiled_pass_smem(T.n);
  cudaError_t e = cudaFuncSetAttribute(tiled_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((T.P + TL_PT - 1) / TL_PT + T.J, T.max_splits);
  count_launch();
  tiled_pass_kernel<<<grid, TL_THREADS, smem, st>>>(T);
  return cudaGetLastError();
}

cudaError_t tiled_reduce(const TiledParams& T, cudaStream_t st) {
  count_launch();
  tiled_reduce_kernel<<<warp_grid(T.P), 256, 0, st>>>(T);
  return cudaGetLastError();
}

cudaError_t tiled_update(const TiledParams& T, cudaStream_t st) {
  const bool rb = T.mode == SOLVER_RBPG;
  if (rb) {
    count_launch();
    tiled_commit_clear_kernel<<<(T.P + 255) / 256, 256, 0, st>>>(T);
  }
  count_launch();
  tiled_update_kernel<<<warp_grid(T.P), 256, 0, st>>>(T);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !rb) return e;
  int maxw = 0;
  // widest block (host copy of the starts is not kept here; bound by m / J rounded up)
  maxw = (T.m + T.J - 1) / T.J + 1;
  int chunks = (maxw / TL_CT + 31) / 32;  // 8 warps x ~4 occupancy tiles per CTA
  chunks = chunks < 1 ? 1 : chunks > 64 ? 64 : chunks;
  dim3 grid(T.P, chunks);
  count_launch();
  tiled_commit_kernel<<<grid, 256, 0, st>>>(T);
  return cudaGetLastError();
}

cudaError_t tiled_finish(const TiledParams& T, cudaStream_t st) {
  int chunks = (T.NT + 31) / 32;  // 8 warps x ~4 tiles per CTA
  chunks = chunks < 1 ? 1 : chunks > 64 ? 64 : chunks;
  dim3 grid(T.P, chunks);
  count_launch();
  tiled_finish_kernel<<<grid, 256, 0, st>>>(T);
  return cudaGetLastError();
}

}  // namespace tb
