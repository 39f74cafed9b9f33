// RBPG with G lanes per pixel (G = 16: two pixels per warp) for dictionaries that fit on chip.
//
// Same algorithm and numerics as warp_solver_kernel's RBPG path (solver.py:250-338; see
// k_warp_solver.cu), re-laid out for throughput: the per-iteration scalar work of RBPG (block draw,
// step-size lookup, backtracking test, monotone acceptance, window stop) is executed once per
// half-warp instead of once per warp, and each pixel slot keeps its extrapolation memory as the
// fp32 difference d_b = x_b - prev_b (y_b = x_b + m_k d_b; exact zero after a rejected visit, so
// the reference's `np.any(dy)` test is reproduced bit-for-bit) next to the fp64 iterate, which
// shrinks a slot to ~9 KB so ~18 pixels are in flight per SM.
#include <float.h>

#include "common.cuh"
#include "solver_params.h"

namespace tb {

template <int G>
__device__ __forceinline__ double group_sum(double v, unsigned gmask) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
  return v;
}

template <int G, int MAXT, int MAXQ, bool ASMEM>
__global__ void __launch_bounds__(320) rbpg_group_kernel(const SolveParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (0xffffu << (16 * grp));
  const int n = P.n, m = P.m, ms = P.ms;
  const int J = P.num_blocks;

  float2* As = reinterpret_cast<float2*>(smem);
  size_t off = ASMEM ? (((size_t)n * ms * sizeof(float2) + 15) & ~(size_t)15) : 0;
  if (ASMEM) {
    for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) {
      int i = idx / m, c = idx - i * m;
      As[(size_t)i * ms + c] = __ldg(&P.A[idx]);
    }
  }
  double* s_cdf = reinterpret_cast<double*>(smem + off);
  double* s_alpha0 = s_cdf + J;
  int* s_bstart = reinterpret_cast<int*>(s_alpha0 + J);
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    s_cdf[j] = P.cdf[j];
    s_alpha0[j] = P.alpha_scale / fmax(P.blk_lip[j], 1e-300);  // solver.py:295
  }
  for (int j = threadIdx.x; j <= J; j += blockDim.x) s_bstart[j] = P.blk_start[j];
  __syncthreads();
  off += block_table_bytes(J);
  const int slot = warp * (32 / G) + grp;
  unsigned char* wb = smem + off + (size_t)slot * rbpg_slot_bytes(n, m, P.max_width, J);
  double2* rv = reinterpret_cast<double2*>(wb);  // residual r (fp64)
  double2* xs = rv + n;                          // x (fp64)
  double2* zs = xs + m;                          // broadcast buffer [max_width]
  float2* ds = reinterpret_cast<float2*>(zs + P.max_width);  // d = x - prev (fp32)
  float2* ryv = ds + m;                          // r_y rounded for the adjoint
  double* ring = reinterpret_cast<double*>(ryv + n + (n & 1));  // last STOP_WINDOW+1 objective values
  double* l1blk = ring + 16;                     // sum |x_b| per block

  auto Arow = [&](int i) -> const float2* { return ASMEM ? As + (size_t)i * ms : P.A + (size_t)i * m; };

  // group-local pixel state
  long long p = -1;
  int k = 0;
  double F = 0.0, l1 = 0.0, lamd = 0.0;
  Philox4x64 rng;
  bool alive = true;

  auto claim = [&]() -> bool {
    unsigned long long pq = 0;
    if (gl == 0) pq = atomicAdd(P.queue, 1ull);
    pq = __shfl_sync(gmask, pq, 0, G);
    if (pq >= (unsigned long long)P.num_pixels) return false;
    p = (long long)pq;
    lamd = (double)P.lam[p];
    for (int c = gl; c < m; c += G) {
      xs[c] = make_double2(0.0, 0.0);
      ds[c] = make_float2(0.f, 0.f);
    }
    double fb = 0.0;
    for (int i = gl; i < n; i += G) {
      const float2 b = P.B[(size_t)p * n + i];
      rv[i] = make_double2(-(double)b.x, -(double)b.y);  // r = -b (solver.py:273)
      fb += (double)b.x * b.x + (double)b.y * b.y;
    }
    for (int j = gl; j < J; j += G) l1blk[j] = 0.0;
    F = group_sum<G>(fb, gmask);
    l1 = 0.0;
    k = 0;
    if (gl == 0) ring[0] = F;
    if (P.hist && gl == 0) P.hist[(size_t)p * P.hist_stride] = F;
    philox_init(rng, P.seeds[p], 0ull);
    __syncwarp(gmask);
    return true;
  };
  auto finish = [&](int status) {
    __syncwarp(gmask);
    for (int c = gl; c < m; c += G) {
      const double2 xv = xs[c];
      P.X[(size_t)p * m + c] = make_float2((float)xv.x, (float)xv.y);
    }
    if (gl == 0) {
      P.f_final[p] = F;
      P.iters[p] = k;
      P.status[p] = status;
    }
    __syncwarp(gmask);
  };

  alive = claim();
  while (__any_sync(0xffffffffu, alive)) {
    if (!alive) continue;
    k += 1;
    // ---- block draw (solver.py:283, 217-219)
    const double u = raw_to_unit(philox_next(rng));
    int blk = 0;
    while (blk < J - 1 && s_cdf[blk] <= u) ++blk;
    const int cs = s_bstart[blk];
    const int width = s_bstart[blk + 1] - cs;
    const double mk = P.mk[k];

    // ---- y = x + m_k d (solver.py:288-289), dy = y - x
    double2 y[MAXT], z[MAXT];
    float2 g[MAXT];
    unsigned masks[MAXT];
    bool any_dy = false;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int cl = gl + G * t;
      y[t] = make_double2(0.0, 0.0);
      bool nz = false;
      if (cl < width) {
        const double2 xv = xs[cs + cl];
        const float2 dv = ds[cs + cl];
        const double2 yv = make_double2(fma(mk, (double)dv.x, xv.x), fma(mk, (double)dv.y, xv.y));
        y[t] = yv;
        const double2 dy = make_double2(yv.x - xv.x, yv.y - xv.y);
        zs[cl] = dy;
        nz = (dy.x != 0.0) || (dy.y != 0.0);
      }
      masks[t] = (__ballot_sync(gmask, nz) >> (G == 32 ? 0 : 16 * grp)) & (G == 32 ? 0xffffffffu : 0xffffu);
      any_dy |= masks[t] != 0u;
    }
    __syncwarp(gmask);

    // forward over the nonzero entries of zs: acc[q] = sum_c A[i][cs+c] zs[c], fp64
    auto forward = [&](double2* acc) {
      const float2* ar[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        acc[q] = make_double2(0.0, 0.0);
        ar[q] = Arow(min(gl + G * q, n - 1)) + cs;
      }
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        unsigned mkk = masks[t];
        while (mkk) {
          const int c = (__ffs(mkk) - 1) + G * t;
          mkk &= mkk - 1;
          const double2 v = zs[c];
#pragma unroll
          for (int q = 0; q < MAXQ; ++q) {
            const float2 a = ASMEM ? ar[q][c] : __ldg(ar[q] + c);
            acc[q].x = fma((double)a.x, v.x, fma(-(double)a.y, v.y, acc[q].x));
            acc[q].y = fma((double)a.x, v.y, fma((double)a.y, v.x, acc[q].y));
          }
        }
      }
    };

    // ---- r_y = r + A_b dy, skipped when dy == 0 (solver.py:290-291)
    double2 ry[MAXQ];
    {
      double2 acc[MAXQ];
      if (any_dy) forward(acc);
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int i = gl + G * q;
        ry[q] = make_double2(0.0, 0.0);
        if (i < n) {
          const double2 r = rv[i];
          ry[q] = any_dy ? make_double2(r.x + acc[q].x, r.y + acc[q].y) : r;
          ryv[i] = make_float2((float)ry[q].x, (float)ry[q].y);
        }
      }
    }
    __syncwarp(gmask);

    // ---- g = 2 A_b^H r_y (solver.py:293), fp32 products
    {
      float2 acc[MAXT];
#pragma unroll
      for (int t = 0; t < MAXT; ++t) acc[t] = make_float2(0.f, 0.f);
      const float2* acol = ASMEM ? As + cs + gl : P.A + cs + gl;
      const int stride = ASMEM ? ms : m;
      int aoff = 0;
      for (int i = 0; i < n; ++i, aoff += stride) {
        const float2 r = ryv[i];
#pragma unroll
        for (int t = 0; t < MAXT; ++t)
          if (gl + G * t < width) cfma_conj(acc[t], ASMEM ? acol[aoff + G * t] : __ldg(acol + aoff + G * t), r);
      }
#pragma unroll
      for (int t = 0; t < MAXT; ++t) g[t] = make_float2(2.f * acc[t].x, 2.f * acc[t].y);
    }

    // ---- backtracking (solver.py:295-314)
    double alpha = s_alpha0[blk];
    bool ok = false;
    double2 adz[MAXQ];
    double l1z = 0.0, fzs = 0.0;
    for (int trial = 0; trial <= P.cap; ++trial) {
      const double tau = alpha * lamd;
      const double tau2 = tau * tau;
      double red[4] = {0.0, 0.0, 0.0, 0.0};  // |dz|^2, sum|z|, ||A dz||^2, ||r_z||^2
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const int cl = gl + G * t;
        bool nz = false;
        z[t] = make_double2(0.0, 0.0);
        if (cl < width) {
          const double2 v = make_double2(fma(-alpha, (double)g[t].x, y[t].x), fma(-alpha, (double)g[t].y, y[t].y));
          const double mag2 = fma(v.x, v.x, v.y * v.y);
          if (mag2 > tau2) {  // soft threshold (prox.py:82-96)
            const double mag = sqrt(mag2);
            const double sc = 1.0 - tau / mag;
            z[t] = make_double2(v.x * sc, v.y * sc);
            red[1] += mag * sc;
          }
          const double2 d = make_double2(z[t].x - y[t].x, z[t].y - y[t].y);
          red[0] += fma(d.x, d.x, d.y * d.y);
          zs[cl] = d;
          nz = (d.x != 0.0) || (d.y != 0.0);
        }
        masks[t] = (__ballot_sync(gmask, nz) >> (G == 32 ? 0 : 16 * grp)) & (G == 32 ? 0xffffffffu : 0xffffu);
      }
      __syncwarp(gmask);
      forward(adz);
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        if (gl + G * q < n) {
          red[2] += adz[q].x * adz[q].x + adz[q].y * adz[q].y;
          const double rx = ry[q].x + adz[q].x, ryy = ry[q].y + adz[q].y;
          red[3] += rx * rx + ryy * ryy;
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int r = 0; r < 4; ++r) red[r] += __shfl_xor_sync(gmask, red[r], o);
      }
      __syncwarp(gmask);
      l1z = red[1];
      fzs = red[3];
      if (red[2] * (2.0 * alpha) <= red[0] * (1.0 + 1e-9)) {  // ||A dz||^2 <= ||dz||^2/(2 alpha)
        ok = true;
        break;
      }
      alpha *= P.c_alpha;
    }
    int status = STATUS_MAX_ITERS;
    bool done = false;
    if (!ok) {
      if (gl == 0) ring[k % (STOP_WINDOW + 1)] = F;  // solver.py:311-314
      if (P.hist && gl == 0) P.hist[(size_t)p * P.hist_stride + k] = F;
      status = STATUS_LINE_SEARCH_FAILURE;
      done = true;
    } else {
      // ---- monotone acceptance with incremental l1 (solver.py:316-325)
      const double l1_new = l1 - l1blk[blk] + l1z;
      const double cand = fzs + lamd * l1_new;
      const bool accept = cand <= F;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const int cl = gl + G * t;
        if (cl < width) {
          if (accept) {
            const double2 xv = xs[cs + cl];
            ds[cs + cl] = make_float2((float)(z[t].x - xv.x), (float)(z[t].y - xv.y));
            xs[cs + cl] = z[t];
          } else {
            ds[cs + cl] = make_float2(0.f, 0.f);  // prev_b <- x_b
          }
        }
      }
      if (accept) {
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = gl + G * q;
          if (i < n) rv[i] = make_double2(ry[q].x + adz[q].x, ry[q].y + adz[q].y);
        }
        l1 = l1_new;
        F = cand;
        if (gl == 0) l1blk[blk] = l1z;
      }
      if (gl == 0) ring[k % (STOP_WINDOW + 1)] = F;
      if (P.hist && gl == 0) P.hist[(size_t)p * P.hist_stride + k] = F;
      __syncwarp(gmask);
      if (!isfinite(F)) {
        status = STATUS_NUMERICAL_FAILURE;
        done = true;
      } else {
        const bool can = k >= STOP_WINDOW;
        const double ref = can ? ring[(k - STOP_WINDOW) % (STOP_WINDOW + 1)] : 0.0;
        const bool conv = can && fabs(F - ref) <= P.tol * fmax(fabs(ref), 1e-300);
        if (!P.fixed && conv) {
          status = STATUS_CONVERGED;
          done = true;
        } else if (k >= P.total_iters) {
          status = conv ? STATUS_CONVERGED : STATUS_MAX_ITERS;  // for-else (solver.py:334-336)
          done = true;
        }
      }
    }
    if (done) {
      finish(status);
      alive = claim();
    }
  }
}

template <int G, int MAXT, int MAXQ, bool ASMEM>
static cudaError_t launch_g(const SolveParams& P, int warps, size_t smem, int grid, cudaStream_t st) {
  auto k = rbpg_group_kernel<G, MAXT, MAXQ, ASMEM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  k<<<grid, warps * 32, smem, st>>>(P);
  return cudaGetLastError();
}

template <int MAXT, bool ASMEM>
static cudaError_t launch_gq(const SolveParams& P, int maxq, int warps, size_t smem, int grid, cudaStream_t st) {
  switch (maxq) {
    case 1: return launch_g<16, MAXT, 1, ASMEM>(P, warps, smem, grid, st);
    case 2: return launch_g<16, MAXT, 2, ASMEM>(P, warps, smem, grid, st);
    case 4: return launch_g<16, MAXT, 4, ASMEM>(P, warps, smem, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

bool rbpg_group_supported(int n, int max_width) { return max_width <= 64 && n <= 64; }

cudaError_t launch_rbpg_group(const SolveParams& P, int num_sms, cudaStream_t st) {
  const int G = 16;
  int maxt = (P.max_width + G - 1) / G;
  int maxq = (P.n + G - 1) / G;
  maxq = maxq <= 1 ? 1 : maxq <= 2 ? 2 : 4;
  const int J = P.num_blocks;
  const size_t slot = rbpg_slot_bytes(P.n, P.m, P.max_width, J);
  const size_t tables = block_table_bytes(J);
  const size_t a_bytes = ((size_t)P.n * P.ms * sizeof(float2) + 15) & ~(size_t)15;
  const size_t cap = 227 * 1024;
  const bool asmem = a_bytes + tables + 8 * slot <= cap;
  const size_t avail = cap - tables - (asmem ? a_bytes : 0);
  int slots = (int)(avail / slot);
  int warps = slots / 2;
  if (warps > 10) warps = 10;
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = (asmem ? a_bytes : 0) + tables + (size_t)warps * 2 * slot;
  long long need = (P.num_pixels + 2 * warps - 1) / (2 * warps);
  int grid = num_sms;
  if (need < grid) grid = (int)need;
  if (grid < 1) grid = 1;
  if (maxt <= 2) return asmem ? launch_gq<2, true>(P, maxq, warps, smem, grid, st) : launch_gq<2, false>(P, maxq, warps, smem, grid, st);
  if (maxt <= 3) return asmem ? launch_gq<3, true>(P, maxq, warps, smem, grid, st) : launch_gq<3, false>(P, maxq, warps, smem, grid, st);
  if (maxt <= 4) return asmem ? launch_gq<4, true>(P, maxq, warps, smem, grid, st) : launch_gq<4, false>(P, maxq, warps, smem, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace tb
