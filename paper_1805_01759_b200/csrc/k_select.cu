// SL1MMER stages 2-3 on device (slimmer.py:77-190), one warp per pixel, fp64 linear algebra.
//
//  detect_support   slimmer.py:77-113  elevation profile (max over motion axes, model.py:210-215),
//                   local maxima (strict left / non-strict right, edges count) above 1e-8 * peak,
//                   top k_max by magnitude with ties resolved to the larger bin (argsort+reverse),
//                   joint argmax over motion bins (first occurrence).
//  model_select     slimmer.py:116-154 rank filter, nested LS refits, BIC = 2N ln(RSS/2N) + pK ln 2N.
//  estimate_params  slimmer.py:157-190 debiased LS amplitudes on the support, grid decode.
// LS is done by an incremental modified Gram-Schmidt QR (two passes) in fp64; RSS is the norm of
// the explicit residual, amplitudes come from back substitution on R.
#include <float.h>

#include "common.cuh"
#include "setup.h"

namespace tb {

constexpr int SEL_MAXQ = 4;   // rows per lane (n <= 128)
constexpr int SEL_MAXK = 8;   // k_max cap

__device__ __forceinline__ double2 zmul_conj(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

__global__ void __launch_bounds__(128) select_kernel(const SelectParams S) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = S.n, m = S.m, ne = S.n_elev, inner = S.inner, kmax = S.k_max;
  const size_t per = select_warp_bytes(n, ne, kmax);
  unsigned char* base = smem + (size_t)warp * per;
  double* prof = reinterpret_cast<double*>(base);
  int* amx = reinterpret_cast<int*>(prof + ne);
  double2* Q = reinterpret_cast<double2*>(base + (((size_t)ne * 12 + 15) & ~(size_t)15));  // [kmax][n]
  double2* Rs = Q + (size_t)kmax * n;  // R[kmax][kmax], row-major, warp-uniform values
#define R(r, c) Rs[(r) * kmax + (c)]

  for (long long p = (long long)blockIdx.x * nw + warp; p < S.num_pixels; p += (long long)gridDim.x * nw) {
    const float2* x = S.X + (size_t)p * m;
    // ---- elevation profile + per-bin argmax over motion bins
    double peak = 0.0;
    if (inner == 1) {
      // elevation-only grids (cfg1-3): the lane's loads of x_hat are issued four at a time -- one
      // dependent global load per loop trip left the warp waiting ~10 DRAM latencies per pixel
      // (long scoreboard was the kernel's top stall); same values, same order of the max
      for (int s0 = lane; s0 < ne; s0 += 128) {
        float2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = s0 + 32 * u < ne ? x[s0 + 32 * u] : make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int s = s0 + 32 * u;
          if (s < ne) {
            const double a = sqrt((double)v[u].x * v[u].x + (double)v[u].y * v[u].y);
            const double best = a > -1.0 ? a : -1.0;  // a NaN magnitude reads as -1, as below
            prof[s] = best;
            amx[s] = 0;
            peak = fmax(peak, best);
          }
        }
      }
    } else
    for (int s = lane; s < ne; s += 32) {
      double best = -1.0;
      int arg = 0;
      for (int j = 0; j < inner; ++j) {
        float2 v = x[(size_t)s * inner + j];
        double a = sqrt((double)v.x * v.x + (double)v.y * v.y);
        if (a > best) {
          best = a;
          arg = j;
        }
      }
      prof[s] = best;
      amx[s] = arg;
      peak = fmax(peak, best);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(TB_FULL_MASK, peak, o));
    __syncwarp();

    // ---- top-k peaks (descending magnitude, ties -> larger bin)
    int cand_bin[SEL_MAXK];
    int ncand = 0;
    if (peak > 0.0) {
      const double floor_v = 1e-8 * peak;
      for (int k = 0; k < kmax; ++k) {
        double bv = -1.0;
        int bs = -1;
        for (int s = lane; s < ne; s += 32) {
          double v = prof[s];
          bool left = (s == 0) || (v > prof[s - 1]);
          bool right = (s == ne - 1) || (v >= prof[s + 1]);
          if (!(left && right && v > floor_v)) continue;
          bool taken = false;
          for (int t = 0; t < ncand; ++t) taken |= (cand_bin[t] == s);
          if (taken) continue;
          if (v > bv || (v == bv && s > bs)) {
            bv = v;
            bs = s;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double ov = __shfl_xor_sync(TB_FULL_MASK, bv, o);
          int os = __shfl_xor_sync(TB_FULL_MASK, bs, o);
          if (ov > bv || (ov == bv && os > bs)) {
            bv = ov;
            bs = os;
          }
        }
        if (bs < 0) break;
        cand_bin[ncand++] = bs;
      }
    }

    // ---- g = b (fp64), ||g||^2
    double2 g[SEL_MAXQ];
    double gg = 0.0;
#pragma unroll
    for (int q = 0; q < SEL_MAXQ; ++q) {
      int i = lane + 32 * q;
      g[q] = make_double2(0.0, 0.0);
      if (i < n) {
        float2 b = S.B[(size_t)p * n + i];
        g[q] = make_double2(b.x, b.y);
        gg += g[q].x * g[q].x + g[q].y * g[q].y;
      }
    }
    gg = warp_sum(gg);

    // ---- rank filter via incremental MGS QR (slimmer.py:116-123)
    long long usable[SEL_MAXK];
    int nu = 0;
    double fro2 = 0.0;
    for (int t = 0; t < ncand; ++t) {
      const long long col = (long long)cand_bin[t] * inner + amx[cand_bin[t]];
      double2 a[SEL_MAXQ];
      double an = 0.0;
#pragma unroll
      for (int q = 0; q < SEL_MAXQ; ++q) {
        int i = lane + 32 * q;
        a[q] = make_double2(0.0, 0.0);
        if (i < n) {
          float2 v = S.A[(size_t)i * m + col];
          a[q] = make_double2(v.x, v.y);
          an += a[q].x * a[q].x + a[q].y * a[q].y;
        }
      }
      an = warp_sum(an);
      double2 rcol[SEL_MAXK];
      for (int j = 0; j < SEL_MAXK; ++j) rcol[j] = make_double2(0.0, 0.0);
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = 0; j < nu; ++j) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int q = 0; q < SEL_MAXQ; ++q) {
            int i = lane + 32 * q;
            if (i < n) {
              double2 c = zmul_conj(Q[(size_t)j * n + i], a[q]);
              re += c.x;
              im += c.y;
            }
          }
          re = warp_sum(re);
          im = warp_sum(im);
#pragma unroll
          for (int q = 0; q < SEL_MAXQ; ++q) {
            int i = lane + 32 * q;
            if (i < n) {
              double2 qq = Q[(size_t)j * n + i];
              a[q].x -= re * qq.x - im * qq.y;
              a[q].y -= re * qq.y + im * qq.x;
            }
          }
          rcol[j].x += re;
          rcol[j].y += im;
        }
      }
      double rn = 0.0;
#pragma unroll
      for (int q = 0; q < SEL_MAXQ; ++q) rn += a[q].x * a[q].x + a[q].y * a[q].y;
      rn = sqrt(warp_sum(rn));
      const double tol = sqrt(fro2 + an) * (double)max(n, nu + 1) * DBL_EPSILON;
      if (rn > tol) {
        const double inv = 1.0 / rn;
#pragma unroll
        for (int q = 0; q < SEL_MAXQ; ++q) {
          int i = lane + 32 * q;
          if (i < n) Q[(size_t)nu * n + i] = make_double2(a[q].x * inv, a[q].y * inv);
        }
        for (int j = 0; j < nu; ++j) R(j, nu) = rcol[j];  // every lane stores the same value
        R(nu, nu) = make_double2(rn, 0.0);
        usable[nu] = col;
        ++nu;
        fro2 += an;
        __syncwarp();
      }
    }

    // ---- nested LS refits + BIC (slimmer.py:140-154)
    const double n2 = 2.0 * n;
    const double pp = (double)S.ppsc;
    double scores[SEL_MAXK + 1];
    double2 tq[SEL_MAXK];
    scores[0] = n2 * log(fmax(gg, 1e-300) / n2);
    double2 res[SEL_MAXQ];
#pragma unroll
    for (int q = 0; q < SEL_MAXQ; ++q) res[q] = g[q];
    for (int k = 1; k <= nu; ++k) {
      const int j = k - 1;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int q = 0; q < SEL_MAXQ; ++q) {
        int i = lane + 32 * q;
        if (i < n) {
          double2 c = zmul_conj(Q[(size_t)j * n + i], res[q]);
          re += c.x;
          im += c.y;
        }
      }
      re = warp_sum(re);
      im = warp_sum(im);
      tq[j] = make_double2(re, im);
      double rss = 0.0;
#pragma unroll
      for (int q = 0; q < SEL_MAXQ; ++q) {
        int i = lane + 32 * q;
        if (i < n) {
          double2 qq = Q[(size_t)j * n + i];
          res[q].x -= re * qq.x - im * qq.y;
          res[q].y -= re * qq.y + im * qq.x;
          rss += res[q].x * res[q].x + res[q].y * res[q].y;
        }
      }
      rss = warp_sum(rss);
      scores[k] = n2 * log(fmax(rss, 1e-300) / n2) + pp * k * log(n2);
    }
    int khat = 0;
    for (int k = 1; k <= nu; ++k)
      if (scores[k] < scores[khat]) khat = k;

    // ---- debiased amplitudes: R[:khat,:khat] coef = t (slimmer.py:173-176)
    double2 coef[SEL_MAXK];
    for (int r = khat - 1; r >= 0; --r) {
      double2 s = tq[r];
      for (int c = r + 1; c < khat; ++c) {
        double2 rr = R(r, c), cc = coef[c];
        s.x -= rr.x * cc.x - rr.y * cc.y;
        s.y -= rr.x * cc.y + rr.y * cc.x;
      }
      double d = R(r, r).x;
      coef[r] = make_double2(s.x / d, s.y / d);
    }

    if (lane == 0) {
      S.order[p] = khat;
      S.n_scores[p] = nu + 1;
      S.err[p] = 0;
      for (int k = 0; k < kmax; ++k) {
        const size_t o = (size_t)p * kmax + k;
        if (k < khat) {
          const long long col = usable[k];
          S.support[o] = col;
          S.amps[o] = coef[k];
          const int s = (int)(col / inner);
          const int jj = (int)(col - (long long)s * inner);
          S.elevs[o] = S.elev[s];
          if (S.n_axes >= 1) {
            const int j0 = S.n_axes == 2 ? jj / S.msize1 : jj;
            S.motion_out[o * S.n_axes + 0] = S.motion[j0];
            if (S.n_axes == 2) S.motion_out[o * S.n_axes + 1] = S.motion[S.msize0 + (jj % S.msize1)];
          }
        } else {
          S.support[o] = -1;
          S.amps[o] = make_double2(0.0, 0.0);
          S.elevs[o] = 0.0;
          for (int a = 0; a < S.n_axes; ++a) S.motion_out[o * S.n_axes + a] = 0.0;
        }
      }
      for (int k = 0; k <= kmax; ++k) S.scores[(size_t)p * (kmax + 1) + k] = (k <= nu) ? scores[k] : __longlong_as_double(0x7ff8000000000000ll);
    }
    __syncwarp();
  }
}

#undef R

cudaError_t launch_select(const SelectParams& S, int num_sms, cudaStream_t st) {
  if (S.num_pixels <= 0) return cudaSuccess;
  if (S.k_max > SEL_MAXK || S.n > 32 * SEL_MAXQ || S.n_axes > 2) return cudaErrorInvalidValue;
  const int warps = 4;
  size_t smem = (size_t)warps * select_warp_bytes(S.n, S.n_elev, S.k_max);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long long blocks = (S.num_pixels + warps - 1) / warps;
  if (blocks > (long long)num_sms * 16) blocks = (long long)num_sms * 16;
  count_launch();
  select_kernel<<<(int)blocks, warps * 32, smem, st>>>(S);
  return cudaGetLastError();
}

}  // namespace tb
