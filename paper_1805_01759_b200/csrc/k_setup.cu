// Per-batch and per-dictionary setup kernels:
//   default_lambda  (prox.py:153-161)      lambda_p = beta * max_k |(A^H b_p)_k|
//   derive_seeds    (cli.py:102, rng.py:17-29)  per-pixel RBPG seeds from (run_seed, pixel_id)
//   power iteration (solver.py:167-188)    sigma_max^2 of column ranges, fp64
#include <float.h>

#include "common.cuh"
#include "setup.h"

namespace tb {

// ------------------------------------------------------------------ default lambda
// lambda_p = beta * max_k |(A^H b_p)_k| as a tiled complex GEMM with a max epilogue: a CTA owns 64
// dictionary columns x 64 pixels; 16-row K slices of A and of the pixel chunk are staged in shared
// memory (converted to fp64 once at staging) and every thread accumulates a 4 x 4 (column x pixel)
// micro-tile (columns tc + 16 i, pixels tp + 16 j: conflict-free / broadcast shared reads), so each
// A element fetched from HBM/L2 serves 64 pixels instead of one.  The products of the complex64
// inputs are exact in fp64 and are accumulated in fp64, as the reference's complex128
// `a.conj().T @ b` does (prox.py:159-161), so lambda is the reference's up to summation order
// (~1e-16 relative) and is carried as a double end to end.  The column max is order-free, so it is
// merged across CTAs with an integer atomicMax on the (non-negative) double bits: deterministic.
constexpr int LT_C = 64, LT_P = 64, LT_K = 16;

__global__ void __launch_bounds__(256) lambda_tile_kernel(const float2* __restrict__ A, int n, int m,
                                                          const float2* __restrict__ B, long long P,
                                                          unsigned long long* __restrict__ bits) {
  __shared__ double2 sa[LT_K][LT_C];
  __shared__ double2 sb[LT_K][LT_P + 1];  // +1: conflict-light transposed staging stores
  const int tid = threadIdx.x, tc = tid & 15, tp = tid >> 4;
  const long long c0 = (long long)blockIdx.x * LT_C;
  for (long long p0 = (long long)blockIdx.y * LT_P; p0 < P; p0 += (long long)gridDim.y * LT_P) {
    double2 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
    for (int k0 = 0; k0 < n; k0 += LT_K) {
      for (int e = tid; e < LT_K * LT_C; e += 256) {
        const int kk = e / LT_C, cc = e % LT_C;
        const long long c = c0 + cc;
        const int i = k0 + kk;
        const float2 v = (i < n && c < m) ? __ldg(&A[(size_t)i * m + c]) : make_float2(0.f, 0.f);
        sa[kk][cc] = make_double2(v.x, v.y);
      }
      for (int e = tid; e < LT_K * LT_P; e += 256) {
        const int pp = e / LT_K, kk = e % LT_K;
        const long long p = p0 + pp;
        const int i = k0 + kk;
        const float2 v = (i < n && p < P) ? __ldg(&B[(size_t)p * n + i]) : make_float2(0.f, 0.f);
        sb[kk][pp] = make_double2(v.x, v.y);
      }
      __syncthreads();
      const int kn = min(LT_K, n - k0);
      for (int kk = 0; kk < kn; ++kk) {
        double2 a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sa[kk][tc + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = sb[kk][tp + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // conj(a) b
            acc[i][j].x = fma(a[i].x, b[j].x, fma(a[i].y, b[j].y, acc[i][j].x));
            acc[i][j].y = fma(a[i].x, b[j].y, fma(-a[i].y, b[j].x, acc[i][j].y));
          }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double best = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (c0 + tc + 16 * i < m) best = fmax(best, hypot(acc[i][j].x, acc[i][j].y));
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(TB_FULL_MASK, best, o));
      const long long p = p0 + tp + 16 * j;
      if (tc == 0 && p < P) atomicMax(&bits[p], (unsigned long long)__double_as_longlong(best));
    }
  }
}

__global__ void lambda_finish_kernel(double* lam, long long P, double beta) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) lam[p] = beta * lam[p];
}

cudaError_t launch_default_lambda(const float2* A, int n, int m, const float2* B, long long P, double beta,
                                  double* lam, int num_sms, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(lam, 0, sizeof(double) * (size_t)P, st);  // +0.0 bits: the max identity
  if (e != cudaSuccess) return e;
  const long long ctiles = (m + LT_C - 1) / LT_C, pchunks = (P + LT_P - 1) / LT_P;
  long long gy = (long long)num_sms * 8 / ctiles;
  if (gy < 1) gy = 1;
  if (gy > pchunks) gy = pchunks;
  if (gy > 65535) gy = 65535;
  if (ctiles > 0x7fffffffll) return cudaErrorInvalidValue;
  count_launch();
  lambda_tile_kernel<<<dim3((unsigned)ctiles, (unsigned)gy), 256, 0, st>>>(A, n, m, B, P, reinterpret_cast<unsigned long long*>(lam));
  count_launch();
  lambda_finish_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(lam, P, beta);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ derive_seed
// integers(0, 2^63-1) on substream(run_seed, pixel_id): Lemire with range 2^63-1.
__global__ void derive_seeds_kernel(uint64_t run_seed, long long first, long long P, uint64_t* seeds) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P) return;
  Philox4x64 s;
  philox_init(s, run_seed, (uint64_t)(first + idx));
  const uint64_t rng_excl = 0x7FFFFFFFFFFFFFFFull;
  for (;;) {
    uint64_t raw = philox_next(s);
    uint64_t lo = raw * rng_excl, hi = __umul64hi(raw, rng_excl);
    if (lo >= 2ull) {
      seeds[idx] = hi;
      return;
    }
  }
}

cudaError_t launch_derive_seeds(uint64_t run_seed, long long first, long long P, uint64_t* seeds, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  count_launch();
  derive_seeds_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(run_seed, first, P, seeds);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ two-scatterer realizations
// The Monte-Carlo realization of simulate.py:297-335 drawn on the device: g = A[:, c0] + e^{j phi}
// A[:, c1] + sqrt(sigma^2 / 2) (N + jN) with unit amplitudes on grid columns c0, c1 (the reference
// snaps both scatterers to the grid, simulate.py:312-322), one warp per realization, lane = row.
// Every realization draws from Philox4x64-10 keyed (seed, stream_id) -- the reference's substream
// (rng.py:17-24) -- in a fixed layout: raw 0 = the phase (numpy's next_double, used when phase is
// NaN), raws 1 + 2i, 2 + 2i = the two uniforms Box-Muller turns into row i's complex normal, raw
// 1 + 2n onwards = the nested RBPG seed (integers(0, 2^63 - 1), Lemire, as derive_seed).  The
// normals are NOT numpy's ziggurat draws, so realizations are statistically (not bit-) equivalent
// to the reference's.
__global__ void synth_pair_kernel(const float2* __restrict__ A, int n, int m, uint64_t seed, const uint64_t* stream_ids,
                                  const int* c0, const int* c1, const float* phase, const float* sigma, long long count,
                                  float2* pixels, uint64_t* seeds) {
  const int lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= count) return;
  const uint64_t sid = stream_ids[r];
  auto raw_at = [&](uint64_t k) {  // raw draw k of Philox(key=[seed, sid]): counter k/4 + 1, lane k % 4
    uint64_t c[4] = {k / 4 + 1, 0ull, 0ull, 0ull};
    philox4x64_10(c, seed, sid);
    const int w = (int)(k & 3ull);
    return w == 0 ? c[0] : w == 1 ? c[1] : w == 2 ? c[2] : c[3];
  };
  double ph = (double)phase[r];
  if (ph != ph) ph = 2.0 * 3.141592653589793 * raw_to_unit(raw_at(0));  // uniform(0, 2 pi)
  double sp, cp;
  sincos(ph, &sp, &cp);
  const double s = (double)sigma[r] * 0.7071067811865476;
  for (int i = lane; i < n; i += 32) {
    const float2 a = A[(size_t)i * m + c0[r]], b = A[(size_t)i * m + c1[r]];
    double gx = (double)a.x + cp * b.x - sp * b.y, gy = (double)a.y + cp * b.y + sp * b.x;
    if (s > 0.0) {
      const double u1 = raw_to_unit(raw_at(1 + 2 * (uint64_t)i)), u2 = raw_to_unit(raw_at(2 + 2 * (uint64_t)i));
      const double rad = sqrt(-2.0 * log1p(-u1));  // 1 - u1 in (0, 1]
      double sn, cn;
      sincospi(2.0 * u2, &sn, &cn);
      gx = fma(s, rad * cn, gx);
      gy = fma(s, rad * sn, gy);
    }
    pixels[(size_t)r * n + i] = make_float2((float)gx, (float)gy);
  }
  if (lane == 0) {
    const uint64_t rng_excl = 0x7FFFFFFFFFFFFFFFull;
    for (uint64_t k = 1 + 2 * (uint64_t)n;; ++k) {
      const uint64_t raw = raw_at(k);
      if (raw * rng_excl >= 2ull) {
        seeds[r] = __umul64hi(raw, rng_excl);
        break;
      }
    }
  }
}

cudaError_t launch_synth_pair(const float2* A, int n, int m, uint64_t seed, const uint64_t* stream_ids, const int* c0,
                              const int* c1, const float* phase, const float* sigma, long long count, float2* pixels,
                              uint64_t* seeds, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  count_launch();
  synth_pair_kernel<<<(unsigned)((count + 7) / 8), 256, 0, st>>>(A, n, m, seed, stream_ids, c0, c1, phase, sigma, count, pixels, seeds);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ power iteration
// Single-CTA-per-range variant: the whole iteration loop runs on device.
// v: complex128 work vectors, one per range, concatenated (initialised with the start vectors).
struct PowerRange {
  long long start, stop, voff;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

__global__ void __launch_bounds__(256) power_iter_small_kernel(const float2* __restrict__ A, int n, int m,
                                                               const PowerRange* ranges, double2* v,
                                                               double2* uscratch, int max_iter, double rtol,
                                                               double* out) {
  extern __shared__ double2 w[];  // [n]
  __shared__ double red[32];
  const PowerRange R = ranges[blockIdx.x];
  const long long width = R.stop - R.start;
  double2* vv = v + R.voff;
  double2* uu = uscratch + R.voff;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (width == 1) {  // solver.py:170-171
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      float2 a = A[(size_t)i * m + R.start];
      s += (double)a.x * a.x + (double)a.y * a.y;
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
    return;
  }
  double prev = 0.0, result = 0.0;
  bool done = false;
  for (int it = 0; it < max_iter && !done; ++it) {
    // w = A v
    for (int i = warp; i < n; i += nw) {
      double re = 0.0, im = 0.0;
      for (long long c = lane; c < width; c += 32) {
        float2 a = A[(size_t)i * m + R.start + c];
        double2 x = vv[c];
        re += (double)a.x * x.x - (double)a.y * x.y;
        im += (double)a.x * x.y + (double)a.y * x.x;
      }
      re = warp_sum(re);
      im = warp_sum(im);
      if (lane == 0) w[i] = make_double2(re, im);
    }
    __syncthreads();
    double s2 = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s2 += w[i].x * w[i].x + w[i].y * w[i].y;
    const double cur = block_sum(s2, red);
    // u = A^H w, ||u||
    double nu2 = 0.0;
    for (long long c = threadIdx.x; c < width; c += blockDim.x) {
      double re = 0.0, im = 0.0;
      for (int i = 0; i < n; ++i) {
        float2 a = A[(size_t)i * m + R.start + c];
        re += (double)a.x * w[i].x + (double)a.y * w[i].y;
        im += (double)a.x * w[i].y - (double)a.y * w[i].x;
      }
      uu[c] = make_double2(re, im);
      nu2 += re * re + im * im;
    }
    const double nu = sqrt(block_sum(nu2, red));
    if (nu == 0.0) {
      result = 0.0;
      done = true;
      break;
    }
    const double inv = 1.0 / nu;
    for (long long c = threadIdx.x; c < width; c += blockDim.x) {
      double2 u = uu[c];
      vv[c] = make_double2(u.x * inv, u.y * inv);
    }
    __syncthreads();
    if (fabs(cur - prev) <= rtol * fmax(cur, 1e-300)) {
      result = cur;
      done = true;
      break;
    }
    prev = cur;
    result = prev;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = result;
}

cudaError_t launch_power_small(const float2* A, int n, int m, const long long* starts, const long long* stops,
                               int num_ranges, double2* v, double2* uscratch, int max_iter, double rtol,
                               double* out_dev, cudaStream_t st) {
  PowerRange* hr = new PowerRange[num_ranges];
  long long off = 0;
  for (int r = 0; r < num_ranges; ++r) {
    hr[r].start = starts[r];
    hr[r].stop = stops[r];
    hr[r].voff = off;
    off += stops[r] - starts[r];
  }
  PowerRange* dr = nullptr;
  cudaError_t e = cudaMallocAsync(&dr, sizeof(PowerRange) * num_ranges, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dr, hr, sizeof(PowerRange) * num_ranges, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  delete[] hr;
  if (e != cudaSuccess) return e;
  size_t smem = (size_t)n * sizeof(double2);
  if (smem > 48 * 1024) cudaFuncSetAttribute(power_iter_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  count_launch();
  power_iter_small_kernel<<<num_ranges, 256, smem, st>>>(A, n, m, dr, v, uscratch, max_iter, rtol, out_dev);
  e = cudaGetLastError();
  cudaFreeAsync(dr, st);
  return e;
}

// Multi-CTA variant for wide ranges (cfg4/cfg5 full dictionaries): host-driven iteration with
// fixed-order partial reductions (deterministic), one convergence read-back per iteration.
constexpr int PW_COLS = 1024;  // columns per CTA of the forward partial
__global__ void __launch_bounds__(256) pw_forward_partial(const float2* __restrict__ A, int n, int m, long long start,
                                                          long long width, const double2* __restrict__ v,
                                                          double inv_scale, double2* partial) {
  // partial[cta][i] = sum_{c in cta tile} A[i][start+c] * v[c] * inv_scale.  The v tile is staged
  // once in shared memory; each warp walks its rows with four independent accumulator chains so
  // four coalesced A loads are in flight per lane (the kernel is an HBM stream of A).
  __shared__ double2 sv[PW_COLS];
  const long long c0 = (long long)blockIdx.x * PW_COLS;
  const int len = (int)min((long long)PW_COLS, width - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = threadIdx.x; c < PW_COLS; c += blockDim.x) sv[c] = c < len ? v[c0 + c] : make_double2(0.0, 0.0);
  __syncthreads();
  for (int i = warp; i < n; i += nw) {
    const float2* arow = A + (size_t)i * m + start + c0;
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    int c = lane;
    for (; c + 96 < len; c += 128) {
      float2 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = __ldg(arow + c + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 x = sv[c + 32 * u];
        re[u] = fma((double)a[u].x, x.x, fma(-(double)a[u].y, x.y, re[u]));
        im[u] = fma((double)a[u].x, x.y, fma((double)a[u].y, x.x, im[u]));
      }
    }
    for (; c < len; c += 32) {
      const float2 a = __ldg(arow + c);
      const double2 x = sv[c];
      re[0] = fma((double)a.x, x.x, fma(-(double)a.y, x.y, re[0]));
      im[0] = fma((double)a.x, x.y, fma((double)a.y, x.x, im[0]));
    }
    double r = warp_sum((re[0] + re[1]) + (re[2] + re[3]));
    double q = warp_sum((im[0] + im[1]) + (im[2] + im[3]));
    if (lane == 0) partial[(size_t)blockIdx.x * n + i] = make_double2(r * inv_scale, q * inv_scale);
  }
}

__global__ void __launch_bounds__(256) pw_reduce_w(const double2* partial, int nparts, int n, double2* w, double* cur) {
  // w[i] = sum over the CTA partials (one warp per row, lanes stride the partials: fixed order)
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < n; i += nw) {
    double re = 0.0, im = 0.0;
    for (int p = lane; p < nparts; p += 32) {
      const double2 t = partial[(size_t)p * n + i];
      re += t.x;
      im += t.y;
    }
    re = warp_sum(re);
    im = warp_sum(im);
    if (lane == 0) w[i] = make_double2(re, im);
  }
  __syncthreads();
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += w[i].x * w[i].x + w[i].y * w[i].y;
  s = block_sum(s, red);
  if (threadIdx.x == 0) *cur = s;
}

__global__ void __launch_bounds__(256) pw_adjoint(const float2* __restrict__ A, int n, int m, long long start,
                                                  long long width, const double2* __restrict__ w, double2* u,
                                                  double* nrm_partial) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < width; c += (long long)gridDim.x * blockDim.x) {
    // four independent row chains: four coalesced A loads in flight per thread
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    const float2* acol = A + start + c;
    int i = 0;
    for (; i + 4 <= n; i += 4) {
      float2 a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) a[q] = __ldg(acol + (size_t)(i + q) * m);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 ww = w[i + q];
        re[q] = fma((double)a[q].x, ww.x, fma((double)a[q].y, ww.y, re[q]));
        im[q] = fma((double)a[q].x, ww.y, fma(-(double)a[q].y, ww.x, im[q]));
      }
    }
    for (; i < n; ++i) {
      const float2 a = __ldg(acol + (size_t)i * m);
      const double2 ww = w[i];
      re[0] = fma((double)a.x, ww.x, fma((double)a.y, ww.y, re[0]));
      im[0] = fma((double)a.x, ww.y, fma(-(double)a.y, ww.x, im[0]));
    }
    const double rr = (re[0] + re[1]) + (re[2] + re[3]), ii = (im[0] + im[1]) + (im[2] + im[3]);
    u[c] = make_double2(rr, ii);
    s += rr * rr + ii * ii;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) nrm_partial[blockIdx.x] = s;
}

__global__ void pw_reduce_norm(const double* nrm_partial, int nparts, double* nrm) {
  __shared__ double red[32];
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) s += nrm_partial[p];
  // fixed-order: strided partial sums then warp/block tree
  s = block_sum(s, red);
  if (threadIdx.x == 0) *nrm = sqrt(s);
}

cudaError_t power_iter_large(const float2* A, int n, int m, long long start, long long stop, double2* v,
                             double2* u, int max_iter, double rtol, double* result, int num_sms, cudaStream_t st) {
  const long long width = stop - start;
  if (width == 1) {
    // handled by the small kernel path in the caller
    return cudaErrorInvalidValue;
  }
  const int nparts = (int)((width + PW_COLS - 1) / PW_COLS);
  const int adj_blocks = num_sms * 4;
  double2 *partial = nullptr, *w = nullptr;
  double *scal = nullptr, *nrm_part = nullptr;
  cudaError_t e = cudaMallocAsync(&partial, sizeof(double2) * (size_t)nparts * n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&w, sizeof(double2) * n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&scal, sizeof(double) * 2, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&nrm_part, sizeof(double) * adj_blocks, st);
  if (e != cudaSuccess) return e;
  double prev = 0.0, res = 0.0, host[2];
  double inv = 1.0;  // v holds the unnormalised u after the first iteration; scale folded in
  bool first = true;
  for (int it = 0; it < max_iter; ++it) {
    count_launch();
    pw_forward_partial<<<nparts, 256, 0, st>>>(A, n, m, start, width, first ? v : u, inv, partial);
    count_launch();
    pw_reduce_w<<<1, 256, 0, st>>>(partial, nparts, n, w, scal);
    count_launch();
    pw_adjoint<<<adj_blocks, 256, 0, st>>>(A, n, m, start, width, w, u, nrm_part);
    count_launch();
    pw_reduce_norm<<<1, 256, 0, st>>>(nrm_part, adj_blocks, scal + 1);
    e = cudaMemcpyAsync(host, scal, sizeof(double) * 2, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) break;
    const double cur = host[0], nu = host[1];
    first = false;
    if (nu == 0.0) {
      res = 0.0;
      break;
    }
    inv = 1.0 / nu;
    if (fabs(cur - prev) <= rtol * fmax(cur, 1e-300)) {
      res = cur;
      break;
    }
    prev = cur;
    res = prev;
  }
  cudaFreeAsync(partial, st);
  cudaFreeAsync(w, st);
  cudaFreeAsync(scal, st);
  cudaFreeAsync(nrm_part, st);
  *result = res;
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

// ------------------------------------------------------------------ steering dictionary
// build_steering_matrix (model.py:296-323): A[i, k] = exp(sign * j 2 pi phase_i(k)) with
// phase_i(k) = xi_i s(k) + sum_a eta_{a,i} p_a(k), k row-major over (elevation, motion axes...).
// The phase is accumulated in the reference's order (outer(xi, s) then += outer(eta_a, p_a)) with
// explicit round-to-nearest ops (no FMA contraction), then 2 pi * phase, cos/sin in fp64, rounded
// to complex64.  Columns [col0, col0 + ncols) of the flat grid are produced (a column shard).
__global__ void steering_kernel(const double* __restrict__ xi, const double* __restrict__ eta, int n, int n_axes,
                                const double* __restrict__ elev, const double* __restrict__ motion, int ms0, int ms1,
                                long long col0, long long ncols, double sign, float2* __restrict__ out) {
  const long long total = (long long)n * ncols;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / ncols);
    const long long c = idx - (long long)i * ncols;
    const long long k = col0 + c;
    const long long inner = (long long)ms0 * ms1;
    const long long s_idx = k / inner;
    const long long rem = k - s_idx * inner;
    double ph = __dmul_rn(xi[i], elev[s_idx]);
    if (n_axes >= 1) {
      const long long j0 = n_axes == 2 ? rem / ms1 : rem;
      ph = __dadd_rn(ph, __dmul_rn(eta[i], motion[j0]));
      if (n_axes == 2) ph = __dadd_rn(ph, __dmul_rn(eta[n + i], motion[ms0 + (rem % ms1)]));
    }
    const double arg = __dmul_rn(sign * 6.283185307179586, ph);
    double sv, cv;
    sincos(arg, &sv, &cv);
    out[(size_t)i * ncols + c] = make_float2((float)cv, (float)sv);
  }
}

cudaError_t launch_steering(const double* xi, const double* eta, int n, int n_axes, const double* elev, const double* motion,
                            int ms0, int ms1, long long col0, long long ncols, double sign, float2* out, int num_sms, cudaStream_t st) {
  if (n <= 0 || ncols <= 0) return cudaSuccess;
  count_launch();
  steering_kernel<<<num_sms * 8, 256, 0, st>>>(xi, eta, n, n_axes, elev, motion, ms0, ms1, col0, ncols, sign, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ linear filter apply
// svd_wiener_solve (solver.py:393-407) with the filter W = V diag(s/(s^2+mu)) U^H precomputed:
// x_p = W b_p for every pixel, fp64 accumulation, complex64 output for the selection stage.
__global__ void __launch_bounds__(256) apply_filter_kernel(const double2* __restrict__ W, int n, int m,
                                                           const float2* __restrict__ B, long long P,
                                                           float2* __restrict__ X) {
  extern __shared__ double2 sbd[];  // [warps][n]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double2* bw = sbd + (size_t)warp * n;
  for (long long p = (long long)blockIdx.x * nw + warp; p < P; p += (long long)gridDim.x * nw) {
    for (int i = lane; i < n; i += 32) {
      const float2 b = B[(size_t)p * n + i];
      bw[i] = make_double2(b.x, b.y);
    }
    __syncwarp();
    for (int c = lane; c < m; c += 32) {
      double re = 0.0, im = 0.0;
      for (int i = 0; i < n; ++i) {
        const double2 w = __ldg(&W[(size_t)c * n + i]);
        const double2 b = bw[i];
        re = fma(w.x, b.x, fma(-w.y, b.y, re));
        im = fma(w.x, b.y, fma(w.y, b.x, im));
      }
      X[(size_t)p * m + c] = make_float2((float)re, (float)im);
    }
    __syncwarp();
  }
}

cudaError_t launch_apply_filter(const double2* W, int n, int m, const float2* B, long long P, float2* X, int num_sms, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  const int warps = 8;
  long long blocks = (P + warps - 1) / warps;
  if (blocks > (long long)num_sms * 8) blocks = (long long)num_sms * 8;
  const size_t smem = (size_t)warps * n * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(apply_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  apply_filter_kernel<<<(int)blocks, warps * 32, smem, st>>>(W, n, m, B, P, X);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- column-major copy of the dictionary
__global__ void transpose_kernel(const float2* __restrict__ A, int n, int m, float2* __restrict__ AT) {
  __shared__ float2 tile[32][33];
  const int c0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, c = c0 + threadIdx.x;
    if (i < n && c < m) tile[r][threadIdx.x] = A[(size_t)i * m + c];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int c = c0 + r, i = i0 + threadIdx.x;
    if (i < n && c < m) AT[(size_t)c * n + i] = tile[threadIdx.x][r];
  }
}
cudaError_t launch_transpose(const float2* A, int n, int m, float2* AT, cudaStream_t st) {
  count_launch();
  transpose_kernel<<<dim3((m + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, st>>>(A, n, m, AT);
  return cudaGetLastError();
}

}  // namespace tb
