// ISTA / FISTA solver with the per-pixel iterate state in TENSOR MEMORY (cfg1-3 shapes: m <= 512).
//
// Reference semantics (paths relative to /root/reference/pkg/src/tomobpdn):
//   _full_vector_pg solver.py:341-376   (ISTA/FISTA, per-iteration backtracking from alpha0)
//   soft_threshold  prox.py:82-96, line_search_ok prox.py:107-119, _window_converged solver.py:227-231
//
// The warp-per-pixel kernel (k_warp_solver.cu) keeps x, d = x - prev and the candidate z of a pixel
// in shared memory: 17.4 KB per pixel on cfg2, so only 9 warps are resident beside the 60 KB
// dictionary and the SM idles on latency (IPC 1.6).  Here one warp still owns one pixel, but
//   * d and z live in tensor memory, used as a lane-private scratchpad: warp w owns TMEM lanes
//     32 (w % 4) .. + 31 and columns 128 (w / 4) .. + 127, lane l keeps its columns l + 32 t as
//     double2 at TMEM columns 4 t (d) and 4 (T + t) (z), T = ceil(m / 32); tcgen05.ld / tcgen05.st
//     (LDTM / STTM) have a ~12-cycle latency and do not use the shared-memory data pipe;
//   * the nonzero entries of z are compacted for the sparse forward product into a 64-entry buffer
//     that is flushed every two column passes (same ascending column order);
//   * per-lane bit masks record where x and d are nonzero (no zero-fill at pixel start);
//   * the column passes of prox and update are rolled loops of 2-pass straight-line chunks (fully
//     unrolled, 16 warps at different places of ~250 KB of code thrashed the instruction cache).
// A slot is 10 KB on cfg2: 16 warps per SM, IPC 2.4, cfg2 FISTA 108 -> 82 ms per 65,536 pixels.
// Variant GT (chosen when it makes more warps resident: cfg3, 12 -> 16): the gradient, which the same
// lane produces and consumes, lives in tensor memory too, and instead of z only its shrink factor.
//
// TEAM = true is the 4-warp-team variant asked for by the round-1 review ("CTA-tiled dense
// contraction"): a team iterates its 4 pixels in lock step and computes G = A^H R_y[:, 4 pixels]
// with CT columns x 4 pixels register tiles (one A load feeds 4 pixels: shared wavefronts 994 -> 758
// per pixel-iteration), synchronising on its own named barrier.  It is bit-identical but SLOWER
// (110 vs 82 ms): the contraction is only 43% of the instructions, the team barrier waits for the
// slowest of 4 prox phases (20% of the stall samples), and a warp executes as many instructions as
// before.  Kept selectable (TB_FISTA_KERNEL=team) with its identity test.
//
// Results are bit-identical to the warp kernel in both modes: every output element sees the same
// sequence of roundings (rows summed in order with the same two packed FFMA2 per row; the fp64
// forward product visits the nonzero columns in ascending order; the same butterfly reductions).
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "solver_params.h"
#include "warp_adjoint.cuh"

namespace tb {

constexpr int FT_TEAM = 4;   // warps (= pixel slots) per team
constexpr int FT_CH = 64;    // compaction buffer entries (flushed every 2 column passes)

// per-slot shared bytes: fp64 A x, A x_prev (n each), fp64 x (m), compaction values (FT_CH), r_y
// quads (n), fp32 gradient (m), fp32 b (n), compaction columns (FT_CH), objective ring (16)
// (gsmem = false: the gradient lives in tensor memory, GT)
__host__ __device__ inline size_t fista_tile_slot_bytes(int n, int m, bool gsmem) {
  size_t b = (size_t)n * 32 + (size_t)m * 16 + (size_t)FT_CH * 16 + (size_t)n * 16 + (gsmem ? (size_t)m * 8 : 0) + (size_t)n * 8 + (size_t)FT_CH * 4 + 16 * 8;
  return (b + 15) & ~(size_t)15;
}

__device__ __forceinline__ void team_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(FT_TEAM * 32) : "memory"); }
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// c = a * b + c on both packed fp32 halves (round to nearest each)
__device__ __forceinline__ void ffma2(unsigned long long& c, unsigned long long a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}

// Tensor memory as a lane-private scratchpad: TMEM lane 32 (warp % 4) + lane, 4 consecutive 32-bit
// columns = one double2 per thread.  LDTM/STTM do not touch the shared-memory data pipe and have a
// ~12-cycle latency; the address is warp-uniform.
__device__ __forceinline__ void tmem_st(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(__double2loint(v.x)),
               "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y))
               : "memory");
}
__device__ __forceinline__ void tmem_ld_issue(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_st_x2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tmem_ld_issue_x2(uint32_t taddr, uint32_t (&r)[2]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double2 tmem_val(const uint32_t (&r)[4]) { return make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2])); }

// ASMEM: the dictionary is staged in shared memory (cfg1, cfg2).  Otherwise (cfg3: 200 KiB) it is
// read from global memory: in the contraction each thread streams its own CT columns (coalesced,
// one load per element per TEAM iteration instead of per pixel iteration), the sparse forward
// product gathers its columns through L1/L2.
// TEAM = false ("solo"): no teams and no barriers -- every warp computes its own pixel's gradient
// with the column-lane adjoint of the warp kernel (warp_adjoint.cuh), keeping this kernel's compact
// slot (d and z in tensor memory, 64-entry compaction buffer: 16 resident warps instead of the warp
// kernel's 9 on cfg2).
// GT (one warp per pixel only): the gradient and the candidate's shrink factor live in tensor memory
// instead of g in shared memory and z in tensor memory; chosen when it makes more warps resident.
template <int CT, int MAXQ, bool ASMEM, bool TEAM, bool GT>
__global__ void __launch_bounds__(512, 1) fista_tile_kernel(const SolveParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int team = warp / FT_TEAM, wt = warp % FT_TEAM;
  const int n = P.n, m = P.m, ms = P.ms;
  const bool ista = P.mode == SOLVER_ISTA;

  // ---- dictionary staged once per CTA, row-major with an odd row stride
  const int as = ASMEM ? ms : m;  // row stride of the dictionary as the kernel reads it
  const float2* As = ASMEM ? reinterpret_cast<const float2*>(smem) : P.A;
  const size_t a_bytes = ASMEM ? (((size_t)n * ms) * sizeof(float2) + 15) & ~(size_t)15 : 0;
  if (ASMEM)
    for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) {
      const int i = idx / m, c = idx - i * m;
      reinterpret_cast<float2*>(smem)[(size_t)i * ms + c] = __ldg(&P.A[idx]);
    }
  int* s_act = reinterpret_cast<int*>(smem + a_bytes);  // [warps] slot-active flags
  const size_t slot_bytes = fista_tile_slot_bytes(n, m, !GT);
  unsigned char* slots = smem + a_bytes + 64 * sizeof(int);
  auto slot_ptr = [&](int s) { return slots + (size_t)s * slot_bytes; };
  const size_t off_xs = (size_t)n * 32, off_zs = off_xs + (size_t)m * 16, off_ry = off_zs + (size_t)FT_CH * 16;
  const size_t off_g = off_ry + (size_t)n * 16, off_b = off_g + (!GT ? (size_t)m * 8 : 0), off_cl = off_b + (size_t)n * 8;
  const size_t off_ring = (off_cl + (size_t)FT_CH * 4 + 7) & ~(size_t)7;
  unsigned char* wb = slot_ptr(warp);
  double2* axv = reinterpret_cast<double2*>(wb);       // A x
  double2* apv = axv + n;                              // A x_prev
  double2* xs = reinterpret_cast<double2*>(wb + off_xs);
  double2* zs = reinterpret_cast<double2*>(wb + off_zs);
  float4* ry4 = reinterpret_cast<float4*>(wb + off_ry);  // (r.x, r.y, r.y, -r.x)
  float2* gs = reinterpret_cast<float2*>(wb + off_g);
  float2* bv = reinterpret_cast<float2*>(wb + off_b);
  int* clist = reinterpret_cast<int*>(wb + off_cl);
  double* ring = reinterpret_cast<double*>(wb + off_ring);
  // tensor memory: the whole 512-column array of this SM (one CTA per SM); warp w owns lanes
  // 32 (w % 4) .. + 31 and columns 128 (w / 4) .. + 127: d = x - prev in columns [0, 4 T), the
  // candidate z in [4 T, 8 T), T = ceil(m / 32) <= 16
  __shared__ uint32_t tmem_base_s;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm_d = tmem_base_s + ((uint32_t)(wt * 32) << 16) + (uint32_t)team * 128u;
  const uint32_t tm_z = tm_d + 4u * (uint32_t)((m + 31) >> 5);
  // GT: with one warp per pixel the gradient is produced and consumed by the same lane, so it can live
  // in tensor memory too (fp32 pair, 2 columns per pass, at [6 T, 8 T)) if instead of the candidate z
  // only its shrink factor sc = 1 - tau / |v| (0 where z = 0) is kept (fp64, [4 T, 6 T)): the update
  // rebuilds z = (y - alpha g) sc from the same operands, bit for bit.  8 T columns as before, and the
  // slot loses the m * 8 bytes of g (cfg3: 16.5 -> 12.5 KB, 16 instead of 12 resident warps: +8%; on
  // cfg2, where 16 warps fit anyway, the rebuilt z costs 9%, so GT is used only when it adds warps).
  const uint32_t tm_s = tm_z, tm_g = tm_z + 2u * (uint32_t)((m + 31) >> 5);

  const double alpha0_full = P.alpha_scale / fmax(P.lip_full, 1e-300);  // solver.py:345
  const unsigned lt_mask = (1u << lane) - 1u;

  // acc[q] += sum over the cnt compacted entries (values zs, columns clist, ascending), lane = row
  auto forward_accum = [&](int cnt, double2* acc) {
    const float2* arow[MAXQ];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) arow[q] = ASMEM ? As + (size_t)min(lane + 32 * q, n - 1) * as : P.AT + min(lane + 32 * q, n - 1);  // global: column-major copy
    int e = 0;
    for (; e + 2 <= cnt; e += 2) {
      const int2 cc = *reinterpret_cast<const int2*>(clist + e);
      const double2 v0 = zs[e], v1 = zs[e + 1];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const float2 a0 = ASMEM ? arow[q][cc.x] : __ldg(arow[q] + (size_t)cc.x * n), a1 = ASMEM ? arow[q][cc.y] : __ldg(arow[q] + (size_t)cc.y * n);
        acc[q].x = fma((double)a0.x, v0.x, fma(-(double)a0.y, v0.y, acc[q].x));
        acc[q].y = fma((double)a0.x, v0.y, fma((double)a0.y, v0.x, acc[q].y));
        acc[q].x = fma((double)a1.x, v1.x, fma(-(double)a1.y, v1.y, acc[q].x));
        acc[q].y = fma((double)a1.x, v1.y, fma((double)a1.y, v1.x, acc[q].y));
      }
    }
    if (e < cnt) {
      const int c = clist[e];
      const double2 v = zs[e];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const float2 a = ASMEM ? arow[q][c] : __ldg(arow[q] + (size_t)c * n);
        acc[q].x = fma((double)a.x, v.x, fma(-(double)a.y, v.y, acc[q].x));
        acc[q].y = fma((double)a.x, v.y, fma((double)a.y, v.x, acc[q].y));
      }
    }
  };

  // per-slot state (registers, warp-uniform except the masks)
  long long p = -1;
  bool active = false;
  int k = 0, ridx = 0, status = STATUS_MAX_ITERS;
  double F = 0.0, lamd = 0.0, mk = 0.0, mk_next = 0.0;
  unsigned xnz = 0u, dnz = 0u;  // bit t: x / d nonzero at column lane + 32 t
  double* hrow = nullptr;

  // ---- initial state: x = 0, prev = 0, A x = 0, F0 = ||b||^2 (solver.py:349)
  auto next_pixel = [&]() {
    unsigned long long pq = 0;
    if (lane == 0) pq = atomicAdd(P.queue, 1ull);
    pq = __shfl_sync(TB_FULL_MASK, pq, 0);
    active = pq < (unsigned long long)P.num_pixels;
    if (!active) return;
    p = (long long)pq;
    lamd = P.lam[p];
    double fb = 0.0;
    for (int i = lane; i < n; i += 32) {
      const float2 b = P.B[(size_t)p * n + i];
      bv[i] = b;
      axv[i] = make_double2(0.0, 0.0);
      apv[i] = make_double2(0.0, 0.0);
      fb += (double)b.x * b.x + (double)b.y * b.y;
    }
    F = warp_sum(fb);
    ring[0] = F;
    hrow = P.hist ? P.hist + (size_t)p * P.hist_stride : nullptr;
    if (hrow) hrow[0] = F;
    xnz = dnz = 0u;
    k = 0;
    ridx = 0;
    status = STATUS_MAX_ITERS;
    mk_next = (ista || P.total_iters < 1) ? 0.0 : __ldg(P.mk + 1);
    __syncwarp();
  };
  next_pixel();

  for (;;) {
    // ---- residual at y (lane = row), fp64: r_y = A y - b, A y = A x + m_k (A x - A x_prev)
    if (active) {
      ++k;
      ridx = ridx == STOP_WINDOW ? 0 : ridx + 1;
      mk = mk_next;  // (k-2)/(k+1), host table (solver.py:222-224); 0 for ISTA
      if (!ista && k < P.total_iters) mk_next = __ldg(P.mk + k + 1);
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int i = lane + 32 * q;
        if (i < n) {
          const double2 ax = axv[i], axp = apv[i];
          const float2 b = bv[i];
          double2 a = ax;
          if (!ista) {
            a.x = fma(mk, ax.x - axp.x, ax.x);
            a.y = fma(mk, ax.y - axp.y, ax.y);
          }
          ry4[i] = conj_operand((float)(a.x - b.x), (float)(a.y - b.y));
        }
      }
    }
    if (!TEAM) {
      if (!active) break;
      __syncwarp();
      // ---- gradient, one warp per pixel: lane = column, ceil(m / 32) passes, rows summed in order
      constexpr int MAXT = 4 * CT;
      float2 acc[MAXT];
#pragma unroll
      for (int t = 0; t < MAXT; ++t) acc[t] = make_float2(0.f, 0.f);
      const int passes = (m + 31) >> 5;
      adjoint_dispatch<1, MAXT, ASMEM, false>(passes, acc, As + lane, as, 32, ry4, n, lane + 32 * (passes - 1) < m);
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (GT) {
          if (32 * t < m) tmem_st_x2(tm_g + 2u * t, __float_as_uint(2.f * acc[t].x), __float_as_uint(2.f * acc[t].y));
        } else if (lane + 32 * t < m) {
          gs[lane + 32 * t] = make_float2(2.f * acc[t].x, 2.f * acc[t].y);
        }
      }
      if (GT)
        tmem_wait_st();
      else
        __syncwarp();
    }
    if (TEAM) {
    if (lane == 0) s_act[warp] = active ? 1 : 0;
    team_bar(team + 1);
    {
      const int4 fl = *reinterpret_cast<const int4*>(s_act + team * FT_TEAM);
      if (!(fl.x | fl.y | fl.z | fl.w)) break;
    }

    // ---- gradient g = 2 A^H r_y for the team's 4 pixels (solver.py:352, prox.py:77-79): fp32,
    //      thread = CT columns (ct + 128 j) x 4 pixels, rows summed in order
    {
      const int ct = wt * 32 + lane;
      unsigned long long acc[CT][FT_TEAM];
      int cj[CT];
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        cj[j] = min(ct + 128 * j, m - 1);
#pragma unroll
        for (int q = 0; q < FT_TEAM; ++q) acc[j][q] = 0ull;
      }
      const unsigned char* rbase = slot_ptr(team * FT_TEAM) + off_ry;
#pragma unroll 5
      for (int i = 0; i < n; ++i) {
        ulonglong2 r[FT_TEAM];
#pragma unroll
        for (int q = 0; q < FT_TEAM; ++q) r[q] = reinterpret_cast<const ulonglong2*>(rbase + (size_t)q * slot_bytes)[i];
        const float2* arow = As + (size_t)i * as;
#pragma unroll
        for (int j = 0; j < CT; ++j) {
          if (j * 128 + wt * 32 < m) {  // warp-uniform: this warp has columns in column set j
            const float2 a = ASMEM ? arow[cj[j]] : __ldg(arow + cj[j]);
            const unsigned long long aa = pack2(a.x, a.x), bb = pack2(a.y, a.y);
#pragma unroll
            for (int q = 0; q < FT_TEAM; ++q) {
              ffma2(acc[j][q], aa, r[q].x);
              ffma2(acc[j][q], bb, r[q].y);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const int c = ct + 128 * j;
        if (c < m) {
#pragma unroll
          for (int q = 0; q < FT_TEAM; ++q) {
            const float2 v = unpack2(acc[j][q]);
            reinterpret_cast<float2*>(slot_ptr(team * FT_TEAM + q) + off_g)[c] = make_float2(2.f * v.x, 2.f * v.y);
          }
        }
      }
    }
    team_bar(team + 1);
    if (!active) continue;
    }  // TEAM

    // ---- backtracking (solver.py:353-361; prox.py:122-150), prox step in fp64
    double2 ay[MAXQ];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int i = lane + 32 * q;
      ay[q] = make_double2(0.0, 0.0);
      if (i < n) {
        const double2 ax = axv[i], axp = apv[i];
        double2 a = ax;
        if (!ista) {
          a.x = fma(mk, ax.x - axp.x, ax.x);
          a.y = fma(mk, ax.y - axp.y, ax.y);
        }
        ay[q] = a;
      }
    }
    // One column pass of the prox step for this lane's column lane + 32 t: z = soft(y - alpha g,
    // alpha lambda) with y = x + m_k d (d from tensor memory; its bits are garbage where dnz is clear)
    auto prox_pass = [&](int t, float2 g, double2 dv, double alpha, double tau, double tau2, double2& yv, double2& zz, double& absz, double& scz) {
      const int cl = lane + 32 * t;
      const bool act = cl < m;
      const int col = act ? cl : m - 1;
      if (!GT) g = gs[col];
      double2 xv = make_double2(0.0, 0.0);
      if ((xnz >> t) & 1u) xv = xs[col];
      yv = xv;
      if ((dnz >> t) & 1u) {
        yv.x = fma(mk, dv.x, xv.x);
        yv.y = fma(mk, dv.y, xv.y);
      }
      const double2 v = make_double2(fma(-alpha, (double)g.x, yv.x), fma(-alpha, (double)g.y, yv.y));
      const double mag2 = fma(v.x, v.x, v.y * v.y);
      zz = make_double2(0.0, 0.0);
      absz = 0.0;
      scz = 0.0;
      // soft_threshold: zero iff |v| <= tau (prox.py:82-96); a NaN v stays NaN
      if (act && !(mag2 <= tau2)) {
        const double rs = rsqrt(mag2);
        const double sc = fma(-tau, rs, 1.0);
        zz = make_double2(v.x * sc, v.y * sc);
        absz = fma(mag2, rs, -tau);
        scz = (zz.x != 0.0 || zz.y != 0.0) ? sc : 0.0;  // NaN z keeps its (NaN) factor
      }
    };
    double alpha = alpha0_full;
    bool ok = false;
    double2 adz[MAXQ];
    double l1z = 0.0, fzs = 0.0;
    for (int trial = 0; trial <= P.cap; ++trial) {
      const double tau = alpha * lamd;
      const double tau2 = tau * tau;
      double red[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // |d|^2, |z|, ||A z - A y||^2, f(z), scale
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) adz[q] = make_double2(0.0, 0.0);
      // column passes run as a rolled loop of 2-pass chunks (fully unrolled, the body thrashed the
      // instruction cache: 16 warps at different places of ~250 KB of code); the two passes of a
      // chunk are straight-line code, so their loads and fp64 chains overlap; the compaction buffer
      // is flushed into the forward product after every chunk
#pragma unroll 1
      for (int t0 = 0; 32 * t0 < m; t0 += 2) {
        const bool two = 32 * (t0 + 1) < m;
        uint32_t dr[2][4], gr[2][2] = {};
        tmem_ld_issue(tm_d + 4u * t0, dr[0]);
        tmem_ld_issue(tm_d + 4u * (two ? t0 + 1 : t0), dr[1]);
        if (GT) {
          tmem_ld_issue_x2(tm_g + 2u * t0, gr[0]);
          tmem_ld_issue_x2(tm_g + 2u * (two ? t0 + 1 : t0), gr[1]);
        }
        tmem_wait_ld();
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int t = t0 + u;
          if (u == 1 && !two) break;
          double2 yv, zz;
          double absz, scz;
          prox_pass(t, make_float2(__uint_as_float(gr[u][0]), __uint_as_float(gr[u][1])), tmem_val(dr[u]), alpha, tau, tau2, yv, zz, absz, scz);
          if (!GT)
            tmem_st(tm_z + 4u * t, zz);
          else
            tmem_st_x2(tm_s + 2u * t, (uint32_t)__double2loint(scz), (uint32_t)__double2hiint(scz));
          const bool act = lane + 32 * t < m;
          red[1] += absz;
          const double2 d = make_double2(zz.x - yv.x, zz.y - yv.y);
          red[0] += act ? fma(d.x, d.x, d.y * d.y) : 0.0;
          const bool nz = act && ((zz.x != 0.0) || (zz.y != 0.0));
          const unsigned mask = __ballot_sync(TB_FULL_MASK, nz);
          if (nz) {
            const int pos = cnt + __popc(mask & lt_mask);
            zs[pos] = zz;
            clist[pos] = lane + 32 * t;
          }
          cnt += __popc(mask);
        }
        if (cnt) {  // warp-uniform
          __syncwarp();
          forward_accum(cnt, adz);  // A z over the nonzero entries, ascending columns
          __syncwarp();
        }
      }
      tmem_wait_st();
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int i = lane + 32 * q;
        if (i < n) {
          // quadratic-bound test in its exact algebraic form ||A d||^2 <= ||d||^2 / (2 alpha)
          const double dx = adz[q].x - ay[q].x, dyy = adz[q].y - ay[q].y;
          red[2] += dx * dx + dyy * dyy;
          const float2 b = bv[i];
          const double fx = adz[q].x - b.x, fy = adz[q].y - b.y;
          red[3] += fx * fx + fy * fy;
          red[4] += fabs(adz[q].x) + fabs(adz[q].y) + fabs(ay[q].x) + fabs(ay[q].y);
        } else {
          adz[q] = make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int r = 0; r < 5; ++r) red[r] += __shfl_xor_sync(TB_FULL_MASK, red[r], o);
      }
      l1z = red[1];
      fzs = red[3];
      if (sqrt(red[2]) <= sqrt(red[0] / (2.0 * alpha)) + 1e-12 * red[4]) {  // fp64 rounding of A z - A y
        ok = true;
        break;
      }
      alpha *= P.c_alpha;
    }
    bool done = false;
    if (!ok) {
      status = STATUS_LINE_SEARCH_FAILURE;  // ISTA/FISTA do not append F (solver.py:357-361)
      done = true;
    } else {
      // ---- update: x_prev <- x, x <- z, F = ||A z - b||^2 + lambda ||z||_1 (solver.py:362-364);
      //      the accepted candidate comes back from tensor memory
#pragma unroll 1
      for (int t0 = 0; 32 * t0 < m; t0 += 2) {
        const bool two = 32 * (t0 + 1) < m;
        uint32_t zr[2][4] = {}, dr[2][4] = {}, gr[2][2] = {}, sr[2][2] = {};
        if (!GT) {
          tmem_ld_issue(tm_z + 4u * t0, zr[0]);
          tmem_ld_issue(tm_z + 4u * (two ? t0 + 1 : t0), zr[1]);
        } else {
          tmem_ld_issue(tm_d + 4u * t0, dr[0]);
          tmem_ld_issue(tm_d + 4u * (two ? t0 + 1 : t0), dr[1]);
          tmem_ld_issue_x2(tm_g + 2u * t0, gr[0]);
          tmem_ld_issue_x2(tm_g + 2u * (two ? t0 + 1 : t0), gr[1]);
          tmem_ld_issue_x2(tm_s + 2u * t0, sr[0]);
          tmem_ld_issue_x2(tm_s + 2u * (two ? t0 + 1 : t0), sr[1]);
        }
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int t = t0 + u;
          if (u == 1 && !two) break;
          const int col = lane + 32 * t;
          const bool xb = (xnz >> t) & 1u;
          double2 xv = make_double2(0.0, 0.0);
          if (xb) xv = xs[col];
          double2 zz;
          if (!GT) {
            zz = tmem_val(zr[u]);  // 0 for lanes past m
          } else {
            // z = (y - alpha g) sc from the operands of the accepted trial: the same roundings
            const double scz = __hiloint2double((int)sr[u][1], (int)sr[u][0]);
            double2 yv = xv;
            if ((dnz >> t) & 1u) {
              const double2 dv = tmem_val(dr[u]);
              yv.x = fma(mk, dv.x, xv.x);
              yv.y = fma(mk, dv.y, xv.y);
            }
            const double vx = fma(-alpha, (double)__uint_as_float(gr[u][0]), yv.x), vy = fma(-alpha, (double)__uint_as_float(gr[u][1]), yv.y);
            zz = scz != 0.0 ? make_double2(vx * scz, vy * scz) : make_double2(0.0, 0.0);
          }
          const bool zb = (zz.x != 0.0) || (zz.y != 0.0);
          const double2 dn = make_double2(zz.x - xv.x, zz.y - xv.y);
          if (zb || xb) xs[col] = zz;  // implies col < m
          const bool nd = !ista && ((dn.x != 0.0) || (dn.y != 0.0));
          tmem_st(tm_d + 4u * t, dn);
          xnz = (xnz & ~(1u << t)) | ((zb ? 1u : 0u) << t);
          dnz = (dnz & ~(1u << t)) | ((nd ? 1u : 0u) << t);
        }
      }
      tmem_wait_st();
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int i = lane + 32 * q;
        if (i < n) {
          apv[i] = axv[i];
          axv[i] = adz[q];
        }
      }
      F = fzs + lamd * l1z;
      // ---- history, failure and window stop (solver.py:366-374)
      ring[ridx] = F;  // every lane stores the same value
      if (hrow) hrow[k] = F;
      __syncwarp();
      if (!isfinite(F)) {
        status = STATUS_NUMERICAL_FAILURE;
        done = true;
      } else if (!P.fixed && k >= STOP_WINDOW) {
        const double ref = ring[ridx == STOP_WINDOW ? 0 : ridx + 1];  // F at k - STOP_WINDOW
        if (fabs(F - ref) <= P.tol * fmax(fabs(ref), 1e-300)) {
          status = STATUS_CONVERGED;
          done = true;
        }
      }
      if (!done && k >= P.total_iters) {  // for-else re-check (solver.py:334-336)
        if (k >= STOP_WINDOW) {
          const double ref = ring[ridx == STOP_WINDOW ? 0 : ridx + 1];
          if (fabs(F - ref) <= P.tol * fmax(fabs(ref), 1e-300)) status = STATUS_CONVERGED;
        }
        done = true;
      }
    }
    if (done) {
      __syncwarp();
#pragma unroll 1
      for (int t = 0; 32 * t < m; ++t) {
        const int col = lane + 32 * t;
        if (col < m) {
          float2 o = make_float2(0.f, 0.f);
          if ((xnz >> t) & 1u) {
            const double2 xv = xs[col];
            o = make_float2((float)xv.x, (float)xv.y);
          }
          P.X[(size_t)p * m + col] = o;
        }
      }
      if (lane == 0) {
        P.f_final[p] = F;
        P.iters[p] = k;
        P.status[p] = status;
      }
      __syncwarp();
      next_pixel();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_s));
}

// Shared-memory plan: the dictionary beside >= 8 slots if it fits, else slots only (A from global)
static bool fista_tile_plan(int n, int m, bool gsmem, bool* asmem) {
  if (m > 512 || n > 128) return false;  // 8 ceil(m / 32) tensor-memory columns per warp <= 128
  const size_t cap = 227 * 1024 - 64, slot = fista_tile_slot_bytes(n, m, gsmem);
  const size_t a_bytes = (((size_t)n * (m | 1)) * sizeof(float2) + 15) & ~(size_t)15;
  const char* ev = getenv("TB_FISTA_TILE_ASMEM");  // 0: force the global-memory dictionary (A/B)
  const bool want = !(ev && atoi(ev) == 0);
  *asmem = want && a_bytes + 64 * sizeof(int) + 2 * FT_TEAM * slot <= cap;
  return *asmem || 64 * sizeof(int) + 2 * FT_TEAM * slot <= cap;
}
static int fista_tile_warps(int n, int m, bool asmem, bool gsmem) {
  const size_t slot = fista_tile_slot_bytes(n, m, gsmem);
  const size_t a_bytes = asmem ? (((size_t)n * (m | 1)) * sizeof(float2) + 15) & ~(size_t)15 : 0;
  const int warps = (int)((227 * 1024 - 64 - a_bytes - 64 * sizeof(int)) / slot);
  return warps > 16 ? 16 : warps / FT_TEAM * FT_TEAM;
}
// One-warp-per-pixel plan: g in shared memory unless g in tensor memory (GT) makes more warps resident
static bool fista_solo_plan(int n, int m, bool* asmem, bool* gt, int* warps) {
  bool as = false, ag = false;
  const bool ok_s = fista_tile_plan(n, m, true, &as), ok_g = fista_tile_plan(n, m, false, &ag);
  const int ws = ok_s ? fista_tile_warps(n, m, as, true) : 0, wg = ok_g ? fista_tile_warps(n, m, ag, false) : 0;
  bool g = ok_g && (!ok_s || (ag == as && wg > ws));
  if (const char* ge = getenv("TB_FISTA_GT")) g = ok_g && (atoi(ge) != 0 || !ok_s);  // A/B
  *gt = g;
  *asmem = g ? ag : as;
  *warps = g ? wg : ws;
  return ok_s || ok_g;
}
bool fista_tile_fits(int n, int m, bool* asmem, int* slots) {
  bool a = false, g = false;
  int w = 0;
  const bool ok = fista_solo_plan(n, m, &a, &g, &w);
  if (asmem) *asmem = a;
  if (slots) *slots = ok ? w : 0;
  return ok;
}

template <int CT, bool ASMEM, bool TEAM, bool GT>
static cudaError_t launch_ft_q(const SolveParams& P, int maxq, int warps, size_t smem, int grid, cudaStream_t st) {
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    count_launch();
    kern<<<grid, warps * 32, smem, st>>>(P);
    return cudaGetLastError();
  };
  switch (maxq) {
    case 1: return go(fista_tile_kernel<CT, 1, ASMEM, TEAM, GT>);
    case 2: return go(fista_tile_kernel<CT, 2, ASMEM, TEAM, GT>);
    case 4: return go(fista_tile_kernel<CT, 4, ASMEM, TEAM, GT>);
    default: return cudaErrorInvalidValue;
  }
}
template <bool ASMEM, bool TEAM, bool GT>
static cudaError_t launch_ft_ct(const SolveParams& P, int ct, int maxq, int warps, size_t smem, int grid, cudaStream_t st) {
  switch (ct) {
    case 1: return launch_ft_q<1, ASMEM, TEAM, GT>(P, maxq, warps, smem, grid, st);
    case 2: return launch_ft_q<2, ASMEM, TEAM, GT>(P, maxq, warps, smem, grid, st);
    case 3: return launch_ft_q<3, ASMEM, TEAM, GT>(P, maxq, warps, smem, grid, st);
    case 4: return launch_ft_q<4, ASMEM, TEAM, GT>(P, maxq, warps, smem, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

// One CTA per SM, up to 16 pixel slots (4 teams); persistent, queue-fed.
cudaError_t launch_fista_tile(const SolveParams& P, int num_sms, cudaStream_t st, int* used_warps, bool team) {
  bool asmem = false, gt = false;
  int warps = 0;
  if (team) {
    if (!fista_tile_plan(P.n, P.m, true, &asmem)) return cudaErrorInvalidValue;
    warps = fista_tile_warps(P.n, P.m, asmem, true);
  } else if (!fista_solo_plan(P.n, P.m, &asmem, &gt, &warps)) {
    return cudaErrorInvalidValue;
  }
  const size_t slot = fista_tile_slot_bytes(P.n, P.m, !gt);
  const size_t a_bytes = asmem ? (((size_t)P.n * P.ms) * sizeof(float2) + 15) & ~(size_t)15 : 0;
  const size_t fixed = a_bytes + 64 * sizeof(int);  // + 16 static bytes (TMEM base), inside the plan's margin
  if (const char* wc = getenv("TB_WARPS_CAP")) {  // tuning/diagnostics
    const int cw = atoi(wc) / FT_TEAM * FT_TEAM;
    if (cw >= FT_TEAM && cw < warps) warps = cw;
  }
  if (warps < FT_TEAM) return cudaErrorInvalidValue;
  // a batch smaller than the resident slots is spread over every SM with fewer teams each
  if (P.num_pixels < (long long)num_sms * warps) {
    const long long per_sm = (P.num_pixels + num_sms - 1) / num_sms;
    warps = (int)((per_sm + FT_TEAM - 1) / FT_TEAM * FT_TEAM);
    if (warps < FT_TEAM) warps = FT_TEAM;
  }
  const size_t smem = fixed + (size_t)warps * slot;
  long long need = (P.num_pixels + warps - 1) / warps;
  int grid = need < num_sms ? (int)need : num_sms;
  if (grid < 1) grid = 1;
  if (used_warps) *used_warps = warps;
  int maxq = (P.n + 31) / 32;
  maxq = maxq <= 1 ? 1 : maxq <= 2 ? 2 : 4;
  const int ct = (P.m + 127) / 128;
  if (team) return asmem ? launch_ft_ct<true, true, false>(P, ct, maxq, warps, smem, grid, st) : launch_ft_ct<false, true, false>(P, ct, maxq, warps, smem, grid, st);
  if (gt) return asmem ? launch_ft_ct<true, false, true>(P, ct, maxq, warps, smem, grid, st) : launch_ft_ct<false, false, true>(P, ct, maxq, warps, smem, grid, st);
  return asmem ? launch_ft_ct<true, false, false>(P, ct, maxq, warps, smem, grid, st) : launch_ft_ct<false, false, false>(P, ct, maxq, warps, smem, grid, st);
}

}  // namespace tb
