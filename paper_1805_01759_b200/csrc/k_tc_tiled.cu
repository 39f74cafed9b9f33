// tcgen05 adjoint for the tiled (large-dictionary) solver: G = A^H r_y (the pass doubles it) for every pending pixel
// tile and every dictionary column of its block, on the 5th-generation tensor cores.
//
//   Gr = Ar^T rr + Ai^T ri,   Gi = Ar^T ri - Ai^T rr          (conj(A) r, solver.py:293 / prox.py:77-79)
//
// as four real GEMM products per K-step with M = 128 dictionary columns, N = 32 pixels, K = 8, each in
// 3xTF32 (hi*hi + hi*lo + lo*hi; fp32 accumulation in TMEM columns [0,32) = Gr, [32,64) = Gi).
// Operands live in HBM already in the canonical K-major SWIZZLE_NONE layout (8-row x 16-byte core
// matrices), in 32-wide K chunks: the dictionary is packed once per (context, partition)
// (tc_pack_dictionary), the pixels' r_y once per round (tc_pack_pixels).  Per CTA (one pixel tile x
// a run of column tiles) one thread streams chunks with cp.async.bulk into a 2-stage shared-memory
// ring (mbarrier complete_tx), another issues tcgen05.mma and tcgen05.commit, and all four warps drain
// TMEM with tcgen05.ld and write G (complex64, [P][m]) for the fp64 epilogue kernel.
#include <stdint.h>

#include "common.cuh"
#include "solver_params.h"
#include "tiled.h"

namespace tb {

namespace {

constexpr int TC_M = 128;                          // dictionary columns per tile
constexpr int TC_N = 32;                           // pixels per tile (= TL_PT)
constexpr int TC_KC = 32;                          // K (complex rows) per chunk
constexpr int TC_AOP = TC_M * TC_KC;               // floats per A operand block
constexpr int TC_BOP = TC_N * TC_KC;               // floats per B operand block
constexpr int TC_ACHUNK = 4 * TC_AOP;              // Ar_hi, Ar_lo, Ai_hi, Ai_lo
constexpr int TC_BCHUNK = 4 * TC_BOP;              // Rr_hi, Rr_lo, Ri_hi, Ri_lo
constexpr uint32_t TC_STAGE_BYTES = (TC_ACHUNK + TC_BCHUNK) * 4;

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ float tf32r(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// canonical K-major offset (floats) of (row r, k) inside one [rows x TC_KC] operand block
__device__ __forceinline__ int koff(int r, int k) { return (r >> 3) * (TC_KC / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  const uint32_t lbo = 128, sbo = (TC_KC / 4) * 128;
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::tf32, fp32 accumulate, K-major A and B, N = 32, M = 128; bit 13 negates A
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((TC_N >> 3) << 17) | ((TC_M >> 4) << 24);
constexpr uint32_t IDESC_NEGA = IDESC | (1u << 13);

__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  const long long t0 = clock64();
  while (!done) {
    if (clock64() - t0 > (1ll << 34)) __trap();  // ~8 s: a lost arrival must fail the launch, never hang the device
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(bar), "r"(parity));
  }
}

}  // namespace

// Packed dictionary: for block b, local tile t (columns bstart[b] + 128 t ...), chunk kc:
// [Ar_hi | Ar_lo | Ai_hi | Ai_lo] blocks at Apk + (tile_base[b] + t) * nck * TC_ACHUNK + kc * TC_ACHUNK.
__global__ void tc_pack_dictionary_kernel(const float2* __restrict__ A, int n, int m, int J, const int* __restrict__ bstart,
                                          const int* __restrict__ tile_base, int nck, float* __restrict__ Apk, long long total_tiles) {
  const long long ntot = total_tiles * nck * (long long)TC_M * TC_KC;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < ntot; idx += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(idx % TC_KC);
    const int r = (int)((idx / TC_KC) % TC_M);
    const long long rest = idx / ((long long)TC_KC * TC_M);
    const int kc = (int)(rest % nck);
    const long long gt = rest / nck;
    int b = 0;
    while (b + 1 < J && tile_base[b + 1] <= gt) ++b;
    const int t = (int)(gt - tile_base[b]);
    const int col = bstart[b] + t * TC_M + r;
    const int row = kc * TC_KC + k;
    float ar = 0.f, ai = 0.f;
    if (col < bstart[b + 1] && row < n) {
      const float2 a = A[(size_t)row * m + col];
      ar = a.x;
      ai = a.y;
    }
    float* base = Apk + ((size_t)gt * nck + kc) * TC_ACHUNK;
    const int o = koff(r, k);
    const float rh = tf32r(ar), ih = tf32r(ai);
    base[0 * TC_AOP + o] = rh;
    base[1 * TC_AOP + o] = tf32r(ar - rh);
    base[2 * TC_AOP + o] = ih;
    base[3 * TC_AOP + o] = tf32r(ai - ih);
  }
}

// Packed r_y of the round's pixel tiles: [tile][chunk][Rr_hi | Rr_lo | Ri_hi | Ri_lo].
__global__ void tc_pack_pixels_kernel(const TiledParams T, int nck, float* __restrict__ Rpk) {
  const int tile = blockIdx.x;
  if (tile >= *T.ntiles) return;
  const int4 td = T.tiles[tile];
  for (int idx = threadIdx.x; idx < nck * TC_N * TC_KC; idx += blockDim.x) {
    const int k = idx % TC_KC, q = (idx / TC_KC) % TC_N, kc = idx / (TC_KC * TC_N);
    const int row = kc * TC_KC + k;
    float rr = 0.f, ri = 0.f;
    if (q < td.z && row < T.n) {
      const int p = T.perm[td.y + q];
      const float2 v = T.ry32[(size_t)p * T.n + row];
      rr = v.x;
      ri = v.y;
    }
    float* base = Rpk + ((size_t)tile * nck + kc) * TC_BCHUNK;
    const int o = koff(q, k);
    const float rh = tf32r(rr), ih = tf32r(ri);
    base[0 * TC_BOP + o] = rh;
    base[1 * TC_BOP + o] = tf32r(rr - rh);
    base[2 * TC_BOP + o] = ih;
    base[3 * TC_BOP + o] = tf32r(ri - ih);
  }
}

// grid (pixel tile, column split); each CTA walks the 128-column tiles of its split of the tile's block.
__global__ void __launch_bounds__(128, 1) tc_adjoint_kernel(const TiledParams T, const float* __restrict__ Apk,
                                                            const float* __restrict__ Rpk, const int* __restrict__ tile_base,
                                                            int nck, int tiles_per_split, float2* __restrict__ G) {
  const int tile = blockIdx.x, split = blockIdx.y;
  if (tile >= *T.ntiles) return;
  const int4 td = T.tiles[tile];
  const int b = td.x;
  const int c_begin = T.bstart[b], c_end = T.bstart[b + 1];
  const int ntile_b = (c_end - c_begin + TC_M - 1) / TC_M;
  const int t0 = split * tiles_per_split;
  if (t0 >= ntile_b) return;
  const int t1 = min(ntile_b, t0 + tiles_per_split);

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[2], empty_bar[2], done_bar;
  __shared__ uint32_t tmem_base;
  __shared__ int s_pid[TC_N];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < TC_N) s_pid[tid] = tid < td.z ? T.perm[td.y + tid] : -1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(s32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full_bar[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty_bar[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const int nchunks = (t1 - t0) * nck;  // flattened (column tile, k chunk) stream
  const float* rbase = Rpk + (size_t)tile * nck * TC_BCHUNK;
  const float* abase = Apk + (size_t)(tile_base[b] + t0) * nck * TC_ACHUNK;

  // producer (thread 0): chunk c goes to stage c & 1 once the MMAs of chunk c - 2 have drained it
  auto load_chunk = [&](int c) {
    const int s = c & 1;
    if (c >= 2) mbar_wait(s32(&empty_bar[s]), ((c >> 1) - 1) & 1);
    const uint32_t fb = s32(&full_bar[s]);
    float* dst = reinterpret_cast<float*>(smem + s * TC_STAGE_BYTES);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(TC_STAGE_BYTES) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)),
                 "l"(abase + (size_t)c * TC_ACHUNK), "r"((uint32_t)(TC_ACHUNK * 4)), "r"(fb)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst + TC_ACHUNK)),
                 "l"(rbase + (size_t)(c % nck) * TC_BCHUNK), "r"((uint32_t)(TC_BCHUNK * 4)), "r"(fb)
                 : "memory");
  };
  int issued = 0;  // producer's next chunk (meaningful in thread 0 only)
  if (tid == 0)
    for (; issued < 2 && issued < nchunks; ++issued) load_chunk(issued);
  for (int t = t0; t < t1; ++t) {
    const int tl = t - t0;
    if (tid == 0)
      for (; issued < (tl + 1) * nck; ++issued) load_chunk(issued);
    if (tid == 32) {  // MMA issuer
      for (int kc = 0; kc < nck; ++kc) {
        const int c = tl * nck + kc, s = c & 1;
        mbar_wait(s32(&full_bar[s]), (c >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a0 = s32(smem + s * TC_STAGE_BYTES);
        const uint32_t b0 = a0 + TC_ACHUNK * 4;
        for (int ks = 0; ks < TC_KC / 8; ++ks) {
          const uint32_t ko = ks * 256;
          const uint64_t arh = desc(a0 + 0 * TC_AOP * 4 + ko), arl = desc(a0 + 1 * TC_AOP * 4 + ko);
          const uint64_t aih = desc(a0 + 2 * TC_AOP * 4 + ko), ail = desc(a0 + 3 * TC_AOP * 4 + ko);
          const uint64_t brh = desc(b0 + 0 * TC_BOP * 4 + ko), brl = desc(b0 + 1 * TC_BOP * 4 + ko);
          const uint64_t bih = desc(b0 + 2 * TC_BOP * 4 + ko), bil = desc(b0 + 3 * TC_BOP * 4 + ko);
          const uint32_t acc = (kc == 0 && ks == 0) ? 0u : 1u;
          // Gr (TMEM cols 0..31) += Ar rr + Ai ri
          mma(tmem, arh, brh, IDESC, acc);
          mma(tmem, arh, brl, IDESC, 1u);
          mma(tmem, arl, brh, IDESC, 1u);
          mma(tmem, aih, bih, IDESC, 1u);
          mma(tmem, aih, bil, IDESC, 1u);
          mma(tmem, ail, bih, IDESC, 1u);
          // Gi (TMEM cols 32..63) += Ar ri - Ai rr
          mma(tmem + 32, arh, bih, IDESC, acc);
          mma(tmem + 32, arh, bil, IDESC, 1u);
          mma(tmem + 32, arl, bih, IDESC, 1u);
          mma(tmem + 32, aih, brh, IDESC_NEGA, 1u);
          mma(tmem + 32, aih, brl, IDESC_NEGA, 1u);
          mma(tmem + 32, ail, brh, IDESC_NEGA, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&empty_bar[s])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&done_bar)));
    }
    mbar_wait(s32(&done_bar), tl & 1);
    if (tid == 0)  // both stages are free: prefetch the next column tile's first chunks under the drain
      for (; issued < nchunks && issued < (tl + 1) * nck + 2; ++issued) load_chunk(issued);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // drain: lane l of warp w holds column 32w + l of this tile, pixels 0..31 (Gr then Gi)
    const int col = c_begin + t * TC_M + 32 * warp + lane;
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t vr[16], vi[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(vr[0]), "=r"(vr[1]), "=r"(vr[2]), "=r"(vr[3]), "=r"(vr[4]), "=r"(vr[5]), "=r"(vr[6]), "=r"(vr[7]), "=r"(vr[8]),
            "=r"(vr[9]), "=r"(vr[10]), "=r"(vr[11]), "=r"(vr[12]), "=r"(vr[13]), "=r"(vr[14]), "=r"(vr[15])
          : "r"(ta + 16 * h));
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(vi[0]), "=r"(vi[1]), "=r"(vi[2]), "=r"(vi[3]), "=r"(vi[4]), "=r"(vi[5]), "=r"(vi[6]), "=r"(vi[7]), "=r"(vi[8]),
            "=r"(vi[9]), "=r"(vi[10]), "=r"(vi[11]), "=r"(vi[12]), "=r"(vi[13]), "=r"(vi[14]), "=r"(vi[15])
          : "r"(ta + 32 + 16 * h));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (col < c_end) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int p = s_pid[16 * h + q];
          if (p >= 0) G[(size_t)p * T.m + col] = make_float2(__uint_as_float(vr[q]), __uint_as_float(vi[q]));
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM drained before the next tile's first (non-accumulating) MMA
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

// host helpers ------------------------------------------------------------------------------------
long long tc_tiles_for(const int* bstart_host, int J, int* tile_base_host) {
  long long tot = 0;
  for (int j = 0; j < J; ++j) {
    tile_base_host[j] = (int)tot;
    tot += (bstart_host[j + 1] - bstart_host[j] + TC_M - 1) / TC_M;
  }
  tile_base_host[J] = (int)tot;
  return tot;
}

size_t tc_dictionary_floats(long long total_tiles, int nck) { return (size_t)total_tiles * nck * TC_ACHUNK; }
size_t tc_pixel_floats(long long max_tiles, int nck) { return (size_t)max_tiles * nck * TC_BCHUNK; }
int tc_chunks(int n) { return (n + TC_KC - 1) / TC_KC; }

cudaError_t tc_pack_dictionary(const float2* A, int n, int m, int J, const int* bstart_dev, const int* tile_base_dev, int nck,
                               float* Apk, long long total_tiles, int num_sms, cudaStream_t st) {
  count_launch();
  tc_pack_dictionary_kernel<<<num_sms * 8, 256, 0, st>>>(A, n, m, J, bstart_dev, tile_base_dev, nck, Apk, total_tiles);
  return cudaGetLastError();
}

cudaError_t tc_adjoint_round(const TiledParams& T, const float* Apk, float* Rpk, const int* tile_base_dev, int nck,
                             int max_tiles, int tiles_per_split, int max_splits, float2* G, cudaStream_t st) {
  count_launch();
  tc_pack_pixels_kernel<<<max_tiles, 256, 0, st>>>(T, nck, Rpk);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = 2 * (size_t)TC_STAGE_BYTES;
  e = cudaFuncSetAttribute(tc_adjoint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  tc_adjoint_kernel<<<dim3(max_tiles, max_splits), 128, smem, st>>>(T, Apk, Rpk, tile_base_dev, nck, tiles_per_split, G);
  return cudaGetLastError();
}

}  // namespace tb
