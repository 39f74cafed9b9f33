// tcgen05 (5th-gen tensor core) prototype of the tiled pass's adjoint product on sm_100a.
//
// G[c][p] = sum_i conj(A[i][c]) r[p][i] for a tile of 64 dictionary columns and 32 pixels, computed
// as the real GEMM D[128 x 32] = Ahat[128 x K] * Rhat[32 x K]^T with K = 2n:
//   Ahat[2c][2i] = Re A_ic, Ahat[2c][2i+1] = Im A_ic, Ahat[2c+1][2i] = -Im A_ic, Ahat[2c+1][2i+1] = Re A_ic
//   Rhat[p][2i]  = Re r_pi, Rhat[p][2i+1]  = Im r_pi
// so D[2c][p] = Re g, D[2c+1][p] = Im g.  3xTF32 split (hi*hi + hi*lo + lo*hi, fp32 accumulation in
// TMEM) keeps fp32-level accuracy.  Operands are staged in shared memory in the canonical K-major
// SWIZZLE_NONE layout (8-row x 16-byte core matrices; LBO = 128 B between the two K-halves of an
// MMA, SBO = K/4*128 B between 8-row groups); one elected thread issues the MMAs, tcgen05.commit
// arrives on an mbarrier, the four warps read their 32-lane TMEM quadrant with tcgen05.ld.
#include <stdint.h>

#include "common.cuh"

namespace tb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// K-major SWIZZLE_NONE operand: element (row r, k) byte offset inside the operand buffer
__device__ __forceinline__ uint32_t kmajor_off(int r, int k, int K) {
  return (uint32_t)((r >> 3) * (K >> 2) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version for sm_100
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

constexpr uint32_t kIdescTF32_M128_N32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__global__ void __launch_bounds__(128, 1) tc_adjoint_proto_kernel(const float2* __restrict__ A, int n, int m, int col0,
                                                                  const float2* __restrict__ R, float2* __restrict__ G,
                                                                  int passes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int K = 2 * n;  // multiple of 8
  const uint32_t a_bytes = 128u * K * 4u, b_bytes = 32u * K * 4u;
  unsigned char* a_hi = sm;
  unsigned char* a_lo = a_hi + a_bytes;
  unsigned char* b_hi = a_lo + a_bytes;
  unsigned char* b_lo = b_hi + b_bytes;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // stage Ahat / Rhat (hi, lo) in the canonical layout
  for (int idx = tid; idx < 64 * n; idx += blockDim.x) {
    const int c = idx % 64, i = idx / 64;
    const float2 a = A[(size_t)i * m + col0 + c];
    const float v[4] = {a.x, a.y, -a.y, a.x};  // (2c,2i) (2c,2i+1) (2c+1,2i) (2c+1,2i+1)
    const int rr[4] = {2 * c, 2 * c, 2 * c + 1, 2 * c + 1};
    const int kk[4] = {2 * i, 2 * i + 1, 2 * i, 2 * i + 1};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float hi = tf32_rna(v[q]);
      const float lo = tf32_rna(v[q] - hi);
      const uint32_t o = kmajor_off(rr[q], kk[q], K);
      *reinterpret_cast<float*>(a_hi + o) = hi;
      *reinterpret_cast<float*>(a_lo + o) = lo;
    }
  }
  for (int idx = tid; idx < 32 * n; idx += blockDim.x) {
    const int p = idx / n, i = idx % n;
    const float2 r = R[(size_t)p * n + i];
    const float v[2] = {r.x, r.y};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float hi = tf32_rna(v[q]);
      const float lo = tf32_rna(v[q] - hi);
      const uint32_t o = kmajor_off(p, 2 * i + q, K);
      *reinterpret_cast<float*>(b_hi + o) = hi;
      *reinterpret_cast<float*>(b_lo + o) = lo;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // make generic-proxy smem writes visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = tmem_base;

  if (tid == 0) {
    const uint32_t lbo = 128, sbo_a = (uint32_t)(K / 4) * 128, sbo_b = sbo_a;
    const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
    int first = 1;
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t koff = (uint32_t)s * 256;
      for (int ps = 0; ps < passes; ++ps) {
        const uint32_t aa = (ps == 2 ? al : ah) + koff;
        const uint32_t bb = (ps == 1 ? bl : bh) + koff;
        const uint64_t da = umma_desc(aa, lbo, sbo_a), db = umma_desc(bb, lbo, sbo_b);
        const uint32_t acc = first ? 0u : 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(taddr),
            "l"(da), "l"(db), "r"(kIdescTF32_M128_N32), "r"(acc));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    for (long long spin = 0; !done; ++spin) {
      if (spin > (1ll << 24)) {  // never hang the device: bail out (output left unwritten)
        done = 2;
        break;
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32-lane quadrant: lane l of warp w holds D[32w + l][0..31]
  uint32_t v[32];
  const uint32_t ta = taddr + ((uint32_t)(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = 32 * warp + lane;  // D row = 2c + part
  const int c = row >> 1, part = row & 1;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    const float mine = __uint_as_float(v[p]);
    const float other = __shfl_xor_sync(TB_FULL_MASK, mine, 1);
    if (part == 0) G[(size_t)c * 32 + p] = make_float2(mine, other);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(taddr));
}

}  // namespace tb

extern "C" int tb_tc_adjoint_proto(const void* A, int n, int m, int col0, const void* R, void* G, int passes, void* stream) {
  if (n < 4 || (2 * n) % 8 != 0 || n > 64) return 1;
  const size_t smem = (size_t)(2 * 128 + 2 * 32) * (2 * n) * 4;
  cudaFuncSetAttribute(tb::tc_adjoint_proto_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tb::count_launch();
  tb::tc_adjoint_proto_kernel<<<1, 128, smem, (cudaStream_t)stream>>>((const float2*)A, n, m, col0, (const float2*)R, (float2*)G, passes);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
