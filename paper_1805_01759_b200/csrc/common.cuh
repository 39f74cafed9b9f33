// Shared device helpers for the tomobpdn_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define TB_FULL_MASK 0xffffffffu

namespace tb {

// Host-side count of this library's kernel launches (tb_launch_count, include/tomobpdn_b200.h).
void count_launch();

// ---------------------------------------------------------------- complex64 arithmetic
struct __align__(8) c64 {
  float x, y;
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// acc += a * b
__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_conj(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
}
// acc += conj(a) * r with r4 = (r.x, r.y, r.y, -r.x): two packed FFMA2 (a.x and a.y as scalar
// broadcast operands), the same per-component rounding sequence as cfma_conj.
__device__ __forceinline__ void cfma_conj_x2(float2& acc, float2 a, float4 r4) {
  asm("{\n\t.reg .b64 c, aa, bb, r01, r23;\n\t"
      "mov.b64 c, {%0, %1};\n\t"
      "mov.b64 aa, {%2, %2};\n\t"
      "mov.b64 bb, {%3, %3};\n\t"
      "mov.b64 r01, {%4, %5};\n\t"
      "mov.b64 r23, {%6, %7};\n\t"
      "fma.rn.f32x2 c, aa, r01, c;\n\t"
      "fma.rn.f32x2 c, bb, r23, c;\n\t"
      "mov.b64 {%0, %1}, c;\n\t}"
      : "+f"(acc.x), "+f"(acc.y)
      : "f"(a.x), "f"(a.y), "f"(r4.x), "f"(r4.y), "f"(r4.z), "f"(r4.w));
}
__device__ __forceinline__ float4 conj_operand(float rx, float ry) { return make_float4(rx, ry, ry, -rx); }
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ float cabsf(float2 a) { return sqrtf(fmaf(a.x, a.x, a.y * a.y)); }

// ---------------------------------------------------------------- warp reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(TB_FULL_MASK, v, o);
  return v;
}
// Warp all-reduce of four doubles by recursive halving: at xor 16 and 8 each lane forwards the
// half it does not keep, so 10 double shuffles (plus 4 broadcasts) replace 20.  Every lane ends
// with the same four sums.
__device__ __forceinline__ void warp_sum4(double v[4]) {
  const int lane = threadIdx.x & 31;
  const bool h16 = lane & 16, h8 = lane & 8;
  double k0 = h16 ? v[2] : v[0], k1 = h16 ? v[3] : v[1];
  const double s0 = h16 ? v[0] : v[2], s1 = h16 ? v[1] : v[3];
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  double kk = h8 ? k1 : k0;
  kk += __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
  kk += __shfl_xor_sync(0xffffffffu, kk, 4);
  kk += __shfl_xor_sync(0xffffffffu, kk, 2);
  kk += __shfl_xor_sync(0xffffffffu, kk, 1);
  // value q = 2 * h16 + h8 now sits in lanes 8q .. 8q + 7
  v[0] = __shfl_sync(0xffffffffu, kk, 0);
  v[1] = __shfl_sync(0xffffffffu, kk, 8);
  v[2] = __shfl_sync(0xffffffffu, kk, 16);
  v[3] = __shfl_sync(0xffffffffu, kk, 24);
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(TB_FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(TB_FULL_MASK, v, o));
  return v;
}

// ---------------------------------------------------------------- Philox4x64-10
// numpy's Philox bit generator (the generator behind rng.substream, rng.py:17-24).
struct Philox4x64 {
  uint64_t k0, k1;
  uint64_t ctr;  // low 64 bits of the 256-bit counter; numpy starts at 0 and pre-increments
  uint64_t buf[4];
  int pos;       // next buffered output, 4 = empty
};

__host__ __device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
#else
    unsigned __int128 p0 = (unsigned __int128)M0 * c[0], p1 = (unsigned __int128)M1 * c[2];
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
#endif
    uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ void philox_init(Philox4x64& s, uint64_t seed, uint64_t stream_id) {
  s.k0 = seed;
  s.k1 = stream_id;
  s.ctr = 0;
  s.pos = 4;
}

__device__ __forceinline__ uint64_t philox_next(Philox4x64& s) {
  if (s.pos == 4) {
    s.ctr += 1;
    uint64_t c[4] = {s.ctr, 0ull, 0ull, 0ull};
    philox4x64_10(c, s.k0, s.k1);
    s.buf[0] = c[0];
    s.buf[1] = c[1];
    s.buf[2] = c[2];
    s.buf[3] = c[3];
    s.pos = 0;
  }
  uint64_t v = s.buf[0];
  // rotate so the buffer stays in registers (no dynamic indexing)
  s.buf[0] = s.buf[1];
  s.buf[1] = s.buf[2];
  s.buf[2] = s.buf[3];
  s.pos += 1;
  return v;
}

// (raw >> 11) * 2^-53: numpy's next_double (Generator.random).
__device__ __forceinline__ double raw_to_unit(uint64_t raw) {
  return (double)(raw >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace tb
