// Parameter block shared by the host launcher (tb_api.cu) and the solver kernels.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime.h>

namespace tb {

enum { SOLVER_RBPG = 0, SOLVER_FISTA = 1, SOLVER_ISTA = 2 };
enum { STATUS_CONVERGED = 0, STATUS_MAX_ITERS = 1, STATUS_LINE_SEARCH_FAILURE = 2, STATUS_NUMERICAL_FAILURE = 3 };
constexpr int STOP_WINDOW = 10;  // solver.py:29

struct SolveParams {
  const float2* A;  // device [n][m] row-major complex64
  const float2* AT; // device [m][n] (column-major copy of A), read by the forward products when A is not in shared memory
  int n, m, ms;     // ms: odd shared-memory row stride (>= m)
  int mode;
  int num_blocks;
  int max_width;          // widest active column range (block or m)
  const int* blk_start;   // device [J+1]
  const double* blk_lip;  // device [J]
  const double* cdf;      // device [J]
  const double* mk;       // device [total_iters + 1]: (k-2)/(k+1)
  double lip_full;
  int total_iters, fixed, cap;
  double tol, c_alpha, alpha_scale;
  const float2* B;
  const double* lam;
  const uint64_t* seeds;
  long long num_pixels;
  float2* X;
  double* f_final;
  double* hist;
  long long hist_stride;
  int* iters;
  int* status;
  unsigned long long* queue;
  double2* dglob;  // RBPG (TB_WS_DCACHE): fp64 extrapolation memory d = x - prev, [slots][m], L2-resident
};

// RBPG keeps d = x - prev in fp64 in global memory (L2) and caches delta_b = A_b d_b per block in
// shared memory, so r_y = r + m_k delta_b needs no forward product (see k_warp_solver.cu).
#ifndef TB_WS_DCACHE
#define TB_WS_DCACHE 1
#endif

// per-warp shared bytes (ISTA/FISTA): 2 fp64 n-vectors, fp64 x (m) + fp64 broadcast buffer (width),
// fp64 d = x - prev (m), fp32 r_y as float4 + fp32 b (n each), 16-double ring, J-double per-block l1
// cache, 32 buffered Philox outputs, width ints (compacted nonzero columns)
__host__ __device__ inline size_t warp_slot_bytes(int n, int m, int width, int J) {
  size_t b = (size_t)n * 32 + (size_t)(m + width) * 16 + (size_t)m * 16 + (size_t)n * 24 + 16 * 8 + (size_t)J * 8 + 32 * 8 + (size_t)width * 4;
  return (b + 15) & ~(size_t)15;
}
// RBPG slot with the delta cache: fp64 r, fp64 x (m), fp64 broadcast buffer (width), r_y quads (n),
// delta_b = A_b d_b for every block (J x n fp64), ring, per-block l1, Philox buffer, column list
__host__ __device__ inline size_t warp_slot_bytes_dc(int n, int m, int width, int J) {
  size_t b = (size_t)n * 16 + (size_t)m * 16 + (size_t)width * 16 + (size_t)n * 16 + (size_t)J * n * 16 + 16 * 8 + (size_t)J * 8 + 32 * 8 + (size_t)width * 4;
  return (b + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t warp_slot_bytes_for(bool rb, int n, int m, int width, int J) {
  return (rb && TB_WS_DCACHE) ? warp_slot_bytes_dc(n, m, width, J) : warp_slot_bytes(n, m, width, J);
}
// per-CTA block tables: cdf, alpha0 (J doubles each) + J+1 block starts
__host__ __device__ inline size_t block_table_bytes(int J) {
  size_t b = (size_t)J * 16 + (size_t)(J + 1) * 4;
  return (b + 15) & ~(size_t)15;
}

cudaError_t launch_warp_solver(const SolveParams& P, int num_sms, cudaStream_t st, int* used_warps);
// ISTA/FISTA kernel with the extrapolation memory and the candidate in tensor memory
// (k_fista_tile.cu): >= 8 pixel slots must fit in shared memory (beside the dictionary: *asmem; else
// it is read from global memory); m <= 512.  *slots = resident pixel slots per SM.  team = the
// 4-warp-team shared contraction (measured slower), else one warp per pixel.
bool fista_tile_fits(int n, int m, bool* asmem, int* slots);
cudaError_t launch_fista_tile(const SolveParams& P, int num_sms, cudaStream_t st, int* used_warps, bool team);

}  // namespace tb
