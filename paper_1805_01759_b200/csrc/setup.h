// Launchers for the setup and selection kernels (k_setup.cu, k_select.cu).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime.h>

namespace tb {

cudaError_t launch_default_lambda(const float2* A, int n, int m, const float2* B, long long P, double beta,
                                  double* lam, int num_sms, cudaStream_t st);
// AT[c][i] = A[i][c] (complex64)
cudaError_t launch_transpose(const float2* A, int n, int m, float2* AT, cudaStream_t st);
cudaError_t launch_derive_seeds(uint64_t run_seed, long long first, long long P, uint64_t* seeds, cudaStream_t st);
cudaError_t launch_synth_pair(const float2* A, int n, int m, uint64_t seed, const uint64_t* stream_ids, const int* c0,
                              const int* c1, const float* phase, const float* sigma, long long count, float2* pixels,
                              uint64_t* seeds, cudaStream_t st);
cudaError_t launch_power_small(const float2* A, int n, int m, const long long* starts, const long long* stops,
                               int num_ranges, double2* v, double2* uscratch, int max_iter, double rtol,
                               double* out_dev, cudaStream_t st);
cudaError_t power_iter_large(const float2* A, int n, int m, long long start, long long stop, double2* v,
                             double2* u, int max_iter, double rtol, double* result, int num_sms, cudaStream_t st);

cudaError_t launch_steering(const double* xi, const double* eta, int n, int n_axes, const double* elev, const double* motion,
                            int ms0, int ms1, long long col0, long long ncols, double sign, float2* out, int num_sms, cudaStream_t st);

cudaError_t launch_apply_filter(const double2* W, int n, int m, const float2* B, long long P, float2* X, int num_sms, cudaStream_t st);

struct SelectParams {
  const float2* A;
  int n, m;
  const float2* X;
  const float2* B;
  long long num_pixels;
  int n_elev, inner, n_axes, msize0, msize1;
  const double* elev;
  const double* motion;
  int k_max, ppsc;
  int* order;
  long long* support;
  double2* amps;
  double* elevs;
  double* motion_out;
  double* scores;
  int* n_scores;
  int* err;
};

// per-warp shared bytes of the selection kernel: profile (double) + argmax (int) + Q[kmax][n] +
// the triangular factor R[kmax][kmax] (warp-uniform values: shared, not per-lane local memory)
__host__ __device__ inline size_t select_warp_bytes(int n, int n_elev, int kmax) {
  size_t a = ((size_t)n_elev * 12 + 15) & ~(size_t)15;
  return a + (size_t)kmax * n * 16 + (size_t)kmax * kmax * 16;
}

cudaError_t launch_select(const SelectParams& S, int num_sms, cudaStream_t st);

}  // namespace tb
