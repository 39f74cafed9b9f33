// Large-dictionary ("tiled") solver: pixel-tiled SIMT GEMMs over dictionary column tiles with the
// iterate state resident in HBM.  Used when A does not fit the warp solver (cfg4: n=100,
// m=160,000; cfg5: m=1,048,576, optionally column-sharded across GPUs).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime.h>

namespace tb {

constexpr int TL_PT = 32;     // pixels per tile
constexpr int TL_CT = 64;     // dictionary columns per column tile
constexpr int TL_THREADS = 256;

enum { PH_PREP = 0, PH_TRIAL = 1, PH_DONE = 2 };

struct TiledParams {
  // problem
  const float2* A;  // [n][m] (local column shard)
  int n, m;         // local columns
  int mode;         // SOLVER_*
  int J;            // blocks (1 for ISTA/FISTA)
  const int* bstart;      // device [J+1] local block starts (column stripes of the global blocks)
  const double* alpha0;   // device [J]: scale / max(L_j, 1e-300)
  const double* cdf;      // device [J]
  const double* mk;       // device [total+1]
  int total_iters, fixed, cap;
  double tol, c_alpha;
  int split_width;  // columns per CTA split (multiple of TL_CT)
  int max_splits;
  // batch (chunk)
  int P;
  const float2* B;       // [P][n]
  const double* lam;     // [P]
  const uint64_t* seeds; // [P]
  double2* X3;           // 3 x [P][m] fp64 state buffers
  // Tile occupancy of the state buffers: occ[buf][p][t] == 0 means TL_CT-column tile t of buffer
  // buf of pixel p is all zero (its memory is then never read, and a zero candidate tile is never
  // written).  Tiles are cut per block from its first column (ftile[b] = first tile of block b), so
  // every pass column tile is exactly one occupancy tile.  L1 iterates are sparse after the first
  // iterations, so this removes most of the fp64 state traffic.
  unsigned char* occ;    // [3][P][NT]
  const int* ftile;      // device [J+1]
  int NT;
  // per-pixel state
  int* phase;
  int* k;
  int* trial;
  int* status;
  int* blk;
  int* roles;     // [P][3]: buffer index of x, prev, z
  int* commit;    // [P]: RBPG block copy after the round (0 none, 1 prev<-x, 2 also x<-z)
  double* F;
  double* l1;
  double* alpha;
  double* ring;   // [P][16]
  double* l1blk;  // [P][J]
  double2* r;     // [P][n]  RBPG residual / FISTA A x
  double2* axp;   // [P][n]  FISTA A x_prev
  double2* ry;    // [P][n]  fp64 r_y (RBPG) / A y (FISTA)
  double2* delta; // [P][J][n] RBPG A_b (x_b - prev_b)
  float2* ry32;   // [P][n]  r_y rounded, adjoint operand
  const float2* G; // [P][m]  A^H r_y from the tensor-core adjoint, or null (SIMT adjoint in the pass)
  // scheduling
  int* perm;      // [P] pending pixels grouped by block
  int4* tiles;    // [P/PT + J]: (block, perm offset, count, 0)
  int* ntiles;    // [1]
  int* remaining; // [1]
  // partials
  double2* part;  // [max_splits][P][n]
  double* psc;    // [max_splits][P][4]
  double2* red;   // [P][n]  reduced forward product (allreduce target when sharded)
  double* redsc;  // [P][4]
  // outputs
  float2* X;      // [P][m] complex64 x_hat (local columns)
  double* f_final;
  double* hist;
  long long hist_stride;
  int* iters;
};

cudaError_t tiled_init(const TiledParams& T, cudaStream_t st);
cudaError_t tiled_prep(const TiledParams& T, cudaStream_t st);
cudaError_t tiled_pass(const TiledParams& T, int num_sms, cudaStream_t st);
cudaError_t tiled_reduce(const TiledParams& T, cudaStream_t st);
cudaError_t tiled_update(const TiledParams& T, cudaStream_t st);
cudaError_t tiled_finish(const TiledParams& T, cudaStream_t st);

// tensor-core adjoint (k_tc_tiled.cu)
long long tc_tiles_for(const int* bstart_host, int J, int* tile_base_host);
size_t tc_dictionary_floats(long long total_tiles, int nck);
size_t tc_pixel_floats(long long max_tiles, int nck);
int tc_chunks(int n);
cudaError_t tc_pack_dictionary(const float2* A, int n, int m, int J, const int* bstart_dev, const int* tile_base_dev, int nck,
                               float* Apk, long long total_tiles, int num_sms, cudaStream_t st);
cudaError_t tc_adjoint_round(const TiledParams& T, const float* Apk, float* Rpk, const int* tile_base_dev, int nck,
                             int max_tiles, int tiles_per_split, int max_splits, float2* G, cudaStream_t st);

}  // namespace tb
