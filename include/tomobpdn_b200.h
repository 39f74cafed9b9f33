/*
 * tomobpdn_b200 -- C ABI of the B200 (sm_100a) batched complex L1-LS library.
 *
 * The reference (`tomobpdn`, pure Python/numpy) has no FFI; its de-facto operator API is the
 * Python solver/pipeline functions.  This header is the boundary those Python entry points
 * bind through ctypes.  Each entry point names the reference interface
 * it replaces (paths relative to /root/reference/pkg/src/tomobpdn).
 *
 * Conventions
 *  - plain pointers + sizes only; complex64 = interleaved float (re, im); complex128 = double.
 *  - "dev" pointers are CUDA device pointers owned by the CALLER; the library never frees
 *    caller memory.  The context owns its dictionary copy and scratch.
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it, outputs are
 *    valid after the stream synchronises.  Calls on one context are not re-entrant.
 *  - return codes: TB_OK, TB_ERR_INVALID (-> ConfigurationError), TB_ERR_CUDA
 *    (-> NumericalError), TB_ERR_CAPACITY (-> CapacityError); tb_last_error() has the text.
 *  - per-pixel solver outcomes are reported in status[] (solver.py:119-123 enum order),
 *    never as return codes (solver.py:311-314, 328-330, 357-361).
 */
#ifndef TOMOBPDN_B200_H
#define TOMOBPDN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_OK 0
#define TB_ERR_INVALID 1
#define TB_ERR_CUDA 2
#define TB_ERR_CAPACITY 3

/* solver kinds (slimmer.py:25 BACKENDS, minus the non-iterative svd_wiener) */
#define TB_SOLVER_RBPG 0  /* solver.py:250 rbpg_solve */
#define TB_SOLVER_FISTA 1 /* solver.py:384 fista_solve */
#define TB_SOLVER_ISTA 2  /* solver.py:379 ista_solve */

/* SolverStatus (solver.py:119-123) */
#define TB_STATUS_CONVERGED 0
#define TB_STATUS_MAX_ITERS 1
#define TB_STATUS_LINE_SEARCH_FAILURE 2
#define TB_STATUS_NUMERICAL_FAILURE 3

typedef struct tb_ctx tb_ctx;
typedef struct tb_tiled tb_tiled;

/* SolverConfig (solver.py:35-97); lambda_reg/seed are per pixel arrays, theta pinned. */
typedef struct tb_solver_config {
  int32_t num_blocks;    /* J, RBPG only (solver.py:50) */
  int32_t max_iters;     /* solver.py:51 */
  int32_t fixed_iters;   /* <= 0 means None (solver.py:56) */
  int32_t backtrack_cap; /* prox.BACKTRACK_CAP = 50 (prox.py:22) */
  double tol;            /* window stop tolerance (solver.py:52, 227-231) */
  double c_alpha;        /* backtracking factor (solver.py:53) */
  double alpha_init_scale; /* alpha0 = scale / L (solver.py:54, 295, 345) */
} tb_solver_config;

const char* tb_version(void);
const char* tb_last_error(void);
/* Number of kernels this library has launched since it was loaded (all entry points, all
   devices).  Instrumentation for the benchmark's gpu_launches claim; no reference counterpart. */
int64_t tb_launch_count(void);
/* Name of the solver kernel family the last tb_solve / tb_tiled_create of this process chose
   ("warp_solver_kernel", "fista_tile_kernel<solo>", "fista_tile_kernel<team>", "tiled_pass_kernel").
   Instrumentation for the benchmark's roofline line; no reference counterpart. */
const char* tb_last_solver_kernel(void);

/* Objective.dictionary (prox.py:25-63): copy a device complex64 [n, m] row-major matrix
 * (row = acquisition, column = flat grid index, model.py:317-323) into a new context. */
int tb_ctx_create(int device, const void* dictionary_dev, int64_t n, int64_t m, tb_ctx** out);
int tb_ctx_destroy(tb_ctx* ctx);

/* spectral_sq_norm (solver.py:167-188) for `num_ranges` column ranges [start, stop) of the
 * context dictionary, fp64 power iteration on A^H A.  v0_dev: device complex128 unit start
 * vectors, concatenated in range order (the reference draws them from
 * substream(0x5EED0F, width)).  sigma2_host: host double[num_ranges]. */
int tb_spectral_sq_norms(tb_ctx* ctx, int32_t num_ranges, const int64_t* starts_host,
                         const int64_t* stops_host, const void* v0_dev, int32_t max_iter,
                         double rtol, double* sigma2_host, void* stream);

/* BlockPartition (solver.py:137-164, 191-214): contiguous ranges + per-block Lipschitz.
 * The context builds the numpy Generator.choice CDF (cumsum(p) / last) used by
 * sample_block (solver.py:217-219).  Host arrays. */
int tb_set_partition(tb_ctx* ctx, int32_t num_blocks, const int64_t* starts_host,
                     const int64_t* stops_host, const double* lipschitz_host);

/* L = 2 spectral_sq_norm(A) for ISTA/FISTA (solver.py:344). */
int tb_set_lipschitz(tb_ctx* ctx, double lipschitz);

/* default_lambda (prox.py:153-161): lambda_p = beta * max_k |(A^H b_p)_k| as a double: the exact
 * products of the complex64 inputs accumulated in fp64, as the reference's complex128 product.
 * pixels_dev: complex64 [P, n] (TSTK1 payload order, stack.py:46-52). */
int tb_default_lambda(tb_ctx* ctx, const void* pixels_dev, int64_t num_pixels, double beta,
                      double* lambda_dev, void* stream);

/* Per-pixel seed rule of the CLI worker (cli.py:102):
 * seeds[i] = derive_seed(substream(run_seed, first_pixel_id + i)) (rng.py:17-29). */
int tb_derive_seeds(uint64_t run_seed, int64_t first_pixel_id, int64_t num_pixels,
                    uint64_t* seeds_dev, void* stream);

/* Monte-Carlo realizations of simulate.py:297-335 on the device (synthesize_pixel, simulate.py:194-205,
 * for the harness's two unit-amplitude scatterers snapped to grid columns col0/col1):
 * pixels[r] = A[:, col0[r]] + e^{j phase[r]} A[:, col1[r]] + sqrt(sigma[r]^2 / 2) (N + jN), complex64 [count][n],
 * phase NaN = drawn uniform(0, 2 pi); seeds[r] = the nested RBPG seed.  Draws come from Philox4x64-10
 * keyed (seed, stream_ids[r]) (rng.py:17-24) with Box-Muller normals: statistically, not bit-,
 * equivalent to the reference's numpy ziggurat draws.  Device arrays. */
int tb_synthesize_pairs(tb_ctx* ctx, uint64_t seed, const uint64_t* stream_ids_dev, const int32_t* col0_dev,
                        const int32_t* col1_dev, const float* phase_dev, const float* sigma_dev, int64_t count,
                        void* pixels_dev, uint64_t* seeds_dev, void* stream);

/* rbpg_solve / fista_solve / ista_solve (solver.py:250-390) over a pixel batch.
 *  pixels_dev  complex64 [P, n];  lambda_dev double [P];  seeds_dev uint64 [P] (RBPG only,
 *  may be NULL otherwise);  x_dev complex64 [P, m] out (Solution.x_hat);
 *  f_final_dev double [P] out (objective_history[-1]);  history_dev double [P, hist_stride]
 *  out or NULL (objective_history, NaN-padded after iterations+1 entries);
 *  iterations_dev int32 [P] out;  status_dev int32 [P] out (TB_STATUS_*).
 *  Asynchronous on `stream`; not re-entrant per context (the context owns the solver workspace:
 *  the RBPG extrapolation memory of the on-chip solver and the tiled solver's state buffers). */
int tb_solve(tb_ctx* ctx, int32_t solver, const tb_solver_config* cfg, const void* pixels_dev,
             const double* lambda_dev, const uint64_t* seeds_dev, int64_t num_pixels, void* x_dev,
             double* f_final_dev, double* history_dev, int64_t hist_stride,
             int32_t* iterations_dev, int32_t* status_dev, void* stream);

/* Large-dictionary solver driven one round at a time (used by tb_solve automatically when the
 * warp-per-pixel plan does not fit, and directly by the column-sharded multi-GPU driver).
 * A round advances every unfinished pixel by one backtracking trial of its current iteration
 * (solver.py:281-333 / 354-371).  round_a = block draw + r_y, fused adjoint/prox/forward pass over
 * the local dictionary columns, split reduction into red_dev; the caller may all-reduce red_dev
 * (sum over column shards) before round_b = test/accept/history/stop.
 *  red_dev: caller-owned device buffer of P*(2n+4) doubles ([P][n] complex128 forward product
 *  followed by [P][4] scalars), or NULL for an internal one.  State lives in HBM (3 fp64 copies
 *  of x per pixel). */
int tb_tiled_create(tb_ctx* ctx, int32_t solver, const tb_solver_config* cfg, const void* pixels_dev,
                    const double* lambda_dev, const uint64_t* seeds_dev, int64_t num_pixels,
                    double* history_dev, int64_t hist_stride, void* red_dev, void* stream,
                    tb_tiled** out);
int tb_tiled_round_a(tb_tiled* h, void* stream);
int tb_tiled_round_b(tb_tiled* h, void* stream);
int tb_tiled_remaining(tb_tiled* h, int64_t* remaining_host, void* stream);
int tb_tiled_finish(tb_tiled* h, void* x_dev, double* f_final_dev, int32_t* iterations_dev,
                    int32_t* status_dev, void* stream);
int tb_tiled_destroy(tb_tiled* h);

/* svd_wiener_solve (solver.py:393-407) batched: x_p = W b_p with the precomputed linear filter
 * W = V diag(s / (s^2 + mu)) U^H (complex128 [m][n], from the dictionary's thin SVD); fp64
 * accumulation, complex64 x_dev [P][m] for the selection stage. */
int tb_apply_filter(tb_ctx* ctx, const void* filter_dev, const void* pixels_dev, int64_t num_pixels,
                    void* x_dev, void* stream);

/* build_steering_matrix (model.py:296-323) on the device: out[i, c] = exp(sign j 2 pi phase_i(col0+c))
 * with phase_i(k) = xi_i s(k) + sum_a eta_{a,i} p_a(k) over the row-major grid (elevation leading);
 * sign = +1 is the reference convention, -1 the BASELINE.json one.  Writes complex64
 * [n][ncols] for the column range [col0, col0 + ncols) -- a whole dictionary or one rank's shard.
 *  xi_dev double [n]; eta_dev double [n_axes][n]; elev_dev double [n_elev];
 *  motion_dev double axis values concatenated; motion_sizes_host int32 [n_axes]. */
int tb_build_steering(int device, const double* xi_dev, const double* eta_dev, int64_t n, int32_t n_axes,
                      const double* elev_dev, int64_t n_elev, const double* motion_dev,
                      const int32_t* motion_sizes_host, int64_t col0, int64_t ncols, double sign,
                      void* out_dev, void* stream);

/* SL1MMER stages 2-3 (slimmer.py:77-190): detect_support -> model_select (BIC over fp64 LS
 * refits, rank filter) -> estimate_params (debiased LS amplitudes, grid decode).
 *  grid: n_elev elevation bins x inner motion bins (inner = prod motion sizes, flat index
 *  row-major with elevation leading, model.py:158-160); elev_dev double [n_elev];
 *  motion_dev double [n_motion_axes][...] concatenated axis values, motion_sizes_host[n_axes].
 *  Outputs (device): model_order int32 [P]; support int64 [P, k_max] (-1 padded);
 *  amplitudes complex128 [P, k_max]; elevations double [P, k_max];
 *  motion double [P, k_max, n_motion_axes]; scores double [P, k_max+1] (NaN padded);
 *  n_scores int32 [P]; error int32 [P] (1 = EstimationError rank deficiency). */
int tb_select(tb_ctx* ctx, const void* x_dev, const void* pixels_dev, int64_t num_pixels,
              int32_t n_elev, int32_t n_motion_axes, const int32_t* motion_sizes_host,
              const double* elev_dev, const double* motion_dev, int32_t k_max,
              int32_t params_per_scatterer, int32_t* model_order_dev, int64_t* support_dev,
              void* amplitudes_dev, double* elevations_dev, double* motion_out_dev,
              double* scores_dev, int32_t* n_scores_dev, int32_t* error_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TOMOBPDN_B200_H */
