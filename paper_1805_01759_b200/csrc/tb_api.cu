// C ABI implementation (include/tomobpdn_b200.h): context management, validation, launches.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/tomobpdn_b200.h"
#include "common.cuh"
#include "setup.h"
#include "solver_params.h"
#include "tiled.h"

struct tb_ctx {
  int device = 0;
  int num_sms = 148;
  int64_t n = 0, m = 0;
  float2* A = nullptr;  // owned copy, [n][m]
  float2* AT = nullptr; // [m][n] transpose, built on first use by the kernels that read A through L1
  // partition
  int num_blocks = 0;
  int* blk_start = nullptr;  // device [J+1]
  double* blk_lip = nullptr; // device [J]
  double* cdf = nullptr;     // device [J]
  int max_block_width = 0;
  double lip_full = 0.0;
  bool has_partition = false, has_lip = false;
  unsigned long long* queue = nullptr;
  double* mk = nullptr;  // momentum table (k-2)/(k+1), k = 0..mk_len-1
  int mk_len = 0;
  std::vector<double> lip_host;  // per-block Lipschitz (host copy)
  std::vector<int> bstart_host;  // J+1
  // tiled-solver workspace, grow-only and kept across solves: re-allocating tens of GB per call
  // costs page mapping time on every solve (one tiled handle per context at a time)
  unsigned char* ws = nullptr;
  size_t ws_size = 0;
  bool ws_busy = false;
  // warp solver RBPG extrapolation memory (fp64 d per warp slot), grow-only
  double2* dglob = nullptr;
  size_t dglob_elems = 0;
  // Ordering of the context's mutable device state (queue counter, dglob, mk, ws) across streams:
  // every launch that uses it records `done` on its stream, and a launch on another stream first
  // waits on `done`, so solves issued on different streams serialise instead of racing; buffers
  // are only freed / reallocated after `done` has completed.
  cudaEvent_t done = nullptr;
  cudaStream_t last = nullptr;
  bool capturing = false;  // inside a graph capture of the tiled rounds: ordering handled around it
};

// Order `st` after the previous user of the context's mutable state (see tb_ctx::done).
static cudaError_t ctx_acquire(tb_ctx* c, cudaStream_t st) {
  if (c->capturing) return cudaSuccess;
  if (c->done && c->last != st) return cudaStreamWaitEvent(st, c->done, 0);
  return cudaSuccess;
}
static cudaError_t ctx_release(tb_ctx* c, cudaStream_t st) {
  if (c->capturing) return cudaSuccess;
  c->last = st;
  return cudaEventRecord(c->done, st);
}
// Wait until no launch uses the context's mutable state (before freeing or reallocating it).
static cudaError_t ctx_drain(tb_ctx* c) { return c->done ? cudaEventSynchronize(c->done) : cudaSuccess; }

struct tb_tiled {
  tb_ctx* ctx = nullptr;
  tb::TiledParams T{};
  void* owned = nullptr;  // single device allocation holding every internal buffer
  bool own_red = false;
  int max_width = 0;
  long long rounds = 0;
  // tensor-core adjoint (k_tc_tiled.cu); G == nullptr selects the SIMT adjoint inside the pass
  float2* G = nullptr;
  float* Apk = nullptr;
  float* Rpk = nullptr;
  int* tile_base = nullptr;
  int nck = 0, tc_max_tiles = 0, tc_tiles_per_split = 1, tc_splits = 1;
};

// TB_TILED_TC=0/1 overrides the default adjoint engine of the tiled path
static bool tiled_use_tc() {
  const char* e = getenv("TB_TILED_TC");
  if (e && *e) return atoi(e) != 0;
  return false;
}

static thread_local std::string g_err;

// numpy's pairwise summation for float64 (the `lip.sum()` of solver.py:156), so the block
// probabilities and the choice CDF are bit-identical to the reference's.
static double numpy_pairwise_sum(const double* a, long long n) {
  if (n < 8) {
    double res = 0.0;
    for (long long i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    long long i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  return numpy_pairwise_sum(a, n2) + numpy_pairwise_sum(a + n2, n - n2);
}

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define TB_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) return fail(TB_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)

static std::atomic<long long> g_launches{0};
void tb::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static void count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// TB_TILED_GRAPH=0 disables the CUDA-graph replay of the tiled round loop (A/B)
static bool tiled_use_graph() {
  const char* e = getenv("TB_TILED_GRAPH");
  return !(e && *e && atoi(e) == 0);
}

extern "C" {

int64_t tb_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
static std::atomic<const char*> g_last_kernel{"none"};
const char* tb_last_solver_kernel(void) { return g_last_kernel.load(std::memory_order_relaxed); }
const char* tb_version(void) { return "tomobpdn_b200 0.1.0 sm_100a"; }
const char* tb_last_error(void) { return g_err.c_str(); }

int tb_ctx_create(int device, const void* dictionary_dev, int64_t n, int64_t m, tb_ctx** out) {
  if (!out || !dictionary_dev) return fail(TB_ERR_INVALID, "null argument");
  if (n < 1 || m < 1) return fail(TB_ERR_INVALID, "dictionary must be a 2-d matrix with n, m >= 1 (got %lld x %lld)", (long long)n, (long long)m);
  if (n > 128) return fail(TB_ERR_INVALID, "n = %lld acquisitions exceeds the supported 128", (long long)n);
  if (n * m >= (1ll << 31)) return fail(TB_ERR_CAPACITY, "dictionary needs %lld entries, device budget is 2^31", (long long)(n * m));
  TB_CUDA(cudaSetDevice(device));
  tb_ctx* c = new tb_ctx();
  c->device = device;
  c->n = n;
  c->m = m;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMalloc(&c->A, sizeof(float2) * n * m);
  if (e == cudaSuccess) e = cudaMemcpy(c->A, dictionary_dev, sizeof(float2) * n * m, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&c->queue, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    cudaFree(c->A);
    delete c;
    return fail(TB_ERR_CUDA, "tb_ctx_create: %s", cudaGetErrorString(e));
  }
  *out = c;
  return TB_OK;
}

int tb_ctx_destroy(tb_ctx* c) {
  if (!c) return TB_OK;
  cudaSetDevice(c->device);
  ctx_drain(c);
  if (c->done) cudaEventDestroy(c->done);
  cudaFree(c->A);
  cudaFree(c->AT);
  cudaFree(c->blk_start);
  cudaFree(c->blk_lip);
  cudaFree(c->cdf);
  cudaFree(c->queue);
  cudaFree(c->mk);
  cudaFree(c->ws);
  cudaFree(c->dglob);
  delete c;
  return TB_OK;
}

int tb_spectral_sq_norms(tb_ctx* c, int32_t num_ranges, const int64_t* starts, const int64_t* stops,
                         const void* v0_dev, int32_t max_iter, double rtol, double* sigma2_host, void* stream) {
  if (!c || !starts || !stops || !v0_dev || !sigma2_host) return fail(TB_ERR_INVALID, "null argument");
  if (num_ranges < 1) return fail(TB_ERR_INVALID, "num_ranges must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  TB_CUDA(cudaSetDevice(c->device));
  long long total = 0;
  std::vector<long long> s(num_ranges), e(num_ranges);
  for (int r = 0; r < num_ranges; ++r) {
    s[r] = starts[r];
    e[r] = stops[r];
    if (s[r] < 0 || e[r] > c->m || e[r] <= s[r]) return fail(TB_ERR_INVALID, "range %d [%lld, %lld) invalid for m = %lld", r, s[r], e[r], (long long)c->m);
    total += e[r] - s[r];
  }
  double2 *v = nullptr, *u = nullptr;
  double* out = nullptr;
  TB_CUDA(cudaMallocAsync(&v, sizeof(double2) * total, st));
  TB_CUDA(cudaMallocAsync(&u, sizeof(double2) * total, st));
  TB_CUDA(cudaMallocAsync(&out, sizeof(double) * num_ranges, st));
  TB_CUDA(cudaMemcpyAsync(v, v0_dev, sizeof(double2) * total, cudaMemcpyDeviceToDevice, st));
  // small ranges on one CTA each (whole loop on device), wide ranges host-driven multi-CTA
  const long long small_limit = 1ll << 18;  // wider ranges use the multi-CTA path (one CTA per range is too slow for cfg4/5 blocks)
  std::vector<long long> ss, se;
  std::vector<int> small_idx;
  std::vector<long long> offs(num_ranges);
  long long off = 0;
  for (int r = 0; r < num_ranges; ++r) {
    offs[r] = off;
    off += e[r] - s[r];
  }
  // the small kernel indexes v by its own concatenation; run it over a compacted copy
  for (int r = 0; r < num_ranges; ++r)
    if ((e[r] - s[r]) * c->n <= small_limit || e[r] - s[r] == 1) {
      ss.push_back(s[r]);
      se.push_back(e[r]);
      small_idx.push_back(r);
    }
  std::vector<double> hres(num_ranges, 0.0);
  if (!small_idx.empty()) {
    long long tot_small = 0;
    for (size_t k = 0; k < ss.size(); ++k) tot_small += se[k] - ss[k];
    double2 *vs = nullptr, *us = nullptr;
    double* os = nullptr;
    TB_CUDA(cudaMallocAsync(&vs, sizeof(double2) * tot_small, st));
    TB_CUDA(cudaMallocAsync(&us, sizeof(double2) * tot_small, st));
    TB_CUDA(cudaMallocAsync(&os, sizeof(double) * ss.size(), st));
    long long o2 = 0;
    for (size_t k = 0; k < ss.size(); ++k) {
      int r = small_idx[k];
      TB_CUDA(cudaMemcpyAsync(vs + o2, v + offs[r], sizeof(double2) * (e[r] - s[r]), cudaMemcpyDeviceToDevice, st));
      o2 += e[r] - s[r];
    }
    TB_CUDA(tb::launch_power_small(c->A, (int)c->n, (int)c->m, ss.data(), se.data(), (int)ss.size(), vs, us, max_iter, rtol, os, st));
    std::vector<double> hs(ss.size());
    TB_CUDA(cudaMemcpyAsync(hs.data(), os, sizeof(double) * ss.size(), cudaMemcpyDeviceToHost, st));
    TB_CUDA(cudaStreamSynchronize(st));
    for (size_t k = 0; k < ss.size(); ++k) hres[small_idx[k]] = hs[k];
    cudaFreeAsync(vs, st);
    cudaFreeAsync(us, st);
    cudaFreeAsync(os, st);
  }
  for (int r = 0; r < num_ranges; ++r) {
    if ((e[r] - s[r]) * c->n <= small_limit || e[r] - s[r] == 1) continue;
    TB_CUDA(tb::power_iter_large(c->A, (int)c->n, (int)c->m, s[r], e[r], v + offs[r], u + offs[r], max_iter, rtol, &hres[r], c->num_sms, st));
  }
  TB_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(v, st);
  cudaFreeAsync(u, st);
  cudaFreeAsync(out, st);
  for (int r = 0; r < num_ranges; ++r) sigma2_host[r] = hres[r];
  return TB_OK;
}

int tb_set_partition(tb_ctx* c, int32_t J, const int64_t* starts, const int64_t* stops, const double* lip) {
  if (!c || !starts || !stops || !lip) return fail(TB_ERR_INVALID, "null argument");
  if (J < 1 || J > c->m) return fail(TB_ERR_INVALID, "num_blocks must lie in [1, %lld], got %d", (long long)c->m, J);
  std::vector<int> bs(J + 1);
  double total = 0.0;
  int maxw = 0;
  for (int j = 0; j < J; ++j) {
    if (starts[j] != (j == 0 ? 0 : stops[j - 1]) || stops[j] <= starts[j]) return fail(TB_ERR_INVALID, "blocks must be contiguous, disjoint, non-empty");
    if (!(lip[j] >= 0.0) || lip[j] != lip[j] || lip[j] > 1.7e308) return fail(TB_ERR_INVALID, "Lipschitz constants must be finite and >= 0");
    bs[j] = (int)starts[j];
    int w = (int)(stops[j] - starts[j]);
    if (w > maxw) maxw = w;
  }
  if (stops[J - 1] != c->m) return fail(TB_ERR_INVALID, "blocks must cover all %lld columns", (long long)c->m);
  total = numpy_pairwise_sum(lip, J);
  if (!(total > 0.0)) return fail(TB_ERR_INVALID, "at least one block must have positive Lipschitz");
  bs[J] = (int)c->m;
  // numpy Generator.choice: p = L / sum(L) (solver.py:156-160), cdf = cumsum(p), cdf /= cdf[-1]
  std::vector<double> p(J), cdf(J);
  for (int j = 0; j < J; ++j) p[j] = lip[j] / total;
  double acc = 0.0;
  for (int j = 0; j < J; ++j) {
    acc += p[j];
    cdf[j] = acc;
  }
  const double last = cdf[J - 1];
  for (int j = 0; j < J; ++j) cdf[j] /= last;
  TB_CUDA(cudaSetDevice(c->device));
  cudaFree(c->blk_start);
  cudaFree(c->blk_lip);
  cudaFree(c->cdf);
  c->blk_start = nullptr;
  c->blk_lip = c->cdf = nullptr;
  TB_CUDA(cudaMalloc(&c->blk_start, sizeof(int) * (J + 1)));
  TB_CUDA(cudaMalloc(&c->blk_lip, sizeof(double) * J));
  TB_CUDA(cudaMalloc(&c->cdf, sizeof(double) * J));
  TB_CUDA(cudaMemcpy(c->blk_start, bs.data(), sizeof(int) * (J + 1), cudaMemcpyHostToDevice));
  TB_CUDA(cudaMemcpy(c->blk_lip, lip, sizeof(double) * J, cudaMemcpyHostToDevice));
  TB_CUDA(cudaMemcpy(c->cdf, cdf.data(), sizeof(double) * J, cudaMemcpyHostToDevice));
  c->num_blocks = J;
  c->max_block_width = maxw;
  c->has_partition = true;
  c->lip_host.assign(lip, lip + J);
  c->bstart_host = bs;
  return TB_OK;
}

int tb_set_lipschitz(tb_ctx* c, double lip) {
  if (!c) return fail(TB_ERR_INVALID, "null context");
  if (!(lip >= 0.0) || lip > 1.7e308) return fail(TB_ERR_INVALID, "Lipschitz constant must be finite and >= 0");
  c->lip_full = lip;
  c->has_lip = true;
  return TB_OK;
}

int tb_default_lambda(tb_ctx* c, const void* pixels, int64_t P, double beta, double* lam, void* stream) {
  if (!c || (P > 0 && (!pixels || !lam))) return fail(TB_ERR_INVALID, "null argument");
  if (P < 0) return fail(TB_ERR_INVALID, "num_pixels must be >= 0");
  TB_CUDA(cudaSetDevice(c->device));
  TB_CUDA(tb::launch_default_lambda(c->A, (int)c->n, (int)c->m, (const float2*)pixels, P, beta, lam, c->num_sms, (cudaStream_t)stream));
  return TB_OK;
}

int tb_synthesize_pairs(tb_ctx* c, uint64_t seed, const uint64_t* stream_ids, const int32_t* col0, const int32_t* col1,
                        const float* phase, const float* sigma, int64_t count, void* pixels, uint64_t* seeds, void* stream) {
  if (!c || count < 0 || (count > 0 && (!stream_ids || !col0 || !col1 || !phase || !sigma || !pixels || !seeds)))
    return fail(TB_ERR_INVALID, "invalid synthesis arguments");
  TB_CUDA(cudaSetDevice(c->device));
  TB_CUDA(tb::launch_synth_pair(c->A, (int)c->n, (int)c->m, seed, stream_ids, col0, col1, phase, sigma, count, (float2*)pixels, seeds,
                                (cudaStream_t)stream));
  return TB_OK;
}

int tb_derive_seeds(uint64_t run_seed, int64_t first, int64_t P, uint64_t* seeds, void* stream) {
  if (P < 0 || (P > 0 && !seeds)) return fail(TB_ERR_INVALID, "invalid seeds arguments");
  TB_CUDA(tb::launch_derive_seeds(run_seed, first, P, seeds, (cudaStream_t)stream));
  return TB_OK;
}

static int check_solve_args(tb_ctx* c, int32_t solver, const tb_solver_config* cfg, const uint64_t* seeds, int64_t P,
                            const double* hist, int64_t hist_stride) {
  if (!c || !cfg) return fail(TB_ERR_INVALID, "null argument");
  if (P < 0) return fail(TB_ERR_INVALID, "num_pixels must be >= 0");
  if (solver != TB_SOLVER_RBPG && solver != TB_SOLVER_FISTA && solver != TB_SOLVER_ISTA) return fail(TB_ERR_INVALID, "unknown solver %d", solver);
  if (cfg->max_iters < 1) return fail(TB_ERR_INVALID, "max_iters must be >= 1, got %d", cfg->max_iters);
  if (!(cfg->tol > 0.0)) return fail(TB_ERR_INVALID, "tol must be > 0");
  if (!(cfg->c_alpha > 0.0 && cfg->c_alpha < 1.0)) return fail(TB_ERR_INVALID, "c_alpha must lie in (0, 1)");
  if (!(cfg->alpha_init_scale > 0.0)) return fail(TB_ERR_INVALID, "alpha_init_scale must be > 0");
  if (cfg->backtrack_cap < 0) return fail(TB_ERR_INVALID, "backtrack_cap must be >= 0");
  const int total = cfg->fixed_iters > 0 ? cfg->fixed_iters : cfg->max_iters;
  if (hist && hist_stride < total + 1) return fail(TB_ERR_INVALID, "hist_stride %lld < iterations + 1", (long long)hist_stride);
  if (solver == TB_SOLVER_RBPG) {
    if (!c->has_partition) return fail(TB_ERR_INVALID, "RBPG needs tb_set_partition first");
    if (cfg->num_blocks != c->num_blocks) return fail(TB_ERR_INVALID, "config num_blocks %d != partition %d", cfg->num_blocks, c->num_blocks);
    if (!seeds && P > 0) return fail(TB_ERR_INVALID, "RBPG needs per-pixel seeds");
  } else if (!c->has_lip) {
    return fail(TB_ERR_INVALID, "ISTA/FISTA need tb_set_lipschitz first");
  }
  return TB_OK;
}

static int ensure_mk(tb_ctx* c, int total, cudaStream_t st) {
  if (c->mk_len >= total + 1) return TB_OK;
  // a live tiled handle points at the current table
  if (c->ws_busy) return fail(TB_ERR_INVALID, "context busy: a tiled solve with fewer iterations is in flight");
  // theta_k = 2/(k+1) collapsed to m_k = (k-2)/(k+1) (solver.py:222-224), IEEE double division
  std::vector<double> h(total + 1);
  for (int k = 0; k <= total; ++k) h[k] = (k - 2.0) / (k + 1.0);
  TB_CUDA(cudaStreamSynchronize(st));
  TB_CUDA(ctx_drain(c));
  cudaFree(c->mk);
  c->mk = nullptr;
  TB_CUDA(cudaMalloc(&c->mk, sizeof(double) * (total + 1)));
  TB_CUDA(cudaMemcpy(c->mk, h.data(), sizeof(double) * (total + 1), cudaMemcpyHostToDevice));
  c->mk_len = total + 1;
  return TB_OK;
}

// Does the warp-per-pixel kernel's shared-memory plan fit this problem?
static bool warp_path_fits(tb_ctx* c, int32_t solver) {
  const int width = solver == TB_SOLVER_RBPG ? c->max_block_width : (int)c->m;
  if ((width + 31) / 32 > 16) return false;
  const int J = solver == TB_SOLVER_RBPG ? c->num_blocks : 1;
  const size_t slot = tb::warp_slot_bytes_for(solver == TB_SOLVER_RBPG, (int)c->n, (int)c->m, width, J);
  return tb::block_table_bytes(J) + 4 * slot <= 227 * 1024 - 64;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int tb_tiled_create(tb_ctx* c, int32_t solver, const tb_solver_config* cfg, const void* pixels, const double* lam,
                    const uint64_t* seeds, int64_t P, double* hist, int64_t hist_stride, void* red_dev,
                    void* stream, tb_tiled** out) {
  int rc = check_solve_args(c, solver, cfg, seeds, P, hist, hist_stride);
  if (rc != TB_OK) return rc;
  if (!out || P < 1 || !pixels || !lam) return fail(TB_ERR_INVALID, "tiled solver needs >= 1 pixel and buffers");
  g_last_kernel.store("tiled_pass_kernel", std::memory_order_relaxed);
  cudaStream_t st = (cudaStream_t)stream;
  TB_CUDA(cudaSetDevice(c->device));
  const int total = cfg->fixed_iters > 0 ? cfg->fixed_iters : cfg->max_iters;
  rc = ensure_mk(c, total, st);
  if (rc != TB_OK) return rc;
  const bool rb = solver == TB_SOLVER_RBPG;
  const int J = rb ? c->num_blocks : 1;
  if (3ll * J * (long long)sizeof(int) > 227ll * 1024)
    return fail(TB_ERR_INVALID, "num_blocks %d exceeds the tiled scheduler's %d-block limit", J, (int)(227 * 1024 / (3 * sizeof(int))));
  const int n = (int)c->n;
  const long long m = c->m;
  const int maxw = rb ? c->max_block_width : (int)m;
  // split width: the pass grid (pixel tiles x splits) should fill whole waves of 2 CTAs/SM: the
  // CTAs are long (each walks its split's column tiles), so a 5th wave that is 10% full costs
  // nearly a whole wave.  Splits = floor(waves / tiles) (TB_TILED_SPLITS=ceil restores the former
  // 4-wave ceil rule, TB_TILED_WAVES overrides the wave count, for A/B); RBPG rounds have
  // ~P/32 + J/2 tiles (a partial tile per block).
  const long long tiles = (P + tb::TL_PT - 1) / tb::TL_PT + (rb ? J : 0);
  const long long tiles_eff = (P + tb::TL_PT - 1) / tb::TL_PT + (rb ? (J + 1) / 2 : 0);
  const char* sm_env = getenv("TB_TILED_SPLITS");
  const bool ceil_rule = sm_env && strcmp(sm_env, "ceil") == 0;
  const char* wv_env = getenv("TB_TILED_WAVES");
  // many pixel tiles (cfg4): 8 shorter waves balance the uneven (sparsity-dependent) CTA work;
  // few tiles (cfg5's 64 RHS): 4 waves, since every extra split adds a [P][n] partial to reduce
  const long long waves = wv_env && atoi(wv_env) > 0 ? atoi(wv_env) : (tiles_eff >= 16 ? 8 : 4);
  long long s_target = ceil_rule ? (4ll * 2 * c->num_sms + tiles - 1) / tiles : (waves * 2 * c->num_sms) / tiles_eff;
  if (s_target < 1) s_target = 1;
  long long sw = (maxw + s_target - 1) / s_target;
  sw = ((sw + tb::TL_CT - 1) / tb::TL_CT) * tb::TL_CT;
  if (sw < tb::TL_CT) sw = tb::TL_CT;
  const int max_splits = (int)((maxw + sw - 1) / sw);

  // one allocation for all internal state
  size_t sz[32];
  int ns = 0;
  sz[ns++] = align256(sizeof(double2) * 3ull * P * m);   // X3
  sz[ns++] = align256(sizeof(int) * P * 6);              // phase k trial status blk perm
  sz[ns++] = align256(sizeof(int) * P * 4);              // roles, commit
  sz[ns++] = align256(sizeof(double) * P * 3);           // F l1 alpha
  sz[ns++] = align256(sizeof(double) * P * 16);          // ring
  sz[ns++] = align256(sizeof(double) * P * J);           // l1blk
  sz[ns++] = align256(sizeof(double2) * P * n * 3);      // r axp ry
  sz[ns++] = align256(sizeof(double2) * P * (rb ? J : 1) * n);  // delta
  sz[ns++] = align256(sizeof(float2) * P * n);           // ry32
  sz[ns++] = align256(sizeof(int4) * (tiles + J + 1));    // tiles
  sz[ns++] = align256(sizeof(int) * 2);                  // ntiles remaining
  sz[ns++] = align256(sizeof(double2) * (size_t)max_splits * P * n);  // part
  sz[ns++] = align256(sizeof(double) * (size_t)max_splits * P * 4);   // psc
  sz[ns++] = red_dev ? 0 : align256(sizeof(double) * P * (2 * n + 4));  // red + redsc
  sz[ns++] = align256(sizeof(double) * J * 2);           // alpha0, cdf
  sz[ns++] = align256(sizeof(int) * (J + 1));            // bstart
  // occupancy tiles: TL_CT-column tiles cut per block from its first column
  std::vector<int> hft(J + 1, 0);
  for (int j = 0; j < J; ++j) {
    const long long w = rb ? (long long)c->bstart_host[j + 1] - c->bstart_host[j] : m;
    hft[j + 1] = hft[j] + (int)((w + tb::TL_CT - 1) / tb::TL_CT);
  }
  const int NT = hft[J];
  sz[ns++] = align256((size_t)3 * P * NT);               // occ
  sz[ns++] = align256(sizeof(int) * (J + 1));            // ftile
  // tensor-core adjoint: packed dictionary, packed r_y, G = A^H r_y, tile bases
  const bool tc = tiled_use_tc();
  std::vector<int> tc_base(J + 1, 0);
  const int nck = tb::tc_chunks(n);
  long long tc_total = 0;
  if (tc) {
    std::vector<int> hb0(J + 1);
    for (int j = 0; j <= J; ++j) hb0[j] = rb ? c->bstart_host[j] : (j == 0 ? 0 : (int)m);
    tc_total = tb::tc_tiles_for(hb0.data(), J, tc_base.data());
  }
  sz[ns++] = tc ? align256(sizeof(float) * tb::tc_dictionary_floats(tc_total, nck)) : 0;  // Apk
  sz[ns++] = tc ? align256(sizeof(float) * tb::tc_pixel_floats(tiles, nck)) : 0;          // Rpk
  sz[ns++] = tc ? align256(sizeof(float2) * (size_t)P * m) : 0;                          // G
  sz[ns++] = tc ? align256(sizeof(int) * (J + 1)) : 0;                                   // tile_base
  size_t tot = 0;
  for (int i = 0; i < ns; ++i) tot += sz[i];
  if (c->ws_busy) return fail(TB_ERR_INVALID, "one tiled solve per context at a time");
  if (c->ws_size < tot) {
    TB_CUDA(cudaStreamSynchronize(st));
    TB_CUDA(ctx_drain(c));
    cudaFree(c->ws);
    c->ws = nullptr;
    c->ws_size = 0;
    size_t fr = 0, tt = 0;
    cudaMemGetInfo(&fr, &tt);
    if (tot > fr) return fail(TB_ERR_CAPACITY, "tiled solver needs %.1f GB for %lld pixels, %.1f GB free", tot / 1e9, (long long)P, fr / 1e9);
    TB_CUDA(cudaMalloc((void**)&c->ws, tot));
    c->ws_size = tot;
  }
  TB_CUDA(ctx_acquire(c, st));
  unsigned char* base = c->ws;
  tb_tiled* h = new tb_tiled();
  h->ctx = c;
  h->owned = nullptr;
  h->own_red = red_dev == nullptr;
  h->max_width = maxw;
  tb::TiledParams& T = h->T;
  unsigned char* q = base;
  int k = 0;
  auto take = [&](size_t) { unsigned char* r = q; q += sz[k++]; return r; };
  T.X3 = (double2*)take(0);
  int* ints = (int*)take(0);
  T.phase = ints;
  T.k = ints + P;
  T.trial = ints + 2 * P;
  T.status = ints + 3 * P;
  T.blk = ints + 4 * P;
  T.perm = ints + 5 * P;
  T.roles = (int*)take(0);
  T.commit = T.roles + 3 * P;
  double* dbl = (double*)take(0);
  T.F = dbl;
  T.l1 = dbl + P;
  T.alpha = dbl + 2 * P;
  T.ring = (double*)take(0);
  T.l1blk = (double*)take(0);
  double2* vec = (double2*)take(0);
  T.r = vec;
  T.axp = vec + (size_t)P * n;
  T.ry = vec + 2 * (size_t)P * n;
  T.delta = (double2*)take(0);
  T.ry32 = (float2*)take(0);
  T.tiles = (int4*)take(0);
  int* cnts = (int*)take(0);
  T.ntiles = cnts;
  T.remaining = cnts + 1;
  T.part = (double2*)take(0);
  T.psc = (double*)take(0);
  double* redp = red_dev ? (double*)red_dev : (double*)take(0);
  if (red_dev) k++;
  T.red = (double2*)redp;
  T.redsc = redp + 2 * (size_t)P * n;
  double* tabs = (double*)take(0);
  int* bst = (int*)take(0);
  T.alpha0 = tabs;
  T.cdf = tabs + J;
  T.bstart = bst;
  T.occ = take(0);
  int* ftl = (int*)take(0);
  T.ftile = ftl;
  T.NT = NT;
  if (tc) {
    h->Apk = (float*)take(0);
    h->Rpk = (float*)take(0);
    h->G = (float2*)take(0);
    h->tile_base = (int*)take(0);
    h->nck = nck;
    h->tc_max_tiles = (int)tiles;
    const long long ntb = (maxw + 127) / 128;
    long long tps = (tiles * ntb + 4ll * c->num_sms - 1) / (4ll * c->num_sms);
    if (tps < 1) tps = 1;
    h->tc_tiles_per_split = (int)tps;
    h->tc_splits = (int)((ntb + tps - 1) / tps);
    T.G = h->G;
  }
  // block tables: alpha0 = scale / max(L, 1e-300) (solver.py:295, 345), cdf, starts
  std::vector<double> ht(2 * J);
  std::vector<int> hb(J + 1);
  std::vector<double> cdf(J);
  if (rb) {
    TB_CUDA(cudaMemcpy(cdf.data(), c->cdf, sizeof(double) * J, cudaMemcpyDeviceToHost));
    for (int j = 0; j < J; ++j) ht[j] = cfg->alpha_init_scale / fmax(c->lip_host[j], 1e-300);
    for (int j = 0; j <= J; ++j) hb[j] = c->bstart_host[j];
  } else {
    ht[0] = cfg->alpha_init_scale / fmax(c->lip_full, 1e-300);
    cdf[0] = 1.0;
    hb[0] = 0;
    hb[1] = (int)m;
  }
  for (int j = 0; j < J; ++j) ht[J + j] = cdf[j];
  TB_CUDA(cudaMemcpyAsync(tabs, ht.data(), sizeof(double) * 2 * J, cudaMemcpyHostToDevice, st));
  TB_CUDA(cudaMemcpyAsync(bst, hb.data(), sizeof(int) * (J + 1), cudaMemcpyHostToDevice, st));
  if (tc) {
    TB_CUDA(cudaMemcpyAsync(h->tile_base, tc_base.data(), sizeof(int) * (J + 1), cudaMemcpyHostToDevice, st));
    TB_CUDA(tb::tc_pack_dictionary(c->A, n, (int)m, J, bst, h->tile_base, nck, h->Apk, tc_total, c->num_sms, st));
  }
  T.A = c->A;
  T.n = n;
  T.m = (int)m;
  T.mode = solver;
  T.J = J;
  T.mk = c->mk;
  T.total_iters = total;
  T.fixed = cfg->fixed_iters > 0;
  T.cap = cfg->backtrack_cap;
  T.tol = cfg->tol;
  T.c_alpha = cfg->c_alpha;
  T.split_width = (int)sw;
  T.max_splits = max_splits;
  T.P = (int)P;
  T.B = (const float2*)pixels;
  T.lam = lam;
  T.seeds = seeds;
  T.hist = hist;
  T.hist_stride = hist_stride;
  // x = prev = 0 (solver.py:270-272, 348): every state tile starts unoccupied (logically zero)
  TB_CUDA(cudaMemsetAsync(T.occ, 0, (size_t)3 * P * NT, st));
  TB_CUDA(cudaMemcpyAsync(ftl, hft.data(), sizeof(int) * (J + 1), cudaMemcpyHostToDevice, st));
  const int rem = (int)P;
  TB_CUDA(cudaMemcpyAsync(T.remaining, &rem, sizeof(int), cudaMemcpyHostToDevice, st));
  TB_CUDA(tb::tiled_init(T, st));
  TB_CUDA(ctx_release(c, st));
  TB_CUDA(cudaStreamSynchronize(st));
  c->ws_busy = true;
  *out = h;
  return TB_OK;
}

int tb_tiled_round_a(tb_tiled* h, void* stream) {
  if (!h) return fail(TB_ERR_INVALID, "null handle");
  cudaStream_t st = (cudaStream_t)stream;
  TB_CUDA(cudaSetDevice(h->ctx->device));
  TB_CUDA(ctx_acquire(h->ctx, st));
  TB_CUDA(tb::tiled_prep(h->T, st));
  if (h->G)
    TB_CUDA(tb::tc_adjoint_round(h->T, h->Apk, h->Rpk, h->tile_base, h->nck, h->tc_max_tiles, h->tc_tiles_per_split,
                                 h->tc_splits, h->G, st));
  TB_CUDA(tb::tiled_pass(h->T, h->ctx->num_sms, st));
  TB_CUDA(tb::tiled_reduce(h->T, st));
  TB_CUDA(ctx_release(h->ctx, st));
  return TB_OK;
}

int tb_tiled_round_b(tb_tiled* h, void* stream) {
  if (!h) return fail(TB_ERR_INVALID, "null handle");
  TB_CUDA(cudaSetDevice(h->ctx->device));
  TB_CUDA(ctx_acquire(h->ctx, (cudaStream_t)stream));
  TB_CUDA(tb::tiled_update(h->T, (cudaStream_t)stream));
  TB_CUDA(ctx_release(h->ctx, (cudaStream_t)stream));
  h->rounds++;
  return TB_OK;
}

int tb_tiled_remaining(tb_tiled* h, int64_t* out, void* stream) {
  if (!h || !out) return fail(TB_ERR_INVALID, "null argument");
  int v = 0;
  TB_CUDA(ctx_acquire(h->ctx, (cudaStream_t)stream));
  TB_CUDA(cudaMemcpyAsync(&v, h->T.remaining, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  TB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  *out = v;
  return TB_OK;
}

int tb_tiled_finish(tb_tiled* h, void* x, double* f_final, int32_t* iters, int32_t* status, void* stream) {
  if (!h || !x || !f_final || !iters || !status) return fail(TB_ERR_INVALID, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  TB_CUDA(cudaSetDevice(h->ctx->device));
  h->T.X = (float2*)x;
  h->T.f_final = f_final;
  h->T.iters = iters;
  TB_CUDA(ctx_acquire(h->ctx, st));
  TB_CUDA(tb::tiled_finish(h->T, st));
  TB_CUDA(cudaMemcpyAsync(status, h->T.status, sizeof(int) * h->T.P, cudaMemcpyDeviceToDevice, st));
  TB_CUDA(ctx_release(h->ctx, st));
  return TB_OK;
}

int tb_tiled_destroy(tb_tiled* h) {
  if (!h) return TB_OK;
  cudaSetDevice(h->ctx->device);
  cudaDeviceSynchronize();
  h->ctx->ws_busy = false;  // the workspace stays with the context
  delete h;
  return TB_OK;
}

// The tiled solver's round loop as CUDA-graph replays: GRAPH_ROUNDS rounds (each the prep, schedule,
// pass, reduce, update[, commit] launches) are captured once per handle on a private stream -- every
// kernel reads its per-round work from device state (pending pixels, tiles), so the same graph is
// valid for the whole solve -- and replayed until the device-side count of unfinished pixels reaches
// 0 (polled once per replay, as the stream loop polls every 16 rounds; rounds past the last pixel
// are no-ops).  Removes the host launch overhead of ~7 launches per round (cfg5 RBPG: ~3,500 rounds).
static constexpr int GRAPH_ROUNDS = 16;
static int run_rounds_graph(tb_tiled* h, long long max_rounds, int total, cudaStream_t st) {
  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  int rc = TB_OK;
  auto cleanup = [&]() {
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (ev) cudaEventDestroy(ev);
    if (cs) cudaStreamDestroy(cs);
  };
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, st);  // the capture stream starts after the caller's work
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev, 0);
  if (e == cudaSuccess) e = ctx_acquire(h->ctx, cs);  // after the context's previous user
  if (e != cudaSuccess) {
    cleanup();
    return fail(TB_ERR_CUDA, "graph setup: %s", cudaGetErrorString(e));
  }
  const long long before = tb_launch_count();
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cleanup();
    return fail(TB_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
  }
  h->ctx->capturing = true;
  for (int r = 0; r < GRAPH_ROUNDS && rc == TB_OK; ++r) {
    rc = tb_tiled_round_a(h, cs);
    if (rc == TB_OK) rc = tb_tiled_round_b(h, cs);
  }
  h->ctx->capturing = false;
  const cudaError_t ee = cudaStreamEndCapture(cs, &g);
  if (rc != TB_OK || ee != cudaSuccess) {
    cleanup();
    return rc != TB_OK ? rc : fail(TB_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ee));
  }
  const long long per_replay = tb_launch_count() - before;  // kernels in one replay
  count_launches(-per_replay);                               // captured, not launched
  h->rounds -= GRAPH_ROUNDS;
  e = cudaGraphInstantiate(&ge, g, 0);
  if (e != cudaSuccess) {
    cleanup();
    return fail(TB_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
  }
  int* rem_h = nullptr;
  e = cudaMallocHost((void**)&rem_h, sizeof(int));
  for (long long r = 0; e == cudaSuccess && r < max_rounds; r += GRAPH_ROUNDS) {
    e = cudaGraphLaunch(ge, cs);
    if (e != cudaSuccess) break;
    count_launches(per_replay);
    h->rounds += GRAPH_ROUNDS;
    if (r + GRAPH_ROUNDS >= total) {  // poll the device-side count once per replay
      e = cudaMemcpyAsync(rem_h, h->T.remaining, sizeof(int), cudaMemcpyDeviceToHost, cs);
      if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
      if (e == cudaSuccess && *rem_h == 0) break;
    }
  }
  if (e == cudaSuccess) e = cudaEventRecord(ev, cs);  // the caller's stream continues after the rounds
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev, 0);
  if (e == cudaSuccess) e = ctx_release(h->ctx, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (rem_h) cudaFreeHost(rem_h);
  cleanup();
  if (e != cudaSuccess) return fail(TB_ERR_CUDA, "graph replay: %s", cudaGetErrorString(e));
  return TB_OK;
}

static int solve_tiled(tb_ctx* c, int32_t solver, const tb_solver_config* cfg, const void* pixels, const double* lam,
                       const uint64_t* seeds, int64_t P, void* x, double* f_final, double* hist, int64_t hist_stride,
                       int32_t* iters, int32_t* status, cudaStream_t st) {
  // pixel chunks sized to the free HBM (state is 3 fp64 copies of x per pixel)
  size_t fr = 0, tt = 0;
  TB_CUDA(cudaMemGetInfo(&fr, &tt));
  fr += c->ws_size;  // the cached tiled workspace is reusable
  const double per_px = (tiled_use_tc() ? 56.0 : 48.0) * (double)c->m + 64.0 * c->n * (solver == TB_SOLVER_RBPG ? c->num_blocks + 4 : 5) + 4096;
  long long chunk = (long long)(0.6 * (double)fr / per_px);
  if (chunk < 1) return fail(TB_ERR_CAPACITY, "not enough device memory for one pixel of m = %lld", (long long)c->m);
  if (chunk > 8192) chunk = 8192;
  const int total = cfg->fixed_iters > 0 ? cfg->fixed_iters : cfg->max_iters;
  for (long long p0 = 0; p0 < P; p0 += chunk) {
    const long long pc = P - p0 < chunk ? P - p0 : chunk;
    tb_tiled* h = nullptr;
    int rc = tb_tiled_create(c, solver, cfg, (const float2*)pixels + p0 * c->n, lam + p0, seeds ? seeds + p0 : nullptr, pc,
                             hist ? hist + p0 * hist_stride : nullptr, hist_stride, nullptr, st, &h);
    if (rc != TB_OK) return rc;
    const long long max_rounds = (long long)total * (cfg->backtrack_cap + 1) + 1;
    if (tiled_use_graph()) {
      rc = run_rounds_graph(h, max_rounds, total, st);
      if (rc != TB_OK) {
        tb_tiled_destroy(h);
        return rc;
      }
    } else {
      for (long long r = 0; r < max_rounds; ++r) {
        rc = tb_tiled_round_a(h, st);
        if (rc == TB_OK) rc = tb_tiled_round_b(h, st);
        if (rc != TB_OK) {
          tb_tiled_destroy(h);
          return rc;
        }
        if ((r + 1) % 16 == 0 || r + 1 >= total) {
          int64_t rem = 0;
          rc = tb_tiled_remaining(h, &rem, st);
          if (rc != TB_OK || rem == 0) break;
        }
      }
    }
    rc = tb_tiled_finish(h, (float2*)x + p0 * c->m, f_final + p0, iters + p0, status + p0, st);
    TB_CUDA(cudaStreamSynchronize(st));
    tb_tiled_destroy(h);
    if (rc != TB_OK) return rc;
  }
  return TB_OK;
}

int tb_solve(tb_ctx* c, int32_t solver, const tb_solver_config* cfg, const void* pixels, const double* lam,
             const uint64_t* seeds, int64_t P, void* x, double* f_final, double* hist, int64_t hist_stride,
             int32_t* iters, int32_t* status, void* stream) {
  int rc = check_solve_args(c, solver, cfg, seeds, P, hist, hist_stride);
  if (rc != TB_OK) return rc;
  if (P == 0) return TB_OK;
  if (!pixels || !lam || !x || !f_final || !iters || !status) return fail(TB_ERR_INVALID, "null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  TB_CUDA(cudaSetDevice(c->device));
  const int total = cfg->fixed_iters > 0 ? cfg->fixed_iters : cfg->max_iters;
  rc = ensure_mk(c, total, st);
  if (rc != TB_OK) return rc;
  if (!warp_path_fits(c, solver))
    return solve_tiled(c, solver, cfg, pixels, lam, seeds, P, x, f_final, hist, hist_stride, iters, status, st);
  tb::SolveParams S{};
  if (!c->AT) {
    // column-major copy for the kernels that read the dictionary through L1 (cfg3): their sparse
    // forward product reads whole columns, contiguous here, one 128-byte line per 16 rows instead
    // of one line per row
    TB_CUDA(cudaMalloc((void**)&c->AT, sizeof(float2) * c->n * c->m));
    TB_CUDA(tb::launch_transpose(c->A, (int)c->n, (int)c->m, c->AT, st));
  }
  S.A = c->A;
  S.AT = c->AT;
  S.n = (int)c->n;
  S.m = (int)c->m;
  S.ms = (int)(c->m | 1);
  S.mode = solver;
  S.max_width = solver == TB_SOLVER_RBPG ? c->max_block_width : (int)c->m;
  S.num_blocks = solver == TB_SOLVER_RBPG ? c->num_blocks : 1;
  S.blk_start = c->blk_start;
  S.blk_lip = c->blk_lip;
  S.cdf = c->cdf;
  S.lip_full = c->lip_full;
  S.total_iters = total;
  S.fixed = cfg->fixed_iters > 0;
  S.cap = cfg->backtrack_cap;
  S.tol = cfg->tol;
  S.c_alpha = cfg->c_alpha;
  S.alpha_scale = cfg->alpha_init_scale;
  S.B = (const float2*)pixels;
  S.lam = lam;
  S.seeds = seeds;
  S.num_pixels = P;
  S.X = (float2*)x;
  S.f_final = f_final;
  S.hist = hist;
  S.hist_stride = hist_stride;
  S.iters = iters;
  S.status = status;
  S.queue = c->queue;
  S.mk = c->mk;
  // ISTA/FISTA: from one full wave of resident pixel slots the tensor-memory kernel (k_fista_tile.cu:
  // 16 resident warps instead of 9 on cfg2, +24-32% on cfg2/cfg3); smaller batches are latency bound
  // and run the unrolled warp kernel.  TB_FISTA_KERNEL=warp|solo|team overrides (A/B, identity tests).
  const char* fk = getenv("TB_FISTA_KERNEL");
  bool tile_asmem = false;
  int tile_slots = 0;
  const bool tile_fits = solver != TB_SOLVER_RBPG && tb::fista_tile_fits((int)c->n, (int)c->m, &tile_asmem, &tile_slots);
  const bool team = fk && strcmp(fk, "team") == 0;
  const bool tile = tile_fits && (fk ? (team || strcmp(fk, "solo") == 0) : P >= (int64_t)c->num_sms * tile_slots);
  if (solver == TB_SOLVER_RBPG && TB_WS_DCACHE) {
    const size_t need = (size_t)c->num_sms * 32 * (size_t)c->m;  // >= resident warp slots x m
    if (c->dglob_elems < need) {
      TB_CUDA(cudaStreamSynchronize(st));
      TB_CUDA(ctx_drain(c));
      cudaFree(c->dglob);
      c->dglob = nullptr;
      c->dglob_elems = 0;
      TB_CUDA(cudaMalloc((void**)&c->dglob, sizeof(double2) * need));
      c->dglob_elems = need;
    }
    S.dglob = c->dglob;
  }
  TB_CUDA(ctx_acquire(c, st));
  TB_CUDA(cudaMemsetAsync(c->queue, 0, sizeof(unsigned long long), st));
  int warps = 0;
  g_last_kernel.store(tile ? (team ? "fista_tile_kernel<team>" : "fista_tile_kernel<solo>") : "warp_solver_kernel", std::memory_order_relaxed);
  if (tile)
    TB_CUDA(tb::launch_fista_tile(S, c->num_sms, st, &warps, team));
  else
    TB_CUDA(tb::launch_warp_solver(S, c->num_sms, st, &warps));
  TB_CUDA(ctx_release(c, st));
  return TB_OK;
}

int tb_apply_filter(tb_ctx* c, const void* filter_dev, const void* pixels_dev, int64_t P, void* x_dev, void* stream) {
  if (!c || (P > 0 && (!filter_dev || !pixels_dev || !x_dev))) return fail(TB_ERR_INVALID, "null argument");
  if (P < 0) return fail(TB_ERR_INVALID, "num_pixels must be >= 0");
  TB_CUDA(cudaSetDevice(c->device));
  TB_CUDA(tb::launch_apply_filter((const double2*)filter_dev, (int)c->n, (int)c->m, (const float2*)pixels_dev, P, (float2*)x_dev, c->num_sms, (cudaStream_t)stream));
  return TB_OK;
}

int tb_build_steering(int device, const double* xi_dev, const double* eta_dev, int64_t n, int32_t n_axes,
                      const double* elev_dev, int64_t n_elev, const double* motion_dev, const int32_t* motion_sizes_host,
                      int64_t col0, int64_t ncols, double sign, void* out_dev, void* stream) {
  if (!xi_dev || !elev_dev || !out_dev || n < 1 || n_elev < 1 || ncols < 0) return fail(TB_ERR_INVALID, "invalid steering arguments");
  if (n_axes < 0 || n_axes > 2 || (n_axes > 0 && (!eta_dev || !motion_dev || !motion_sizes_host)))
    return fail(TB_ERR_INVALID, "1 elevation + at most 2 motion axes supported");
  if (!(sign == 1.0 || sign == -1.0)) return fail(TB_ERR_INVALID, "sign must be +1 or -1");
  const int ms0 = n_axes >= 1 ? motion_sizes_host[0] : 1, ms1 = n_axes >= 2 ? motion_sizes_host[1] : 1;
  const long long m = n_elev * (long long)ms0 * ms1;
  if (col0 < 0 || col0 + ncols > m) return fail(TB_ERR_INVALID, "column range [%lld, %lld) outside grid of %lld", (long long)col0, (long long)(col0 + ncols), m);
  TB_CUDA(cudaSetDevice(device));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  TB_CUDA(tb::launch_steering(xi_dev, eta_dev, (int)n, n_axes, elev_dev, motion_dev, ms0, ms1, col0, ncols, sign, (float2*)out_dev, sms, (cudaStream_t)stream));
  return TB_OK;
}

int tb_select(tb_ctx* c, const void* x, const void* pixels, int64_t P, int32_t n_elev, int32_t n_axes,
              const int32_t* msizes, const double* elev, const double* motion, int32_t k_max, int32_t ppsc,
              int32_t* order, int64_t* support, void* amps, double* elevs, double* motion_out, double* scores,
              int32_t* n_scores, int32_t* err, void* stream) {
  if (!c) return fail(TB_ERR_INVALID, "null context");
  if (k_max < 1) return fail(TB_ERR_INVALID, "k_max must be >= 1, got %d", k_max);
  if (k_max > 8) return fail(TB_ERR_INVALID, "k_max %d exceeds the supported 8", k_max);
  if (n_axes < 0 || n_axes > 2) return fail(TB_ERR_INVALID, "1 elevation + at most 2 motion axes supported");
  long long inner = 1;
  for (int a = 0; a < n_axes; ++a) inner *= msizes[a];
  if ((long long)n_elev * inner != c->m) return fail(TB_ERR_INVALID, "grid size %lld != dictionary columns %lld", (long long)n_elev * inner, (long long)c->m);
  if (P == 0) return TB_OK;
  tb::SelectParams S{};
  S.A = c->A;
  S.n = (int)c->n;
  S.m = (int)c->m;
  S.X = (const float2*)x;
  S.B = (const float2*)pixels;
  S.num_pixels = P;
  S.n_elev = n_elev;
  S.inner = (int)inner;
  S.n_axes = n_axes;
  S.msize0 = n_axes >= 1 ? msizes[0] : 1;
  S.msize1 = n_axes >= 2 ? msizes[1] : 1;
  S.elev = elev;
  S.motion = motion;
  S.k_max = k_max;
  S.ppsc = ppsc;
  S.order = order;
  S.support = (long long*)support;
  S.amps = (double2*)amps;
  S.elevs = elevs;
  S.motion_out = motion_out;
  S.scores = scores;
  S.n_scores = n_scores;
  S.err = err;
  TB_CUDA(cudaSetDevice(c->device));
  TB_CUDA(tb::launch_select(S, c->num_sms, (cudaStream_t)stream));
  return TB_OK;
}

}  // extern "C"
