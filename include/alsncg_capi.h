/*
 * alsncg_capi.h -- the C-ABI drop-in boundary of the B200 ALS-NCG core.
 *
 * Plain C, plain pointers and sizes, no torch/CUDA types.  Everything the
 * reference's C++ solver API (/root/reference/proj/include/alsncg/) does on
 * the hot path is reachable here; include/alsncg/ (the .hpp headers) re-declares that C++
 * API on top of this ABI (see INTEGRATION.md for the ctypes / C++ bindings).
 *
 * Conventions
 *  - Every entry point returns an int status (ALSNCG_OK == 0); on failure
 *    alsncg_last_error() returns a thread-local message.  The C++ shim maps
 *    ALSNCG_EINVAL -> std::invalid_argument, ALSNCG_EDATA -> DataError,
 *    ALSNCG_EDUP -> DuplicateRatingError, everything else -> std::runtime_error,
 *    mirroring the reference's exception types.
 *  - "Flat vectors" on host buffers use the reference layout (factors.hpp:49-79):
 *    n_f*n_u user values (user i at [i*n_f, (i+1)*n_f)) followed by n_f*n_m
 *    item values.  Device buffers (alsncg_dev_*) use the padded row layout
 *    described at alsncg_row_stride().
 *  - Calls on one context are synchronous w.r.t. the host unless named
 *    *_async; one host thread per context.
 */
#ifndef ALSNCG_CAPI_H
#define ALSNCG_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ALSNCG_OK = 0,
  ALSNCG_EINVAL = 1,       /* shape / config error  (std::invalid_argument) */
  ALSNCG_EDATA = 2,        /* malformed ratings     (alsncg::DataError)     */
  ALSNCG_EDUP = 3,         /* duplicate rating      (DuplicateRatingError)  */
  ALSNCG_ECUDA = 4,        /* CUDA runtime error / no device                */
  ALSNCG_ENCCL = 5,        /* NCCL error                                    */
  ALSNCG_ENOMEM = 6,       /* device allocation failed                      */
  ALSNCG_EUNSUPPORTED = 7, /* n_f beyond the compiled kernel range          */
  ALSNCG_ELOGIC = 8        /* trace ordering (std::logic_error)             */
};

typedef struct alsncg_ctx alsncg_ctx;
typedef struct alsncg_ratings alsncg_ratings;
typedef struct alsncg_solver alsncg_solver;

/* SolverConfig (config.hpp:29-50) + NcgOverrides (ncg.hpp:52-55). */
typedef struct {
  double lambda;
  int n_f;
  int max_iters;
  double tol;
  uint64_t seed;
  double alpha0;
  double armijo_c;
  double tau;
  int max_backtracks;
  int n_blocks;
  int n_workers;
  int trace_every;
  int snapshot_every;
  int paper_timing;
  int has_fixed_alpha;
  double fixed_alpha;
  int force_beta_zero;
} alsncg_config;

/* TraceRecord (config.hpp:52-60). */
typedef struct {
  int iter;
  double loss;
  double grad_norm;
  double elapsed_seconds;
  int backtracks;
  int64_t shuffled_columns;
  int restarted;
} alsncg_trace_record;

/* SolveResult counters (config.hpp:88-98). */
typedef struct {
  int converged;
  int iterations;
  double final_loss;
  double final_grad_norm;
  int restarts;
  int fallback_steps;
  int fallback_columns;
} alsncg_result;

/* SnapshotSink (config.hpp:84-86): called with host copies of the factors. */
typedef void (*alsncg_snapshot_fn)(int iter, int n_f, int n_u, int n_m, const double* user_data,
                                   const double* item_data, void* user);

const char* alsncg_last_error(void);
int alsncg_abi_version(void);
/* Padded device row stride for rank n_f: n_f rounded up to even, so each
 * user/item row starts 16-byte aligned; pad entries are kept at zero. */
int alsncg_row_stride(int n_f);
/* Largest n_f the compiled half-sweep kernels accept. */
int alsncg_max_rank(void);

/* ---------------- host-side data (no device needed) ---------------- */

/* RatingsMatrix::from_triples (ratings.cpp:28-89): validate, sort by
 * (user,item), reject duplicates, CSR + stable-count CSC.  Output arrays are
 * caller-allocated: uptr[n_u+1], iptr[n_m+1], uidx/uval/iidx/ival[nnz].
 * Bit-identical to the reference. */
int alsncg_csr_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
                     const double* values, int single_precision_storage, int64_t* uptr,
                     int* uidx, double* uval, int64_t* iptr, int* iidx, double* ival,
                     int* dup_user, int* dup_item);

/* random_init (factors.cpp:24-32): items first then users, U[0,1)/sqrt(n_f). */
int alsncg_random_init(int n_f, int n_u, int n_m, uint64_t seed, double* user, double* item);

/* Seeded BASELINE.json workload generator:
 * rank-10 truth, Zipf(1) items, >= min_per_user ratings per user, half-star
 * values.  Emits exactly nnz user-major triples. */
int alsncg_synth_generate(int n_u, int n_m, int64_t nnz, int min_per_user, uint64_t seed,
                          int* users, int* items, double* values);

/* backtracking_search (linesearch.cpp:115-131); returns the LineSearchStatus
 * (0 accepted, 1 not descent, 2 max backtracks) or -ALSNCG_EINVAL. */
int alsncg_backtracking_search(const double c[5], double slope, double alpha0, double armijo_c,
                               double tau, int max_backtracks, double* alpha, int* backtracks);

/* ---------------- device context ---------------- */

int alsncg_ctx_create(int device, alsncg_ctx** out);
/* Multi-GPU: one process per GPU; rank 0 calls alsncg_nccl_unique_id and the
 * 128 bytes are broadcast by the caller (torch.distributed / MPI / files). */
int alsncg_nccl_unique_id(unsigned char id[128]);
int alsncg_ctx_create_dist(int device, int rank, int world, const unsigned char id[128],
                           alsncg_ctx** out);
/* ranking::mean_ranking_accuracy (ranking.cpp:90-109): mean over users of the
 * top-t Kendall-tau accuracy of model_k's item ranking against the final
 * model's (FactorModel layout: n_f doubles per user / item column).  Scores
 * use the reference's exact arithmetic, so ties and orders are the
 * reference's; the per-user values are summed in user order on the host.
 * ALSNCG_EINVAL for t outside [1, n_m] or no users. */
int alsncg_mean_ranking_accuracy(alsncg_ctx* ctx, int n_f, int n_u, int n_m, const double* user_k,
                                 const double* item_k, const double* user_final, const double* item_final,
                                 int t, double* out);

/* Trace CSV of one run (harness.cpp:80-118: header
 * "iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns", %.17g doubles;
 * the restarted flag is not part of the file).  read returns the record count
 * in *n and fills min(*n, cap) records; ALSNCG_EDATA on unreadable / malformed
 * files, ALSNCG_ELOGIC on out-of-order iterations. */
int alsncg_write_trace_csv(const char* path, const alsncg_trace_record* recs, int n);
int alsncg_read_trace_csv(const char* path, alsncg_trace_record* recs, int cap, int* n);

/* Testing aid (no reference counterpart): an in-process stand-in for the NCCL
 * communicator.  `world` contexts on one or more devices of ONE process, each
 * driven by its own host thread, exchange factor shards and scalar partials
 * through device-to-device copies; every collective drains all ranks' streams
 * first, so the sharded code path runs end to end with its GPU work serialised
 * (used by the -m gpu tests to check world = 2 against world = 1 bitwise on a
 * single GPU). */
typedef struct alsncg_loopgroup alsncg_loopgroup;
int alsncg_loopgroup_create(int world, alsncg_loopgroup** out);
int alsncg_loopgroup_destroy(alsncg_loopgroup* group);
int alsncg_ctx_create_loopback(int device, int rank, alsncg_loopgroup* group, alsncg_ctx** out);
int alsncg_ctx_destroy(alsncg_ctx* ctx);
int alsncg_ctx_info(alsncg_ctx* ctx, int* device, int* rank, int* world);
/* The cudaStream_t (as void*) every kernel of this context is launched on. */
void* alsncg_ctx_stream(alsncg_ctx* ctx);
int alsncg_ctx_synchronize(alsncg_ctx* ctx);
/* Per-kernel CUDA-event timing (off by default). */
int alsncg_ctx_set_profiling(alsncg_ctx* ctx, int on);
int alsncg_ctx_reset_stats(alsncg_ctx* ctx);
/* Number of distinct kernel names recorded; name/launch count/total ms. */
int alsncg_ctx_stat_count(alsncg_ctx* ctx);
int alsncg_ctx_stat(alsncg_ctx* ctx, int k, const char** name, int64_t* launches, double* ms);
/* Launches of this library's kernels since the last reset (always counted). */
int64_t alsncg_ctx_launches(alsncg_ctx* ctx);

/* ---------------- device-resident ratings ---------------- */

/* Uploads the dual CSR/CSC store.  With a distributed context each rank
 * keeps only its nnz-balanced user and item row ranges. */
int alsncg_ratings_upload(alsncg_ctx* ctx, int n_u, int n_m, int64_t nnz, const int64_t* uptr,
                          const int* uidx, const double* uval, const int64_t* iptr,
                          const int* iidx, const double* ival, alsncg_ratings** out);
/* Downloads the CSR/CSC arrays back (full store; single-GPU contexts). */
int alsncg_ratings_download(alsncg_ratings* r, int64_t* uptr, int* uidx, double* uval,
                            int64_t* iptr, int* iidx, double* ival);
/* Local shard: users [u0,u1) and items [m0,m1) owned by this rank. */
int alsncg_ratings_shard(alsncg_ratings* r, int* u0, int* u1, int* m0, int* m1);
/* Host only (no device): the shard bounds every rank computes for a CSR/CSC
 * pointer array -- world+1 row bounds, nnz-balanced, interior bounds rounded
 * to multiples of `align` rows (the quartic/loss tile size, 64).  Replaces the
 * reference's block routing (parallel.cpp:57-142) for the row-sharded layout. */
int alsncg_partition_rows(int n_rows, const int64_t* ptr, int world, int align, int* bounds);
int alsncg_ratings_free(alsncg_ratings* r);

/* ---------------- hot-path kernels, HOST buffers (reference-facing) -------- */

/* ncg::loss (ncg.cpp:43-68). */
int alsncg_loss(alsncg_ratings* r, int n_f, const double* x, double lambda, double* out);
/* ncg::gradient (ncg.cpp:70-116). */
int alsncg_gradient(alsncg_ratings* r, int n_f, const double* x, double lambda, double* g);
/* linesearch::quartic_coefficients (linesearch.cpp:46-111). */
int alsncg_quartic(alsncg_ratings* r, int n_f, const double* x, const double* p, double lambda,
                   double c[5]);
/* One half-sweep (als.cpp:85-121 / parallel.cpp:144-185): kind 0 recomputes
 * the user columns from src = item factors (n_f*n_m), kind 1 the item columns
 * from src = user factors.  out has n_f*n_dest entries. */
int alsncg_half_sweep(alsncg_ratings* r, int kind, int n_f, const double* src, double lambda,
                      double* out, int* fallback_columns);
/* als_sweep = P(x) (als.cpp:123-128). */
int alsncg_als_sweep(alsncg_ratings* r, int n_f, const double* x, double lambda, double* out,
                     int* fallback_columns);

/* ---------------- hot-path kernels, DEVICE buffers ---------------- */
/* Device flat vectors: (n_u + n_m) rows of alsncg_row_stride(n_f) doubles,
 * user rows first; pad entries must be zero on input and stay zero. */
int alsncg_dev_loss(alsncg_ratings* r, int n_f, const double* d_x, double lambda, double* out);
int alsncg_dev_gradient(alsncg_ratings* r, int n_f, const double* d_x, double lambda,
                        double* d_g);
int alsncg_dev_quartic(alsncg_ratings* r, int n_f, const double* d_x, const double* d_p,
                       double lambda, double c[5]);
int alsncg_dev_half_sweep(alsncg_ratings* r, int kind, int n_f, const double* d_src,
                          double lambda, double* d_out, int* fallback_columns);
/* Fused vector ops over n doubles (ncg.cpp:118-136, factors.cpp:80-105). */
int alsncg_dev_dot(alsncg_ctx* ctx, int64_t n, const double* d_x, const double* d_y,
                   double* out);
/* Reference summation order (one device thread, index order, no FMA):
 * bit-identical to the reference's dot (factors.cpp:95-103) and beta_bar
 * (ncg.cpp:118-132).  Backs the API-level host-vector utilities. */
int alsncg_dev_dot_seq(alsncg_ctx* ctx, int64_t n, const double* d_x, const double* d_y,
                       double* out);
int alsncg_dev_beta_bar_seq(alsncg_ctx* ctx, int64_t n, const double* d_gn, const double* d_gp,
                            const double* d_bn, const double* d_bp, double* out);
int alsncg_dev_axpby(alsncg_ctx* ctx, int64_t n, double a, const double* d_x, double b,
                     const double* d_y, double* d_out);
int alsncg_dev_beta_bar(alsncg_ctx* ctx, int64_t n, const double* d_gn, const double* d_gp,
                        const double* d_bn, const double* d_bp, double* out);
/* Device memory helpers (so ctypes callers need no CUDA bindings). */
int alsncg_dev_malloc(alsncg_ctx* ctx, size_t bytes, void** ptr);
int alsncg_dev_free(alsncg_ctx* ctx, void* ptr);
int alsncg_memcpy_h2d(alsncg_ctx* ctx, void* dst, const void* src, size_t bytes);
int alsncg_memcpy_d2h(alsncg_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Packed host flat vector <-> padded device flat vector. */
int alsncg_flat_h2d(alsncg_ctx* ctx, int n_f, int n_u, int n_m, const double* host,
                    double* d_dev);
int alsncg_flat_d2h(alsncg_ctx* ctx, int n_f, int n_u, int n_m, const double* d_dev,
                    double* host);

/* ---------------- drivers ---------------- */

/* ncg::als_ncg_solve (ncg.cpp:138-307) on the device.  model_out (host,
 * n_f*(n_u+n_m), may be NULL) receives unflatten(x); trace receives up to
 * trace_cap records, *trace_len the total count. */
int alsncg_ncg_solve(alsncg_ratings* r, const alsncg_config* cfg, alsncg_snapshot_fn snap,
                     void* user, alsncg_result* res, double* model_out,
                     alsncg_trace_record* trace, int trace_cap, int* trace_len);
/* als::als_solve (als.cpp:130-195) on the device. */
int alsncg_als_solve(alsncg_ratings* r, const alsncg_config* cfg, alsncg_snapshot_fn snap,
                     void* user, alsncg_result* res, double* model_out,
                     alsncg_trace_record* trace, int trace_cap, int* trace_len);

/* Stepping interface over the same driver (benchmarks, custom stopping):
 * create = validate + setup through P(x0) (ncg.cpp:140-192); step runs up to
 * n outer iterations (stops early on convergence) and returns how many ran. */
int alsncg_solver_create(alsncg_ratings* r, const alsncg_config* cfg, alsncg_solver** out);
int alsncg_solver_step(alsncg_solver* s, int n, int* ran);
int alsncg_solver_state(alsncg_solver* s, int* iterations, int* converged, double* grad_norm,
                        int* restarts, int* fallback_steps, int* fallback_columns);
int alsncg_solver_trace(alsncg_solver* s, alsncg_trace_record* trace, int cap, int* len);
/* Host copy of the current iterate (packed flat layout). */
int alsncg_solver_model(alsncg_solver* s, double* model_out);
int alsncg_solver_destroy(alsncg_solver* s);

#ifdef __cplusplus
}
#endif
#endif /* ALSNCG_CAPI_H */
