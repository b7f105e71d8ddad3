/*
 * alsncg_oracle.h -- CPU ORACLE for the ALS-NCG hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This is a plain-C restatement of the reference algorithm (arXiv 1508.03110
 * C++ reference under /root/reference/proj).  It exists only as the checker
 * for the CUDA product path: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * library (paper_1508_03110_b200/) never links or calls it.
 *
 * Arithmetic follows the reference operation for operation (FP64, no FMA,
 * sequential sums in source order), so on the functions whose reference
 * source compiles here (everything but als.cpp, which needs the absent
 * Eigen3) the port is pinned BITWISE against oracle/_ref (the reference
 * sources compiled in place, see oracle/Makefile) by tests/test_oracle.py.
 * The dense column solve restates Eigen's LLT as an unblocked Cholesky and
 * Eigen's CompleteOrthogonalDecomposition as a pseudo-inverse (Jacobi
 * eigensolver) least-norm solve; that part is pinned by the reference's
 * property tests only (see DESIGN.md "parity unpinned" note for Eigen).
 */
#ifndef ALSNCG_ORACLE_H
#define ALSNCG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Read-only view of the dual CSR/CSC store (ratings.hpp:98-104). */
typedef struct {
  int n_u, n_m;
  int64_t nnz;
  const int64_t* uptr; const int* uidx; const double* uval;
  const int64_t* iptr; const int* iidx; const double* ival;
} orc_ratings;

/* SolverConfig (config.hpp:29-50) + NcgOverrides (ncg.hpp:52-55). */
typedef struct {
  double lambda; int n_f; int max_iters; double tol; uint64_t seed;
  double alpha0, armijo_c, tau; int max_backtracks;
  int n_blocks, n_workers, trace_every, snapshot_every, paper_timing;
  int has_fixed_alpha; double fixed_alpha; int force_beta_zero;
} orc_config;

/* TraceRecord (config.hpp:52-60). */
typedef struct {
  int iter; double loss, grad_norm, elapsed_seconds; int backtracks;
  int64_t shuffled_columns; int restarted;
} orc_trace_rec;

/* SolveResult counters (config.hpp:88-98). */
typedef struct {
  int converged, iterations; double final_loss, final_grad_norm;
  int restarts, fallback_steps, fallback_columns;
} orc_result;

/* ---- rng.hpp / rng.cpp: mt19937_64 + derived draws ---- */
typedef struct { uint64_t mt[312]; int mti; int has_spare; double spare; } orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
uint64_t orc_rng_uniform_below(orc_rng* r, uint64_t n);
double orc_rng_normal(orc_rng* r);
int orc_sample_cumulative(const double* cum, int n, double u);

/* ---- ratings.cpp:28-89 from_triples.  Returns 0 ok, 1 out of range /
 * negative dims, 2 non-finite value, 3 duplicate (dup_user/dup_item set). */
int orc_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
              const double* values, int single_precision,
              int64_t* uptr, int* uidx, double* uval,
              int64_t* iptr, int* iidx, double* ival, int* dup_user, int* dup_item);

/* ---- BASELINE workload generator (restated recipe, no
 * reference counterpart).  Returns 0 ok, 1 bad dimensions / nnz. */
int orc_synth_generate(int n_u, int n_m, int64_t nnz, int min_per_user, uint64_t seed,
                       int* users, int* items, double* values);

/* ---- factors.cpp ---- */
void orc_random_init(int n_f, int n_u, int n_m, uint64_t seed, double* user, double* item);
/* FlatVector ops over (user part, item part) with nu = n_f*n_u, nm = n_f*n_m. */
void orc_axpby(int64_t nu, int64_t nm, double a, const double* xu, const double* xm,
               double b, const double* yu, const double* ym, double* ou, double* om);
double orc_dot(int64_t nu, int64_t nm, const double* xu, const double* xm,
               const double* yu, const double* ym);

/* ---- ncg.cpp ---- */
double orc_loss(const orc_ratings* r, int n_f, const double* xu, const double* xm, double lambda);
void orc_gradient(const orc_ratings* r, int n_f, const double* xu, const double* xm,
                  double lambda, int n_workers, double* gu, double* gm);
double orc_beta_bar(int64_t nu, int64_t nm, const double* gnu, const double* gnm,
                    const double* gpu, const double* gpm, const double* bnu,
                    const double* bnm, const double* bpu, const double* bpm);

/* ---- linesearch.cpp ---- */
void orc_quartic(const orc_ratings* r, int n_f, const double* xu, const double* xm,
                 const double* pu, const double* pm, double lambda, int n_chunks,
                 int n_workers, double c[5]);
/* status: 0 accepted, 1 not descent, 2 max backtracks (linesearch.hpp:36-40) */
int orc_backtracking(const double c[5], double slope, double alpha0, double cc, double tau,
                     int max_backtracks, double* alpha, int* backtracks);

/* ---- als.cpp (restated without Eigen) ---- */
void orc_solve_normal_column(const int* idx, const double* vals, int count,
                             const double* const* cols, int n_f, double lambda,
                             double* out, int* fallback_columns);
void orc_update_users(const orc_ratings* r, int n_f, const double* item_data,
                      double lambda, int n_workers, double* out, int* fallback_columns);
void orc_update_items(const orc_ratings* r, int n_f, const double* user_data,
                      double lambda, int n_workers, double* out, int* fallback_columns);

/* ---- parallel.cpp:69-111: routing-table column totals (T_u, T_m). */
void orc_routing_totals(const orc_ratings* r, int n_blocks, int64_t* tu_total, int64_t* tm_total);

/* ---- drivers: ncg.cpp:138-307, als.cpp:130-195.  model_u/model_m receive
 * the final factors; trace receives up to trace_cap records.  Returns 0, or
 * -1 on invalid config (config.cpp:21-34). */
int orc_ncg_solve(const orc_ratings* r, const orc_config* cfg, double* model_u,
                  double* model_m, orc_trace_rec* trace, int trace_cap, int* trace_len,
                  orc_result* res);
int orc_als_solve(const orc_ratings* r, const orc_config* cfg, double* model_u,
                  double* model_m, orc_trace_rec* trace, int trace_cap, int* trace_len,
                  orc_result* res);

#ifdef __cplusplus
}
#endif
#endif
