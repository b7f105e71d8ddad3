// engine.h -- internal device engine of the B200 ALS-NCG core.
//
// Owns the CUDA context state (device, stream, optional NCCL communicator,
// scratch, per-kernel timing), the device-resident dual CSR/CSC store with
// its work plans, and declares the kernel launchers implemented in k_*.cu.
// Nothing here is part of the public ABI (include/alsncg_capi.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "alsncg_capi.h"
#include "nccl_shim.h"

namespace ab2 {

// ---------------------------------------------------------------- errors --
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AB2_CUDA(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::ab2::Error(e_ == cudaErrorMemoryAllocation ? ALSNCG_ENOMEM : ALSNCG_ECUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));           \
  } while (0)

#define AB2_NCCL(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw ::ab2::Error(ALSNCG_ENCCL,                                                   \
                         std::string(#expr) + ": " + ::ab2::nccl().GetErrorString(r_)); \
  } while (0)

inline int row_stride(int n_f) { return (n_f + 1) & ~1; }
// Number of 8-wide blocks of the augmented Gram [m ; r] (rhs at column ld).
inline int gram_blocks(int n_f) { return (row_stride(n_f) + 1 + 7) / 8; }
constexpr int kMaxGramBlocks = 26;  // n_f <= 206
constexpr int kMaxRank = 206;

// -------------------------------------------------------------- context --
struct Ctx;

// In-process stand-in for an NCCL communicator (tests only): `world` contexts
// in one process, each driven by its own host thread, exchange through
// device-to-device copies between their buffers.  Every collective is
// barrier -> every rank's stream drained -> barrier -> copies -> barrier, so
// no rank touches a buffer a peer still reads.  It exercises exactly the
// sharded code paths (partition_rows, per-shard kernels, ragged row
// exchange, rank-ordered tile sums) with the GPU work serialised.
struct LoopGroup {
  explicit LoopGroup(int w);
  int world;
  std::vector<Ctx*> ranks;  // registered by the contexts
  std::vector<void*> slot;  // per-rank buffer pointer of the current collective
  void barrier();
 private:
  std::mutex m_;
  std::condition_variable cv_;
  int arrived_ = 0;
  unsigned gen_ = 0;
};

struct KernelStat {
  std::string name;
  int64_t launches = 0;
  double ms = 0.0;
};

struct Ctx {
  int device = 0;
  int rank = 0;
  int world = 1;
  cudaStream_t stream = nullptr;
  // Side stream for work that is independent of the main chain (the NCG
  // gradient at x_{k+1} runs beside the two half-sweeps P(x_{k+1})).
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // Work to enqueue on `side` once the next half-sweep has launched its first
  // Gram kernel (it then overlaps that batch's latency-bound solve, not the
  // DMMA-bound Gram); the main stream joins before the following Gram.
  std::function<void()> side_work;
  bool side_join = false;
  ncclComm_t comm = nullptr;
  LoopGroup* loop = nullptr;  // in-process communicator (tests), instead of comm
  bool profiling = false;
  int64_t launches = 0;
  const char* launch_name = nullptr;  // last begin_launch (error messages)
  std::vector<KernelStat> stats;
  struct Pending {
    int stat;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  // Growable scratch slots (device), pinned host staging.
  std::vector<void*> scratch_ptr;
  std::vector<size_t> scratch_size;
  double* d_red = nullptr;      // reduction partials (block-level, double-double)
  unsigned* d_counters = nullptr;
  double* d_scalars = nullptr;  // small result slots
  double* h_scalars = nullptr;  // pinned mirror
  int sm_count = 148;
  // per-device caches (one Ctx per device): L2 persistence limits and the
  // set of kernels whose dynamic shared-memory limit was raised on this device
  int l2_max_persist = -1, l2_max_window = 0;
  std::map<const void*, int> kernel_attr;  // kernel -> occupancy (CTAs per SM) after the attribute was set
  // Raises `fn`'s dynamic shared-memory limit on this context's device once
  // and returns its occupancy (CTAs per SM) at `threads`/`smem` (>= 1).
  int prepare_kernel(const void* fn, int smem_limit, int threads, size_t smem);

  explicit Ctx(int dev);
  ~Ctx();
  void* scratch(int slot, size_t bytes);
  // Stream-ordered allocations from the device pool (its release threshold
  // is raised in the constructor, so per-solve / per-upload buffers are
  // recycled instead of going through cudaMalloc/cudaFree every call).
  void* alloc(size_t bytes);
  void release(void* p);
  // Kernel launch bookkeeping: call before/after each launch.
  int begin_launch(const char* name);
  void end_launch(int token);
  void collect_stats();  // syncs and folds pending events into stats
  void sync();
  void fetch_scalars(int n);  // d_scalars[0..n) -> h_scalars (synchronous)
  // d_counters[slot] summed over the ranks (NCCL all-reduce when world > 1;
  // uses counter slot 24 as the receive buffer), read back synchronously.
  unsigned counter_total(int slot);
};

// -------------------------------------------------------- device ratings --
// One compressed view (CSR by user or CSC by item) restricted to this rank's
// row range [row0, row0+nrows); ptr is rebased so ptr[0] == 0.
struct View {
  int row0 = 0;
  int nrows = 0;
  int64_t nnz = 0;
  int64_t* ptr = nullptr;  // device, nrows+1
  int* idx = nullptr;      // device, nnz
  double* val = nullptr;   // device, nnz
  std::vector<int64_t> h_ptr;  // host copy of ptr (plans are built on the host)
};

// Rows cut into segments of at most S ratings (heavy rows -> several
// segments whose partials are reduced in segment order: deterministic).
struct SegPlan {
  int S = 0;
  int n_seg = 0;
  int n_multi = 0;  // rows with >1 segment
  int n_slots = 0;  // segments belonging to multi rows
  int* seg_row = nullptr;   // local row
  int64_t* seg_beg = nullptr;
  int* seg_len = nullptr;
  int* seg_slot = nullptr;  // -1 for single-segment rows
  int* m_row = nullptr;
  int* m_slot0 = nullptr;
  int* m_nslot = nullptr;
  void* block = nullptr;  // single device allocation backing the arrays
};

constexpr int kTileRows = 64;  // quartic/loss tile height (rows per CTA)

// Half-sweep work plan for the split Gram / solve kernels: rows are grouped
// into batches whose partial-Gram slots fit a memory budget; within a batch
// every segment owns one slot, a row's slots are contiguous (row_slot0,
// row_nslot, local to the batch) and segments are ordered heavy-first.
struct HsBatch {
  int row0, row1;      // local rows [row0, row1)
  int seg0, seg1;      // segments of the batch
  int nslots;
  int multi0, multi1;  // rows with more than one partial slot: multi_rows[multi0, multi1)
};
struct HsPlan {
  int S = 0;
  std::vector<HsBatch> batches;
  int* seg_row = nullptr;
  int64_t* seg_beg = nullptr;
  int* seg_len = nullptr;
  int* seg_slot = nullptr;
  int* row_slot0 = nullptr;
  int* row_nslot = nullptr;
  int* multi_rows = nullptr;
  int max_batch_slots = 0;
  void* block = nullptr;
};

struct DevRatings {
  Ctx* ctx = nullptr;
  int n_u = 0, n_m = 0;
  int64_t nnz = 0;
  View users, items;
  // Shard bounds of every rank (identical on all ranks).
  std::vector<int> ub, mb;  // size world+1
  std::map<int, std::unique_ptr<SegPlan>> plans[2];
  std::map<std::pair<int, int64_t>, std::unique_ptr<HsPlan>> hs_plans[2];
  std::map<int, std::pair<int64_t, int64_t>> routing;  // n_blocks -> (T_u, T_m)
  ~DevRatings();
  const View& view(int kind) const { return kind == 0 ? users : items; }
  const SegPlan& plan(int kind, int S);
  const HsPlan& hs_plan(int kind, int S, int64_t max_slots);
  int n_rows(int kind) const { return kind == 0 ? n_u : n_m; }
  std::pair<int64_t, int64_t> routing_totals(int n_blocks);
};

DevRatings* upload_ratings(Ctx* ctx, int n_u, int n_m, int64_t nnz, const int64_t* uptr,
                           const int* uidx, const double* uval, const int64_t* iptr,
                           const int* iidx, const double* ival);
// nnz-balanced contiguous ranges aligned to `align` rows (identical on every rank).
std::vector<int> partition_rows(int n_rows, const int64_t* ptr, int world, int align);

// Scoped L2 access-policy window on ctx->stream: marks [base, base+bytes) as
// persisting (up to the device's persisting-L2 limit) and restores the
// stream's default policy on exit.
struct L2Window {
  Ctx* ctx;
  bool set = false;
  L2Window(Ctx* c, const void* base, size_t bytes);
  ~L2Window();
};

// ------------------------------------------------------------- kernels --
// All launchers enqueue on ctx->stream.  Device flat vectors: (n_u+n_m) rows
// of ld = row_stride(n_f) doubles, user rows first.

// Gradient rows of this rank's shard (both views) -> g (ncg.cpp:70-116).
void launch_gradient(DevRatings& R, int n_f, const double* x, double lambda, double* g);
// Tile partials of the quartic (linesearch.cpp:46-111) or of the loss
// (ncg.cpp:43-68) for this rank's tiles; result reduced in global tile order
// into ctx->d_scalars[slot..slot+5) (quartic) / [slot] (loss).
void launch_quartic(DevRatings& R, int n_f, const double* x, const double* p, double lambda,
                    int slot);
void launch_loss(DevRatings& R, int n_f, const double* x, double lambda, int slot);
// Half-sweep for this rank's rows of `kind` (0 users from item rows of src,
// 1 items from user rows of src); writes rows of `out` (same flat layout).
// Adds the number of least-norm fallback columns to d_counters[counter].
void launch_half_sweep(DevRatings& R, int kind, int n_f, const double* src_rows,
                       double lambda, double* out_rows, int counter);

// Deterministic compensated reductions over n doubles.  Results land in
// ctx->d_scalars[slot + k].
enum VecOp {
  kDot = 0,        // s0 = sum x*y
  kGbarFused = 1,  // out = x - px; s0 = sum out*(g - gprev); s1 = sum out*g;
                   // s2 = sum g*g; s3 = -sum g*out
  kDirFused = 2,   // out = -gbar + beta*p; s0 = sum g*out
  kBetaParts = 3,  // s0 = sum bn*(gn - gp); s1 = sum bp*gp
};
void launch_vec(Ctx* ctx, VecOp op, int64_t n, const double* a, const double* b,
                const double* c, const double* d, double beta, double* out, int slot);
// Reference-order sums (single thread): s0 = sum a*(b - c) (c may be null:
// sum a*b), s1 = sum d*c (d may be null) into d_scalars[slot], [slot+1].
void launch_seq_dots(Ctx* ctx, int64_t n, const double* a, const double* b, const double* c,
                     const double* d, int slot);
// out = a*x + b*y elementwise (no FMA: reference rounding, factors.cpp:88-91).
void launch_axpby(Ctx* ctx, int64_t n, double a, const double* x, double b, const double* y,
                  double* out);
// Routing-table totals (parallel.cpp:69-111) for this rank's rows.
void launch_routing_count(DevRatings& R, int n_blocks, unsigned long long* d_out2);
// Packed <-> padded row layout conversions.
void launch_pad_rows(Ctx* ctx, int64_t rows, int n_f, const double* packed, double* padded);
// x0 = flatten(random_init(seed)) straight into the padded flat vector x.
void launch_random_init(Ctx* ctx, int n_f, int n_u, int n_m, uint64_t seed, double* x);
void launch_unpad_rows(Ctx* ctx, int64_t rows, int n_f, const double* padded, double* packed);

// Multi-GPU: replicate row ranges [b[r], b[r+1]) of a row-major buffer from
// their owning rank to all ranks (grouped in-place broadcasts over NCCL).
void allgather_rows(Ctx* ctx, double* rows, const std::vector<int>& bounds, int ld);
// ranking::mean_ranking_accuracy (k_ranking.cu): per-user accuracies into
// d_q[n_u]; models in FactorModel layout (n_f doubles per user / item).
void launch_mean_ranking(Ctx* ctx, int n_f, int n_u, int n_m, const double* d_uk, const double* d_mk,
                         const double* d_uf, const double* d_mf, int t, double* d_q);
// In-place sum over the ranks of n unsigned 32/64-bit counters (NCCL
// all-reduce, or the loopback group).
void allreduce_sum_u32(Ctx* ctx, const unsigned* send, unsigned* recv, int n);
void allreduce_sum_u64(Ctx* ctx, const unsigned long long* send, unsigned long long* recv, int n);

}  // namespace ab2
