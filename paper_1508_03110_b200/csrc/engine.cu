// engine.cu -- context, device-resident ratings, work plans, sharding.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "engine.h"

namespace ab2 {

// ------------------------------------------------------------------ Ctx --
Ctx::Ctx(int dev) : device(dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw Error(ALSNCG_ECUDA, "no CUDA device visible (the product path has no CPU fallback)");
  if (dev < 0 || dev >= n) throw Error(ALSNCG_EINVAL, "device index out of range");
  AB2_CUDA(cudaSetDevice(dev));
  AB2_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
  AB2_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  AB2_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  AB2_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  AB2_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  AB2_CUDA(cudaMalloc(&d_red, sizeof(double) * 2 * 8 * 4 * 148));
  AB2_CUDA(cudaMalloc(&d_counters, sizeof(unsigned) * 64));
  AB2_CUDA(cudaMemset(d_counters, 0, sizeof(unsigned) * 64));
  AB2_CUDA(cudaMalloc(&d_scalars, sizeof(double) * 64));
  AB2_CUDA(cudaMemset(d_scalars, 0, sizeof(double) * 64));
  AB2_CUDA(cudaMallocHost(&h_scalars, sizeof(double) * 64));
  cudaMemPool_t pool;
  AB2_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = UINT64_MAX;
  AB2_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
}

void* Ctx::alloc(size_t bytes) {
  void* p = nullptr;
  AB2_CUDA(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), stream));
  return p;
}

void Ctx::release(void* p) {
  if (p) cudaFreeAsync(p, stream);
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (auto& p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  for (void* p : scratch_ptr)
    if (p) cudaFree(p);
  cudaFree(d_red);
  cudaFree(d_counters);
  cudaFree(d_scalars);
  cudaFreeHost(h_scalars);
  if (comm) nccl().CommDestroy(comm);
  if (side) {
    cudaStreamSynchronize(side);
    cudaStreamDestroy(side);
  }
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (stream) cudaStreamDestroy(stream);
}

void* Ctx::scratch(int slot, size_t bytes) {
  if (slot >= static_cast<int>(scratch_ptr.size())) {
    scratch_ptr.resize(slot + 1, nullptr);
    scratch_size.resize(slot + 1, 0);
  }
  if (scratch_size[slot] < bytes) {
    if (scratch_ptr[slot]) {
      AB2_CUDA(cudaStreamSynchronize(stream));
      AB2_CUDA(cudaFree(scratch_ptr[slot]));
      scratch_ptr[slot] = nullptr;
    }
    const size_t want = std::max(bytes, scratch_size[slot] + scratch_size[slot] / 2);
    AB2_CUDA(cudaMalloc(&scratch_ptr[slot], want));
    scratch_size[slot] = want;
  }
  return scratch_ptr[slot];
}

int Ctx::begin_launch(const char* name) {
  ++launches;
  launch_name = name;
  if (!profiling) return -1;
  int k = 0;
  for (; k < static_cast<int>(stats.size()); ++k)
    if (stats[k].name == name) break;
  if (k == static_cast<int>(stats.size())) stats.push_back({name, 0, 0.0});
  Pending p;
  p.stat = k;
  auto take = [&]() {
    cudaEvent_t e;
    if (!event_pool.empty()) {
      e = event_pool.back();
      event_pool.pop_back();
    } else {
      AB2_CUDA(cudaEventCreate(&e));
    }
    return e;
  };
  p.a = take();
  p.b = take();
  AB2_CUDA(cudaEventRecord(p.a, stream));
  pending.push_back(p);
  return static_cast<int>(pending.size()) - 1;
}

void Ctx::end_launch(int token) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(ALSNCG_ECUDA, std::string("kernel launch (") + (launch_name ? launch_name : "?") +
                                  "): " + cudaGetErrorString(e));
  if (token >= 0) AB2_CUDA(cudaEventRecord(pending[token].b, stream));
}

void Ctx::collect_stats() {
  AB2_CUDA(cudaStreamSynchronize(stream));
  for (auto& p : pending) {
    float ms = 0.f;
    AB2_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    stats[p.stat].launches += 1;
    stats[p.stat].ms += ms;
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}

void Ctx::sync() { AB2_CUDA(cudaStreamSynchronize(stream)); }

unsigned Ctx::counter_total(int slot) {
  unsigned* d = d_counters + slot;
  if (world > 1) {
    allreduce_sum_u32(this, d, d_counters + 24, 1);
    d = d_counters + 24;
  }
  unsigned h = 0;
  AB2_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, stream));
  sync();
  return h;
}

int Ctx::prepare_kernel(const void* fn, int smem_limit, int threads, size_t smem) {
  auto it = kernel_attr.find(fn);
  if (it != kernel_attr.end()) return it->second;
  AB2_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_limit));
  int per_sm = 0;
  if (threads > 0) AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  per_sm = std::max(per_sm, 1);
  kernel_attr.emplace(fn, per_sm);
  return per_sm;
}

void Ctx::fetch_scalars(int n) {
  AB2_CUDA(cudaMemcpyAsync(h_scalars, d_scalars, sizeof(double) * n, cudaMemcpyDeviceToHost, stream));
  AB2_CUDA(cudaStreamSynchronize(stream));
}

L2Window::L2Window(Ctx* c, const void* base, size_t bytes) : ctx(c) {
  // per-context (= per-device) limits, queried once per context
  if (c->l2_max_persist < 0) {
    int mp = 0, mw = 0;
    if (cudaDeviceGetAttribute(&mp, cudaDevAttrMaxPersistingL2CacheSize, c->device) != cudaSuccess) mp = 0;
    if (cudaDeviceGetAttribute(&mw, cudaDevAttrMaxAccessPolicyWindowSize, c->device) != cudaSuccess) mw = 0;
    if (mp > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(mp));
    cudaGetLastError();
    c->l2_max_window = mw;
    c->l2_max_persist = mp;
  }
  const int max_persist = c->l2_max_persist, max_window = c->l2_max_window;
  if (max_persist <= 0 || max_window <= 0 || bytes == 0) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c->stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
    return;  // stream attributes and the persisting-L2 reset are not graph operations
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  v.accessPolicyWindow.num_bytes = std::min(bytes, static_cast<size_t>(max_window));
  v.accessPolicyWindow.hitRatio =
      std::min(1.0f, static_cast<float>(max_persist) / static_cast<float>(v.accessPolicyWindow.num_bytes));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  set = cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
  cudaGetLastError();
}

L2Window::~L2Window() {
  if (!set) return;
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaCtxResetPersistingL2Cache();
  cudaGetLastError();
}

// ------------------------------------------------------------ sharding --
std::vector<int> partition_rows(int n_rows, const int64_t* ptr, int world, int align) {
  std::vector<int> b(world + 1, 0);
  b[world] = n_rows;
  const int64_t total = ptr[n_rows];
  for (int r = 1; r < world; ++r) {
    const int64_t target = total * r / world;
    int row = static_cast<int>(std::lower_bound(ptr, ptr + n_rows + 1, target) - ptr);
    row = std::min(n_rows, ((row + align / 2) / align) * align);
    b[r] = std::max(b[r - 1], row);
  }
  return b;
}

LoopGroup::LoopGroup(int w) : world(w), ranks(w, nullptr), slot(w, nullptr) {}

void LoopGroup::barrier() {
  std::unique_lock<std::mutex> lk(m_);
  const unsigned g = gen_;
  if (++arrived_ == world) {
    arrived_ = 0;
    ++gen_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return gen_ != g; });
  }
}

namespace {
// Loopback collective skeleton: publish this rank's buffer, drain every
// stream, run `body` (reads peers' published buffers), drain, release.
template <typename F>
void loop_collective(Ctx* ctx, void* buf, F&& body) {
  LoopGroup& G = *ctx->loop;
  G.slot[ctx->rank] = buf;
  ctx->sync();
  G.barrier();
  body(G);
  ctx->sync();
  G.barrier();
}

template <typename T>
void loop_allreduce(Ctx* ctx, const T* send, T* recv, int n) {
  loop_collective(ctx, const_cast<T*>(send), [&](LoopGroup& G) {
    std::vector<T> acc(n, 0), h(n);
    for (int r = 0; r < G.world; ++r) {  // rank order
      AB2_CUDA(cudaMemcpy(h.data(), G.slot[r], sizeof(T) * n, cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) acc[i] += h[i];
    }
    G.barrier();  // every rank has read every send buffer (send may alias recv)
    AB2_CUDA(cudaMemcpy(recv, acc.data(), sizeof(T) * n, cudaMemcpyHostToDevice));
  });
}
}  // namespace

void allreduce_sum_u32(Ctx* ctx, const unsigned* send, unsigned* recv, int n) {
  if (ctx->loop) return loop_allreduce(ctx, send, recv, n);
  AB2_NCCL(nccl().AllReduce(send, recv, n, ncclUint32, ncclSum, ctx->comm, ctx->stream));
}

void allreduce_sum_u64(Ctx* ctx, const unsigned long long* send, unsigned long long* recv, int n) {
  if (ctx->loop) return loop_allreduce(ctx, send, recv, n);
  AB2_NCCL(nccl().AllReduce(send, recv, n, ncclUint64, ncclSum, ctx->comm, ctx->stream));
}

void allgather_rows(Ctx* ctx, double* rows, const std::vector<int>& bounds, int ld) {
  if (ctx->world <= 1) return;
  if (ctx->loop) {  // every peer's rows [bounds[r], bounds[r+1]) into this rank's buffer
    loop_collective(ctx, rows, [&](LoopGroup& G) {
      for (int r = 0; r < G.world; ++r) {
        const size_t count = static_cast<size_t>(bounds[r + 1] - bounds[r]) * ld;
        if (r == ctx->rank || count == 0) continue;
        const size_t off = static_cast<size_t>(bounds[r]) * ld;
        AB2_CUDA(cudaMemcpyAsync(rows + off, static_cast<double*>(G.slot[r]) + off, sizeof(double) * count,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
      }
    });
    return;
  }
  AB2_NCCL(nccl().GroupStart());
  for (int r = 0; r < ctx->world; ++r) {
    const size_t count = static_cast<size_t>(bounds[r + 1] - bounds[r]) * ld;
    if (count == 0) continue;
    double* p = rows + static_cast<size_t>(bounds[r]) * ld;
    AB2_NCCL(nccl().Broadcast(p, p, count, ncclDouble, r, ctx->comm, ctx->stream));
  }
  AB2_NCCL(nccl().GroupEnd());
}

// -------------------------------------------------------------- upload --
namespace {

void upload_view(Ctx* ctx, View& v, int row0, int row1, const int64_t* ptr, const int* idx,
                 const double* val) {
  v.row0 = row0;
  v.nrows = row1 - row0;
  const int64_t base = ptr[row0];
  v.nnz = ptr[row1] - base;
  v.h_ptr.resize(v.nrows + 1);
  for (int r = 0; r <= v.nrows; ++r) v.h_ptr[r] = ptr[row0 + r] - base;
  v.ptr = static_cast<int64_t*>(ctx->alloc(sizeof(int64_t) * (v.nrows + 1)));
  v.idx = static_cast<int*>(ctx->alloc(sizeof(int) * std::max<int64_t>(v.nnz, 1)));
  v.val = static_cast<double*>(ctx->alloc(sizeof(double) * std::max<int64_t>(v.nnz, 1)));
  AB2_CUDA(cudaMemcpyAsync(v.ptr, v.h_ptr.data(), sizeof(int64_t) * (v.nrows + 1),
                           cudaMemcpyHostToDevice, ctx->stream));
  if (v.nnz > 0) {
    AB2_CUDA(cudaMemcpyAsync(v.idx, idx + base, sizeof(int) * v.nnz, cudaMemcpyHostToDevice, ctx->stream));
    AB2_CUDA(cudaMemcpyAsync(v.val, val + base, sizeof(double) * v.nnz, cudaMemcpyHostToDevice, ctx->stream));
  }
}

void free_view(Ctx* ctx, View& v) {
  ctx->release(v.ptr);
  ctx->release(v.idx);
  ctx->release(v.val);
  v.ptr = nullptr;
  v.idx = nullptr;
  v.val = nullptr;
}

}  // namespace

DevRatings* upload_ratings(Ctx* ctx, int n_u, int n_m, int64_t nnz, const int64_t* uptr,
                           const int* uidx, const double* uval, const int64_t* iptr,
                           const int* iidx, const double* ival) {
  if (n_u < 0 || n_m < 0 || nnz < 0) throw Error(ALSNCG_EINVAL, "negative ratings dimensions");
  if (uptr[0] != 0 || uptr[n_u] != nnz || iptr[0] != 0 || iptr[n_m] != nnz)
    throw Error(ALSNCG_EDATA, "CSR/CSC pointers do not span nnz");
  AB2_CUDA(cudaSetDevice(ctx->device));
  auto R = std::make_unique<DevRatings>();
  R->ctx = ctx;
  R->n_u = n_u;
  R->n_m = n_m;
  R->nnz = nnz;
  R->ub = partition_rows(n_u, uptr, ctx->world, kTileRows);
  R->mb = partition_rows(n_m, iptr, ctx->world, kTileRows);
  upload_view(ctx, R->users, R->ub[ctx->rank], R->ub[ctx->rank + 1], uptr, uidx, uval);
  upload_view(ctx, R->items, R->mb[ctx->rank], R->mb[ctx->rank + 1], iptr, iidx, ival);
  ctx->sync();
  return R.release();
}

DevRatings::~DevRatings() {
  if (ctx) cudaSetDevice(ctx->device);
  free_view(ctx, users);
  free_view(ctx, items);
  for (auto& m : plans)
    for (auto& kv : m) ctx->release(kv.second->block);
  for (auto& m : hs_plans)
    for (auto& kv : m) ctx->release(kv.second->block);
}

const SegPlan& DevRatings::plan(int kind, int S) {
  auto& m = plans[kind];
  auto it = m.find(S);
  if (it != m.end()) return *it->second;
  const View& v = view(kind);
  auto P = std::make_unique<SegPlan>();
  P->S = S;
  std::vector<int> row, len, slot;
  std::vector<int64_t> beg;
  std::vector<int> mrow, mslot0, mnslot;
  // heavy rows first (their segments), then single-segment rows by
  // descending count: big work items are scheduled first.
  std::vector<int> singles;
  int n_slots = 0;
  for (int r = 0; r < v.nrows; ++r) {
    const int64_t c = v.h_ptr[r + 1] - v.h_ptr[r];
    if (c > S) {
      const int ns = static_cast<int>((c + S - 1) / S);
      mrow.push_back(r);
      mslot0.push_back(n_slots);
      mnslot.push_back(ns);
      for (int s = 0; s < ns; ++s) {
        row.push_back(r);
        beg.push_back(v.h_ptr[r] + static_cast<int64_t>(s) * S);
        len.push_back(static_cast<int>(std::min<int64_t>(S, c - static_cast<int64_t>(s) * S)));
        slot.push_back(n_slots + s);
      }
      n_slots += ns;
    } else {
      singles.push_back(r);
    }
  }
  // descending count, stable (counting sort: counts of single-segment rows are <= S)
  {
    std::vector<int> bucket(static_cast<size_t>(S) + 2, 0);
    for (int r : singles) ++bucket[S - (v.h_ptr[r + 1] - v.h_ptr[r])];
    int run = 0;
    for (int& b : bucket) {
      const int c = b;
      b = run;
      run += c;
    }
    std::vector<int> sorted(singles.size());
    for (int r : singles) sorted[bucket[S - (v.h_ptr[r + 1] - v.h_ptr[r])]++] = r;
    singles.swap(sorted);
  }
  for (int r : singles) {
    row.push_back(r);
    beg.push_back(v.h_ptr[r]);
    len.push_back(static_cast<int>(v.h_ptr[r + 1] - v.h_ptr[r]));
    slot.push_back(-1);
  }
  P->n_seg = static_cast<int>(row.size());
  P->n_multi = static_cast<int>(mrow.size());
  P->n_slots = n_slots;
  const size_t ns = std::max<size_t>(row.size(), 1), nm = std::max<size_t>(mrow.size(), 1);
  const size_t bytes = ns * (8 + 4 + 4 + 4) + nm * 12 + 64;
  // stream-ordered pool memory: no device-wide synchronisation on alloc / free
  char* blk = static_cast<char*>(ctx->alloc(bytes));
  P->block = blk;
  P->seg_beg = reinterpret_cast<int64_t*>(blk);
  P->seg_row = reinterpret_cast<int*>(blk + ns * 8);
  P->seg_len = P->seg_row + ns;
  P->seg_slot = P->seg_len + ns;
  P->m_row = P->seg_slot + ns;
  P->m_slot0 = P->m_row + nm;
  P->m_nslot = P->m_slot0 + nm;
  // stream-ordered with the kernels that read the plan (ctx->stream is a
  // non-blocking stream, so a legacy-stream cudaMemcpy would not order them)
  auto up = [&](void* d, const void* h, size_t n) {
    if (n) AB2_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, ctx->stream));
  };
  up(P->seg_beg, beg.data(), beg.size() * 8);
  up(P->seg_row, row.data(), row.size() * 4);
  up(P->seg_len, len.data(), len.size() * 4);
  up(P->seg_slot, slot.data(), slot.size() * 4);
  up(P->m_row, mrow.data(), mrow.size() * 4);
  up(P->m_slot0, mslot0.data(), mslot0.size() * 4);
  up(P->m_nslot, mnslot.data(), mnslot.size() * 4);
  ctx->sync();  // the host vectors go out of scope
  const SegPlan& ref = *P;
  m.emplace(S, std::move(P));
  return ref;
}

const HsPlan& DevRatings::hs_plan(int kind, int S, int64_t max_slots) {
  auto key = std::make_pair(S, max_slots);
  auto& m = hs_plans[kind];
  auto it = m.find(key);
  if (it != m.end()) return *it->second;
  const View& v = view(kind);
  auto P = std::make_unique<HsPlan>();
  P->S = S;
  std::vector<int> row_slot0(std::max(v.nrows, 1), 0), row_nslot(std::max(v.nrows, 1), 0);
  std::vector<int> srow, slen, sslot, multi;
  std::vector<int64_t> sbeg;
  int r = 0;
  while (r < v.nrows) {
    HsBatch b;
    b.row0 = r;
    b.multi0 = static_cast<int>(multi.size());
    b.seg0 = static_cast<int>(srow.size());
    int slots = 0;
    std::vector<int> order;  // segment ids of this batch
    const size_t first = srow.size();
    while (r < v.nrows) {
      const int64_t c = v.h_ptr[r + 1] - v.h_ptr[r];
      const int ns = c == 0 ? 0 : static_cast<int>((c + S - 1) / S);
      if (slots > 0 && slots + ns > max_slots) break;
      row_slot0[r] = slots;
      row_nslot[r] = ns;
      if (ns > 1) multi.push_back(r);
      for (int s2 = 0; s2 < ns; ++s2) {
        srow.push_back(r);
        sbeg.push_back(v.h_ptr[r] + static_cast<int64_t>(s2) * S);
        slen.push_back(static_cast<int>(std::min<int64_t>(S, c - static_cast<int64_t>(s2) * S)));
        sslot.push_back(slots + s2);
      }
      slots += ns;
      ++r;
    }
    // heavy-first order inside the batch (load balance of the Gram kernel)
    // descending length, stable (counting sort: lengths are <= S)
    std::vector<int> perm(srow.size() - first);
    {
      std::vector<int> bucket(static_cast<size_t>(S) + 2, 0);
      for (size_t id = first; id < srow.size(); ++id) ++bucket[S - slen[id]];
      int run = 0;
      for (int& bb : bucket) {
        const int c = bb;
        bb = run;
        run += c;
      }
      for (size_t id = first; id < srow.size(); ++id) perm[bucket[S - slen[id]]++] = static_cast<int>(id);
    }
    std::vector<int> r2, l2, s2v;
    std::vector<int64_t> b2v;
    for (int id : perm) {
      r2.push_back(srow[id]);
      l2.push_back(slen[id]);
      s2v.push_back(sslot[id]);
      b2v.push_back(sbeg[id]);
    }
    std::copy(r2.begin(), r2.end(), srow.begin() + first);
    std::copy(l2.begin(), l2.end(), slen.begin() + first);
    std::copy(s2v.begin(), s2v.end(), sslot.begin() + first);
    std::copy(b2v.begin(), b2v.end(), sbeg.begin() + first);
    b.row1 = r;
    b.multi1 = static_cast<int>(multi.size());
    b.seg1 = static_cast<int>(srow.size());
    b.nslots = slots;
    P->max_batch_slots = std::max(P->max_batch_slots, slots);
    P->batches.push_back(b);
  }
  const size_t ns = std::max<size_t>(srow.size(), 1), nr = std::max<size_t>(v.nrows, 1);
  const size_t nm = std::max<size_t>(multi.size(), 1);
  char* blk = static_cast<char*>(ctx->alloc(ns * (8 + 4 + 4 + 4) + nr * 8 + nm * 4 + 64));
  P->block = blk;
  P->seg_beg = reinterpret_cast<int64_t*>(blk);
  P->seg_row = reinterpret_cast<int*>(blk + ns * 8);
  P->seg_len = P->seg_row + ns;
  P->seg_slot = P->seg_len + ns;
  P->row_slot0 = P->seg_slot + ns;
  P->row_nslot = P->row_slot0 + nr;
  P->multi_rows = P->row_nslot + nr;
  // stream-ordered with the kernels that read the plan (ctx->stream is a
  // non-blocking stream, so a legacy-stream cudaMemcpy would not order them)
  auto up = [&](void* d, const void* h, size_t n) {
    if (n) AB2_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, ctx->stream));
  };
  up(P->seg_beg, sbeg.data(), sbeg.size() * 8);
  up(P->seg_row, srow.data(), srow.size() * 4);
  up(P->seg_len, slen.data(), slen.size() * 4);
  up(P->seg_slot, sslot.data(), sslot.size() * 4);
  up(P->row_slot0, row_slot0.data(), static_cast<size_t>(v.nrows) * 4);
  up(P->row_nslot, row_nslot.data(), static_cast<size_t>(v.nrows) * 4);
  up(P->multi_rows, multi.data(), multi.size() * 4);
  ctx->sync();  // the host vectors go out of scope
  const HsPlan& ref = *P;
  m.emplace(key, std::move(P));
  return ref;
}

std::pair<int64_t, int64_t> DevRatings::routing_totals(int n_blocks) {
  auto it = routing.find(n_blocks);
  if (it != routing.end()) return it->second;
  unsigned long long* d = static_cast<unsigned long long*>(ctx->scratch(5, 16));
  launch_routing_count(*this, n_blocks, d);
  if (ctx->world > 1) allreduce_sum_u64(ctx, d, d, 2);
  unsigned long long h[2];
  AB2_CUDA(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  auto v = std::make_pair(static_cast<int64_t>(h[0]), static_cast<int64_t>(h[1]));
  routing[n_blocks] = v;
  return v;
}

}  // namespace ab2
