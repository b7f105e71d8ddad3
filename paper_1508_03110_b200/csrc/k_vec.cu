// k_vec.cu -- K8: fused NCG vector work (ncg.cpp:118-136, 186-275;
// factors.cpp:80-105) as single-pass kernels with deterministic compensated
// reductions, plus layout helpers and the routing-table counter.
//
// Elementwise results are bit-identical to the reference (each op is one
// IEEE multiply or add in the reference's order, no FMA); reductions are
// double-double per thread -> block -> last-block finalise in block order.
// Roofline: HBM-bound; algorithmic bytes = 8 B x (#streams read + written)
// per element (K8).
#include "common.cuh"

#include <cmath>

namespace ab2 {

namespace {

constexpr int kVecThreads = 256;
constexpr int kVecMaxBlocks = 4 * 148;

template <int OP>
struct VecNS {
  static constexpr int value = OP == kDot ? 1 : OP == kGbarFused ? 4 : OP == kDirFused ? 1 : 2;
};

template <int OP>
__device__ __forceinline__ void vec_elem(int64_t i, const double* __restrict__ a,
                                         const double* __restrict__ b,
                                         const double* __restrict__ c,
                                         const double* __restrict__ d, double beta,
                                         double* __restrict__ out, dd (&acc)[VecNS<OP>::value]) {
  if constexpr (OP == kDot) {
    dd_add(acc[0], __dmul_rn(a[i], b[i]));
  } else if constexpr (OP == kGbarFused) {
    // gbar_next = 1*x_next + (-1)*P(x_next)         (ncg.cpp:257)
    const double g = c[i];
    const double o = __dsub_rn(a[i], b[i]);
    out[i] = o;
    dd_add(acc[0], __dmul_rn(o, __dsub_rn(g, d[i])));  // beta numerator   (ncg.cpp:126-129)
    dd_add(acc[1], __dmul_rn(o, g));                   // next denominator (ncg.cpp:123)
    dd_add(acc[2], __dmul_rn(g, g));                   // ||g||^2          (ncg.cpp:134-136)
    dd_add(acc[3], __dmul_rn(g, -o));                  // g.p for p=-gbar  (ncg.cpp:270)
  } else if constexpr (OP == kDirFused) {
    // p_next = -1*gbar_next + beta*p                   (ncg.cpp:267)
    const double o = __dadd_rn(-a[i], __dmul_rn(beta, b[i]));
    out[i] = o;
    dd_add(acc[0], __dmul_rn(c[i], o));                // g_next.p_next    (ncg.cpp:270)
  } else {
    dd_add(acc[0], __dmul_rn(a[i], __dsub_rn(b[i], c[i])));
    dd_add(acc[1], __dmul_rn(d[i], c[i]));
  }
}

template <int OP>
__global__ void __launch_bounds__(kVecThreads)
    k_vec(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
          const double* __restrict__ c, const double* __restrict__ d, double beta,
          double* __restrict__ out, dd* __restrict__ partials, unsigned* counter,
          double* result) {
  constexpr int NS = VecNS<OP>::value;
  __shared__ dd sh[(kVecThreads / 32) * NS];
  __shared__ bool last;
  dd acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = {0.0, 0.0};
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    vec_elem<OP>(i, a, b, c, d, beta, out, acc);
  block_sum_dd<NS>(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) partials[blockIdx.x * NS + k] = acc[k];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = {0.0, 0.0};
  for (int blk = threadIdx.x; blk < gridDim.x; blk += blockDim.x)
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const volatile dd* p = partials + blk * NS + k;
      acc[k] = dd_plus(acc[k], dd{p->hi, p->lo});
    }
  block_sum_dd<NS>(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) result[k] = dd_value(acc[k]);
    *counter = 0u;
  }
}

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}

__global__ void k_pad_rows(int64_t rows, int n_f, int ld, const double* __restrict__ packed,
                           double* __restrict__ padded) {
  const int64_t n = rows * ld;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / ld;
    const int k = static_cast<int>(i - r * ld);
    padded[i] = k < n_f ? packed[r * n_f + k] : 0.0;
  }
}

__global__ void k_unpad_rows(int64_t rows, int n_f, int ld, const double* __restrict__ padded,
                             double* __restrict__ packed) {
  const int64_t n = rows * n_f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / n_f;
    const int k = static_cast<int>(i - r * n_f);
    packed[i] = padded[r * ld + k];
  }
}

// parallel.cpp:69-111: a column is listed once per distinct destination
// block among its neighbours; totals = sum over rows of #distinct(idx % nb).
__global__ void k_routing_count(int nrows, const int64_t* __restrict__ ptr,
                                const int* __restrict__ idx, int nb,
                                unsigned long long* __restrict__ out) {
  extern __shared__ unsigned bits[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int words = (nb + 31) / 32;
  unsigned* my = bits + warp * words;
  unsigned long long total = 0;
  for (int r = blockIdx.x * (blockDim.x / 32) + warp; r < nrows; r += gridDim.x * (blockDim.x / 32)) {
    for (int w = lane; w < words; w += 32) my[w] = 0u;
    __syncwarp();
    for (int64_t t = ptr[r] + lane; t < ptr[r + 1]; t += 32) {
      const int d = idx[t] % nb;
      atomicOr(&my[d >> 5], 1u << (d & 31));
    }
    __syncwarp();
    int c = 0;
    for (int w = lane; w < words; w += 32) c += __popc(my[w]);
    total += static_cast<unsigned long long>(c);
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(kFull, total, off);
  if (lane == 0) atomicAdd(out, total);
}

// Reference summation order (factors.cpp:95-103, ncg.cpp:118-132): one
// thread walks the vector in index order with separately rounded multiply
// and add, reproducing the reference's dot / beta_bar bit for bit.  Used by
// the API-level host-vector utilities only; the driver uses k_vec.
__global__ void k_seq_dots(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ c, const double* __restrict__ d, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    s0 = __dadd_rn(s0, __dmul_rn(a[i], c ? __dsub_rn(b[i], c[i]) : b[i]));
    if (d) s1 = __dadd_rn(s1, __dmul_rn(d[i], c[i]));
  }
  out[0] = s0;
  out[1] = s1;
}

int vec_blocks(int64_t n) {
  int64_t b = (n + kVecThreads * 8 - 1) / (kVecThreads * 8);
  if (b < 1) b = 1;
  if (b > kVecMaxBlocks) b = kVecMaxBlocks;
  return static_cast<int>(b);
}

int ew_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return static_cast<int>(b);
}

}  // namespace

void launch_vec(Ctx* ctx, VecOp op, int64_t n, const double* a, const double* b, const double* c,
                const double* d, double beta, double* out, int slot) {
  const int blocks = vec_blocks(n);
  dd* partials = reinterpret_cast<dd*>(ctx->d_red);
  double* res = ctx->d_scalars + slot;
  unsigned* cnt = ctx->d_counters;
  switch (op) {
    case kDot: {
      const int t = ctx->begin_launch("vec_dot");
      k_vec<kDot><<<blocks, kVecThreads, 0, ctx->stream>>>(n, a, b, c, d, beta, out, partials, cnt, res);
      ctx->end_launch(t);
      break;
    }
    case kGbarFused: {
      const int t = ctx->begin_launch("vec_gbar_fused");
      k_vec<kGbarFused><<<blocks, kVecThreads, 0, ctx->stream>>>(n, a, b, c, d, beta, out, partials, cnt, res);
      ctx->end_launch(t);
      break;
    }
    case kDirFused: {
      const int t = ctx->begin_launch("vec_dir_fused");
      k_vec<kDirFused><<<blocks, kVecThreads, 0, ctx->stream>>>(n, a, b, c, d, beta, out, partials, cnt, res);
      ctx->end_launch(t);
      break;
    }
    case kBetaParts: {
      const int t = ctx->begin_launch("vec_beta_parts");
      k_vec<kBetaParts><<<blocks, kVecThreads, 0, ctx->stream>>>(n, a, b, c, d, beta, out, partials, cnt, res);
      ctx->end_launch(t);
      break;
    }
  }
}

void launch_seq_dots(Ctx* ctx, int64_t n, const double* a, const double* b, const double* c,
                     const double* d, int slot) {
  const int t = ctx->begin_launch("vec_seq_dot");
  k_seq_dots<<<1, 32, 0, ctx->stream>>>(n, a, b, c, d, ctx->d_scalars + slot);
  ctx->end_launch(t);
}

void launch_axpby(Ctx* ctx, int64_t n, double a, const double* x, double b, const double* y,
                  double* out) {
  const int t = ctx->begin_launch("vec_axpby");
  k_axpby<<<ew_blocks(n), 256, 0, ctx->stream>>>(n, a, x, b, y, out);
  ctx->end_launch(t);
}

void launch_pad_rows(Ctx* ctx, int64_t rows, int n_f, const double* packed, double* padded) {
  const int t = ctx->begin_launch("pad_rows");
  k_pad_rows<<<ew_blocks(rows * row_stride(n_f)), 256, 0, ctx->stream>>>(rows, n_f, row_stride(n_f),
                                                                          packed, padded);
  ctx->end_launch(t);
}

void launch_unpad_rows(Ctx* ctx, int64_t rows, int n_f, const double* padded, double* packed) {
  const int t = ctx->begin_launch("unpad_rows");
  k_unpad_rows<<<ew_blocks(rows * n_f), 256, 0, ctx->stream>>>(rows, n_f, row_stride(n_f), padded,
                                                               packed);
  ctx->end_launch(t);
}

void launch_routing_count(DevRatings& R, int n_blocks, unsigned long long* d_out2) {
  Ctx* ctx = R.ctx;
  AB2_CUDA(cudaMemsetAsync(d_out2, 0, 2 * sizeof(unsigned long long), ctx->stream));
  const int words = (n_blocks + 31) / 32;
  const size_t smem = static_cast<size_t>(8) * words * sizeof(unsigned);
  // T_u: user columns -> item destination blocks (neighbours are items).
  for (int kind = 0; kind < 2; ++kind) {
    const View& v = R.view(kind);
    if (v.nrows == 0) continue;
    const int blocks = std::min(148 * 8, (v.nrows + 7) / 8);
    const int t = ctx->begin_launch("routing_count");
    k_routing_count<<<blocks, 256, smem, ctx->stream>>>(v.nrows, v.ptr, v.idx, n_blocks, d_out2 + kind);
    ctx->end_launch(t);
  }
}

// ------------------------------------------------------------ random_init --
// x0 = flatten(random_init(seed)) (factors.cpp:24-32) generated on the device:
// the mt19937_64 stream of std::mt19937_64(seed) (state seeded on the host),
// items first then users, u = (draw >> 11) * 2^-53 * (1/sqrt(n_f)) -- the
// same operations as the host Rng::uniform, so x0 is bitwise the reference's.
//
// The draw stream is cut into chunks of kMtChunk = 312*256 draws, one CTA per
// chunk walking the sequential twist chain (ping-pong state, two barriers per
// 312-draw block).  The state at each chunk start comes from jump-ahead: with
// T the one-step transition of the 19937-bit state, T^J s = g_J(T) s for
// g_J(x) = x^J mod phi(x) (phi the characteristic polynomial), and g(T) s is
// the XOR, over the set coefficients i of g, of the state window at word i of
// the sequence continuing s.  mt_jump_table.inc (tools/gen_mt_jump.py, which
// also checks each polynomial against stepping the generator) holds g_J for
// J = 1, 8, 64, 512 chunks; chunk states are filled level by level (at most 7
// dependent jumps per level), every jump of a step in its own CTA.
namespace {
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull,
                   kMtLower = 0x000000007FFFFFFFull;
constexpr int kMtDeg = 19937;
constexpr int kMtChunkTwists = 256;
constexpr int64_t kMtChunk = 312 * static_cast<int64_t>(kMtChunkTwists);  // draws per chunk
constexpr int kMtSeqWords = 128 * 156 + 312;  // >= kMtDeg + 312 words of the continued sequence
constexpr int kJumpParts = 3, kJumpThreads = kJumpParts * 320;

__device__ const uint64_t g_mt_jump[4][312] = {
#include "mt_jump_table.inc"
};

__device__ __forceinline__ uint64_t mt_twist(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t y = (cur & kMtUpper) | (next & kMtLower);
  return far ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}

// states[dst] = g(T) states[src], src = src0 + blockIdx.x * src_stride, dst = src + dst_off.
__global__ void __launch_bounds__(kJumpThreads) k_mt_jump(uint64_t* __restrict__ states, int n_chunks,
                                                           int src0, int src_stride, int dst_off,
                                                           int poly) {
  extern __shared__ uint64_t jw[];  // [kMtSeqWords] sequence + [kJumpParts][312] partial windows
  const int src = src0 + static_cast<int>(blockIdx.x) * src_stride, dst = src + dst_off;
  if (dst >= n_chunks) return;
  const int tid = threadIdx.x;
  if (tid < 312) jw[tid] = states[static_cast<int64_t>(src) * 312 + tid];
  __syncthreads();
  // continue the word sequence: 156 new words per step (w[k+312] needs w[k], w[k+1], w[k+156])
  for (int base = 0; base + 312 < kMtSeqWords; base += 156) {
    if (tid < 156) jw[base + 312 + tid] = mt_twist(jw[base + tid], jw[base + tid + 1], jw[base + tid + 156]);
    __syncthreads();
  }
  // window k of the result: XOR of w[i + k] over the set coefficients i; the
  // coefficient words are split over kJumpParts thread groups
  const int part = tid / 320, k = tid % 320;
  constexpr int WPP = 312 / kJumpParts;
  uint64_t r = 0;
  if (k < 312) {
    for (int wi = part * WPP; wi < (part + 1) * WPP; ++wi) {
      uint64_t bits = g_mt_jump[poly][wi];
      const uint64_t* w = jw + 64 * wi + k;
      while (bits) {
        const int b = __ffsll(static_cast<long long>(bits)) - 1;
        bits &= bits - 1;
        r ^= w[b];
      }
    }
    jw[kMtSeqWords + part * 312 + k] = r;
  }
  __syncthreads();
  if (tid < 312) {
    uint64_t v = 0;
#pragma unroll
    for (int q = 0; q < kJumpParts; ++q) v ^= jw[kMtSeqWords + q * 312 + tid];
    states[static_cast<int64_t>(dst) * 312 + tid] = v;
  }
}

// One CTA per chunk: draws [chunk * kMtChunk, min(n_draws, (chunk + 1) * kMtChunk)).
__global__ void __launch_bounds__(320) k_mt_random_init(const uint64_t* __restrict__ states,
                                                          int64_t n_item_draws, int64_t n_draws,
                                                          int n_f, int ld, int n_u, double scale,
                                                          double* __restrict__ x) {
  __shared__ uint64_t S[2][312];  // ping-pong state: two barriers per 312 draws
  const int tid = threadIdx.x;
  if (tid < 312) S[0][tid] = states[static_cast<int64_t>(blockIdx.x) * 312 + tid];
  __syncthreads();
  int cur = 0;
  const int64_t base0 = static_cast<int64_t>(blockIdx.x) * kMtChunk;
  const int64_t end = min(n_draws, base0 + kMtChunk);
  // draw k = base + tid -> (q, col) = divmod(k, n_f), kept incrementally (one
  // 64-bit division per CTA): q < n_m are item rows, the rest user rows
  int64_t q = (base0 + tid) / n_f;
  int col = static_cast<int>((base0 + tid) % n_f);
  const int dq = 312 / n_f, dc = 312 % n_f;
  const int64_t n_m = n_item_draws / n_f;
  for (int64_t base = base0; base < end; base += 312) {
    const int nx = cur ^ 1;
    if (tid < 156) S[nx][tid] = mt_twist(S[cur][tid], S[cur][tid + 1], S[cur][tid + 156]);
    __syncthreads();
    if (tid >= 156 && tid < 311) S[nx][tid] = mt_twist(S[cur][tid], S[cur][tid + 1], S[nx][tid - 156]);
    if (tid == 311) S[nx][311] = mt_twist(S[cur][311], S[nx][0], S[nx][155]);
    __syncthreads();
    cur = nx;
    const int64_t k = base + tid;
    if (tid < 312 && k < end) {
      uint64_t z = S[cur][tid];
      z ^= (z >> 29) & 0x5555555555555555ull;
      z ^= (z << 17) & 0x71D67FFFEDA60000ull;
      z ^= (z << 37) & 0xFFF7EEE000000000ull;
      z ^= z >> 43;
      const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
      const double val = __dmul_rn(u, scale);
      const int64_t row = k < n_item_draws ? n_u + q : q - n_m;
      x[row * ld + col] = val;
    }
    q += dq;
    col += dc;
    if (col >= n_f) {
      col -= n_f;
      ++q;
    }
  }
}
}  // namespace

void launch_random_init(Ctx* ctx, int n_f, int n_u, int n_m, uint64_t seed, double* x) {
  // std::mt19937_64 seeding (linear recurrence, 312 words) on the host
  uint64_t st[312];
  st[0] = seed;
  for (int i = 1; i < 312; ++i) st[i] = 6364136223846793005ull * (st[i - 1] ^ (st[i - 1] >> 62)) + i;
  const int64_t nm = static_cast<int64_t>(n_f) * n_m, nu = static_cast<int64_t>(n_f) * n_u;
  const int64_t n_draws = nm + nu;
  const int n_chunks = static_cast<int>(std::max<int64_t>(1, (n_draws + kMtChunk - 1) / kMtChunk));
  uint64_t* states = static_cast<uint64_t*>(ctx->scratch(7, sizeof(uint64_t) * 312 * static_cast<size_t>(n_chunks)));
  AB2_CUDA(cudaMemcpyAsync(states, st, sizeof st, cudaMemcpyHostToDevice, ctx->stream));
  const int ld = row_stride(n_f);
  AB2_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (static_cast<size_t>(n_u) + n_m) * ld, ctx->stream));
  if (n_chunks > 1) {
    // chunk states by jump-ahead: strides 512, 64, 8, 1 chunks (polynomials 3..0)
    const size_t smem = sizeof(uint64_t) * (kMtSeqWords + kJumpParts * 312);
    ctx->prepare_kernel(reinterpret_cast<const void*>(k_mt_jump), static_cast<int>(smem), 0, 0);
    const int tok = ctx->begin_launch("random_init_jump");
    for (int a = 1; a * 512 < n_chunks; ++a)
      k_mt_jump<<<1, kJumpThreads, smem, ctx->stream>>>(states, n_chunks, (a - 1) * 512, 0, 512, 3);
    const int strides[4] = {512, 64, 8, 1};
    for (int lvl = 1; lvl < 4; ++lvl) {
      const int big = strides[lvl - 1], small = strides[lvl];
      if (small >= n_chunks) continue;
      const int n_src = (n_chunks + big - 1) / big;
      for (int step = 1; step < 8; ++step)
        k_mt_jump<<<n_src, kJumpThreads, smem, ctx->stream>>>(states, n_chunks, (step - 1) * small, big,
                                                                small, 3 - lvl);
    }
    ctx->end_launch(tok);
  }
  const int t = ctx->begin_launch("random_init");
  k_mt_random_init<<<n_chunks, 320, 0, ctx->stream>>>(states, nm, n_draws, n_f, ld, n_u,
                                                     1.0 / std::sqrt(static_cast<double>(n_f)), x);
  ctx->end_launch(t);
  // (no sync: a copy from pageable memory returns once `st` has been staged,
  // so the host goes on to build the work plans while the kernels run)
}

}  // namespace ab2
