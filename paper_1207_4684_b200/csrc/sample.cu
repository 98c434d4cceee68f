// sample.cu -- K4/K6: Bernoulli l1 row sampling with ascending compaction
//   phat_i = min(1, m p_i), keep iff u_i < phat_i, D_ii = 1/phat_i
// Decisions are exact fp64 comparisons; u_i comes from the counter-based generator keyed by the
// GLOBAL row (K6, bit-identical to the host generator) or from an explicit array.  Compaction is
// integer: per-tile counts -> exclusive scan -> ordered writes, so idx/weight are bit-exact.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kRowsPerThread = 8;
constexpr int kTile = kThreads * kRowsPerThread;  // 2048 rows per tile

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct Decide {
  const float* p;
  const double* u;   // explicit uniforms or nullptr
  int64_t row_base;
  double m;
  uint64_t key;      // mix64(seed + G * (9 + 1))
  __device__ __forceinline__ bool operator()(int64_t i, double& phat) const {
    const double mp = m * (double)p[i];
    phat = mp < 1.0 ? mp : (mp >= 1.0 ? 1.0 : 0.0);   // NaN p: never sampled (R31)
    double ui;
    if (u) ui = u[i];
    else ui = (double)(mix64(key + 0x9E3779B97F4A7C15ULL * (uint64_t)(row_base + i + 1)) >> 11) * 0x1.0p-53;
    return ui < phat;
  }
  // the same decision from an already-rounded p value
  __device__ __forceinline__ bool decide_p(float pi, int64_t i, double& phat) const {
    const double mp = m * (double)pi;
    phat = mp < 1.0 ? mp : (mp >= 1.0 ? 1.0 : 0.0);
    const double ui = (double)(mix64(key + 0x9E3779B97F4A7C15ULL * (uint64_t)(row_base + i + 1)) >> 11) * 0x1.0p-53;
    return ui < phat;
  }
};

__global__ void __launch_bounds__(kThreads) count_kernel(Decide dec, int64_t n, int64_t* __restrict__ counts) {
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * kTile + (int64_t)threadIdx.x * kRowsPerThread;
  int c = 0;
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    const int64_t i = base + r;
    double ph;
    if (i < n && dec(i, ph)) ++c;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    counts[tile] = t;
  }
}

// single-CTA exclusive scan of ntiles counts (in place) and total -> *count
__global__ void __launch_bounds__(1024) scan_kernel(int64_t* __restrict__ counts, int64_t ntiles,
                                                    int64_t* __restrict__ count) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < ntiles ? counts[i] : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive prefix of warp totals
    }
    __syncthreads();
    const int64_t excl = carry + (warp > 0 ? warp_tot[warp - 1] : 0) + x - v;
    if (i < ntiles) counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = carry;
}

__global__ void __launch_bounds__(kThreads) write_kernel(Decide dec, int64_t n, const int64_t* __restrict__ offsets,
                                                          int64_t* __restrict__ idx, double* __restrict__ weight,
                                                          int64_t capacity) {
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * kTile + (int64_t)threadIdx.x * kRowsPerThread;
  unsigned keep = 0u;
  double ph[kRowsPerThread];
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    const int64_t i = base + r;
    ph[r] = 1.0;
    if (i < n && dec(i, ph[r])) keep |= 1u << r;
  }
  const int c = __popc(keep);
  // block exclusive scan of c
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __shared__ int wt[kThreads / 32];
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  int wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += wt[w];
  int64_t pos = offsets[tile] + wpre + x - c;
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    if ((keep >> r) & 1u) {
      if (pos < capacity) {
        idx[pos] = dec.row_base + base + r;
        weight[pos] = 1.0 / ph[r];
      }
      ++pos;
    }
  }
}


// ------------------------------------------------------------------------------------------------
// Single-pass fused probabilities + sampling for the pipeline (a9 + a10 in one kernel):
//   p_i = (float)((double)lambda_i / total)   (exactly l1_probs), then the same exact fp64 decision and
//   ascending compaction as count/scan/write, with the tile offsets from a decoupled look-back:
// tile t (taken in launch order from an atomic ticket, so every predecessor is already running)
// publishes its count as an AGGREGATE, walks back over predecessors summing aggregates until it meets an
// INCLUSIVE prefix, publishes its own INCLUSIVE prefix and writes its kept rows.  Integer arithmetic
// only -> idx / weight / count bit-identical to the three-kernel path.  Reads lambda once, writes p once.
constexpr uint64_t kAgg = 1ull << 62, kInc = 2ull << 62, kValMask = (1ull << 62) - 1;
// 32 rows per thread, 8192 per tile: the look-back chain (each tile waits for a predecessor's inclusive prefix) was
// the bound with 2048-row tiles (ncu: 45 % of the stall samples at the barrier behind warp 0's look-back, DRAM
// throughput 16 %); phat is recomputed for the few kept rows instead of being held for all 32
constexpr int kFRows = 32, kFTile = kThreads * kFRows;

__global__ void __launch_bounds__(kThreads) probs_sample_kernel(const float* __restrict__ lambda,
                                                                 const double* __restrict__ total, float* __restrict__ p,
                                                                 Decide dec, int64_t n, int64_t ntiles,
                                                                 unsigned long long* __restrict__ state,
                                                                 unsigned* __restrict__ ticket, int64_t* __restrict__ idx,
                                                                 double* __restrict__ weight, int64_t capacity,
                                                                 int64_t* __restrict__ count, int vec) {
  __shared__ int64_t s_tile, s_excl;
  __shared__ int wt[kThreads / 32];
  if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const double tot = *total;
  const int64_t base = tile * kFTile + (int64_t)threadIdx.x * kFRows;
  unsigned keep = 0u;
  if (vec && base + kFRows <= n) {
#pragma unroll
    for (int q = 0; q < kFRows; q += 4) {
      const float4 l = *(const float4*)(lambda + base + q);
      const float lv[4] = {l.x, l.y, l.z, l.w};
      float pv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pv[r] = (float)((double)lv[r] / tot);
      *(float4*)(p + base + q) = make_float4(pv[0], pv[1], pv[2], pv[3]);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double ph;
        if (dec.decide_p(pv[r], base + q + r, ph)) keep |= 1u << (q + r);
      }
    }
  } else {
#pragma unroll 4
    for (int r = 0; r < kFRows; ++r) {
      const int64_t i = base + r;
      if (i < n) {
        const float pv = (float)((double)lambda[i] / tot);
        p[i] = pv;
        double ph;
        if (dec.decide_p(pv, i, ph)) keep |= 1u << r;
      }
    }
  }
  const int c = __popc(keep);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  int wpre = 0, agg = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) wpre += wt[w];
    agg += wt[w];
  }
  if (warp == 0) {
    // warp-parallel look-back: lane j inspects tile (t - 1 - j) of the current window of 32
    volatile unsigned long long* st = state;
    if (tile == 0) {
      if (lane == 0) {
        st[0] = kInc | (uint64_t)agg;
        s_excl = 0;
      }
    } else {
      if (lane == 0) {
        st[tile] = kAgg | (uint64_t)agg;
        __threadfence();
      }
      __syncwarp();
      int64_t excl = 0;
      int64_t t = tile - 1 - lane;
      while (true) {
        uint64_t v = kInc;   // past tile 0: nothing to add, acts as the terminating prefix
        if (t >= 0)
          do { v = st[t]; } while ((v >> 62) == 0);
        const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 32;          // nearest inclusive prefix in the window
        int64_t add = (lane <= stop && t >= 0) ? (int64_t)(v & kValMask) : 0;
        for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        excl += add;
        if (inc) break;
        t -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st[tile] = kInc | (uint64_t)(excl + agg);
        s_excl = excl;
      }
    }
    if (lane == 0 && tile == ntiles - 1) *count = s_excl + agg;
  }
  __syncthreads();
  int64_t pos = s_excl + wpre + x - c;
  for (unsigned kb = keep; kb; kb &= kb - 1u) {   // kept rows (few): phat again from the same p
    const int r = __ffs(kb) - 1;
    if (pos < capacity) {
      const float pv = (float)((double)lambda[base + r] / tot);
      double ph;
      dec.decide_p(pv, base + r, ph);
      idx[pos] = dec.row_base + base + r;
      weight[pos] = 1.0 / ph;
    }
    ++pos;
  }
}

fct_status sample_impl(const float* p, const double* u, int64_t n, int64_t row_base, int64_t m, uint64_t seed,
                       int64_t* idx, double* weight, int64_t capacity, int64_t* count, void* ws, size_t wsb,
                       cudaStream_t st) {
  FCT_CHECK_ARG(p && count && (capacity == 0 || (idx && weight)), FCT_ERR_ARG, "l1_sample: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && row_base >= 0 && capacity >= 0, FCT_ERR_SHAPE, "l1_sample: n=%lld row_base=%lld",
                (long long)n, (long long)row_base);
  FCT_CHECK_ARG(m >= 1 && m <= (1LL << 29), FCT_ERR_ARG, "l1_sample: m=%lld not in [1, 2^29]", (long long)m);
  const size_t need = l1_sample_workspace_bytes(n);
  FCT_CHECK_ARG(ws && wsb >= need, FCT_ERR_WORKSPACE, "l1_sample: workspace %zu < %zu bytes", wsb, need);
  const int64_t ntiles = (n + kTile - 1) / kTile;
  FCT_CHECK_ARG(ntiles <= 0x7fffffffLL, FCT_ERR_SHAPE, "l1_sample: n too large");
  int64_t* counts = (int64_t*)ws;
  Decide dec{p, u, row_base, (double)m, mix64(seed + 0x9E3779B97F4A7C15ULL * 10ULL)};
  count_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(dec, n, counts);
  FCT_LAUNCHED("count_kernel", st);
  scan_kernel<<<1, 1024, 0, st>>>(counts, ntiles, count);
  FCT_LAUNCHED("scan_kernel", st);
  write_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(dec, n, counts, idx, weight, capacity);
  FCT_LAUNCHED("write_kernel", st);
  return FCT_OK;
}

}  // namespace

extern "C" size_t l1_sample_workspace_bytes(int64_t n) {
  if (n < 1) return 0;
  return fct::align256(sizeof(int64_t) * (size_t)((n + kTile - 1) / kTile));
}

extern "C" fct_status l1_sample(const float* p, int64_t n, int64_t row_base, int64_t m, uint64_t seed, int64_t* idx,
                                double* weight, int64_t capacity, int64_t* count, void* workspace,
                                size_t workspace_bytes, void* stream) {
  return sample_impl(p, nullptr, n, row_base, m, seed, idx, weight, capacity, count, workspace, workspace_bytes,
                     (cudaStream_t)stream);
}

extern "C" fct_status l1_sample_u(const float* p, const double* u, int64_t n, int64_t row_base, int64_t m,
                                  int64_t* idx, double* weight, int64_t capacity, int64_t* count, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(u, FCT_ERR_ARG, "l1_sample_u: u is NULL");
  return sample_impl(p, u, n, row_base, m, 0, idx, weight, capacity, count, workspace, workspace_bytes,
                     (cudaStream_t)stream);
}

extern "C" size_t l1_probs_sample_workspace_bytes(int64_t n) {
  if (n < 1) return 0;
  return fct::align256(sizeof(unsigned long long) * (size_t)((n + kTile - 1) / kTile)) + fct::align256(sizeof(unsigned));
}

extern "C" fct_status l1_probs_sample(const float* lambda, int64_t n, const double* lambda_total, int64_t row_base,
                                      int64_t m, uint64_t seed, float* p, int64_t* idx, double* weight,
                                      int64_t capacity, int64_t* count, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  FCT_CHECK_ARG(lambda && lambda_total && p && count && (capacity == 0 || (idx && weight)), FCT_ERR_ARG,
                "l1_probs_sample: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && row_base >= 0 && capacity >= 0, FCT_ERR_SHAPE, "l1_probs_sample: n=%lld row_base=%lld",
                (long long)n, (long long)row_base);
  FCT_CHECK_ARG(m >= 1 && m <= (1LL << 29), FCT_ERR_ARG, "l1_probs_sample: m=%lld not in [1, 2^29]", (long long)m);
  const size_t need = l1_probs_sample_workspace_bytes(n);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_WORKSPACE, "l1_probs_sample: workspace %zu < %zu bytes",
                workspace_bytes, need);
  const int64_t ntiles = (n + kFTile - 1) / kFTile;
  FCT_CHECK_ARG(ntiles <= 0x7fffffffLL, FCT_ERR_SHAPE, "l1_probs_sample: n too large");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* state = (unsigned long long*)workspace;
  unsigned* ticket = (unsigned*)((char*)workspace + fct::align256(sizeof(unsigned long long) * (size_t)ntiles));
  FCT_CUDA_RET(cudaMemsetAsync(workspace, 0, need, st));
  Decide dec{nullptr, nullptr, row_base, (double)m, mix64(seed + 0x9E3779B97F4A7C15ULL * 10ULL)};
  probs_sample_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(lambda, lambda_total, p, dec, n, ntiles, state, ticket,
                                                              idx, weight, capacity, count,
                                                              (((uintptr_t)lambda | (uintptr_t)p) & 15) == 0);
  FCT_LAUNCHED("probs_sample_kernel", st);
  return FCT_OK;
}

// ------------------------------------------------------------------------------------------------
// NEXT-4: multinomial sampling -- m i.i.d. draws proportional to p from an exact
// fixed-point CDF; integer arithmetic only, bit-exact with the oracle (oracle.c or_sample_multinomial):
//   F = 62 - ceil(log2 n) - e (max p < 2^e),  W_i = floor(p_i 2^F),  CDF = inclusive scan of W (uint64),
//   target_j = (X_j T) >> 53 with X_j = rng_u64(seed, 10, j) >> 11,  idx_j = first i with CDF_i > target_j,
//   weight_j = (double)T / ((double)m (double)W_idx).
namespace {

__global__ void mn_max_kernel(const float* __restrict__ p, int64_t n, unsigned* __restrict__ mbits) {
  unsigned m = 0u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = p[i];
    if (v > 0.f) m = max(m, __float_as_uint(v));   // positive floats order like their bit patterns
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(mbits, m);
}
__device__ __forceinline__ int mn_F(const unsigned* mbits, int lg) {
  int e = 0;
  frexp((double)__uint_as_float(*mbits), &e);
  return 62 - lg - e;
}
__device__ __forceinline__ uint64_t mn_W(float v, int F) {
  return v > 0.f ? (uint64_t)floor(ldexp((double)v, F)) : 0ull;
}
constexpr int kMnTile = 2048, kMnThreads = 256, kMnPer = kMnTile / kMnThreads;

__global__ void __launch_bounds__(kMnThreads) mn_tile_sum_kernel(const float* __restrict__ p, int64_t n,
                                                                  const unsigned* __restrict__ mbits, int lg,
                                                                  uint64_t* __restrict__ tsum) {
  if (*mbits == 0u) return;
  const int F = mn_F(mbits, lg);
  const int64_t base = (int64_t)blockIdx.x * kMnTile;
  uint64_t s = 0;
  for (int r = threadIdx.x; r < kMnTile; r += kMnThreads)
    if (base + r < n) s += mn_W(p[base + r], F);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ uint64_t red[kMnThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kMnThreads / 32; ++w) t += red[w];
    tsum[blockIdx.x] = t;
  }
}
// single CTA: exclusive scan of the tile sums in place, total -> *T (0 when no positive p)
__global__ void __launch_bounds__(1024) mn_scan_kernel(uint64_t* __restrict__ tsum, int64_t ntiles,
                                                        const unsigned* __restrict__ mbits, uint64_t* __restrict__ T) {
  __shared__ uint64_t warp_tot[32];
  __shared__ uint64_t carry;
  if (*mbits == 0u) {
    if (threadIdx.x == 0) *T = 0;
    return;
  }
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < ntiles; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const uint64_t v = i < ntiles ? tsum[i] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    const uint64_t excl = carry + (warp > 0 ? warp_tot[warp - 1] : 0) + x - v;
    if (i < ntiles) tsum[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *T = carry;
}
__global__ void __launch_bounds__(kMnThreads) mn_cdf_kernel(const float* __restrict__ p, int64_t n,
                                                             const unsigned* __restrict__ mbits, int lg,
                                                             const uint64_t* __restrict__ toff, uint64_t* __restrict__ cdf) {
  if (*mbits == 0u) return;
  const int F = mn_F(mbits, lg);
  const int64_t base = (int64_t)blockIdx.x * kMnTile + (int64_t)threadIdx.x * kMnPer;
  uint64_t w[kMnPer], s = 0;
#pragma unroll
  for (int r = 0; r < kMnPer; ++r) {
    w[r] = base + r < n ? mn_W(p[base + r], F) : 0;
    s += w[r];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __shared__ uint64_t wt[kMnThreads / 32];
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  uint64_t pre = toff[blockIdx.x];
  for (int q = 0; q < warp; ++q) pre += wt[q];
  uint64_t c = pre + x - s;
#pragma unroll
  for (int r = 0; r < kMnPer; ++r) {
    c += w[r];
    if (base + r < n) cdf[base + r] = c;
  }
}
__global__ void mn_draw_kernel(const uint64_t* __restrict__ cdf, int64_t n, const uint64_t* __restrict__ Tp, int64_t m,
                               uint64_t key, int64_t row_base, int64_t* __restrict__ idx, double* __restrict__ weight) {
  const uint64_t T = *Tp;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    if (T == 0) {
      idx[j] = -1;
      weight[j] = 0.0;
      continue;
    }
    const uint64_t X = mix64(key + 0x9E3779B97F4A7C15ULL * (uint64_t)(j + 1)) >> 11;
    const uint64_t hi = __umul64hi(X, T), lo = X * T;
    const uint64_t target = (hi << 11) | (lo >> 53);
    int64_t a = 0, b = n - 1;
    while (a < b) {
      const int64_t mid = a + (b - a) / 2;
      if (cdf[mid] > target) b = mid; else a = mid + 1;
    }
    const uint64_t W = cdf[a] - (a > 0 ? cdf[a - 1] : 0ull);
    idx[j] = row_base + a;
    weight[j] = (double)T / ((double)m * (double)W);
  }
}

}  // namespace

extern "C" size_t l1_sample_multinomial_workspace_bytes(int64_t n) {
  if (n < 1) return 0;
  const size_t ntiles = (size_t)((n + kMnTile - 1) / kMnTile);
  return fct::align256(sizeof(uint64_t) * (size_t)n) + fct::align256(sizeof(uint64_t) * ntiles) + fct::align256(8);
}

extern "C" fct_status l1_sample_multinomial(const float* p, int64_t n, int64_t m, uint64_t seed, int64_t row_base,
                                            int64_t* idx, double* weight, uint64_t* total, void* workspace,
                                            size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(p && idx && weight && total, FCT_ERR_ARG, "l1_sample_multinomial: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && row_base >= 0, FCT_ERR_SHAPE, "l1_sample_multinomial: n=%lld", (long long)n);
  FCT_CHECK_ARG(m >= 1, FCT_ERR_ARG, "l1_sample_multinomial: m=%lld", (long long)m);
  const size_t need = l1_sample_multinomial_workspace_bytes(n);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_WORKSPACE,
                "l1_sample_multinomial: workspace %zu < %zu bytes", workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ntiles = (n + kMnTile - 1) / kMnTile;
  fct::Carver cv(workspace);
  uint64_t* cdf = cv.take<uint64_t>((size_t)n);
  uint64_t* tsum = cv.take<uint64_t>((size_t)ntiles);
  unsigned* mbits = cv.take<unsigned>(2);
  int lg = 0;
  while ((1LL << lg) < n) ++lg;
  FCT_CUDA_RET(cudaMemsetAsync(mbits, 0, sizeof(unsigned), st));
  mn_max_kernel<<<fct::num_sms() * 4, 256, 0, st>>>(p, n, mbits);
  FCT_LAUNCHED("mn_max_kernel", st);
  mn_tile_sum_kernel<<<(unsigned)ntiles, kMnThreads, 0, st>>>(p, n, mbits, lg, tsum);
  FCT_LAUNCHED("mn_tile_sum_kernel", st);
  mn_scan_kernel<<<1, 1024, 0, st>>>(tsum, ntiles, mbits, total);
  FCT_LAUNCHED("mn_scan_kernel", st);
  mn_cdf_kernel<<<(unsigned)ntiles, kMnThreads, 0, st>>>(p, n, mbits, lg, tsum, cdf);
  FCT_LAUNCHED("mn_cdf_kernel", st);
  const uint64_t key = mix64(seed + 0x9E3779B97F4A7C15ULL * 11ULL);   // stream 10
  mn_draw_kernel<<<(unsigned)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, st>>>(cdf, n, total, m, key, row_base,
                                                                                      idx, weight);
  FCT_LAUNCHED("mn_draw_kernel", st);
  return FCT_OK;
}
