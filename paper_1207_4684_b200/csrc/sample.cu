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
    phat = mp < 1.0 ? mp : 1.0;
    double ui;
    if (u) ui = u[i];
    else ui = (double)(mix64(key + 0x9E3779B97F4A7C15ULL * (uint64_t)(row_base + i + 1)) >> 11) * 0x1.0p-53;
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
