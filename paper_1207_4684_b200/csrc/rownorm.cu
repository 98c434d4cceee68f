// rownorm.cu -- K2/K3: l1 row-norm estimation and sampling probabilities
//   lambda_i = median_j |(A (Rinv Pi2))_ij|,  p_i = lambda_i / sum lambda
//
// Precision scheme:
//   1. v_j = |fl32(sum_l a_l m~_lj)| by a sequential fp32 FMA chain with m~ = fp32(M).
//   2. rigorous error bound e_j >= |v_j - |sum_l a_l m_lj||:
//        e_j = (d+3) u 1.1 * min(||a||_2 ||m~_j||_2, ||a||_1 ||m~_j||_inf) + tiny absolute term,
//      (gamma_d for the FMA chain + u for rounding M to fp32; 10% covers rounding of the bound).
//   3. with lo = v - e, hi = v + e, the true m-th order statistic lies in [L_m, H_m] (the m-th
//      smallest lo / hi).  Entries whose interval misses [L_m1, H_m2] are certainly below or
//      above the middle order statistic(s); the remaining "candidates" (1-2 per row in practice)
//      are recomputed exactly in fp64 with the fp64 M, and the median is selected among them.
//   => lambda is the exact median up to fp64 rounding, then rounded once to fp32.
#include <math.h>
#include "common.cuh"

namespace {

constexpr int kRowThreads = 256;  // 8 warps, one row per thread, 32 rows per warp per step

// M = Rinv * Pi2 in fp64; also the fp32 copy (padded to KP columns, zeros) and
// per-column bounds (||m~_j||_2 rounded up, ||m~_j||_inf).
__global__ void form_m_kernel(const double* __restrict__ Rinv, const float* __restrict__ Pi2, int d,
                              int k, int KP, double* __restrict__ M64T, float* __restrict__ M32,
                              float* __restrict__ colb) {
  // one thread per (l, j); M64T stored transposed [k][d] for the candidate recompute
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d * KP; e += gridDim.x * blockDim.x) {
    const int l = e / KP, j = e - l * KP;
    double acc = 0.0;
    if (j < k)
      for (int q = 0; q < d; ++q) acc = fma(Rinv[l * d + q], (double)Pi2[q * k + j], acc);
    M32[l * KP + j] = (float)acc;   // zero for the padding columns j >= k
    if (j < k) M64T[j * d + l] = acc;
  }
}

__global__ void colbound_kernel(const float* __restrict__ M32, int d, int k, int KP, float* __restrict__ colb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= KP) return;
  double s2 = 0.0, mx = 0.0;
  for (int l = 0; l < d; ++l) {
    const double m = fabs((double)M32[l * KP + j]);
    s2 += m * m;
    mx = fmax(mx, m);
  }
  colb[2 * j] = __double2float_ru(sqrt(s2) * (1.0 + 1e-12));
  colb[2 * j + 1] = (float)mx;
}

__device__ __forceinline__ void cswap(float& a, float& b) {
  const float lo = fminf(a, b), hi = fmaxf(a, b);
  a = lo;
  b = hi;
}

// Batcher odd-even merge sort of N (power of two) registers, ascending
template <int N>
__device__ __forceinline__ void sort_net(float (&a)[N]) {
#pragma unroll
  for (int p = 1; p < N; p <<= 1)
#pragma unroll
    for (int kk = p; kk >= 1; kk >>= 1)
#pragma unroll
      for (int j = kk % p; j + kk < N; j += 2 * kk)
#pragma unroll
        for (int i = 0; i < kk; ++i)
          if (j + i + kk < N && (j + i) / (2 * p) == (j + i + kk) / (2 * p)) cswap(a[j + i], a[j + i + kk]);
}

template <int K>
struct SortN {
  static constexpr int value = K <= 8 ? 8 : (K <= 16 ? 16 : 32);
};

// K = padded column count (multiple of 4, >= k); NS = sorting width (power of two >= K)
template <int K>
__global__ void __launch_bounds__(kRowThreads)
rownorm_kernel(const float* __restrict__ A, int64_t n, int d, int64_t lda, const float* __restrict__ M32g,
               const double* __restrict__ M64Tg, const float* __restrict__ colbg, int k, float gam,
               float* __restrict__ lambda, double* __restrict__ partial) {
  constexpr int NS = SortN<K>::value;
  extern __shared__ unsigned char smraw[];
  float* M32 = (float*)smraw;                                   // [d][K]   (16-byte aligned rows)
  float* colb = M32 + (size_t)d * K;                            // [K][2]
  double* M64T = (double*)(colb + 2 * K);                       // [k][d]
  float* tiles = (float*)(M64T + (size_t)k * d);                // [8 warps][32][d+1]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ldt = d + 1;
  float* tile = tiles + (size_t)warp * 32 * ldt;

  for (int e = threadIdx.x; e < k * d; e += blockDim.x) M64T[e] = M64Tg[e];
  for (int e = threadIdx.x; e < d * K; e += blockDim.x) M32[e] = M32g[e];
  for (int e = threadIdx.x; e < 2 * K; e += blockDim.x) colb[e] = colbg[e];
  __syncthreads();

  const int m1 = (k - 1) / 2;       // 0-based lower middle order statistic
  const int m2 = k / 2;             // 0-based upper middle (== m1 for odd k)
  double local = 0.0;
  const int64_t ntiles = (n + 31) / 32;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tileid = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; tileid < ntiles; tileid += wstride) {
    const int64_t row0 = tileid * 32;
    const int nr = (int)(n - row0 < 32 ? n - row0 : 32);
    __syncwarp();
    for (int r = 0; r < nr; ++r) {
      const float* src = A + (row0 + r) * lda;
      for (int l = lane; l < d; l += 32) tile[r * ldt + l] = src[l];
    }
    __syncwarp();
    if (lane < nr) {
      const float* a = tile + lane * ldt;
      float acc[K];
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] = 0.f;
      float n1 = 0.f, n2 = 0.f;
      for (int l = 0; l < d; ++l) {
        const float al = a[l];
        n1 += fabsf(al);
        n2 = fmaf(al, al, n2);
        const float4* mrow = (const float4*)(M32 + l * K);
#pragma unroll
        for (int j4 = 0; j4 < K / 4; ++j4) {
          const float4 mv = mrow[j4];
          acc[4 * j4 + 0] = fmaf(al, mv.x, acc[4 * j4 + 0]);
          acc[4 * j4 + 1] = fmaf(al, mv.y, acc[4 * j4 + 1]);
          acc[4 * j4 + 2] = fmaf(al, mv.z, acc[4 * j4 + 2]);
          acc[4 * j4 + 3] = fmaf(al, mv.w, acc[4 * j4 + 3]);
        }
      }
      float lam;
      if (n1 == 0.f) {
        lam = 0.f;
      } else {
        const float nrm2 = __fsqrt_ru(n2) * 1.0001f;
        float lo[NS], hi[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          if (j < K && j < k) {
            const float v = fabsf(acc[j]);
            float e = gam * fminf(nrm2 * colb[2 * j], n1 * colb[2 * j + 1]) + 1e-37f;
            if (!isfinite(v) || !isfinite(e)) e = INFINITY;
            lo[j] = fmaxf(v - e, 0.f);
            hi[j] = v + e;
          } else {
            lo[j] = INFINITY;
            hi[j] = INFINITY;
          }
        }
        float slo[NS], shi[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) { slo[j] = lo[j]; shi[j] = hi[j]; }
        sort_net<NS>(slo);
        sort_net<NS>(shi);
        float L = 0.f, H = 0.f;
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          if (j == m1) L = slo[j];
          if (j == m2) H = shi[j];
        }
        // candidates overlap [L, H]; count the entries certainly below
        int below = 0;
        unsigned cmask = 0u;
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          if (j < k) {
            if (hi[j] < L) ++below;
            else if (lo[j] <= H) cmask |= 1u << j;
          }
        }
        // exact fp64 values of the candidates; select ranks (m1 - below), (m2 - below)
        const int r1 = m1 - below, r2 = m2 - below;
        double x1 = 0.0, x2 = 0.0;
        const int nc = __popc(cmask);
        if (nc <= 2) {
          double c0 = INFINITY, c1 = INFINITY;
          unsigned mm = cmask;
          while (mm) {
            const int j = __ffs(mm) - 1;
            mm &= mm - 1;
            const double* mc = M64T + (size_t)j * d;
            double s = 0.0;
            for (int l = 0; l < d; ++l) s = fma((double)a[l], mc[l], s);
            if (c0 == INFINITY) c0 = fabs(s); else c1 = fabs(s);
          }
          const double cmin = fmin(c0, c1), cmax = fmax(c0, c1);
          x1 = r1 == 0 ? cmin : cmax;
          x2 = r2 == 0 ? cmin : cmax;
        } else {
          // general path (rare): exact values of all candidates, then rank by counting
          double ex[NS];
#pragma unroll
          for (int j = 0; j < NS; ++j) {
            ex[j] = INFINITY;
            if ((cmask >> j) & 1u) {
              const double* mc = M64T + (size_t)j * d;
              double s = 0.0;
              for (int l = 0; l < d; ++l) s = fma((double)a[l], mc[l], s);
              ex[j] = fabs(s);
            }
          }
#pragma unroll
          for (int j = 0; j < NS; ++j) {
            if ((cmask >> j) & 1u) {
              int rank = 0;
#pragma unroll
              for (int i = 0; i < NS; ++i)
                rank += ((cmask >> i) & 1u) && (ex[i] < ex[j] || (ex[i] == ex[j] && i < j));
              if (rank == r1) x1 = ex[j];
              if (rank == r2) x2 = ex[j];
            }
          }
        }
        lam = (float)(0.5 * (x1 + x2));
      }
      lambda[row0 + lane] = lam;
      local += (double)lam;
    }
  }
  // CTA reduction of the fp32 lambdas in fp64 (fixed order -> deterministic)
  __shared__ double red[kRowThreads / 32];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __syncthreads();
  if (lane == 0) red[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kRowThreads / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int np, double* __restrict__ out,
                                    int zero_first) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += partial[i];  // fixed assignment
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = zero_first ? t : *out + t;
  }
}

__global__ void probs_kernel(const float* __restrict__ lambda, int64_t n, const double* __restrict__ total,
                             float* __restrict__ p) {
  const double tot = *total;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (float)((double)lambda[i] / tot);
}

int pad_k(int k) { return (k + 3) / 4 * 4; }

size_t smem_bytes(int d, int k, int K) {
  return sizeof(double) * (size_t)k * d + sizeof(float) * ((size_t)d * K + 2 * K) +
         sizeof(float) * (size_t)(kRowThreads / 32) * 32 * (d + 1);
}

int rownorm_grid() { return fct::num_sms() * 2; }

template <int K>
fct_status launch_rownorm(const float* A, int64_t n, int d, int64_t lda, const float* M32, const double* M64T,
                          const float* colb, int k, float* lambda, double* partial, int grid, cudaStream_t st) {
  const size_t smem = smem_bytes(d, k, K);
  auto kern = rownorm_kernel<K>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const float u = 5.9604645e-08f;  // 2^-24
  const float gam = (float)(d + 3) * u * 1.1f;
  kern<<<grid, kRowThreads, smem, st>>>(A, n, d, lda, M32, M64T, colb, k, gam, lambda, partial);
  FCT_LAUNCHED("rownorm_kernel", st);
  return FCT_OK;
}

}  // namespace

extern "C" size_t l1_rownorm_workspace_bytes(int64_t n, int64_t d, int32_t k) {
  (void)n;
  if (d < 1 || k < 1) return 0;
  const int K = pad_k(k);
  return fct::align256(sizeof(double) * (size_t)k * d) + fct::align256(sizeof(float) * (size_t)d * K) +
         fct::align256(sizeof(float) * 2 * K) + fct::align256(sizeof(double) * (size_t)rownorm_grid()) +
         fct::align256(sizeof(double));
}

fct_status fct_rownorm_impl(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                            const float* Pi2, int32_t k, float* lambda, double* lambda_sum, bool zero_sum,
                            void* ws, size_t wsb, cudaStream_t st) {
  FCT_CHECK_ARG(A && Rinv && Pi2 && lambda, FCT_ERR_ARG, "l1_rownorm: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && d >= 1 && d <= FCT_MAX_D && lda >= d, FCT_ERR_SHAPE,
                "l1_rownorm: bad shape n=%lld d=%lld lda=%lld (d <= %d)", (long long)n, (long long)d,
                (long long)lda, FCT_MAX_D);
  FCT_CHECK_ARG(k >= 1 && k <= FCT_MAX_K, FCT_ERR_ARG, "l1_rownorm: k=%d not in [1, %d]", k, FCT_MAX_K);
  const size_t need = l1_rownorm_workspace_bytes(n, d, k);
  FCT_CHECK_ARG(ws && wsb >= need, FCT_ERR_WORKSPACE, "l1_rownorm: workspace %zu < %zu bytes", wsb, need);
  const int K = pad_k(k);
  fct::Carver cv(ws);
  double* M64T = cv.take<double>((size_t)k * d);
  float* M32 = cv.take<float>((size_t)d * K);
  float* colb = cv.take<float>(2 * K);
  const int grid = rownorm_grid();
  double* partial = cv.take<double>(grid);
  double* tmp_sum = cv.take<double>(1);
  form_m_kernel<<<(d * K + 127) / 128, 128, 0, st>>>(Rinv, Pi2, (int)d, k, K, M64T, M32, colb);
  FCT_LAUNCHED("form_m_kernel", st);
  colbound_kernel<<<1, 32, 0, st>>>(M32, (int)d, k, K, colb);
  FCT_LAUNCHED("colbound_kernel", st);
  fct_status rc;
  switch (K) {
#define CASE_K(KK) case KK: rc = launch_rownorm<KK>(A, n, (int)d, lda, M32, M64T, colb, k, lambda, partial, grid, st); break;
    CASE_K(4) CASE_K(8) CASE_K(12) CASE_K(16) CASE_K(20) CASE_K(24) CASE_K(28) CASE_K(32)
#undef CASE_K
    default: rc = FCT_ERR_UNSUPPORTED; fct::set_error("l1_rownorm: k=%d", k);
  }
  if (rc != FCT_OK) return rc;
  double* out = lambda_sum ? lambda_sum : tmp_sum;
  sum_partials_kernel<<<1, 256, 0, st>>>(partial, grid, out, (zero_sum || !lambda_sum) ? 1 : 0);
  FCT_LAUNCHED("sum_partials_kernel", st);
  return FCT_OK;
}

extern "C" fct_status l1_rownorm(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                                 const float* Pi2, int32_t k, float* lambda, double* lambda_sum,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(lambda_sum, FCT_ERR_ARG, "l1_rownorm: lambda_sum is NULL");
  return fct_rownorm_impl(A, n, d, lda, Rinv, Pi2, k, lambda, lambda_sum, false, workspace, workspace_bytes,
                          (cudaStream_t)stream);
}

extern "C" fct_status l1_probs(const float* lambda, int64_t n, const double* lambda_total, float* p,
                               void* stream) {
  FCT_CHECK_ARG(lambda && lambda_total && p, FCT_ERR_ARG, "l1_probs: NULL pointer");
  FCT_CHECK_ARG(n >= 1, FCT_ERR_SHAPE, "l1_probs: n=%lld", (long long)n);
  cudaStream_t st = (cudaStream_t)stream;
  probs_kernel<<<fct::num_sms() * 4, 256, 0, st>>>(lambda, n, lambda_total, p);
  FCT_LAUNCHED("probs_kernel", st);
  return FCT_OK;
}

extern "C" fct_status l1_rownorm_probs(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                                       const float* Pi2, int32_t k, float* lambda, float* p, double* lambda_sum,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  FCT_CHECK_ARG(p, FCT_ERR_ARG, "l1_rownorm_probs: p is NULL");
  // the total lives in the workspace when the caller passes NULL
  const size_t need = l1_rownorm_workspace_bytes(n, d, k);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_WORKSPACE,
                "l1_rownorm_probs: workspace %zu < %zu bytes", workspace_bytes, need);
  double* total = lambda_sum;
  if (!total) total = (double*)((char*)workspace + need - fct::align256(sizeof(double)));
  fct_status rc = fct_rownorm_impl(A, n, d, lda, Rinv, Pi2, k, lambda, total, true, workspace, workspace_bytes, st);
  if (rc != FCT_OK) return rc;
  return l1_probs(lambda, n, total, p, stream);
}
