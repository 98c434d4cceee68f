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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include "common.cuh"
#include "sortnet.cuh"
#include "selnet.cuh"

namespace {

constexpr int kRowThreads = 256;  // 8 warps, one row per thread, 32 rows per warp per step

// M = Rinv * Pi2 in fp64; also the fp32 copy (padded to KP columns, zeros) and
// per-column bounds (||m~_j||_2 rounded up, ||m~_j||_inf).
__global__ void form_m_kernel(const double* __restrict__ Rinv, const float* __restrict__ Pi2, int d,
                              int k, int KP, double* __restrict__ M64, float* __restrict__ M32,
                              float* __restrict__ colb) {
  // one thread per (l, j); M64 stored row-major [d][k]: a candidate column j is read with stride k, so
  // lanes with different candidates hit different banks (and equal candidates broadcast)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d * KP; e += gridDim.x * blockDim.x) {
    const int l = e / KP, j = e - l * KP;
    double acc = 0.0;
    if (j < k)
      for (int q = 0; q < d; ++q) acc = fma(Rinv[l * d + q], (double)Pi2[q * k + j], acc);
    M32[l * KP + j] = (float)acc;   // zero for the padding columns j >= k
    if (j < k) M64[l * k + j] = acc;
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

// Batcher odd-even merge sort of N (power of two) registers, ascending (explicit network, sortnet.cuh)
struct CSwap {
  __device__ __forceinline__ void operator()(float& a, float& b) const { cswap(a, b); }
};
template <int N>
__device__ __forceinline__ void sort_net(float (&a)[N]) {
  if constexpr (N == 8) sortnet8(a, CSwap{});
  else if constexpr (N == 16) sortnet16(a, CSwap{});
  else sortnet32(a, CSwap{});
}

template <int K>
struct SortN {
  static constexpr int value = K <= 8 ? 8 : (K <= 16 ? 16 : 32);
};

// K = padded column count (multiple of 4, >= k); NS = sorting width (power of two >= K)
template <int K>
__global__ void __launch_bounds__(kRowThreads)
rownorm_kernel(const float* __restrict__ A, int64_t n, int d, int64_t lda, const float* __restrict__ M32g,
               const double* __restrict__ M64g, const float* __restrict__ colbg, int k, float gam,
               float* __restrict__ lambda, double* __restrict__ partial) {
  constexpr int NS = SortN<K>::value;
  extern __shared__ unsigned char smraw[];
  float* M32 = (float*)smraw;                                   // [d][K]   (16-byte aligned rows)
  float* colb = M32 + (size_t)d * K;                            // [K][2]
  double* M64 = (double*)(colb + 2 * K);                       // [k][d]
  float* tiles = (float*)(M64 + (size_t)k * d);                // [8 warps][32][d+1]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ldt = d + 1;
  float* tile = tiles + (size_t)warp * 32 * ldt;

  for (int e = threadIdx.x; e < k * d; e += blockDim.x) M64[e] = M64g[e];
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
            double s = 0.0;
            for (int l = 0; l < d; ++l) s = fma((double)a[l], M64[l * k + j], s);
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
              double s = 0.0;
              for (int l = 0; l < d; ++l) s = fma((double)a[l], M64[l * k + j], s);
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

// ------------------------------------------------------------------------------------------------
// v1 (aligned rows, d % 4 == 0): warp tiles of 64 rows staged with cp.async (coalesced 16-B chunks)
// into a padded shared layout (conflict-free LDS.128 per row), 2 rows per thread so every broadcast
// LDS.128 of M feeds 8 FMAs; one sorting network per row (v only) and the certified-candidate rule
//   L' = v_(m1) - E, H' = v_(m2) + E, E = max_j e_j   (L' <= L_m1, H' >= H_m2: a candidate superset)
// followed by the exact fp64 recompute of the candidates.
// exact |sum_l a_l M_lj| in fp64 with 4 independent partial sums (short dependency chains)
__device__ __forceinline__ double exact_abs_dot(const float* __restrict__ arow, const double* __restrict__ mc, int k,
                                                int d) {
  // arow: 16-byte aligned row in shared memory (d % 4 == 0 in the v1 kernel); mc = &M64[0][j], stride k
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int l = 0; l < d; l += 4) {
    const float4 a = *(const float4*)(arow + l);
    s0 = fma((double)a.x, mc[(l + 0) * k], s0);
    s1 = fma((double)a.y, mc[(l + 1) * k], s1);
    s2 = fma((double)a.z, mc[(l + 2) * k], s2);
    s3 = fma((double)a.w, mc[(l + 3) * k], s3);
  }
  return fabs((s0 + s1) + (s2 + s3));
}

template <int K>
__device__ __forceinline__ float certified_median(const float (&acc)[K], float n1, float n2, const float* __restrict__ colb,
                                                  float gam, int k, int m1, int m2, const float* __restrict__ arow,
                                                  int d, const double* __restrict__ M64) {
  if (n1 == 0.f) return 0.f;
  const float nrm2 = __fsqrt_ru(n2) * 1.0001f;
  float srt[K];
  float E = 0.f;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const float v = fabsf(acc[j]);
    const float ej = j < k ? gam * fminf(nrm2 * colb[2 * j], n1 * colb[2 * j + 1]) + 1e-37f : 0.f;
    bad |= !(isfinite(v) && isfinite(ej));
    E = fmaxf(E, ej);
    srt[j] = j < k ? v : INFINITY;
  }
  // median-selection network for exactly k inputs (k in (K-4, K]; uniform across the grid)
  switch (K - k) {
    case 0: selnet<K>(srt, CSwap{}); break;
    case 1: if constexpr (K >= 2) selnet<(K >= 2 ? K - 1 : 1)>(srt, CSwap{}); break;
    case 2: if constexpr (K >= 3) selnet<(K >= 3 ? K - 2 : 1)>(srt, CSwap{}); break;
    default: if constexpr (K >= 4) selnet<(K >= 4 ? K - 3 : 1)>(srt, CSwap{}); break;
  }
  float v1 = 0.f, v2 = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j == m1) v1 = srt[j];
    if (j == m2) v2 = srt[j];
  }
  // L' = min over {j : v_j >= v_(m1)} of (v_j - e_j) <= L_m1 and H' = max over {j : v_j <= v_(m2)} of
  // (v_j + e_j) >= H_m2 (at most m1 lower bounds can lie below the first set's minimum, and symmetrically)
  float L = INFINITY, H = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < k) {
      const float v = fabsf(acc[j]);
      const float ej = gam * fminf(nrm2 * colb[2 * j], n1 * colb[2 * j + 1]) + 1e-37f;
      if (v >= v1) L = fminf(L, v - ej);
      if (v <= v2) H = fmaxf(H, v + ej);
    }
  }
  if (bad) { L = 0.f; H = INFINITY; }
  (void)E;
  int below = 0;
  unsigned cmask = 0u;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < k) {
      const float v = fabsf(acc[j]);
      const float ej = gam * fminf(nrm2 * colb[2 * j], n1 * colb[2 * j + 1]) + 1e-37f;
      if (!bad && v + ej < L) ++below;
      else if (bad || v - ej <= H) cmask |= 1u << j;
    }
  }
  const int r1 = m1 - below, r2 = m2 - below;
  const int nc = __popc(cmask);
  double x1 = 0.0, x2 = 0.0;
  if (nc <= 2) {
    const int j0 = __ffs(cmask) - 1;
    const double c0 = exact_abs_dot(arow, M64 + j0, k, d);
    double c1 = INFINITY;
    if (nc == 2) c1 = exact_abs_dot(arow, M64 + (31 - __clz(cmask)), k, d);
    const double cmin = fmin(c0, c1), cmax = fmax(c0, c1);
    x1 = r1 == 0 ? cmin : cmax;
    x2 = r2 == 0 ? cmin : cmax;
  } else {
    // rare: several candidates -- exact value of each once (local array), then rank by counting
    double ex[32];
    int idx[32];
    int m = 0;
    unsigned mj = cmask;
    while (mj) {
      const int j = __ffs(mj) - 1;
      mj &= mj - 1;
      ex[m] = exact_abs_dot(arow, M64 + j, k, d);
      idx[m++] = j;
    }
    for (int a = 0; a < m; ++a) {
      int rank = 0;
      for (int b = 0; b < m; ++b) rank += (ex[b] < ex[a]) || (ex[b] == ex[a] && idx[b] < idx[a]);
      if (rank == r1) x1 = ex[a];
      if (rank == r2) x2 = ex[a];
    }
  }
  return (float)(0.5 * (x1 + x2));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}

template <int K>
__global__ void __launch_bounds__(256)
rownorm_v1_kernel(const float* __restrict__ A, int64_t n, int d, int64_t lda, const float* __restrict__ M32g,
                  const double* __restrict__ M64g, const float* __restrict__ colbg, int k, float gam, int ldt,
                  float* __restrict__ lambda, double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float* M32 = (float*)smraw;                                     // [d][K]
  float* colb = M32 + (size_t)d * K;                              // [K][2]
  double* M64 = (double*)(colb + 2 * K);                         // [k][d]
  float* tiles = (float*)(M64 + (size_t)k * d);                  // [warps][64][ldt]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* tile = tiles + (size_t)warp * 64 * ldt;
  for (int e = threadIdx.x; e < k * d; e += blockDim.x) M64[e] = M64g[e];
  for (int e = threadIdx.x; e < d * K; e += blockDim.x) M32[e] = M32g[e];
  for (int e = threadIdx.x; e < 2 * K; e += blockDim.x) colb[e] = colbg[e];
  __syncthreads();
  const int m1 = (k - 1) / 2, m2 = k / 2;
  const int q4 = d >> 2;                  // 16-B chunks per row
  double local = 0.0;
  const int64_t ntiles = (n + 63) / 64;
  for (int64_t tid = (int64_t)blockIdx.x * nw + warp; tid < ntiles; tid += (int64_t)gridDim.x * nw) {
    const int64_t row0 = tid * 64;
    const int nr = (int)(n - row0 < 64 ? n - row0 : 64);
    __syncwarp();
    for (int q = lane; q < 64 * q4; q += 32) {
      const int r = q / q4, c4 = q - r * q4;
      const bool ok = r < nr;
      cp_async16(tile + r * ldt + 4 * c4, A + (row0 + (ok ? r : 0)) * lda + 4 * c4, ok);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    const float* ar0 = tile + lane * ldt;
    const float* ar1 = tile + (lane + 32) * ldt;
    float acc0[K], acc1[K];
#pragma unroll
    for (int j = 0; j < K; ++j) { acc0[j] = 0.f; acc1[j] = 0.f; }
    float n10 = 0.f, n20 = 0.f, n11 = 0.f, n21 = 0.f;
#pragma unroll 2
    for (int l4 = 0; l4 < q4; ++l4) {
      const float4 a0 = *(const float4*)(ar0 + 4 * l4);
      const float4 a1 = *(const float4*)(ar1 + 4 * l4);
      n10 += fabsf(a0.x) + fabsf(a0.y) + fabsf(a0.z) + fabsf(a0.w);
      n11 += fabsf(a1.x) + fabsf(a1.y) + fabsf(a1.z) + fabsf(a1.w);
      n20 = fmaf(a0.x, a0.x, fmaf(a0.y, a0.y, fmaf(a0.z, a0.z, fmaf(a0.w, a0.w, n20))));
      n21 = fmaf(a1.x, a1.x, fmaf(a1.y, a1.y, fmaf(a1.z, a1.z, fmaf(a1.w, a1.w, n21))));
      const float av0[4] = {a0.x, a0.y, a0.z, a0.w}, av1[4] = {a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int ll = 0; ll < 4; ++ll) {
        const float4* mrow = (const float4*)(M32 + (4 * l4 + ll) * K);
#pragma unroll
        for (int j4 = 0; j4 < K / 4; ++j4) {
          const float4 mv = mrow[j4];
          acc0[4 * j4 + 0] = fmaf(av0[ll], mv.x, acc0[4 * j4 + 0]);
          acc0[4 * j4 + 1] = fmaf(av0[ll], mv.y, acc0[4 * j4 + 1]);
          acc0[4 * j4 + 2] = fmaf(av0[ll], mv.z, acc0[4 * j4 + 2]);
          acc0[4 * j4 + 3] = fmaf(av0[ll], mv.w, acc0[4 * j4 + 3]);
          acc1[4 * j4 + 0] = fmaf(av1[ll], mv.x, acc1[4 * j4 + 0]);
          acc1[4 * j4 + 1] = fmaf(av1[ll], mv.y, acc1[4 * j4 + 1]);
          acc1[4 * j4 + 2] = fmaf(av1[ll], mv.z, acc1[4 * j4 + 2]);
          acc1[4 * j4 + 3] = fmaf(av1[ll], mv.w, acc1[4 * j4 + 3]);
        }
      }
    }
    if (lane < nr) {
      const float lam = certified_median<K>(acc0, n10, n20, colb, gam, k, m1, m2, ar0, d, M64);
      lambda[row0 + lane] = lam;
      local += (double)lam;
    }
    if (lane + 32 < nr) {
      const float lam = certified_median<K>(acc1, n11, n21, colb, gam, k, m1, m2, ar1, d, M64);
      lambda[row0 + lane + 32] = lam;
      local += (double)lam;
    }
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) red[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0;
    for (int w = 0; w < nw; ++w) s2 += red[w];
    partial[blockIdx.x] = s2;
  }
}

// ------------------------------------------------------------------------------------------------
// tc: helpers for the tcgen05 row-norm kernel below (ws; the ws2 kernel in rownorm_ws2.cu is the default for
// the five configurations' k).  The contraction Lambda = A M runs on the 5th-generation tensor cores
// (kind::tf32, 3xTF32): D = A*M_hi + A*M_lo + A_lo*M_hi, A_hi = trunc_tf32(A) (the MMA's own operand
// truncation), A_lo = A - A_hi (exact in fp32, written to TMEM by the threads), M_hi/M_lo likewise.
// Tiles = 128 rows x Kp (Kp = d rounded up to 32) fp32, TMA-loaded with SWIZZLE_128B (K-major canonical
// layout for the UMMA descriptor); D lives in TMEM; error bound of the 3xTF32 evaluation: measured max
// |err| = 1.9e-6 * sum|a m| on the box, bound used 2^-14 * 1.05 * min(||a||_2 ||m~_j||_2, ||a||_1 ||m~_j||_inf).
// (The single-role double-buffered tc kernel that preceded ws was superseded by it and removed in round 2.)
namespace tc {
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(const void* p) {   // K-major SWIZZLE_128B, SBO = 1024 B
  const uint64_t a = (su32(p) >> 4) & 0x3FFF;
  return a | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ float trunc_tf32(float x) { return __int_as_float(__float_as_int(x) & 0xFFFFE000); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nTW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra TW_%=;\n}\n" ::"r"(
                   su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_tile(float* dst, const CUtensorMap* map, int nchunk, int row0, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(nchunk * 16384) : "memory");
  for (int q = 0; q < nchunk; ++q)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(dst + q * 128 * 32)), "l"(map), "r"(q * 32), "r"(row0), "r"(su32(bar)) : "memory");
}
#define TC_R32 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32}"
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " TC_R32 ";" ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]),
               "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]),
               "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
               "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
               "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                 "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                 "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                 "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
}  // namespace tc

// ------------------------------------------------------------------------------------------------
// ws: warp-specialised tcgen05 row-norm (one persistent CTA per SM, 16 warps).
//   warps 0-3  ("split"): wait for the TMA'd tile, thread r <-> row r <-> TMEM lane r: norms -> smem,
//              A_lo = A - trunc_tf32(A) -> TMEM; thread 0 issues the 3xTF32 MMAs into a rotating D buffer
//              and the TMA loads (NA tile buffers ahead).
//   warps 4-15 (3 epilogue groups of 4): group g takes tiles i = g (mod 3): tcgen05.ld D, certified
//              median (candidates recomputed in fp64 from the row in global memory / L2), lambda.
// All hand-offs are mbarriers; no CTA-wide barrier in the steady state.
namespace wsk {
constexpr int kSplitWarps = 4, kEpiGroups = 3, kThreads = 32 * (kSplitWarps + 4 * kEpiGroups);
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nWW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra WW_%=;\n}\n"
               ::"r"(tc::su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc::su32(b)) : "memory");
}
// exact |sum_l a_l M_lj| in fp64, row from global memory (16-byte aligned, d % 4 == 0)
__device__ __forceinline__ double exact_abs_dot_g(const float* __restrict__ arow, const double* __restrict__ mc, int k,
                                                  int d) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int l = 0; l < d; l += 4) {
    const float4 a = __ldg((const float4*)(arow + l));
    s0 = fma((double)a.x, mc[(l + 0) * k], s0);
    s1 = fma((double)a.y, mc[(l + 1) * k], s1);
    s2 = fma((double)a.z, mc[(l + 2) * k], s2);
    s3 = fma((double)a.w, mc[(l + 3) * k], s3);
  }
  return fabs((s0 + s1) + (s2 + s3));
}
}  // namespace wsk

template <int K>
__device__ __forceinline__ float certified_median_g(const float (&acc)[K], float n1, float n2,
                                                    const float* __restrict__ colb, float gam, int k, int m1, int m2,
                                                    const float* __restrict__ arow, int d,
                                                    const double* __restrict__ M64) {
  if (n1 == 0.f) return 0.f;
  const float nrm2 = __fsqrt_ru(n2) * 1.0001f;
  float srt[K], e[K];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const float v = fabsf(acc[j]);
    e[j] = j < k ? gam * fminf(nrm2 * colb[2 * j], n1 * colb[2 * j + 1]) + 1e-37f : 0.f;
    bad |= !(isfinite(v) && isfinite(e[j]));
    srt[j] = j < k ? v : INFINITY;
  }
  switch (K - k) {
    case 0: selnet<K>(srt, CSwap{}); break;
    case 1: if constexpr (K >= 2) selnet<(K >= 2 ? K - 1 : 1)>(srt, CSwap{}); break;
    case 2: if constexpr (K >= 3) selnet<(K >= 3 ? K - 2 : 1)>(srt, CSwap{}); break;
    default: if constexpr (K >= 4) selnet<(K >= 4 ? K - 3 : 1)>(srt, CSwap{}); break;
  }
  float v1 = 0.f, v2 = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j == m1) v1 = srt[j];
    if (j == m2) v2 = srt[j];
  }
  float L = INFINITY, H = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < k) {
      const float v = fabsf(acc[j]);
      if (v >= v1) L = fminf(L, v - e[j]);
      if (v <= v2) H = fmaxf(H, v + e[j]);
    }
  }
  if (bad) { L = 0.f; H = INFINITY; }
  int below = 0;
  unsigned cmask = 0u;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < k) {
      const float v = fabsf(acc[j]);
      if (!bad && v + e[j] < L) ++below;
      else if (bad || v - e[j] <= H) cmask |= 1u << j;
    }
  }
  const int r1 = m1 - below, r2 = m2 - below;
  const int nc = __popc(cmask);
  double x1 = 0.0, x2 = 0.0;
  if (nc <= 2) {
    const int j0 = __ffs(cmask) - 1;
    const double c0 = wsk::exact_abs_dot_g(arow, M64 + j0, k, d);
    double c1 = INFINITY;
    if (nc == 2) c1 = wsk::exact_abs_dot_g(arow, M64 + (31 - __clz(cmask)), k, d);
    const double cmin = fmin(c0, c1), cmax = fmax(c0, c1);
    x1 = r1 == 0 ? cmin : cmax;
    x2 = r2 == 0 ? cmin : cmax;
  } else {
    double ex[32];
    int idx[32];
    int m = 0;
    unsigned mj = cmask;
    while (mj) {
      const int j = __ffs(mj) - 1;
      mj &= mj - 1;
      ex[m] = wsk::exact_abs_dot_g(arow, M64 + j, k, d);
      idx[m++] = j;
    }
    for (int a = 0; a < m; ++a) {
      int rank = 0;
      for (int b = 0; b < m; ++b) rank += (ex[b] < ex[a]) || (ex[b] == ex[a] && idx[b] < idx[a]);
      if (rank == r1) x1 = ex[a];
      if (rank == r2) x2 = ex[a];
    }
  }
  return (float)(0.5 * (x1 + x2));
}

template <int K>
__global__ void __launch_bounds__(wsk::kThreads, 1)
rownorm_ws_kernel(const __grid_constant__ CUtensorMap tmA, const float* __restrict__ A, int64_t n, int d, int64_t lda,
                  const float* __restrict__ M32g, const double* __restrict__ M64g, const float* __restrict__ colbg,
                  int k, float gam, int NA, int ND, float* __restrict__ lambda, double* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* base = smraw + ((1024u - (tc::su32(smraw) & 1023u)) & 1023u);
  const int nch = (d + 31) >> 5;
  const int KP = nch * 32;
  const int tile_floats = nch * 128 * 32;
  float* sA = (float*)base;                          // [NA][nch][128][32] (SW128)
  float* sMhi = sA + NA * tile_floats;               // [nch][32][32] (SW128)
  float* sMlo = sMhi + nch * 32 * 32;
  double* M64 = (double*)(sMlo + nch * 32 * 32);     // [d][k]
  float* colb = (float*)(M64 + (size_t)d * k);       // [K][2]
  float* norms = colb + 2 * K;                       // [ND][128][2]
  uint64_t* bars = (uint64_t*)(norms + (size_t)ND * 256 + 2);   // 8-aligned (offsets are multiples of 8 B)
  uint64_t* tma_full = bars;                 // [NA]
  uint64_t* a_free = tma_full + NA;          // [NA]   MMA done with the smem tile
  uint64_t* alo_free = a_free + NA;          // [2]    MMA done with the TMEM A_lo buffer
  uint64_t* d_full = alo_free + 2;           // [ND]   MMA result ready
  uint64_t* n_full = d_full + ND;            // [ND]   norms written (128 arrivals)
  uint64_t* d_free = n_full + ND;            // [ND]   epilogue done (4 arrivals)
  __shared__ uint32_t tbase;
  __shared__ double red[wsk::kThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int i = 0; i < NA; ++i) { wsk::init(&tma_full[i], 1); wsk::init(&a_free[i], 1); }
    for (int i = 0; i < 2; ++i) wsk::init(&alo_free[i], 1);
    for (int i = 0; i < ND; ++i) { wsk::init(&d_full[i], 1); wsk::init(&n_full[i], 128); wsk::init(&d_free[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int e = tid; e < 32 * KP; e += blockDim.x) {
    const int j = e / KP, l = e - j * KP;
    const float m = (j < K && l < d) ? M32g[l * K + j] : 0.f;
    const float hi = tc::trunc_tf32(m), lo = m - hi;
    const int off = (l >> 5) * 32 * 32 + j * 32 + ((((l & 31) >> 2) ^ (j & 7)) << 2) + (l & 3);
    sMhi[off] = hi;
    sMlo[off] = lo;
  }
  for (int e = tid; e < k * d; e += blockDim.x) M64[e] = M64g[e];
  for (int e = tid; e < 2 * K; e += blockDim.x) colb[e] = colbg[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t dcol0 = 2u * KP;   // D buffers after the two A_lo buffers
  const int64_t ntiles = (n + 127) / 128;
  const int64_t t0 = blockIdx.x, tstep = gridDim.x;
  const int64_t my_tiles = t0 < ntiles ? (ntiles - 1 - t0) / tstep + 1 : 0;
  double local = 0.0;

  if (warp < wsk::kSplitWarps) {
    // ------------------------------------------------------------------ split + MMA issue + TMA
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int ksteps = (d + 7) >> 3;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    if (tid == 0)
      for (int64_t i = 0; i < my_tiles && i < NA; ++i)
        tc::tma_tile(sA + (i % NA) * tile_floats, &tmA, nch, (int)((t0 + i * tstep) * 128), &tma_full[i % NA]);
    for (int64_t i = 0; i < my_tiles; ++i) {
      const int sa = (int)(i % NA), sd = (int)(i % ND), sl = (int)(i & 1);
      wsk::wait(&tma_full[sa], (unsigned)((i / NA) & 1));
      if (i >= 2) wsk::wait(&alo_free[sl], (unsigned)(((i - 2) >> 1) & 1));
      if (i >= ND) wsk::wait(&d_free[sd], (unsigned)(((i - ND) / ND) & 1));
      const float* tile = sA + sa * tile_floats;
      float s1 = 0.f, s2 = 0.f;
      for (int q = 0; q < nch; ++q) {
        uint32_t lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *(const float4*)(tile + q * 128 * 32 + tid * 32 + ((c ^ (tid & 7)) << 2));
          const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            s1 += fabsf(a[w]);
            s2 = fmaf(a[w], a[w], s2);
            lo[c * 4 + w] = __float_as_uint(a[w] - tc::trunc_tf32(a[w]));
          }
        }
        tc::st32(tm + lane_off + (uint32_t)(sl * KP + q * 32), lo);
      }
      norms[(sd * 128 + tid) * 2] = s1;
      norms[(sd * 128 + tid) * 2 + 1] = s2;
      wsk::arrive(&n_full[sd]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tD = tm + dcol0 + (uint32_t)(sd * 32);
        int cnt = 0;
        for (int pass = 0; pass < 3; ++pass) {
          const float* Bm = pass == 1 ? sMlo : sMhi;
          for (int ks = 0; ks < ksteps; ++ks) {
            const int q = ks >> 2, kin = ks & 3;
            const uint64_t bd = tc::sdesc((const unsigned char*)(Bm + q * 32 * 32) + kin * 32);
            const uint32_t accf = cnt > 0 ? 1u : 0u;
            if (pass < 2) {
              const uint64_t ad = tc::sdesc((const unsigned char*)(tile + q * 128 * 32) + kin * 32);
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                           ::"r"(tD), "l"(ad), "l"(bd), "r"(idesc), "r"(accf));
            } else {
              const uint32_t ta = tm + (uint32_t)(sl * KP + ks * 8);
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                           ::"r"(tD), "r"(ta), "l"(bd), "r"(idesc), "r"(accf));
            }
            ++cnt;
          }
        }
        wsk::commit(&d_full[sd]);
        wsk::commit(&alo_free[sl]);
        wsk::commit(&a_free[sa]);
        // refill the tile buffer of the previous tile once its MMA is done
        if (i >= 1 && i - 1 + NA < my_tiles) {
          const int pa = (int)((i - 1) % NA);
          wsk::wait(&a_free[pa], (unsigned)(((i - 1) / NA) & 1));
          tc::tma_tile(sA + pa * tile_floats, &tmA, nch, (int)((t0 + (i - 1 + NA) * tstep) * 128), &tma_full[pa]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue groups
    const int ew = warp - wsk::kSplitWarps;
    const int g = ew >> 2, qd = ew & 3;
    const int m1 = (k - 1) / 2, m2 = k / 2;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    for (int64_t i = g; i < my_tiles; i += wsk::kEpiGroups) {
      const int sd = (int)(i % ND);
      const unsigned ph = (unsigned)((i / ND) & 1);
      wsk::wait(&d_full[sd], ph);
      wsk::wait(&n_full[sd], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t dv[32];
      tc::ld32(tm + lane_off + dcol0 + (uint32_t)(sd * 32), dv);
      const int r = qd * 32 + lane;
      const float n1 = norms[(sd * 128 + r) * 2], n2 = norms[(sd * 128 + r) * 2 + 1];
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) wsk::arrive(&d_free[sd]);   // D and the norms are in registers
      float acc[K];
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] = __uint_as_float(dv[j]);
      const int64_t row = (t0 + i * tstep) * 128 + r;
      if (row < n) {
        const float lam = certified_median_g<K>(acc, n1, n2, colb, gam, k, m1, m2, A + row * lda, d, M64);
        lambda[row] = lam;
        local += (double)lam;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) red[warp] = local;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < wsk::kThreads / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
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

int v1_ldt(int d) {
  int q = d / 4 + 1;
  if (!(q & 1)) ++q;   // odd number of 16-B chunks per staged row -> conflict-free LDS.128
  return 4 * q;
}
size_t v1_fixed_smem(int d, int k, int K) {
  return sizeof(float) * ((size_t)d * K + 2 * K) + sizeof(double) * (size_t)k * d;
}
int v1_warps(int d, int k, int K) {
  const size_t per = sizeof(float) * 64 * (size_t)v1_ldt(d);
  const size_t budget = 200 * 1024;
  const size_t fixed = v1_fixed_smem(d, k, K);
  if (fixed + per > budget) return 0;
  return (int)std::min<size_t>(8, (budget - fixed) / per);
}
bool v1_ok(const float* A, int d, int64_t lda, int k, int K) {
  return d % 4 == 0 && lda % 4 == 0 && ((uintptr_t)A & 15) == 0 && v1_warps(d, k, K) >= 1;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

bool tc_ok(const float* A, int64_t n, int d, int64_t lda) {
  return !getenv("FCT_ROWNORM_SIMT") && d % 4 == 0 && d <= 128 && lda % 4 == 0 && ((uintptr_t)A & 15) == 0 &&
         n < (1LL << 31) && encode_fn() != nullptr;
}

template <int K>
fct_status launch_ws(const float* A, int64_t n, int d, int64_t lda, const float* M32, const double* M64,
                     const float* colb, int k, float* lambda, double* partial, int grid, cudaStream_t st) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(float)};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  FCT_CHECK_ARG(cr == CUDA_SUCCESS, FCT_ERR_CUDA, "l1_rownorm: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  const int nch = (d + 31) / 32, KP = nch * 32;
  const int ND = (512 - 2 * KP) / 32;               // D buffers in TMEM after two A_lo buffers
  const size_t fixed = 1024 + sizeof(float) * (2 * (size_t)nch * 32 * 32) + sizeof(double) * (size_t)k * d +
                       sizeof(float) * (2 * K + (size_t)ND * 256 + 2) + sizeof(uint64_t) * (3 * (size_t)ND + 2 + 2 * 4);
  const size_t tileb = sizeof(float) * (size_t)nch * 128 * 32;
  const size_t budget = 232448 - 2048;
  int NA = (int)std::min<size_t>(4, (budget - fixed) / tileb);
  if (NA < 2 || ND < 4) return FCT_ERR_UNSUPPORTED;
  const size_t smem = fixed + tileb * NA;
  auto kern = rownorm_ws_kernel<K>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int g = std::max(1, std::min(grid, fct::num_sms()));
  if (fct::debug_sync()) fprintf(stderr, "[fct] rownorm_ws: grid %d NA %d ND %d smem %zu\n", g, NA, ND, smem);
  const float gam = 6.103515625e-05f * 1.05f;   // 3xTF32 bound (see the tc helpers above)
  FCT_CUDA_RET(cudaMemsetAsync(partial, 0, sizeof(double) * grid, st));
  kern<<<g, wsk::kThreads, smem, st>>>(map, A, n, d, lda, M32, M64, colb, k, gam, NA, ND, lambda, partial);
  FCT_LAUNCHED("rownorm_ws_kernel", st);
  return FCT_OK;
}

template <int K>
fct_status launch_rownorm(const float* A, int64_t n, int d, int64_t lda, const float* M32, const double* M64,
                          const float* colb, int k, float* lambda, double* partial, int grid, cudaStream_t st) {
  // dispatch: ws2 (instances for the configurations' k) -> ws (any k; tcgen05) -> v1 / SIMT (unaligned A,
  // d % 4 != 0, d > 128, or a shared-memory budget ws cannot meet)
  if (tc_ok(A, n, d, lda)) {
    const fct_status r2 = fct_rownorm_ws2(A, n, d, lda, M32, K, M64, colb, k, partial, grid, lambda, st);
    if (r2 != FCT_ERR_UNSUPPORTED) return r2;
    const fct_status r = launch_ws<K>(A, n, d, lda, M32, M64, colb, k, lambda, partial, grid, st);
    if (r != FCT_ERR_UNSUPPORTED) return r;
  }
  const float u = 5.9604645e-08f;  // 2^-24
  const float gam1 = (float)(d + 3) * u * 1.1f;
  if (v1_ok(A, d, lda, k, K)) {
    const int nw = v1_warps(d, k, K);
    const int ldt = v1_ldt(d);
    const size_t smem1 = v1_fixed_smem(d, k, K) + sizeof(float) * 64 * (size_t)ldt * nw;
    auto kern1 = rownorm_v1_kernel<K>;
    FCT_CUDA_RET(cudaFuncSetAttribute(kern1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
    int occ = 1;
    FCT_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern1, nw * 32, smem1));
    const int g1 = std::max(1, std::min(grid, fct::num_sms() * std::max(occ, 1)));
    FCT_CUDA_RET(cudaMemsetAsync(partial, 0, sizeof(double) * grid, st));
    kern1<<<g1, nw * 32, smem1, st>>>(A, n, d, lda, M32, M64, colb, k, gam1, ldt, lambda, partial);
    FCT_LAUNCHED("rownorm_v1_kernel", st);
    return FCT_OK;
  }
  const size_t smem = smem_bytes(d, k, K);
  auto kern = rownorm_kernel<K>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kRowThreads, smem, st>>>(A, n, d, lda, M32, M64, colb, k, gam1, lambda, partial);
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
  double* M64 = cv.take<double>((size_t)k * d);
  float* M32 = cv.take<float>((size_t)d * K);
  float* colb = cv.take<float>(2 * K);
  const int grid = rownorm_grid();
  double* partial = cv.take<double>(grid);
  double* tmp_sum = cv.take<double>(1);
  form_m_kernel<<<(d * K + 127) / 128, 128, 0, st>>>(Rinv, Pi2, (int)d, k, K, M64, M32, colb);
  FCT_LAUNCHED("form_m_kernel", st);
  colbound_kernel<<<1, 32, 0, st>>>(M32, (int)d, k, K, colb);
  FCT_LAUNCHED("colbound_kernel", st);
  fct_status rc;
  switch (K) {
#define CASE_K(KK) case KK: rc = launch_rownorm<KK>(A, n, (int)d, lda, M32, M64, colb, k, lambda, partial, grid, st); break;
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
