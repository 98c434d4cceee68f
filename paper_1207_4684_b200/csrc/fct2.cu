// fct2.cu -- NEXT-3: the FCT2 sketch  Y = Pi1 A,  Pi1 = (8/r1) sqrt(pi t/(2s)) C H~
// (Sec. 3.2; running time P:L839-854).
//   H~ = blockdiag(G, ..., G) over t-row blocks (the SAME G in every block), G the SRHT of the
//   paper's experiments: G = sqrt(t/s) R (H_t / sqrt t) D_t, R = the rows `sel` of H_t.
//   C  = r1 x (nb s) i.i.d. Cauchy, passed in (row-major, ldc).
// Two kernels:
//   srht_kernel   one CTA per (t-block, column slice): the block's rows x DT columns in shared memory (swizzled
//                 column-major), D_t, in-place Walsh-Hadamard in register passes of up to 5 index bits
//                 (3 passes for t = 8192), rows `sel` scaled by 1/sqrt(s) -> Z (nb s x d)
//   cz_kernel     Y += C Z: split-K over the nb s columns of C, 64 x 64 output tiles, 4 x 4 fp32 register
//                 micro-tiles (a 128 x 64 tile with 8 x 4 micro-tiles measured slower: 34.0 vs 31.2 ms at cfg 4); the fp32 partials are folded into fp64 every 256 K (hierarchical accumulation as
//                 in K1) and added into an fp64 workspace; a last kernel writes Y = (float)(kappa W).
// This is the first correct version: the contraction is FP32-SIMT bound (r1 d nb s FMA).
#include <math.h>
#include "common.cuh"
#include "tc.cuh"

namespace {

constexpr int kSrhtThreads = 512;

// tile layout: column-major [DT][t] with the row index swizzled inside each 32-row chunk, phys(r) = r ^ ((r >> 5) & 31):
// a thread holding 32 consecutive rows (lanes = consecutive chunks) and a warp reading 32 consecutive rows
// (lanes = consecutive rows) both hit 32 distinct banks
__device__ __forceinline__ int phys(int r) { return r ^ ((r >> 5) & 31); }

// one radix-2^lb pass of the unnormalised Walsh-Hadamard transform over index bits [lo, lo + lb) of every
// column: a thread loads the R = 2^lb elements base + (i << lo), transforms them in registers, stores them back
template <int LB>
__device__ __forceinline__ void wht_pass(float* __restrict__ T, int t, int CS, int DT, int lo) {
  constexpr int R = 1 << LB;
  const int lgroups = __ffs(t) - 1 - LB;           // log2(groups per column)
  for (int g = threadIdx.x; g < (DT << lgroups); g += blockDim.x) {
    const int c = g >> lgroups, q = g & ((1 << lgroups) - 1);
    const int base = (q & ((1 << lo) - 1)) | ((q >> lo) << (lo + LB));
    float* col = T + (size_t)c * CS;
    float v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = col[phys(base + (i << lo))];
#pragma unroll
    for (int h = 1; h < R; h <<= 1)
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (!(i & h)) {
          const float a = v[i], b = v[i + h];
          v[i] = a + b;
          v[i + h] = a - b;
        }
#pragma unroll
    for (int i = 0; i < R; ++i) col[phys(base + (i << lo))] = v[i];
  }
}

template <int LDT>   // DT = 2^LDT columns per CTA
__global__ void __launch_bounds__(kSrhtThreads)
srht_kernel(const float* __restrict__ A, int64_t n, int d, int64_t lda, const int8_t* __restrict__ signs_t,
            const int32_t* __restrict__ sel, int t, int s, float inv_sqrt_s, float* __restrict__ Z, int ldz,
            float* __restrict__ Zh, float* __restrict__ Zl, int64_t ldzt) {
  constexpr int DT = 1 << LDT;
  extern __shared__ float T[];   // [DT][CS], rows swizzled (phys); CS = t + 8 spreads the columns over the banks
  const int CS = t + 8;
  const int c0 = blockIdx.x * DT;
  const int64_t b = blockIdx.y;
  const int64_t row0 = b * t;
  // load D_t A_b: 8 independent global loads in flight per thread before the shared stores
  const int total = t << LDT;
  for (int e0 = threadIdx.x; e0 < total; e0 += 8 * kSrhtThreads) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kSrhtThreads;
      const int r = e >> LDT, c = e & (DT - 1);
      const int64_t row = row0 + r;
      const int col = c0 + c;
      v[u] = (e < total && row < n && col < d) ? __ldg(A + row * lda + col) * (float)__ldg(signs_t + r) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kSrhtThreads;
      if (e < total) T[(e & (DT - 1)) * CS + phys(e >> LDT)] = v[u];
    }
  }
  __syncthreads();
  // index bits in ceil(lt / 5) balanced passes of at most 5 bits (t = 2048: 4 + 4 + 3, t = 8192: 5 + 4 + 4)
  const int lt = __ffs(t) - 1;
  const int np = (lt + 4) / 5;
  for (int lo = 0, pi = 0; lo < lt; ++pi) {
    const int lb = (lt - lo + (np - pi) - 1) / (np - pi);
    switch (lb) {
      case 5: wht_pass<5>(T, t, CS, DT, lo); break;
      case 4: wht_pass<4>(T, t, CS, DT, lo); break;
      case 3: wht_pass<3>(T, t, CS, DT, lo); break;
      case 2: wht_pass<2>(T, t, CS, DT, lo); break;
      default: wht_pass<1>(T, t, CS, DT, lo); break;
    }
    __syncthreads();
    lo += lb;
  }
  if (Zh) {
    // transposed tf32 split for the tensor-core contraction: Zh[col][b s + i] = tf32(z), Zl = z - tf32(z)
    for (int e = threadIdx.x; e < (s << LDT); e += blockDim.x) {
      const int c = e / s, i = e - c * s;
      const int col = c0 + c;
      if (col < d) {
        const float v = T[c * CS + phys(__ldg(sel + i))] * inv_sqrt_s;
        const float hi = tcx::trunc_tf32(v);
        Zh[(int64_t)col * ldzt + b * s + i] = hi;
        Zl[(int64_t)col * ldzt + b * s + i] = v - hi;
      }
    }
    return;
  }
  for (int e = threadIdx.x; e < (s << LDT); e += blockDim.x) {
    const int i = e >> LDT, c = e & (DT - 1);
    const int col = c0 + c;
    if (col < d) Z[(b * s + i) * ldz + col] = T[c * CS + phys(__ldg(sel + i))] * inv_sqrt_s;
  }
}

constexpr int BM = 64, BN = 64, BK = 16, FLUSH = 16;   // flush the fp32 partials every FLUSH * BK = 256 K

__global__ void __launch_bounds__(256)
cz_kernel(const float* __restrict__ C, int64_t ldc, const float* __restrict__ Z, int ldz, int r1, int d, int64_t K,
          int64_t kchunk, double* __restrict__ W) {
  __shared__ float Cs[BK][BM + 4];
  __shared__ float Zs[BK][BN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int64_t kb = (int64_t)blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  float acc[4][4];
  double acc64[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[i][j] = 0.f;
      acc64[i][j] = 0.0;
    }
  int steps = 0;
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {   // C tile: 64 rows x 16 k, thread -> (row, 4 k)
      const int e = threadIdx.x * 4 + u;
      const int rr = e / BK, kk = e - rr * BK;
      const int64_t k = k0 + kk;
      Cs[kk][rr] = (m0 + rr < r1 && k < ke) ? __ldg(C + (int64_t)(m0 + rr) * ldc + k) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {   // Z tile: 16 k x 64 columns
      const int e = threadIdx.x * 4 + u;
      const int kk = e / BN, cc = e - kk * BN;
      const int64_t k = k0 + kk;
      Zs[kk][cc] = (k < ke && n0 + cc < d) ? __ldg(Z + k * ldz + n0 + cc) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], z[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Cs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) z[j] = Zs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], z[j], acc[i][j]);
    }
    __syncthreads();
    if (++steps == FLUSH) {
      steps = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc64[i][j] += (double)acc[i][j];
          acc[i][j] = 0.f;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      const double v = acc64[i][j] + (double)acc[i][j];
      if (r < r1 && c < d && v != 0.0) atomicAdd(&W[(int64_t)r * d + c], v);
    }
}

__global__ void finalize_kernel(const double* __restrict__ W, int64_t count, double kappa, float* __restrict__ Y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    Y[i] = (float)(kappa * W[i]);
}

int slice_width(int t) { return std::max(1, std::min(8, 32768 / t)); }   // <= 128 KB tile (DT = 2 at t = 8192: 25.1 vs 20.8 ms)

template <int LDT>
fct_status launch_srht(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs_t, const int32_t* sel,
                       int t, int s, float* Z, float* Zh, float* Zl, int64_t ldzt, int64_t nb, cudaStream_t st) {
  constexpr int DT = 1 << LDT;
  const size_t smem = (size_t)DT * (t + 8) * sizeof(float);
  FCT_CUDA_RET(cudaFuncSetAttribute(srht_kernel<LDT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  srht_kernel<LDT><<<dim3((unsigned)((d + DT - 1) / DT), (unsigned)nb), kSrhtThreads, smem, st>>>(
      A, n, (int)d, lda, signs_t, sel, t, s, (float)(1.0 / sqrt((double)s)), Z, (int)d, Zh, Zl, ldzt);
  FCT_LAUNCHED("fct2 srht_kernel", st);
  return FCT_OK;
}

}  // namespace

extern "C" size_t fct2_workspace_bytes(int64_t n, int64_t d, int32_t t, int32_t s, int32_t r1) {
  if (n < 1 || d < 1 || t < 1 || s < 1 || r1 < 1) return 0;
  const int64_t nb = (n + t - 1) / t;
  const int64_t K = nb * s, ldzt = (K + 3) / 4 * 4;
  fct::Carver c(nullptr);
  c.take<float>(std::max((size_t)K * (size_t)d, 2 * (size_t)d * (size_t)ldzt));   // Z, or Z^T hi | lo
  c.take<double>((size_t)r1 * (size_t)d);                                       // W
  return c.off;
}

extern "C" fct_status fct2_sketch(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs_t,
                                  const int32_t* sel, const float* C, int64_t ldc, int32_t t, int32_t s, int32_t r1,
                                  float* Y, void* workspace, size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(A && signs_t && sel && C && Y, FCT_ERR_ARG, "fct2_sketch: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && d >= 1 && lda >= d && r1 >= 1, FCT_ERR_SHAPE, "fct2_sketch: n=%lld d=%lld lda=%lld r1=%d",
                (long long)n, (long long)d, (long long)lda, r1);
  FCT_CHECK_ARG(fct::is_pow2(t) && t <= 32768 && s >= 1 && s <= t, FCT_ERR_ARG,
                "fct2_sketch: t=%d must be a power of two <= 32768 and 1 <= s=%d <= t", t, s);
  const int64_t nb = (n + t - 1) / t, K = nb * s;
  FCT_CHECK_ARG(ldc >= K, FCT_ERR_SHAPE, "fct2_sketch: ldc=%lld < nb*s=%lld", (long long)ldc, (long long)K);
  FCT_CHECK_ARG(nb <= 65535, FCT_ERR_UNSUPPORTED, "fct2_sketch: %lld blocks > 65535", (long long)nb);
  const size_t need = fct2_workspace_bytes(n, d, t, s, r1);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_ARG, "fct2_sketch: workspace %zu < %zu bytes",
                workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  fct::Carver cv(workspace);
  const int64_t ldzt = (K + 3) / 4 * 4;
  float* Z = cv.take<float>(std::max((size_t)K * (size_t)d, 2 * (size_t)d * (size_t)ldzt));
  double* W = cv.take<double>((size_t)r1 * (size_t)d);
  FCT_CUDA_RET(cudaMemsetAsync(W, 0, sizeof(double) * (size_t)r1 * d, st));
  // tensor-core contraction unless its TMA constraints fail (or FCT2_SIMT=1)
  const bool tc = !getenv("FCT2_SIMT") && ldc % 4 == 0 && ((uintptr_t)C & 15) == 0 && K < (1LL << 31);
  auto srht = [&](float* Zr, float* Zh, float* Zl) -> fct_status {
    switch (slice_width(t)) {
      case 8: return launch_srht<3>(A, n, d, lda, signs_t, sel, t, s, Zr, Zh, Zl, ldzt, nb, st);
      case 4: return launch_srht<2>(A, n, d, lda, signs_t, sel, t, s, Zr, Zh, Zl, ldzt, nb, st);
      case 2: return launch_srht<1>(A, n, d, lda, signs_t, sel, t, s, Zr, Zh, Zl, ldzt, nb, st);
      default: return launch_srht<0>(A, n, d, lda, signs_t, sel, t, s, Zr, Zh, Zl, ldzt, nb, st);
    }
  };
  fct_status rc = FCT_ERR_UNSUPPORTED;
  if (tc) {
    float* Zh = Z;
    float* Zl = Z + (size_t)d * ldzt;
    // 1. Z^T = (H~ A)^T split into tf32 hi / lo;  2. W = C Z on tcgen05
    rc = srht(nullptr, Zh, Zl);
    if (rc != FCT_OK) return rc;
    rc = fct2_cz_tc(C, ldc, Zh, Zl, ldzt, K, r1, (int)d, W, st);
    if (rc != FCT_OK && rc != FCT_ERR_UNSUPPORTED) return rc;
  }
  if (rc == FCT_ERR_UNSUPPORTED) {
    // 1. Z = H~ A;  2. W = C Z (SIMT, fp32 partials folded into fp64), split-K to fill the GPU
    rc = srht(Z, nullptr, nullptr);
    if (rc != FCT_OK) return rc;
    const int mt = (r1 + BM - 1) / BM, ntl = (int)((d + BN - 1) / BN);
    int64_t splits = std::max<int64_t>(1, (int64_t)fct::num_sms() * 4 / (mt * ntl));
    int64_t kchunk = (K + splits - 1) / splits;
    kchunk = (kchunk + BK - 1) / BK * BK;
    splits = (K + kchunk - 1) / kchunk;
    FCT_CHECK_ARG(splits <= 65535, FCT_ERR_UNSUPPORTED, "fct2_sketch: too many K splits");
    cz_kernel<<<dim3(mt, ntl, (unsigned)splits), 256, 0, st>>>(C, ldc, Z, (int)d, r1, (int)d, K, kchunk, W);
    FCT_LAUNCHED("fct2 cz_kernel", st);
  }
  // 3. Y = kappa W
  const double kappa = 8.0 / r1 * sqrt(M_PI * (double)t / (2.0 * (double)s));
  const int64_t cnt = (int64_t)r1 * d;
  finalize_kernel<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, 4096), 256, 0, st>>>(W, cnt, kappa, Y);
  FCT_LAUNCHED("fct2 finalize_kernel", st);
  return FCT_OK;
}
