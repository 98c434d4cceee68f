// condition.cu -- K5: R and R^-1 of the sketch Y = Pi1 A (FastL1Basis)
// CholeskyQR2 in fp64:  G1 = Y^T Y = R1^T R1;  Q1 = Y R1^-1;  G2 = Q1^T Q1 = R2^T R2;
//                       R = R2 R1 (diag > 0),  R^-1 = R1^-1 R2^-1.
// The second pass restores the accuracy a single Gram-matrix Cholesky loses (error ~ u cond(Y)
// instead of u cond(Y)^2), matching Householder QR (the oracle) to fp64 rounding x cond(Y).
#include <math.h>
#include "common.cuh"

namespace {

constexpr int kT = 32;       // Gram tile
constexpr int kChunk = 256;  // rows of Y per partial Gram

// Gp[c][i][j] = sum_{r in chunk c} X[r][i] X[r][j] for the (ti, tj) tile; X fp32 or fp64
template <typename T>
__global__ void __launch_bounds__(kT * 8) gram_kernel(const T* __restrict__ X, int r1, int d, double* __restrict__ Gp) {
  const int ti = blockIdx.x, tj = blockIdx.y, c = blockIdx.z;
  if (tj < ti) return;
  __shared__ double xa[kT][kT + 1], xb[kT][kT + 1];
  const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;  // 32 x 8
  double acc[4] = {0, 0, 0, 0};
  const int rbeg = c * kChunk, rend = min(r1, rbeg + kChunk);
  for (int r0 = rbeg; r0 < rend; r0 += kT) {
    for (int q = ty; q < kT; q += 8) {
      const int r = r0 + q;
      const int ci = ti * kT + tx, cj = tj * kT + tx;
      xa[q][tx] = (r < rend && ci < d) ? (double)X[(size_t)r * d + ci] : 0.0;
      xb[q][tx] = (r < rend && cj < d) ? (double)X[(size_t)r * d + cj] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < kT; ++q) {
      const double bj = xb[q][tx];
#pragma unroll
      for (int s = 0; s < 4; ++s) acc[s] = fma(xa[q][ty + 8 * s], bj, acc[s]);
    }
    __syncthreads();
  }
  const int j = tj * kT + tx;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int i = ti * kT + ty + 8 * s;
    if (i < d && j < d) Gp[((size_t)c * d + i) * d + j] = acc[s];
  }
}

// Q = Y * Rinv1  (r1 x d fp64), one thread per output entry
__global__ void apply_rinv_kernel(const float* __restrict__ Y, const double* __restrict__ Rinv, int r1, int d,
                                  double* __restrict__ Q) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)r1 * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / d), j = (int)(e - (int64_t)r * d);
    double s = 0.0;
    for (int l = 0; l <= j; ++l) s = fma((double)Y[(size_t)r * d + l], Rinv[l * d + j], s);
    Q[e] = s;
  }
}

// Single CTA: G = sum of partial Grams (fixed order, upper triangle), Cholesky G = Rk^T Rk,
// Rk^-1; then R = Rk * Rprev, Rinv = Rprev_inv * Rk^-1 (or Rk, Rk^-1 if Rprev == nullptr).
__global__ void __launch_bounds__(1024) chol_kernel(const double* __restrict__ Gp, int nchunks, int d,
                                                    const double* __restrict__ Rprev,
                                                    const double* __restrict__ Rprev_inv, double* Rk_out,
                                                    double* Rkinv_out, double* R, double* Rinv,
                                                    int* __restrict__ info, int big) {  // R/Rk_out may alias
  extern __shared__ double G[];  // d x d (+ 2 d x d when big)
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (Rprev && *info != 0) return;  // first pass already failed: keep its info
  if (tid == 0) fail = 0;
  for (int e = tid; e < d * d; e += nt) {
    const int i = e / d, j = e - i * d;
    double s = 0.0;
    if (j >= i)
      for (int c = 0; c < nchunks; ++c) s += Gp[(size_t)c * d * d + e];
    G[e] = s;
  }
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    if (tid == 0) {
      const double piv = G[j * d + j];
      if (!(piv > 0.0) || !isfinite(piv)) {
        fail = j + 1;
      } else {
        G[j * d + j] = sqrt(piv);
      }
    }
    __syncthreads();
    if (fail) break;
    const double rjj = G[j * d + j];
    for (int i = j + 1 + tid; i < d; i += nt) G[j * d + i] /= rjj;
    __syncthreads();
    const int m = d - j - 1;  // trailing block size
    for (int e = tid; e < m * m; e += nt) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l >= i) G[i * d + l] -= G[j * d + i] * G[j * d + l];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) *info = fail;
    return;
  }
  // Rk^-1 by back substitution, column c by thread c, in shared memory when two more d x d arrays fit
  // (X = Rk^-1, S = staging for the previous factor); otherwise in the global outputs
  double* X = big ? G + d * d : Rkinv_out;
  double* S = big ? G + 2 * d * d : nullptr;
  for (int c = tid; c < d; c += nt) {
    for (int i = d - 1; i >= 0; --i) {
      double v = 0.0;
      if (i <= c) {
        double s = (i == c) ? 1.0 : 0.0;
        for (int l = i + 1; l <= c; ++l) s = fma(-G[i * d + l], X[l * d + c], s);
        v = s / G[i * d + i];
      }
      X[i * d + c] = v;
    }
  }
  __syncthreads();
  for (int e = tid; e < d * d; e += nt) {
    const int i = e / d, j = e - i * d;
    Rk_out[e] = j >= i ? G[e] : 0.0;
    if (big) Rkinv_out[e] = X[e];
  }
  // combine with the previous factor: R = Rk Rprev, R^-1 = Rprev^-1 Rk^-1 (all upper triangular)
  if (Rprev) {
    const double* P = Rprev;
    if (big) {
      for (int e = tid; e < d * d; e += nt) S[e] = Rprev[e];
      __syncthreads();
      P = S;
    }
    for (int e = tid; e < d * d; e += nt) {
      const int i = e / d, j = e - i * d;
      double r = 0.0;
      if (j >= i)
        for (int l = i; l <= j; ++l) r = fma(G[i * d + l], P[l * d + j], r);
      R[e] = r;
    }
    __syncthreads();
    if (big) {
      for (int e = tid; e < d * d; e += nt) S[e] = Rprev_inv[e];
      __syncthreads();
      P = S;
    } else {
      P = Rprev_inv;
    }
    for (int e = tid; e < d * d; e += nt) {
      const int i = e / d, j = e - i * d;
      double ri = 0.0;
      if (j >= i)
        for (int l = i; l <= j; ++l) ri = fma(P[i * d + l], X[l * d + j], ri);
      Rinv[e] = ri;
    }
  } else {
    for (int e = tid; e < d * d; e += nt) {
      const int i = e / d, j = e - i * d;
      R[e] = j >= i ? G[e] : 0.0;
      Rinv[e] = X[e];
    }
  }
  if (tid == 0) *info = 0;
}

}  // namespace

extern "C" size_t fct_condition_workspace_bytes(int32_t r1, int64_t d) {
  if (r1 < 1 || d < 1) return 0;
  const size_t nch = (size_t)((r1 + kChunk - 1) / kChunk);
  return fct::align256(sizeof(double) * nch * d * d) + fct::align256(sizeof(double) * (size_t)r1 * d) +
         4 * fct::align256(sizeof(double) * d * d);
}

extern "C" fct_status fct_condition(const float* Y, int32_t r1, int64_t d, double* R, double* Rinv, int32_t* info,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(Y && R && Rinv && info, FCT_ERR_ARG, "fct_condition: NULL pointer");
  FCT_CHECK_ARG(d >= 1 && d <= FCT_MAX_D && r1 >= d, FCT_ERR_SHAPE,
                "fct_condition: need 1 <= d <= %d and r1 >= d (r1=%d d=%lld)", FCT_MAX_D, r1, (long long)d);
  const size_t need = fct_condition_workspace_bytes(r1, d);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_WORKSPACE,
                "fct_condition: workspace %zu < %zu bytes", workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = (r1 + kChunk - 1) / kChunk;
  fct::Carver cv(workspace);
  double* Gp = cv.take<double>((size_t)nch * d * d);
  double* Q = cv.take<double>((size_t)r1 * d);
  double* R1 = cv.take<double>((size_t)d * d);
  double* R1inv = cv.take<double>((size_t)d * d);
  double* R2 = cv.take<double>((size_t)d * d);
  double* R2inv = cv.take<double>((size_t)d * d);
  const int dd = (int)d;
  const int nt = (dd + kT - 1) / kT;
  const int big = 3 * sizeof(double) * (size_t)d * d <= 200 * 1024 ? 1 : 0;
  const size_t smem = sizeof(double) * (size_t)d * d * (big ? 3 : 1);
  FCT_CUDA_RET(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gram_kernel<float><<<dim3(nt, nt, nch), kT * 8, 0, st>>>(Y, r1, dd, Gp);
  FCT_LAUNCHED("gram_kernel<float>", st);
  chol_kernel<<<1, 1024, smem, st>>>(Gp, nch, dd, nullptr, nullptr, R1, R1inv, R1, R1inv, info, big);
  FCT_LAUNCHED("chol_kernel(1)", st);
  apply_rinv_kernel<<<fct::num_sms() * 4, 256, 0, st>>>(Y, R1inv, r1, dd, Q);
  FCT_LAUNCHED("apply_rinv_kernel", st);
  gram_kernel<double><<<dim3(nt, nt, nch), kT * 8, 0, st>>>(Q, r1, dd, Gp);
  FCT_LAUNCHED("gram_kernel<double>", st);
  chol_kernel<<<1, 1024, smem, st>>>(Gp, nch, dd, R1, R1inv, R2, R2inv, R, Rinv, info, big);
  FCT_LAUNCHED("chol_kernel(2)", st);
  return FCT_OK;
}
