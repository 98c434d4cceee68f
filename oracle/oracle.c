/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct fp64 CPU
 * implementation of the FCT1 hot path of arXiv 1207.4684, written from PAPER.md.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code with the CUDA path
 * (paper_1207_4684_b200/csrc): no FWHT, no blocking, no fusion.
 *
 * Functions and the passages they follow ("P:L" = PAPER.md line):
 *   or_sketch   Y = 4 B C H~ D A           FCT1 construction, Sec. 3.1
 *               (explicit Hadamard entries (-1)^popcount(r&l)/sqrt(s), the Sylvester
 *                matrix of P:L2273-2284; H~ = blockdiag([H_s; I_s]) P:L2246-2266;
 *                D = Rademacher signs, the north_star addition, reading R1)
 *   or_rownorm  lambda_i = median_j |(A R^-1 Pi2)_ij|, with R^-1 Pi2 formed first
 *   or_rownorm_exact  lambda_i = ||(A R^-1)_i||_1 (the exact row norms of Sec. 6.2)
 *               P:L2921-2938
 *   or_sample   phat_i = min(1, m p_i), keep i w.p. phat_i, weight 1/phat_i
 *               l1 sampling lemma P:L1258-1268, use P:L2028-2033
 * Pins: tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- own copy of the counter-based generator (stream 9 = sampling uniforms) ---- */
static uint64_t or_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t or_rng_u64(uint64_t seed, uint64_t stream, uint64_t i) {
  const uint64_t g = 0x9E3779B97F4A7C15ULL;
  return or_mix(or_mix(seed + g * (stream + 1)) + g * (i + 1));
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* (-1)^{popcount(r & l)}: entry (r, l) of the unnormalised Sylvester Hadamard matrix */
static inline double had_sign(uint32_t r, uint32_t l) {
  return (__builtin_popcount(r & l) & 1) ? -1.0 : 1.0;
}

/*
 * Y (r1 x d, fp64, row-major) = 4 B C H~ D A_pad, with A_pad = A zero-padded to
 * n' = s*ceil(n/s) rows (P:L2255-2256 assumes n/s integral; reading R7).
 * H~-row 2sb+r (r<s) is row r of H_s applied to block b, 2sb+s+r is the identity row r.
 * cauchy[2n'] = diag(C), hash[2n'] = bucket of each column of B.
 * Mbound (optional) = the same sum with every factor replaced by its absolute value.
 * Blocks [b0, b1) only (b1 = -1: all); result is ADDED into Y / Mbound.
 */
int or_sketch(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
              const float* cauchy, const int32_t* hash, int32_t s, int32_t r1,
              int64_t b0, int64_t b1, double* Y, double* Mbound) {
  if (n < 1 || d < 1 || lda < d || s < 1 || (s & (s - 1)) || r1 < 1) return -1;
  const int64_t nb = (n + s - 1) / s;
  if (b1 < 0 || b1 > nb) b1 = nb;
  const double inv_sqrt_s = 1.0 / sqrt((double)s);
  int nt = or_num_threads();
  const size_t cells = (size_t)r1 * (size_t)d;
  double* accY = (double*)calloc((size_t)nt * cells, sizeof(double));
  double* accM = Mbound ? (double*)calloc((size_t)nt * cells, sizeof(double)) : NULL;
  if (!accY || (Mbound && !accM)) { free(accY); free(accM); return -2; }
#pragma omp parallel
  {
#ifdef _OPENMP
    const int tid = omp_get_thread_num();
#else
    const int tid = 0;
#endif
    double* y = accY + (size_t)tid * cells;
    double* mb = accM ? accM + (size_t)tid * cells : NULL;
    double* z = (double*)malloc(sizeof(double) * (size_t)s * (size_t)d);
    double* h = (double*)malloc(sizeof(double) * (size_t)d);
    double* ha = (double*)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = b0; b < b1; ++b) {
      /* z = D_b A_b (zero rows past n) */
      for (int64_t l = 0; l < s; ++l) {
        const int64_t row = b * s + l;
        for (int64_t j = 0; j < d; ++j)
          z[l * d + j] = row < n ? (double)signs[row] * (double)A[row * lda + j] : 0.0;
      }
      for (int64_t r = 0; r < s; ++r) {
        /* Hadamard half: (H_s z)_r = sum_l (-1)^{popcount(r&l)} z_l / sqrt(s) */
        for (int64_t j = 0; j < d; ++j) { h[j] = 0.0; ha[j] = 0.0; }
        for (int64_t l = 0; l < s; ++l) {
          const double sg = had_sign((uint32_t)r, (uint32_t)l);
          for (int64_t j = 0; j < d; ++j) { h[j] += sg * z[l * d + j]; ha[j] += fabs(z[l * d + j]); }
        }
        const int64_t ih = 2 * s * b + r;        /* H~-row of the Hadamard half */
        const int64_t ii = 2 * s * b + s + r;    /* H~-row of the identity half */
        const double ch = 4.0 * (double)cauchy[ih], ci = 4.0 * (double)cauchy[ii];
        double* yh = y + (size_t)hash[ih] * d;
        double* yi = y + (size_t)hash[ii] * d;
        for (int64_t j = 0; j < d; ++j) {
          yh[j] += ch * (h[j] * inv_sqrt_s);
          yi[j] += ci * z[r * d + j];
        }
        if (mb) {
          double* mh = mb + (size_t)hash[ih] * d;
          double* mi = mb + (size_t)hash[ii] * d;
          for (int64_t j = 0; j < d; ++j) {
            mh[j] += fabs(ch) * (ha[j] * inv_sqrt_s);
            mi[j] += fabs(ci) * fabs(z[r * d + j]);
          }
        }
      }
    }
    free(z); free(h); free(ha);
  }
  for (int t = 0; t < nt; ++t) {
    const double* y = accY + (size_t)t * cells;
    for (size_t c = 0; c < cells; ++c) Y[c] += y[c];
    if (Mbound) {
      const double* mb = accM + (size_t)t * cells;
      for (size_t c = 0; c < cells; ++c) Mbound[c] += mb[c];
    }
  }
  free(accY); free(accM);
  return 0;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/*
 * lambda_i = median_j |Lambda_ij|, Lambda = A (Rinv Pi2) with M = Rinv Pi2 formed first
 * (P:L2169-2171); even k: mean of the two middle order statistics (reading R11).
 * Rinv: d x d fp64 row-major; Pi2: d x k fp32 row-major.  *lambda_sum = sum_i lambda_i.
 * bound (optional): bound_i = max_j sum_l |A_il| |M_lj| (magnitude of the dot products).
 */
int or_rownorm(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
               const float* Pi2, int32_t k, double* lambda, double* lambda_sum, double* bound) {
  if (n < 0 || d < 1 || lda < d || k < 1) return -1;
  double* M = (double*)malloc(sizeof(double) * (size_t)d * (size_t)k);
  if (!M) return -2;
  for (int64_t l = 0; l < d; ++l)
    for (int64_t j = 0; j < k; ++j) {
      double acc = 0.0;
      for (int64_t m = 0; m < d; ++m) acc += Rinv[l * d + m] * (double)Pi2[m * k + j];
      M[l * k + j] = acc;
    }
  double total = 0.0;
#pragma omp parallel reduction(+ : total)
  {
    double* v = (double*)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double bmax = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        double acc = 0.0, mag = 0.0;
        for (int64_t l = 0; l < d; ++l) {
          acc += (double)A[i * lda + l] * M[l * k + j];
          mag += fabs((double)A[i * lda + l]) * fabs(M[l * k + j]);
        }
        v[j] = fabs(acc);
        if (mag > bmax) bmax = mag;
      }
      qsort(v, (size_t)k, sizeof(double), cmp_double);
      const double med = (k & 1) ? v[k / 2] : 0.5 * (v[k / 2 - 1] + v[k / 2]);
      lambda[i] = med;
      if (bound) bound[i] = bmax;
      total += med;
    }
    free(v);
  }
  free(M);
  if (lambda_sum) *lambda_sum = total;
  return 0;
}

/*
 * Exact l1 row norms of U = A R^-1 ("we compute the row norms of U exactly instead
 * of estimating them"; U of FastL1Basis P:L2771-2796):  lambda_i = sum_j |sum_l A_il Rinv_lj|  (fp64).
 * bound (optional): bound_i = sum_j sum_l |A_il| |Rinv_lj|  (magnitude of the dot products).
 */
int or_rownorm_exact(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv, double* lambda,
                     double* lambda_sum, double* bound) {
  if (n < 0 || d < 1 || lda < d) return -1;
  double total = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : total)
  for (int64_t i = 0; i < n; ++i) {
    double lam = 0.0, mag = 0.0;
    for (int64_t j = 0; j < d; ++j) {
      double u = 0.0;
      for (int64_t l = 0; l < d; ++l) {
        u += (double)A[i * lda + l] * Rinv[l * d + j];
        mag += fabs((double)A[i * lda + l]) * fabs(Rinv[l * d + j]);
      }
      lam += fabs(u);
    }
    lambda[i] = lam;
    if (bound) bound[i] = mag;
    total += lam;
  }
  if (lambda_sum) *lambda_sum = total;
  return 0;
}

/*
 * Bernoulli l1 sampling (Lemma P:L1258-1268 with s := m, t_i := p_i):
 * phat_i = min(1, m * p_i) computed in fp64 from the fp32 p_i (exact: m <= 2^29, 24-bit p);
 * keep i iff u_i < phat_i with u_i = u53(rng_u64(seed, 9, row_base + i)) (or given u[]);
 * weight = 1/phat_i; idx ascending GLOBAL rows.  Returns count; writes at most capacity.
 */
int64_t or_sample(const float* p, const double* u, int64_t n, int64_t row_base, int64_t m,
                  uint64_t seed, int64_t* idx, double* weight, int64_t capacity) {
  int64_t count = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double pi = (double)p[i];
    const double mp = (double)m * pi;
    const double phat = mp < 1.0 ? mp : (mp >= 1.0 ? 1.0 : 0.0);   /* NaN p_i: never sampled (R31) */
    double ui;
    if (u) ui = u[i];
    else ui = (double)(or_rng_u64(seed, 9, (uint64_t)(row_base + i)) >> 11) * 0x1.0p-53;
    if (ui < phat) {
      if (count < capacity) { idx[count] = row_base + i; weight[count] = 1.0 / phat; }
      ++count;
    }
  }
  return count;
}

/*
 * NEXT-4: m i.i.d. draws with probability proportional to p_i from an exact fixed-point
 * CDF (the multinomial reading of "sample m rows with probabilities p", P:L1258-1268 / P:L2178-2188):
 *   F = 62 - ceil(log2 n) - e,  max_i p_i < 2^e (frexp)        -> sum_i W_i < 2^62
 *   W_i = floor(p_i 2^F) (exact in fp64 -> uint64),  CDF_i = sum_{t <= i} W_t,  T = CDF_{n-1}
 *   X_j = rng_u64(seed, 10, j) >> 11,  target_j = floor(X_j T / 2^53)   (128-bit product)
 *   idx_j = row_base + min{i : CDF_i > target_j},  weight_j = (double)T / ((double)m (double)W_i)
 * Returns T (0: no positive p) and writes F.  Integer arithmetic only: bit-exact.
 */
uint64_t or_sample_multinomial(const float* p, int64_t n, int64_t m, uint64_t seed, int64_t row_base, int64_t* idx,
                               double* weight, int32_t* F_out) {
  float mx = 0.f;
  for (int64_t i = 0; i < n; ++i) if (p[i] > mx) mx = p[i];
  if (!(mx > 0.f)) return 0;
  int e = 0;
  frexp((double)mx, &e);
  int lg = 0;
  while (((int64_t)1 << lg) < n) ++lg;
  const int F = 62 - lg - e;
  if (F_out) *F_out = F;
  uint64_t* cdf = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  uint64_t* W = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  uint64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double v = p[i] > 0.f ? floor(ldexp((double)p[i], F)) : 0.0;
    W[i] = (uint64_t)v;
    acc += W[i];
    cdf[i] = acc;
  }
  const uint64_t T = acc;
  for (int64_t j = 0; j < m && T > 0; ++j) {
    const uint64_t X = or_rng_u64(seed, 10, (uint64_t)j) >> 11;
    const uint64_t target = (uint64_t)(((unsigned __int128)X * (unsigned __int128)T) >> 53);
    int64_t lo = 0, hi = n - 1;             /* first i with cdf[i] > target */
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (cdf[mid] > target) hi = mid; else lo = mid + 1;
    }
    idx[j] = row_base + lo;
    weight[j] = (double)T / ((double)m * (double)W[lo]);
  }
  free(cdf);
  free(W);
  return T;
}
