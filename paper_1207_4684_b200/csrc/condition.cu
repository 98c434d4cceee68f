// condition.cu -- K5: R and R^-1 of the sketch Y = Pi1 A (FastL1Basis: "construct Pi1 A and an
// R such that Pi1 A = QR ... for example using a QR-factorization of Pi1 A"; cost P:L1046-1048).
//
// CholeskyQR2 in fp64, with shifted CholeskyQR3 as the device-side fallback:
//   pass k:  X_k = Y R_cum^-1 (X_1 = Y),  G_k = X_k^T X_k (+ sigma I on pass 1 of the shifted variant),
//            G_k = R_k^T R_k (Cholesky),  R_cum <- R_k R_cum,  R_cum^-1 <- R_cum^-1 R_k^-1.
//   2 passes (CholeskyQR2) restore the accuracy a single Gram Cholesky loses (error ~ u cond(Y) instead of
//   u cond(Y)^2) and match Householder QR (the oracle) to fp64 rounding x cond(Y) while cond(Y) < ~u^-1/2.
//   When a pivot is not positive/finite, or the second Gram is far from I (cond(Y) beyond that range), the
//   whole computation restarts with sigma = 11 (r1 d + d(d+1)) u ||Y||_F^2 added to the first Gram and runs 3
//   passes (shifted CholeskyQR3, Fukaya et al.), stable up to cond(Y) ~ u^-1.  Only if the shifted Cholesky
//   fails too (non-finite Y) is info > 0; R and R^-1 are then NaN so nothing downstream can look valid.
//
// One cooperative persistent kernel (one CTA per SM, grid-wide barriers between phases, nothing returns to the
// host).  Per pass:
//   1 [all CTAs]  partial Gram of the CTA's contiguous rows of X_k: rows staged in shared memory (fp64),
//                 X_k = Y R_cum^-1 formed there with 4x4 register tiles, Gram accumulated in 4x4 register tiles;
//   2 [all CTAs]  fixed-order reduction of the per-CTA records (8 warps x c-slices, then a fixed combine);
//   3 [CTA 0]     right-looking Cholesky and triangular inverse on the register-resident triangle (16 x 16
//                 cyclic thread grid, one published row and one barrier per step);
//   4 [all CTAs]  R_cum <- R_k R_cum, R_cum^-1 <- R_cum^-1 R_k^-1 (packed triangular products).
// Deterministic: every sum has a fixed order.
#include <cooperative_groups.h>
#include <math.h>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int NT = 256;        // threads per CTA (8 warps)
constexpr int NW = NT / 32;
constexpr int ROWS = 32;       // rows of Y staged per sub-chunk
constexpr int NBLK_MAX = FCT_MAX_D / 16;   // register blocks per thread and dimension in the factorisation
constexpr int MAXB = FCT_MAX_D / 4;                             // 4-wide column blocks
constexpr int MAXTILE = (MAXB * (MAXB + 1) / 2 + NT - 1) / NT;  // Gram tiles per thread

// packed upper-triangular index of (i, j), j >= i
__device__ __forceinline__ int pk(int i, int j, int d) { return i * d - (i * (i - 1)) / 2 + (j - i); }

struct Args {
  const float* Y;
  int r1, d, T;            // T = d (d + 1) / 2
  int nb, ntile;           // 4-wide blocks of d (padded), Gram tiles nb (nb + 1) / 2
  double* Gp;              // [grid][ntile * 16] partial Gram records
  double* G;               // [ntile * 16] reduced Gram
  double* R;               // [d][d] output
  double* Rinv;            // [d][d] output
  int* info;
  int* state;              // [1]: 0 ok, 1 restart with shift, 2 failed
  int series;              // near-identity Grams of passes >= 1 by the second-order series (R32)
  double* Rk;              // [T] packed R_k of the current pass
  double* Rki;             // [T] packed R_k^-1
  double* C[2];            // ping-pong [T] packed cumulative R
  double* Ci[2];           // ping-pong [T] packed cumulative R^-1
  unsigned long long* ts;  // optional phase timestamps (globaltimer, CTA 0 thread 0)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// row of packed entry e of an n x n upper triangle (the largest i with i n - i (i - 1) / 2 <= e)
__device__ __forceinline__ int tri_row(int e, int n) {
  const double b = 2.0 * n + 1.0;
  int i = max(0, min(n - 1, (int)floor((b - sqrt(b * b - 8.0 * e)) / 2.0)));
  while (i > 0 && pk(i, i, n) > e) --i;
  while (i + 1 < n && pk(i + 1, i + 1, n) <= e) ++i;
  return i;
}

// NBLK = ceil(d / 16) rounded up to a power of two: the factorisation's register blocks per thread and dimension
template <int NBLK>
__global__ void __launch_bounds__(NT, 1) cond_kernel(Args a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int d = a.d, T = a.T, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int DP = 4 * a.nb;     // padded row length
  const int V = a.ntile * 16;  // values per Gram record
  // phase-1 shared layout: Rinv full [d][DP] | xs [ROWS][DP] | qs [ROWS][DP]
  double* sRi = sm;
  double* xs = sRi + (size_t)d * DP;
  double* qs = xs + ROWS * DP;
  const int rows_per = (a.r1 + gridDim.x - 1) / gridDim.x;
  const int rb = min(a.r1, blockIdx.x * rows_per), re = min(a.r1, rb + rows_per);
  const double u = 0x1.0p-53;

  int shifted = 0, npass = 2, nts = 0;
  const double* Rci = nullptr;   // packed cumulative R^-1 used to form X_k; nullptr on pass 0
  auto stamp = [&]() {
    if (a.ts && blockIdx.x == 0 && tid == 0 && nts < 56) a.ts[nts++] = gtimer();
  };
  stamp();
  for (int pass = 0; pass < npass; ++pass) {
    // ================= phase 1: partial Gram of X = Y R_cum^-1 over this CTA's rows
    if (pass > 0)
      for (int e = tid; e < d * DP; e += NT) {
        const int i = e / DP, j = e - i * DP;
        sRi[e] = (j >= i && j < d) ? Rci[pk(i, j, d)] : 0.0;
      }
    double acc[MAXTILE][16];
    int tbi[MAXTILE], tbj[MAXTILE];
#pragma unroll
    for (int q = 0; q < MAXTILE; ++q) {
#pragma unroll
      for (int v = 0; v < 16; ++v) acc[q][v] = 0.0;
      const int t = min(tid + q * NT, a.ntile - 1);
      tbi[q] = tri_row(t, a.nb);
      tbj[q] = tbi[q] + (t - pk(tbi[q], tbi[q], a.nb));
    }
    for (int r0 = rb; r0 < re; r0 += ROWS) {
      const int nr = min(ROWS, re - r0);
      __syncthreads();
      for (int e = tid; e < ROWS * DP; e += NT) {
        const int r = e / DP, c = e - r * DP;
        xs[e] = (r < nr && c < d) ? (double)a.Y[(size_t)(r0 + r) * d + c] : 0.0;
      }
      __syncthreads();
      const double* X = xs;
      if (pass > 0) {   // q[r][j] = sum_{l <= j} y[r][l] Rinv[l][j], 4 x 4 register tiles
        for (int t = tid; t < (ROWS / 4) * a.nb; t += NT) {
          const int br = t / a.nb, bc = t - br * a.nb;
          double o[4][4];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) o[x][y] = 0.0;
          const int lmax = min(d, 4 * bc + 4);
          for (int l = 0; l < lmax; ++l) {
            const double2 r01 = *(const double2*)(sRi + (size_t)l * DP + 4 * bc);
            const double2 r23 = *(const double2*)(sRi + (size_t)l * DP + 4 * bc + 2);
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const double xv = xs[(4 * br + x) * DP + l];
              o[x][0] = fma(xv, r01.x, o[x][0]);
              o[x][1] = fma(xv, r01.y, o[x][1]);
              o[x][2] = fma(xv, r23.x, o[x][2]);
              o[x][3] = fma(xv, r23.y, o[x][3]);
            }
          }
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            *(double2*)(qs + (4 * br + x) * DP + 4 * bc) = make_double2(o[x][0], o[x][1]);
            *(double2*)(qs + (4 * br + x) * DP + 4 * bc + 2) = make_double2(o[x][2], o[x][3]);
          }
        }
        __syncthreads();
        X = qs;
      }
#pragma unroll
      for (int q = 0; q < MAXTILE; ++q) {
        const int t = tid + q * NT;
        if (t < a.ntile) {
          const int bi = tbi[q], bj = tbj[q];
#pragma unroll 2
          for (int r = 0; r < ROWS; ++r) {
            const double2 p01 = *(const double2*)(X + r * DP + 4 * bi), p23 = *(const double2*)(X + r * DP + 4 * bi + 2);
            const double2 q01 = *(const double2*)(X + r * DP + 4 * bj), q23 = *(const double2*)(X + r * DP + 4 * bj + 2);
            const double pv[4] = {p01.x, p01.y, p23.x, p23.y}, qv[4] = {q01.x, q01.y, q23.x, q23.y};
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) acc[q][4 * x + y] = fma(pv[x], qv[y], acc[q][4 * x + y]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < MAXTILE; ++q) {
      const int t = tid + q * NT;
      if (t < a.ntile)
#pragma unroll
        for (int v = 0; v < 16; v += 2)
          *(double2*)(a.Gp + (size_t)blockIdx.x * V + 16 * t + v) = make_double2(acc[q][v], acc[q][v + 1]);
    }
    grid.sync();
    stamp();
    // ================= phase 2: fixed-order reduction of the records (lanes: values, warps: record slices)
    {
      double* red = sm;   // [NW][32]
      const int per = ((int)gridDim.x + NW - 1) / NW;
      const int c0 = warp * per, c1 = min((int)gridDim.x, c0 + per);
      for (int v0 = blockIdx.x * 32; v0 < V; v0 += gridDim.x * 32) {
        const int v = v0 + lane;
        double s = 0.0;
        if (v < V)
          for (int c = c0; c < c1; ++c) s += a.Gp[(size_t)c * V + v];
        __syncthreads();
        red[warp * 32 + lane] = s;
        __syncthreads();
        if (warp == 0 && v < V) {
          double t = 0.0;
          for (int w = 0; w < NW; ++w) t += red[w * 32 + lane];
          a.G[v] = t;
        }
      }
    }
    grid.sync();
    stamp();
    // ================= phase 3' (passes >= 1, all CTAs): a Gram within 2^-26 of I entrywise -- the common case,
    // X_k is already orthonormal to ~u cond(Y) -- is factored by its series instead of d serial steps
    // (R32).  G = I + E, F1 = up(E) (strict upper part, half the diagonal), U = up(F1^T F1):
    //   R_k = I + F1 - U,   R_k^-1 = I - F1 + U + F1^2   (dropped terms O(d^2 max|E|^3) <= 2^-64).
    // Every CTA checks the same reduced Gram, so all take the same branch.
    bool near = false;
    if (pass >= 1 && a.series) {
      int far = 0;
      for (int e = tid; e < a.nb * a.nb * 16; e += NT) {
        const int bij = e >> 4, x = (e >> 2) & 3, y = e & 3;
        const int bi = bij / a.nb, bj = bij - bi * a.nb;
        const int i = 4 * bi + x, c = 4 * bj + y;
        if (bj >= bi && i <= c && c < d && !(fabs(a.G[16 * pk(bi, bj, a.nb) + (e & 15)] - (i == c ? 1.0 : 0.0)) <= 0x1p-26))
          far = 1;
      }
      near = !__syncthreads_or(far);
    }
    if (near) {
      const int nbk = a.nb;
      auto F1 = [&](int i, int c) -> double {   // i <= c
        const double v = a.G[16 * pk(i >> 2, c >> 2, nbk) + 4 * (i & 3) + (c & 3)];
        return i == c ? 0.5 * (v - 1.0) : v;
      };
      for (int e = blockIdx.x * NT + tid; e < T; e += gridDim.x * NT) {
        const int i = tri_row(e, d), c = i + (e - pk(i, i, d));
        double u0 = 0.0, u1 = 0.0, q0 = 0.0, q1 = 0.0;
        int l = 0;
        for (; l + 1 <= i; l += 2) {   // U[i][c] = sum_{l <= i} F1[l][i] F1[l][c]
          u0 = fma(F1(l, i), F1(l, c), u0);
          u1 = fma(F1(l + 1, i), F1(l + 1, c), u1);
        }
        if (l <= i) u0 = fma(F1(l, i), F1(l, c), u0);
        for (l = i; l + 1 <= c; l += 2) {   // (F1^2)[i][c] = sum_{i <= l <= c} F1[i][l] F1[l][c]
          q0 = fma(F1(i, l), F1(l, c), q0);
          q1 = fma(F1(i, l + 1), F1(l + 1, c), q1);
        }
        if (l <= c) q0 = fma(F1(i, l), F1(l, c), q0);
        const double f1 = F1(i, c), uu = (i == c ? 0.5 : 1.0) * (u0 + u1), id = i == c ? 1.0 : 0.0;
        a.Rk[e] = id + f1 - uu;
        a.Rki[e] = id - f1 + uu + (q0 + q1);
      }
    }
    // ================= phase 3 (CTA 0): register-resident Cholesky and triangular inverse
    // The d x d upper triangle lives in the registers of the CTA's 256 threads on a 16 x 16 cyclic grid:
    // thread (ti, tc) = (tid / 16, tid % 16) owns the entries (ti + 16 a, tc + 16 b), a, b < nblk.  Each step of
    // the right-looking factorisation (and of the inverse) publishes one row through shared memory and costs one
    // barrier: d steps of ~nblk^2 FMAs per thread instead of a serial panel chain (round 2: 59 -> ~10 us / pass).
    if (!near && blockIdx.x == 0) {
      double* Rs = sm;            // packed [T]: R_k
      double* buf = sm + 2 * T;   // [2][DPAD]: the published row of the current step (double-buffered)
      const int DPAD = 16 * NBLK;
      __shared__ int fail;
      __shared__ double sigma;
      const int ti = tid >> 4, tc = tid & 15;
      constexpr int nblk = NBLK;
      double g[NBLK][NBLK];
      // own entries of G from the tile record (entry (i, c), i <= c: tile (i / 4, c / 4), element 4 (i % 4) + c % 4)
#pragma unroll
      for (int x = 0; x < NBLK; ++x)
#pragma unroll
        for (int y = 0; y < NBLK; ++y) {
          const int i = ti + 16 * x, c = tc + 16 * y;
          g[x][y] = (x < nblk && y < nblk && i <= c && c < d)
                        ? a.G[16 * pk(i >> 2, c >> 2, a.nb) + 4 * (i & 3) + (c & 3)] : 0.0;
        }
      if (tid == 0) { fail = 0; sigma = 0.0; }
      __syncthreads();
      if (pass == 0 && shifted) {   // sigma = 11 (r1 d + d (d + 1)) u ||Y||_F^2, ||Y||_F^2 = trace(G) (fixed order)
#pragma unroll
        for (int x = 0; x < NBLK; ++x)
          if (x < nblk && ti == tc && ti + 16 * x < d) buf[ti + 16 * x] = g[x][x];
        __syncthreads();
        if (tid == 0) {
          double tr = 0.0;
          for (int i = 0; i < d; ++i) tr += buf[i];
          sigma = 11.0 * ((double)a.r1 * d + (double)d * (d + 1)) * u * tr;
        }
        __syncthreads();
#pragma unroll
        for (int x = 0; x < NBLK; ++x)
          if (x < nblk && ti == tc) g[x][x] += sigma;
      }
      if (pass == 1 && !shifted) {  // CholeskyQR2's second Gram must be close to I
        int bad = 0;
#pragma unroll
        for (int x = 0; x < NBLK; ++x)
#pragma unroll
          for (int y = 0; y < NBLK; ++y) {
            const int i = ti + 16 * x, c = tc + 16 * y;
            if (x < nblk && y < nblk && i <= c && c < d && !(fabs(g[x][y] - (i == c ? 1.0 : 0.0)) <= 0.5)) bad = 1;
          }
        if (__syncthreads_or(bad) && tid == 0) fail = 1;
        __syncthreads();
      }
      stamp();
      // ---- right-looking Cholesky G = R^T R without a division or square root on the step chain: the trailing
      // matrix is kept as H = C_j S^(j) (S^(j) the Schur complement, C_j = prod_{k<j} m_k, m_k = H[k][k] 2^-e_k in
      // [1, 2) with 2^e_k the binade of H[k][k], both exact bit operations).  Step j publishes row j of H and every
      // owner of (i, c), i > j, forms H[i][c] <- m_j H[i][c] - (H[j][i] 2^-e_j) H[j][c]  (= m_j (S - S_ji S_jc / s_j)
      // scaled by C_j).  Afterwards R[j][c] = H[j][c] / sqrt(C_j H[j][j]).  A pivot that is not a positive normal
      // number (< 2^-1000 included) fails -> shifted CholeskyQR3.
      __shared__ double mv[FCT_MAX_D], pv[FCT_MAX_D];
      int jf = fail ? 0 : d;   // steps done
      if (!fail)
        for (int j = 0; j < d; ++j) {
          double* bj = buf + (j & 1) * DPAD;
          const int xj = j >> 4;
          if constexpr (NBLK >= 8) {   // publish row j (the row's owners select block row xj; measured faster at 8)
            if (ti == (j & 15)) {
#pragma unroll
              for (int x = 0; x < NBLK; ++x)
                if (x == xj)
#pragma unroll
                  for (int y = 0; y < NBLK; ++y) {
                    const int c = tc + 16 * y;
                    if (c >= j && c < d) bj[c] = g[x][y];
                  }
            }
          } else {   // publish row j: block row xj selected branch-free (compile-time register indices)
            double pr[NBLK];
#pragma unroll
            for (int y = 0; y < NBLK; ++y) pr[y] = g[0][y];
#pragma unroll
            for (int x = 1; x < NBLK; ++x)
#pragma unroll
              for (int y = 0; y < NBLK; ++y) pr[y] = x == xj ? g[x][y] : pr[y];
            const bool pub = ti == (j & 15);
#pragma unroll
            for (int y = 0; y < NBLK; ++y) {
              const int c = tc + 16 * y;
              if (pub && c >= j && c < d) bj[c] = pr[y];
            }
          }
          __syncthreads();
          const double piv = bj[j];
          if (!(piv >= 0x1p-1000) || !(piv <= 0x1p+1000)) {
            jf = j;
            break;
          }
          const long long pb = __double_as_longlong(piv);
          const double m = __longlong_as_double((pb & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);   // [1, 2)
          const double sc = __longlong_as_double((long long)(2046 - ((pb >> 52) & 0x7FF)) << 52);     // 2^-e
          if (tid == 0) { mv[j] = m; pv[j] = piv; }
          // every entry takes the update; outside the trailing triangle the factor is 0 and the multiplier 1, so
          // finished rows are unchanged and entries below the diagonal collect garbage that is never read
          double fc[NBLK];
#pragma unroll
          for (int y = 0; y < NBLK; ++y) {
            const int c = tc + 16 * y;
            const double v = bj[min(c, d - 1)];
            fc[y] = (c > j && c < d) ? v : 0.0;
          }
#pragma unroll
          for (int x = 0; x < NBLK; ++x) {
            const int i = ti + 16 * x;
            const bool live = i > j && i < d;
            const double v = bj[min(i, d - 1)];
            const double fi = live ? v * sc : 0.0, mu = live ? m : 1.0;
#pragma unroll
            for (int y = 0; y < NBLK; ++y) g[x][y] = fma(-fi, fc[y], g[x][y] * mu);
          }
        }
      __syncthreads();
      // rinv_i = 1 / sqrt(C_i H_ii): C by a fixed-order scan of the m_k, then R[i][c] = H[i][c] rinv_i and
      // 1 / R[i][i] = C_i rinv_i
      double* cs = buf + 2 * DPAD;   // [DPAD] C_i, then 1 / R[i][i]
      double* ri = buf;              // [DPAD] rinv_i (the publication buffers are free now)
      if (jf == d && !fail) {
        if (tid < d) cs[tid] = tid == 0 ? 1.0 : mv[tid - 1];
        __syncthreads();
        for (int off = 1; off < d; off <<= 1) {   // inclusive product scan (Hillis-Steele)
          const double v = (tid < d && tid >= off) ? cs[tid - off] : 1.0;
          __syncthreads();
          if (tid < d) cs[tid] *= v;
          __syncthreads();
        }
        if (tid < d) {
          const double r = rsqrt(cs[tid] * pv[tid]);
          ri[tid] = r;
          cs[tid] = cs[tid] * r;
        }
        __syncthreads();
#pragma unroll
        for (int x = 0; x < NBLK; ++x)
#pragma unroll
          for (int y = 0; y < NBLK; ++y) {
            const int i = ti + 16 * x, c = tc + 16 * y;
            if (i <= c && c < d) Rs[pk(i, c, d)] = g[x][y] * ri[i];
          }
      }
      if (jf < d && tid == 0 && !fail) fail = jf + 1;
      __syncthreads();
      if (fail) {
        if (tid == 0) {
          if (!shifted) a.state[1] = 1;                 // restart with the shift (shifted CholeskyQR3)
          else { a.state[1] = 2; *a.info = fail; }
        }
      } else {
        stamp();
        // R_k^-1 is formed grid-parallel in phase 3b (one warp per column); hand over 1 / R[p][p] in a.G
        for (int i = tid; i < d; i += NT) a.G[i] = cs[i];
        __syncthreads();
        stamp();
        for (int e = tid; e < T; e += NT) a.Rk[e] = Rs[e];
        if (tid == 0) a.state[1] = 0;
      }
    }
    grid.sync();
    stamp();
    const int st1 = ((volatile int*)a.state)[1];
    if (st1 == 2) break;                                                            // failed even with the shift
    if (st1 == 1) { shifted = 1; npass = 3; pass = -1; Rci = nullptr; continue; }   // restart: shifted CholeskyQR3
    // ================= phase 3b (all CTAs, after a Cholesky): X = R_k^-1 column by column, one warp per column c
    // (R X[:, c] = e_c by backward substitution: lane l keeps the partial sums of rows l + 32 k; step p finalises
    // X[p][c] = s_p / R[p][p], broadcasts it, and the lanes subtract R[r][p] X[p][c] for r < p); R_k staged in
    // shared memory by every CTA that owns a column
    if (!near) {
      const int c = blockIdx.x * NW + warp;
      if (blockIdx.x * NW < d) {
        double* sR = sm;       // packed [T]
        double* sD = sm + T;   // [d] 1 / R[p][p]
        for (int e = tid; e < T; e += NT) sR[e] = a.Rk[e];
        for (int i = tid; i < d; i += NT) sD[i] = a.G[i];
        __syncthreads();
        if (c < d) {
          constexpr int KR = FCT_MAX_D / 32;
          double sv[KR];
          int rb[KR];   // pk(r, r) - r: R[r][p] = sR[rb + p]
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int r = lane + 32 * k;
            sv[k] = r == c ? 1.0 : 0.0;
            rb[k] = r < d ? pk(r, r, d) - r : 0;
          }
          const long long ck0 = clock64();
          // branch-free steps (selects only): the loads of R[.][p] do not depend on the chain and are issued first
          // (one step ahead), so a step costs the SHFL -> DMUL -> DFMA chain
          double rv[KR], dp = sD[c];
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int r = lane + 32 * k;
            rv[k] = sR[r < c ? rb[k] + c : 0];
          }
          for (int p = c; p >= 0; --p) {
            double rn[KR];
            const int pn = p > 0 ? p - 1 : 0;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
              const int r = lane + 32 * k;
              rn[k] = sR[r < pn ? rb[k] + pn : 0];
            }
            const double dn = sD[pn];
            const int kp = p >> 5;
            double own = sv[0];
#pragma unroll
            for (int k = 1; k < KR; ++k) own = k == kp ? sv[k] : own;
            const double xp = __shfl_sync(0xffffffffu, own, p & 31) * dp;   // X[p][c]
#pragma unroll
            for (int k = 0; k < KR; ++k) {
              const int r = lane + 32 * k;
              const double f = r < p ? rv[k] : 0.0;
              const double v = fma(-f, xp, sv[k]);
              sv[k] = r == p ? xp : v;
              rv[k] = rn[k];
            }
            dp = dn;
          }
          if (a.ts && c == d - 1 && lane == 0) {   // diagnostics (FCT_COND_TIMING): cycles of the longest column
            a.ts[60] = (unsigned long long)(clock64() - ck0);
            a.ts[61] = (unsigned long long)(c + 1);
          }
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int r = lane + 32 * k;
            if (r <= c) a.Rki[pk(r, c, d)] = sv[k];
          }
        }
      }
      grid.sync();
      stamp();
    }
    // ================= phase 4 (all CTAs): after pass p the cumulative factors live in C[p & 1], Ci[p & 1]
    {
      const int pp = pass & 1;
      double* Rn = a.C[pp];
      double* Rin = a.Ci[pp];
      const double* Rc = a.C[pp ^ 1];
      const double* Ric = a.Ci[pp ^ 1];
      for (int e = blockIdx.x * NT + tid; e < T; e += gridDim.x * NT) {
        if (pass == 0) { Rn[e] = a.Rk[e]; Rin[e] = a.Rki[e]; continue; }
        const int i = tri_row(e, d), j = i + (e - pk(i, i, d));
        double r = 0.0, ri = 0.0;
        for (int l = i; l <= j; ++l) {
          r = fma(a.Rk[pk(i, l, d)], Rc[pk(l, j, d)], r);
          ri = fma(Ric[pk(i, l, d)], a.Rki[pk(l, j, d)], ri);
        }
        Rn[e] = r;
        Rin[e] = ri;
      }
      Rci = Rin;
    }
    grid.sync();
    stamp();
  }
  // outputs: unpack the cumulative factors (or NaN when even the shifted fallback failed)
  const int st1 = ((volatile int*)a.state)[1];
  const double* Rf = a.C[(npass - 1) & 1];
  const double* Rif = a.Ci[(npass - 1) & 1];
  for (int e = blockIdx.x * NT + tid; e < d * d; e += gridDim.x * NT) {
    const int i = e / d, j = e - i * d;
    if (st1 == 2) {
      a.R[e] = a.Rinv[e] = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      a.R[e] = j >= i ? Rf[pk(i, j, d)] : 0.0;
      a.Rinv[e] = j >= i ? Rif[pk(i, j, d)] : 0.0;
    }
  }
  if (blockIdx.x == 0 && tid == 0 && st1 != 2) *a.info = shifted ? -1 : 0;
  stamp();
}

int cond_grid() {
  static int g = 0;
  if (g) return g;
  int dev = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  g = coop ? std::min(fct::num_sms(), 1024) : 0;
  return g;
}

size_t cond_smem(int d) {
  const size_t DP = (size_t)(d + 3) / 4 * 4, T = (size_t)d * (d + 1) / 2;
  const size_t p1 = (size_t)d * DP + 2 * (size_t)ROWS * DP;
  return sizeof(double) * std::max(std::max(p1, 2 * T + 3 * 16 * (size_t)NBLK_MAX), (size_t)NW * 32);
}

size_t ntile_of(int64_t d) {
  const size_t nb = (size_t)(d + 3) / 4;
  return nb * (nb + 1) / 2;
}

}  // namespace

extern "C" size_t fct_condition_workspace_bytes(int32_t r1, int64_t d) {
  if (r1 < 1 || d < 1) return 0;
  const size_t T = (size_t)d * (d + 1) / 2, V = ntile_of(d) * 16;
  return fct::align256(sizeof(double) * 1024 * V) + fct::align256(sizeof(double) * V) +
         6 * fct::align256(sizeof(double) * T) + fct::align256(4 * sizeof(int)) +
         fct::align256(64 * sizeof(unsigned long long));
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
  const int grid = cond_grid();
  FCT_CHECK_ARG(grid >= 1, FCT_ERR_CUDA, "fct_condition: cooperative launch not supported");
  const size_t T = (size_t)d * (d + 1) / 2;
  Args a;
  a.Y = Y; a.r1 = r1; a.d = (int)d; a.T = (int)T;
  a.nb = (int)((d + 3) / 4); a.ntile = (int)ntile_of(d);
  fct::Carver cv(workspace);
  a.Gp = cv.take<double>((size_t)1024 * a.ntile * 16);
  a.G = cv.take<double>((size_t)a.ntile * 16);
  a.Rk = cv.take<double>(T);
  a.Rki = cv.take<double>(T);
  for (int q = 0; q < 2; ++q) { a.C[q] = cv.take<double>(T); a.Ci[q] = cv.take<double>(T); }
  a.state = cv.take<int>(4);
  unsigned long long* ts = cv.take<unsigned long long>(64);
  a.ts = getenv("FCT_COND_TIMING") ? ts : nullptr;
  a.series = getenv("FCT_COND_NOSERIES") ? 0 : 1;
  a.R = R; a.Rinv = Rinv; a.info = info;
  FCT_CUDA_RET(cudaMemsetAsync(a.state, 0, 4 * sizeof(int), st));
  const size_t smem = cond_smem((int)d);
  const int nblk = d <= 16 ? 1 : d <= 32 ? 2 : d <= 64 ? 4 : 8;
  auto kern = nblk == 1 ? cond_kernel<1> : nblk == 2 ? cond_kernel<2> : nblk == 4 ? cond_kernel<4> : cond_kernel<8>;
  static size_t smem_set[4] = {0, 0, 0, 0};
  const int ki = nblk == 1 ? 0 : nblk == 2 ? 1 : nblk == 4 ? 2 : 3;
  if (smem > smem_set[ki]) {
    FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set[ki] = smem;
  }
  void* args[] = {&a};
  FCT_CUDA_RET(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(NT), args, smem, st));
  FCT_LAUNCHED("cond_kernel", st);
  return FCT_OK;
}
