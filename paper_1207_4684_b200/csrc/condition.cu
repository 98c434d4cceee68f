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
//   3 [CTA 0]     blocked Cholesky (8-row panels: one warp factors the panel, all warps apply the rank-8
//                 trailing update, 2 barriers per panel) and blocked triangular inverse (same shape);
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
constexpr int NB = 8;          // Cholesky / inverse panel height
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
    if (a.ts && blockIdx.x == 0 && tid == 0 && nts < 64) a.ts[nts++] = gtimer();
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
    // ================= phase 3 (CTA 0): blocked Cholesky and blocked triangular inverse
    if (blockIdx.x == 0) {
      double* Gs = sm;        // packed [T]: G, then R_k (rows scaled)
      double* Xs = sm + T;    // packed [T]: R_k^-1
      __shared__ int fail;
      __shared__ double sigma;
      __shared__ double dinv[FCT_MAX_D];   // 1 / R_k[i][i]
      if (tid == 0) { fail = 0; sigma = 0.0; }
      for (int e = tid; e < a.nb * a.nb * 16; e += NT) {   // unpack the tile record into the packed upper triangle
        const int bij = e >> 4, x = (e >> 2) & 3, y = e & 3;
        const int bi = bij / a.nb, bj = bij - bi * a.nb;
        const int i = 4 * bi + x, j = 4 * bj + y;
        if (bj >= bi && i < d && j < d && j >= i) Gs[pk(i, j, d)] = a.G[16 * pk(bi, bj, a.nb) + (e & 15)];
      }
      __syncthreads();
      if (pass == 0 && shifted) {   // sigma = 11 (r1 d + d (d + 1)) u ||Y||_F^2, ||Y||_F^2 = trace(G)
        if (tid == 0) {
          double tr = 0.0;
          for (int i = 0; i < d; ++i) tr += Gs[pk(i, i, d)];
          sigma = 11.0 * ((double)a.r1 * d + (double)d * (d + 1)) * u * tr;
        }
        __syncthreads();
        for (int i = tid; i < d; i += NT) Gs[pk(i, i, d)] += sigma;
        __syncthreads();
      }
      if (pass == 1 && !shifted) {  // CholeskyQR2's second Gram must be close to I
        for (int i = warp; i < d; i += NW) {
          const double* rowi = Gs + pk(i, i, d) - i;
          for (int c = i + lane; c < d; c += 32)
            if (!(fabs(rowi[c] - (c == i ? 1.0 : 0.0)) <= 0.5)) fail = 1;
        }
        __syncthreads();
      }
      stamp();
      // ---- blocked right-looking Cholesky, G = R^T R on the packed upper triangle (row i: rowi[c], c >= i)
      for (int jb = 0; jb < d && !fail; jb += NB) {
        const int jn = min(NB, d - jb);
        if (warp == 0) {   // panel rows jb .. jb+jn-1 in registers (lane: columns lane + 32k), factored by one warp
          double v[NB][4];
#pragma unroll
          for (int q = 0; q < NB; ++q)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane + 32 * k, i = jb + q;
              v[q][k] = (q < jn && c >= i && c < d) ? Gs[pk(i, c, d)] : 0.0;
            }
#pragma unroll
          for (int p = 0; p < NB; ++p) {
            if (p < jn) {
              const int j = jb + p, kj = j >> 5;
              const double vj = kj == 0 ? v[p][0] : kj == 1 ? v[p][1] : kj == 2 ? v[p][2] : v[p][3];
              const double piv = __shfl_sync(0xffffffffu, vj, j & 31);
              if (!(piv > 0.0) || !isfinite(piv)) {
                if (lane == 0 && !fail) fail = j + 1;
              } else {
                const double rs = rsqrt(piv);   // R row j = G row j / sqrt(piv); rows below: G_q -= R_j[q] R_j
#pragma unroll
                for (int k = 0; k < 4; ++k) v[p][k] *= rs;
                if (lane == 0) dinv[j] = rs;
#pragma unroll
                for (int q = p + 1; q < NB; ++q) {
                  if (q < jn) {
                    const int i = jb + q, ki = i >> 5;
                    const double wi = ki == 0 ? v[p][0] : ki == 1 ? v[p][1] : ki == 2 ? v[p][2] : v[p][3];
                    const double f = __shfl_sync(0xffffffffu, wi, i & 31);
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[q][k] = fma(-f, v[p][k], v[q][k]);
                  }
                }
              }
            }
          }
#pragma unroll
          for (int q = 0; q < NB; ++q)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane + 32 * k, i = jb + q;
              if (q < jn && c >= i && c < d) Gs[pk(i, c, d)] = v[q][k];
            }
        }
        __syncthreads();
        if (fail) break;
        // trailing rank-jn update of rows i >= jb + jn: G[i][c] -= sum_q R[jb+q][i] R[jb+q][c]
        const int i0 = jb + jn;
        if (i0 < d) {
          double P[NB][4];
#pragma unroll
          for (int q = 0; q < NB; ++q)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane + 32 * k, j = jb + q;
              P[q][k] = (q < jn && c >= i0 && c < d) ? Gs[pk(j, c, d)] : 0.0;
            }
          for (int i = i0 + warp; i < d; i += NW) {
            double f[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) f[q] = q < jn ? Gs[pk(jb + q, i, d)] : 0.0;
            double* rowi = Gs + pk(i, i, d) - i;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int c = lane + 32 * k;
              if (c >= i && c < d) {
                double v = rowi[c];
#pragma unroll
                for (int q = 0; q < NB; ++q) v = fma(-f[q], P[q][k], v);
                rowi[c] = v;
              }
            }
          }
        }
        __syncthreads();
      }
      __syncthreads();
      if (fail) {
        if (tid == 0) {
          if (!shifted) a.state[1] = 1;                 // restart with the shift (shifted CholeskyQR3)
          else { a.state[1] = 2; *a.info = fail; }
        }
      } else {
        stamp();
        // ---- blocked inverse X = R^-1 (upper): acc = I; panels from the bottom: (a) one warp finalises the
        // panel rows by back substitution inside the panel, (b) all warps subtract the panel's contribution
        // from the rows above: acc[r][c] -= sum_{l in panel} R[r][l] X[l][c]
        for (int e = tid; e < T; e += NT) Xs[e] = 0.0;
        __syncthreads();
        for (int i = tid; i < d; i += NT) Xs[pk(i, i, d)] = 1.0;
        __syncthreads();
        const int last = ((d - 1) / NB) * NB;
        for (int pr = last; pr >= 0; pr -= NB) {
          const int pn = min(NB, d - pr);
          if (warp == 0) {   // panel rows pr .. pr+pn-1 of acc in registers; back substitution inside the panel
            double x[NB][4];
#pragma unroll
            for (int q = 0; q < NB; ++q)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k, i = pr + q;
                x[q][k] = (q < pn && c >= i && c < d) ? Xs[pk(i, c, d)] : 0.0;
              }
#pragma unroll
            for (int p = NB - 1; p >= 0; --p) {
              if (p < pn) {
                const int i = pr + p;
#pragma unroll
                for (int l = p + 1; l < NB; ++l)
                  if (l < pn) {
                    const double rl = Gs[pk(i, pr + l, d)];
#pragma unroll
                    for (int k = 0; k < 4; ++k) x[p][k] = fma(-rl, x[l][k], x[p][k]);
                  }
                const double di = dinv[i];
#pragma unroll
                for (int k = 0; k < 4; ++k) x[p][k] *= di;
              }
            }
#pragma unroll
            for (int q = 0; q < NB; ++q)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k, i = pr + q;
                if (q < pn && c >= i && c < d) Xs[pk(i, c, d)] = x[q][k];
              }
          }
          __syncthreads();
          if (pr > 0) {
            double Xp[NB][4];
#pragma unroll
            for (int q = 0; q < NB; ++q)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k, l = pr + q;
                Xp[q][k] = (q < pn && c >= l && c < d) ? Xs[pk(l, c, d)] : 0.0;
              }
            for (int r = warp; r < pr; r += NW) {
              double f[NB];
#pragma unroll
              for (int q = 0; q < NB; ++q) f[q] = q < pn ? Gs[pk(r, pr + q, d)] : 0.0;
              double* xr = Xs + pk(r, r, d) - r;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                if (c >= pr && c < d) {
                  double v = xr[c];
#pragma unroll
                  for (int q = 0; q < NB; ++q) v = fma(-f[q], Xp[q][k], v);
                  xr[c] = v;
                }
              }
            }
          }
          __syncthreads();
        }
        stamp();
        for (int e = tid; e < T; e += NT) { a.Rk[e] = Gs[e]; a.Rki[e] = Xs[e]; }
        if (tid == 0) a.state[1] = 0;
      }
    }
    grid.sync();
    stamp();
    const int st1 = ((volatile int*)a.state)[1];
    if (st1 == 2) break;                                                            // failed even with the shift
    if (st1 == 1) { shifted = 1; npass = 3; pass = -1; Rci = nullptr; continue; }   // restart: shifted CholeskyQR3
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
  return sizeof(double) * std::max(std::max(p1, 2 * T), (size_t)NW * 32);
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
  a.R = R; a.Rinv = Rinv; a.info = info;
  FCT_CUDA_RET(cudaMemsetAsync(a.state, 0, 4 * sizeof(int), st));
  const size_t smem = cond_smem((int)d);
  static size_t smem_set = 0;
  if (smem > smem_set) {
    FCT_CUDA_RET(cudaFuncSetAttribute(cond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  void* args[] = {&a};
  FCT_CUDA_RET(cudaLaunchCooperativeKernel((const void*)cond_kernel, dim3(grid), dim3(NT), args, smem, st));
  FCT_LAUNCHED("cond_kernel", st);
  return FCT_OK;
}
