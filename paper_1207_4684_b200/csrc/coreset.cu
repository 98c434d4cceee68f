// coreset.cu -- NEXT-2: FastCauchyRegression steps 6-8 (PAPER.md P:L2178-2188,
// Thm P:L2955-2980): build the coreset DA, Db from the sampler's (idx, weight) and solve
//     x_hat = argmin_x ||D(Ax - b)||_1 = argmin_x sum_j |Z_j . [x; 1]|,   Z = D [A, -b].
//
// l1_coreset_gather: Z_j = weight_j * X[idx_j - row_base]   (fp64, one rounding per entry; data-parallel)
// l1_lad_solve:      the l1 regression as the LP  min 1'u + 1'v  s.t.  At x + u - v = bt,  u, v >= 0
//                    (At = Z[:, :p], bt = -Z[:, p]) and its dual  max bt'y  s.t.  At'y = 0, -1 <= y <= 1,
//                    by a primal-dual path-following interior-point method with Mehrotra's predictor-
//                    corrector.  Newton system per iteration, with theta_i = 1 / (u_i/su_i + v_i/sv_i),
//                    su = 1 - y, sv = 1 + y (dual slacks):
//                        (At' Theta At) dx = At' Theta q + At' y,      dy = theta (q - At dx),
//                        du = (gu + u dy) / su,   dv = (gv - v dy) / sv,
//                    with q = rho - u + v - gu/su + gv/sv, rho = bt - At x;  gu = sigma mu - u su (- du_a dsu_a),
//                    gv = sigma mu - v sv (- dv_a dsv_a) (predictor: sigma = 0, no second-order term).
//                    Stopping: f(x) - sum_i y_i rho_i(x) <= tol * max(f(x), 1e-5 f(0)) (f(x) = sum |rho_i(x)| the
//                    true objective; sum y rho is the dual value b'y - (At'y)'x, exact weak-duality bound when
//                    At'y = 0).
// One persistent cooperative kernel: each CTA owns a contiguous row range; per iteration the rows are
// streamed twice for the weighted Gram (tcgen05 is not used: the Gram is fp64, m p^2 DFMA, and tiny next to
// the path), per-CTA partials are reduced in a fixed order (deterministic), CTA 0 factors the p x p system
// (Cholesky in shared memory, kept there for the corrector solve), grid-wide barriers separate the phases.
#include <cooperative_groups.h>
#include <math.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int NT = 256;       // threads per CTA
constexpr int RC = 64;        // rows per shared-memory chunk (NT / RC = 4 threads per row for the dot)
static_assert(NT == 4 * RC, "phase A row dot uses 4 threads per row");
constexpr int MAXQ = 128;     // q <= 128  ->  p <= 127
constexpr int MT = 3;         // max 4x4 Gram tiles per thread (ceil(561 / 256))
constexpr int NSC = 8;        // scalar partials per CTA

struct Geom {
  int q, p, P4, nb, T, NG, PE, SW;  // SW = chunk row stride (doubles, odd)
  __host__ __device__ Geom(int q_) : q(q_), p(q_ - 1) {
    P4 = (q + 3) / 4 * 4;                 // augmented vector [a (p), rho] has q entries
    nb = P4 / 4;
    T = nb * (nb + 1) / 2;                // upper-triangle 4x4 tiles
    NG = T >= NT ? 1 : NT / T;            // row groups sharing the tiles
    PE = 16 * T + P4 + NSC;               // partial record: tiles | At'y | scalars
    SW = P4 + 1;
  }
};

__device__ __forceinline__ void tile_jk(int t, int nb, int& J, int& K) {
  // inverse of t = J*nb - J(J-1)/2 + (K - J), J <= K
  J = 0;
  while (t >= nb - J) {
    t -= nb - J;
    ++J;
  }
  K = J + t;
}

struct Ws {
  double *u, *v, *y, *su, *sv, *th, *rho, *dya, *du, *dv, *dy;
  double *part, *red, *rat, *mus;   // per-CTA partials, reduced record, ratio / mu partials
  double *x, *dx, *dxa;             // p each
  double* scal;                     // misc scalars
};

__device__ __forceinline__ void ratio_min(double val, double dval, double& amin) {
  if (dval < 0.0) amin = fmin(amin, -val / dval);
}

// block-wide reductions (NT threads)
__device__ double block_sum(double v, double* red_s) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red_s[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < NT / 32; ++w) s += red_s[w];
  return s;
}
__device__ double block_min(double v, double* red_s) {
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red_s[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = red_s[0];
  for (int w = 1; w < NT / 32; ++w) s = fmin(s, red_s[w]);
  return s;
}

// rows [c0, c0 + nr) of Z, columns [0, nc), into S (row stride SW), zero-padded to RC x P4; the loads of a
// thread are issued together (8 in flight) before the shared stores
__device__ __forceinline__ void load_chunk(double* __restrict__ S, const double* __restrict__ Z, int64_t ldz, int64_t c0,
                                           int nr, int nc, int P4, int SW) {
  const int total = RC * P4;
  for (int e0 = threadIdx.x; e0 < total; e0 += 8 * NT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * NT;
      const int r = e / P4, j = e - r * P4;
      v[u] = (e < total && r < nr && j < nc) ? Z[(c0 + r) * ldz + j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * NT;
      if (e < total) {
        const int r = e / P4, j = e - r * P4;
        S[r * SW + j] = v[u];
      }
    }
  }
}

// a_i . xs for row i of Z with 4 threads per row (lanes 4r..4r+3), result in all four lanes
__device__ __forceinline__ double row_dot4(const double* __restrict__ a, const double* __restrict__ xs, int p, bool ok) {
  const int sub = threadIdx.x & 3;
  double d = 0.0;
  if (ok)
    for (int j = sub; j < p; j += 4) d = fma(a[j], xs[j], d);
  d += __shfl_xor_sync(0xffffffffu, d, 1);
  d += __shfl_xor_sync(0xffffffffu, d, 2);
  return d;
}

// reductions over the per-CTA partials: one load per thread, then a fixed-shape tree (deterministic)
__device__ double parts_sum(const double* a, int n, double* red_s) {
  double v = 0.0;
  for (int c = threadIdx.x; c < n; c += NT) v += a[c];
  return block_sum(v, red_s);
}
__device__ double parts_min(const double* a, int n, int stride, double* red_s) {
  double v = 1e300;
  for (int c = threadIdx.x; c < n; c += NT) v = fmin(v, a[(size_t)c * stride]);
  return block_min(v, red_s);
}
// warp-cooperative sum of column e over n records of length PE (lanes take records c = lane, lane + 32, ...)
__device__ __forceinline__ double warp_col_sum(const double* part, int n, int PE, int e) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int c = lane; c < n; c += 32) v += part[(size_t)c * PE + e];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(NT, 1)
lad_ipm_kernel(const double* __restrict__ Z, int64_t ldz, const int64_t* __restrict__ mptr, int64_t capacity, int q,
               int max_iter, double tol, Ws w, double* __restrict__ xout, double* __restrict__ info) {
  cg::grid_group grid = cg::this_grid();
  const Geom g(q);
  const int p = g.p, tid = threadIdx.x, cta = blockIdx.x, ncta = gridDim.x;
  extern __shared__ __align__(16) double sm[];
  // [chunk S: RC x SW] [theta_s RC] [y_s RC] [x_s MAXQ] [red_s 32] [D0, RH, IV: MAXQ] [G: p x (p+1), CTA 0]
  double* S = sm;
  double* ths = S + (RC * g.SW > NT * 16 ? RC * g.SW : NT * 16);  // chunk | group-reduction staging
  double* yss = ths + RC;
  double* xs = yss + RC;
  double* red_s = xs + MAXQ;
  double* D0 = red_s + 32;
  double* RH = D0 + MAXQ;
  double* IV = RH + MAXQ;  // 1 / L_kk
  double* G = IV + MAXQ;
  const int GS = p + 1;  // row stride of G

  int64_t m = mptr ? *mptr : capacity;
  if (m > capacity) m = capacity;
  if (m < 0) m = 0;
  const int64_t r0 = m * cta / ncta, r1 = m * (cta + 1) / ncta;

  // tile assignment
  int myT[MT], myJ[MT], myK[MT], ntile = 0, grp = 0;
  if (g.T >= NT) {
    for (int t = tid; t < g.T && ntile < MT; t += NT) myT[ntile++] = t;
  } else if (tid < g.NG * g.T) {
    myT[ntile++] = tid % g.T;
    grp = tid / g.T;
  }
  for (int i = 0; i < ntile; ++i) tile_jk(myT[i], g.nb, myJ[i], myK[i]);

  // ---- initial point: x = 0, rho = bt, u - v = rho with both >= delta = mean |rho|, y = 0
  double loc = 0.0;
  for (int64_t i = r0 + tid; i < r1; i += NT) loc += fabs(Z[i * ldz + p]);
  loc = block_sum(loc, red_s);
  if (tid == 0) w.mus[cta] = loc;
  if (cta == 0)
    for (int j = tid; j < p; j += NT) w.x[j] = 0.0;
  grid.sync();
  const double tot = parts_sum(w.mus, ncta, red_s);
  const double delta = m > 0 ? fmax(tot / (double)m, 1e-300) : 1.0;
  for (int64_t i = r0 + tid; i < r1; i += NT) {
    const double rh = -Z[i * ldz + p];
    w.u[i] = fmax(rh, 0.0) + delta;
    w.v[i] = fmax(-rh, 0.0) + delta;
    w.y[i] = 0.0;
    w.su[i] = 1.0;
    w.sv[i] = 1.0;
  }
  grid.sync();

  int it = 0, status = 1, nsing = 0;
  double f = 0.0, dual = 0.0, gnorm = 0.0;
  const double f0 = tot;  // objective at x = 0 (scale of the absolute floor of the stopping test)
  const double eta = 0.99995;
  for (;; ++it) {
    // ================= A: rho, theta, Gram of [a, rho] weighted by theta, At'y, scalars
    for (int j = tid; j < MAXQ; j += NT) xs[j] = j < p ? w.x[j] : 0.0;
    double acc[MT][16];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[i][e] = 0.0;
    double gy = 0.0, s_f = 0.0, s_yr = 0.0, s_comp = 0.0, s_rp = 0.0;
    __syncthreads();
    for (int64_t c0 = r0; c0 < r1; c0 += RC) {
      const int nr = (int)min((int64_t)RC, r1 - c0);
      load_chunk(S, Z, ldz, c0, nr, q, g.P4, g.SW);
      __syncthreads();
      {
        // rho_r = -(a_r . x + z_rp): 4 threads per row, lanes 4r..4r+3 take columns sub, sub + 4, ...
        const int rr = tid >> 2, sub = tid & 3;
        const double* a = S + rr * g.SW;
        double d0 = 0.0;
        for (int j = sub; j < p; j += 4) d0 = fma(a[j], xs[j], d0);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 1);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 2);
        double th = 0.0, yv = 0.0;
        if (sub == 0 && rr < nr) {
          const int64_t i = c0 + rr;
          const double rh = -(d0 + a[p]);
          const double u = w.u[i], v = w.v[i], su = w.su[i], sv = w.sv[i];
          yv = w.y[i];
          th = 1.0 / (u / su + v / sv);
          w.th[i] = th;
          w.rho[i] = rh;
          s_f += fabs(rh);
          s_yr += yv * rh;
          s_comp += u * su + v * sv;
          s_rp += fabs(rh - u + v);
        }
        __syncthreads();  // every lane of the row has read a[p] before it is replaced by rho
        if (sub == 0) {
          if (rr < nr) S[rr * g.SW + p] = -(d0 + a[p]);
          ths[rr] = th;
          yss[rr] = yv;
        }
      }
      __syncthreads();
      for (int i = 0; i < ntile; ++i) {
        const int J = myJ[i], K = myK[i];
        for (int r = grp; r < nr; r += g.NG) {
          const double* a = S + r * g.SW;
          const double t = ths[r];
          const double aj0 = t * a[4 * J], aj1 = t * a[4 * J + 1], aj2 = t * a[4 * J + 2], aj3 = t * a[4 * J + 3];
          const double ak0 = a[4 * K], ak1 = a[4 * K + 1], ak2 = a[4 * K + 2], ak3 = a[4 * K + 3];
          double* A_ = acc[i];
          A_[0] = fma(aj0, ak0, A_[0]); A_[1] = fma(aj0, ak1, A_[1]); A_[2] = fma(aj0, ak2, A_[2]); A_[3] = fma(aj0, ak3, A_[3]);
          A_[4] = fma(aj1, ak0, A_[4]); A_[5] = fma(aj1, ak1, A_[5]); A_[6] = fma(aj1, ak2, A_[6]); A_[7] = fma(aj1, ak3, A_[7]);
          A_[8] = fma(aj2, ak0, A_[8]); A_[9] = fma(aj2, ak1, A_[9]); A_[10] = fma(aj2, ak2, A_[10]); A_[11] = fma(aj2, ak3, A_[11]);
          A_[12] = fma(aj3, ak0, A_[12]); A_[13] = fma(aj3, ak1, A_[13]); A_[14] = fma(aj3, ak2, A_[14]); A_[15] = fma(aj3, ak3, A_[15]);
        }
      }
      if (tid < p)
        for (int r = 0; r < nr; ++r) gy = fma(yss[r], S[r * g.SW + tid], gy);
      __syncthreads();
    }
    // CTA partial record
    double* P = w.part + (size_t)cta * g.PE;
    if (g.NG == 1) {
      for (int i = 0; i < ntile; ++i)
        for (int e = 0; e < 16; ++e) P[16 * myT[i] + e] = acc[i][e];
    } else {
      // reduce the NG row groups through shared memory (the chunk region is free now)
      for (int e = 0; e < 16; ++e) {
        if (ntile) S[(size_t)tid * 16 + e] = acc[0][e];
      }
      __syncthreads();
      for (int e = tid; e < 16 * g.T; e += NT) {
        const int t = e >> 4, k = e & 15;
        double s = 0.0;
        for (int gg = 0; gg < g.NG; ++gg) s += S[(size_t)(gg * g.T + t) * 16 + k];
        P[e] = s;
      }
    }
    if (tid < g.P4) P[16 * g.T + tid] = tid < p ? gy : 0.0;
    {
      const double a0 = block_sum(s_f, red_s);
      const double a1 = block_sum(s_yr, red_s);
      const double a2 = block_sum(s_comp, red_s);
      const double a3 = block_sum(s_rp, red_s);
      if (tid == 0) {
        double* sc = P + 16 * g.T + g.P4;
        sc[0] = a0; sc[1] = a1; sc[2] = a2; sc[3] = a3;
      }
    }
    grid.sync();
    // ================= B: fixed-order reduction of the partial records
    for (int e = cta * (NT / 32) + (tid >> 5); e < g.PE; e += ncta * (NT / 32)) {
      const double s = warp_col_sum(w.part, ncta, g.PE, e);
      if ((tid & 31) == 0) w.red[e] = s;
    }
    grid.sync();
    const double* scr = w.red + 16 * g.T + g.P4;
    f = scr[0];
    dual = scr[1];
    const double comp = scr[2];
    // relative gap, with an absolute floor at 1e-5 of the x = 0 objective (exact fits: f -> 0)
    const bool conv = m == 0 || f <= 1e-300 || (f - dual) <= tol * fmax(f, 1e-5 * f0);
    if (conv || it >= max_iter || !isfinite(f)) {
      status = conv ? 0 : (isfinite(f) ? 1 : 2);
      for (int j = 0; j < p; ++j) gnorm = fmax(gnorm, fabs(w.red[16 * g.T + j]));
      break;
    }
    const double mu = comp / (2.0 * (double)m);
    if (!(mu > 0.0)) {
      status = 2;
      break;
    }
    // ================= C: CTA 0 factors G = At' Theta At and solves for the predictor direction
    // (everything in shared memory: G/L, the original diagonal D0 and the right-hand side RH)
    if (cta == 0) {
      auto gram = [&](int j, int k) -> double {  // augmented Gram entry, j <= k
        const int J = j >> 2, K = k >> 2;
        const int t = J * g.nb - J * (J - 1) / 2 + (K - J);
        return w.red[16 * t + 4 * (j & 3) + (k & 3)];
      };
      for (int e = tid; e < p * p; e += NT) {
        const int j = e / p, k = e - j * p;
        if (k <= j) G[j * GS + k] = gram(k, j);  // lower triangle
      }
      for (int j = tid; j < p; j += NT) {
        D0[j] = gram(j, j);
        RH[j] = gram(j, p) + w.red[16 * g.T + j];  // rhs: At'Theta rho + At'y
      }
      __syncthreads();
      // Cholesky (lower, in place), blocked by 8 columns: the diagonal block by warp 0 (warp-synchronous),
      // the panel below it by one thread per row, the trailing update by warps over rows -- three CTA
      // barriers per 8 columns.  A pivot that collapses relative to its original diagonal is replaced by
      // 1e128 (that component of the step is dropped) -- the usual safeguard near the optimal face.
      const int wid = tid >> 5, lane = tid & 31;
      for (int k0 = 0; k0 < p; k0 += 8) {
        const int kb = min(8, p - k0), ke = k0 + kb;
        if (wid == 0) {
          for (int k = k0; k < ke; ++k) {
            if (lane == 0) {
              double piv = G[k * GS + k];
              if (!(piv > 1e-14 * D0[k]) || !isfinite(piv)) {
                piv = 1e128;
                ++nsing;
              }
              const double lkk = sqrt(piv);
              G[k * GS + k] = lkk;
              IV[k] = 1.0 / lkk;
            }
            __syncwarp();
            if (lane < ke - k - 1) G[(k + 1 + lane) * GS + k] *= IV[k];
            __syncwarp();
            for (int e = lane; e < 64; e += 32) {   // rows i, cols j of the block, k < j <= i < ke
              const int i = k + 1 + (e >> 3), j = k + 1 + (e & 7);
              if (i < ke && j <= i) G[i * GS + j] -= G[i * GS + k] * G[j * GS + k];
            }
            __syncwarp();
          }
        }
        __syncthreads();
        // panel: rows i >= ke solve X L_bb^T = G[i, k0:ke] (forward substitution over the block's columns)
        for (int i = ke + tid; i < p; i += NT) {
          double x[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if (kk < kb) {
              double v = G[i * GS + k0 + kk];
              for (int jj = 0; jj < kk; ++jj) v -= x[jj] * G[(k0 + kk) * GS + k0 + jj];
              x[kk] = v * IV[k0 + kk];
              G[i * GS + k0 + kk] = x[kk];
            }
          }
        }
        __syncthreads();
        // trailing update G[i][j] -= sum_kk G[i][k0+kk] G[j][k0+kk], ke <= j <= i < p
        for (int i = ke + wid; i < p; i += NT / 32) {
          double li[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) li[kk] = kk < kb ? G[i * GS + k0 + kk] : 0.0;
          for (int j = ke + lane; j <= i; j += 32) {
            double acc = G[i * GS + j];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              if (kk < kb) acc -= li[kk] * G[j * GS + k0 + kk];
            G[i * GS + j] = acc;
          }
        }
        __syncthreads();
      }
    }
    auto solve = [&](double* out) {  // CTA 0: RH := (L L')^-1 RH (blocked by 8), then out := RH
      const int wid = tid >> 5, lane = tid & 31;
      for (int k0 = 0; k0 < p; k0 += 8) {  // forward: L w = RH
        const int ke = min(p, k0 + 8);
        if (wid == 0) {
          for (int k = k0; k < ke; ++k) {
            const double wk = RH[k] * IV[k];
            __syncwarp();
            if (lane == 0) RH[k] = wk;
            if (lane < ke - k - 1) RH[k + 1 + lane] -= G[(k + 1 + lane) * GS + k] * wk;
            __syncwarp();
          }
        }
        __syncthreads();
        for (int i = ke + tid; i < p; i += NT) {
          double v = RH[i];
          for (int k = k0; k < ke; ++k) v -= G[i * GS + k] * RH[k];
          RH[i] = v;
        }
        __syncthreads();
      }
      for (int kb0 = (p - 1) / 8 * 8; kb0 >= 0; kb0 -= 8) {  // backward: L' x = w
        const int ke = min(p, kb0 + 8);
        if (wid == 0) {
          for (int k = ke - 1; k >= kb0; --k) {
            const double wk = RH[k] * IV[k];
            __syncwarp();
            if (lane == 0) RH[k] = wk;
            if (lane < k - kb0) RH[kb0 + lane] -= G[k * GS + kb0 + lane] * wk;
            __syncwarp();
          }
        }
        __syncthreads();
        for (int i = tid; i < kb0; i += NT) {
          double v = RH[i];
          for (int k = kb0; k < ke; ++k) v -= G[k * GS + i] * RH[k];
          RH[i] = v;
        }
        __syncthreads();
      }
      for (int j = tid; j < p; j += NT) out[j] = RH[j];
      __threadfence();
    };
    if (cta == 0) solve(w.dxa);
    grid.sync();
    // ================= D: affine-scaling direction per row, step-length ratios
    for (int j = tid; j < MAXQ; j += NT) xs[j] = j < p ? w.dxa[j] : 0.0;
    __syncthreads();
    double ap = 1e300, ad = 1e300;
    for (int64_t b0 = r0; b0 < r1; b0 += NT / 4) {
      const int64_t i = b0 + (tid >> 2);
      const bool ok = i < r1;
      const double ad_ = row_dot4(Z + (ok ? i : r0) * ldz, xs, p, ok);
      if (ok && (tid & 3) == 0) {
        const double u = w.u[i], v = w.v[i], su = w.su[i], sv = w.sv[i];
        const double dy = w.th[i] * (w.rho[i] - ad_);
        const double du = -u + u * dy / su, dv = -v - v * dy / sv;
        w.dya[i] = dy;
        ratio_min(u, du, ap);
        ratio_min(v, dv, ap);
        ratio_min(su, -dy, ad);
        ratio_min(sv, dy, ad);
      }
    }
    ap = block_min(ap, red_s);
    ad = block_min(ad, red_s);
    if (tid == 0) {
      w.rat[2 * cta] = ap;
      w.rat[2 * cta + 1] = ad;
    }
    grid.sync();
    // ================= E: mu_aff
    ap = parts_min(w.rat, ncta, 2, red_s);
    ad = parts_min(w.rat + 1, ncta, 2, red_s);
    const double apa = fmin(1.0, ap), ada = fmin(1.0, ad);
    double smu = 0.0;
    for (int64_t i = r0 + tid; i < r1; i += NT) {
      const double u = w.u[i], v = w.v[i], su = w.su[i], sv = w.sv[i], dy = w.dya[i];
      const double du = -u + u * dy / su, dv = -v - v * dy / sv;
      smu += (u + apa * du) * (su - ada * dy) + (v + apa * dv) * (sv + ada * dy);
    }
    smu = block_sum(smu, red_s);
    if (tid == 0) w.mus[cta] = smu;
    grid.sync();
    // ================= F: corrector right-hand side At' Theta q_c
    const double mua = parts_sum(w.mus, ncta, red_s) / (2.0 * (double)m);
    double sig = mua / mu;
    sig = fmin(1.0, sig * sig * sig);
    const double tau = sig * mu;
    double hc = 0.0;
    for (int64_t c0 = r0; c0 < r1; c0 += RC) {
      const int nr = (int)min((int64_t)RC, r1 - c0);
      load_chunk(S, Z, ldz, c0, nr, p, g.P4, g.SW);
      if (tid < RC) {
        double tq = 0.0;
        if (tid < nr) {
          const int64_t i = c0 + tid;
          const double u = w.u[i], v = w.v[i], su = w.su[i], sv = w.sv[i], dya = w.dya[i];
          const double dua = -u + u * dya / su, dva = -v - v * dya / sv;
          const double gu = tau - u * su + dua * dya, gv = tau - v * sv - dva * dya;
          const double qc = (w.rho[i] - u + v) - gu / su + gv / sv;
          tq = w.th[i] * qc;
        }
        ths[tid] = tq;
      }
      __syncthreads();
      if (tid < p)
        for (int r = 0; r < nr; ++r) hc = fma(ths[r], S[r * g.SW + tid], hc);
      __syncthreads();
    }
    if (tid < g.P4) w.part[(size_t)cta * g.PE + tid] = tid < p ? hc : 0.0;
    grid.sync();
    // ================= G: reduce, CTA 0 solves with the kept factor
    if (cta == 0) {
      for (int j = tid >> 5; j < p; j += NT / 32) {
        const double s = warp_col_sum(w.part, ncta, g.PE, j);
        if ((tid & 31) == 0) RH[j] = s + w.red[16 * g.T + j];
      }
      __syncthreads();
      solve(w.dx);
    }
    grid.sync();
    // ================= H: combined direction per row, step-length ratios
    for (int j = tid; j < MAXQ; j += NT) xs[j] = j < p ? w.dx[j] : 0.0;
    __syncthreads();
    ap = 1e300;
    ad = 1e300;
    for (int64_t b0 = r0; b0 < r1; b0 += NT / 4) {
      const int64_t i = b0 + (tid >> 2);
      const bool ok = i < r1;
      const double adx = row_dot4(Z + (ok ? i : r0) * ldz, xs, p, ok);
      if (ok && (tid & 3) == 0) {
        const double u = w.u[i], v = w.v[i], su = w.su[i], sv = w.sv[i], dya = w.dya[i];
        const double dua = -u + u * dya / su, dva = -v - v * dya / sv;
        const double gu = tau - u * su + dua * dya, gv = tau - v * sv - dva * dya;
        const double qc = (w.rho[i] - u + v) - gu / su + gv / sv;
        const double dy = w.th[i] * (qc - adx);
        const double du = (gu + u * dy) / su, dv = (gv - v * dy) / sv;
        w.du[i] = du;
        w.dv[i] = dv;
        w.dy[i] = dy;
        ratio_min(u, du, ap);
        ratio_min(v, dv, ap);
        ratio_min(su, -dy, ad);
        ratio_min(sv, dy, ad);
      }
    }
    ap = block_min(ap, red_s);
    ad = block_min(ad, red_s);
    if (tid == 0) {
      w.rat[2 * cta] = ap;
      w.rat[2 * cta + 1] = ad;
    }
    grid.sync();
    // ================= I: step
    ap = parts_min(w.rat, ncta, 2, red_s);
    ad = parts_min(w.rat + 1, ncta, 2, red_s);
    const double alp = fmin(1.0, eta * ap), ald = fmin(1.0, eta * ad);
    for (int64_t i = r0 + tid; i < r1; i += NT) {
      w.u[i] += alp * w.du[i];
      w.v[i] += alp * w.dv[i];
      const double dy = w.dy[i];
      w.y[i] += ald * dy;
      w.su[i] -= ald * dy;
      w.sv[i] += ald * dy;
    }
    if (cta == 0)
      for (int j = tid; j < p; j += NT) w.x[j] += alp * w.dx[j];
    grid.sync();
  }
  if (cta == 0) {
    for (int j = tid; j < p; j += NT) xout[j] = w.x[j];
    if (tid == 0) {
      info[0] = f;
      info[1] = dual;
      info[2] = f > 0.0 ? (f - dual) / f : 0.0;
      info[3] = (double)it;
      info[4] = gnorm;
      info[5] = (double)status;
      info[6] = (double)m;
      info[7] = (double)nsing;
    }
  }
}

__global__ void coreset_gather_kernel(const float* __restrict__ X, int64_t n, int q, int64_t ldx,
                                      const int64_t* __restrict__ idx, const double* __restrict__ weight,
                                      const int64_t* __restrict__ count, int64_t row_base, int64_t capacity,
                                      double* __restrict__ Z, int64_t ldz) {
  int64_t m = count ? *count : capacity;
  if (m > capacity) m = capacity;
  const int64_t total = m * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / q;
    const int c = (int)(e - j * q);
    const int64_t row = (idx ? idx[j] : j) - row_base;
    const double wj = weight ? weight[j] : 1.0;
    Z[j * ldz + c] = (row >= 0 && row < n) ? wj * (double)X[row * ldx + c] : __longlong_as_double(0x7ff8000000000000LL);
  }
}

size_t lad_smem_bytes(int q) {
  const Geom g(q);
  const size_t base = (size_t)RC * g.SW + 2 * RC + 4 * MAXQ + 32;
  const size_t stage = (size_t)NT * 16;  // group-reduction staging aliases the chunk region
  const size_t chunk = std::max((size_t)RC * g.SW, stage);
  return (chunk - (size_t)RC * g.SW + base + (size_t)g.p * (g.p + 1)) * sizeof(double);
}

int lad_grid() {  // one CTA per SM; the attribute is set once for the largest q
  static int grid = 0;
  if (grid) return grid;
  const size_t smem = lad_smem_bytes(MAXQ);
  if (cudaFuncSetAttribute(lad_ipm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lad_ipm_kernel, NT, smem) != cudaSuccess || per < 1) return 0;
  return grid = std::min(fct::num_sms(), 1024);
}

}  // namespace

extern "C" fct_status l1_coreset_gather(const float* X, int64_t n, int64_t q, int64_t ldx, const int64_t* idx,
                                        const double* weight, const int64_t* count, int64_t row_base,
                                        int64_t capacity, double* Z, int64_t ldz, void* stream) {
  FCT_CHECK_ARG(X && Z, FCT_ERR_ARG, "l1_coreset_gather: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && q >= 1 && ldx >= q && ldz >= q && capacity >= 0 && row_base >= 0, FCT_ERR_SHAPE,
                "l1_coreset_gather: n=%lld q=%lld ldx=%lld ldz=%lld capacity=%lld", (long long)n, (long long)q,
                (long long)ldx, (long long)ldz, (long long)capacity);
  if (capacity == 0) return FCT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = capacity * q;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)fct::num_sms() * 8);
  coreset_gather_kernel<<<blocks, 256, 0, st>>>(X, n, (int)q, ldx, idx, weight, count, row_base, capacity, Z, ldz);
  FCT_LAUNCHED("l1_coreset_gather", st);
  return FCT_OK;
}

extern "C" size_t l1_lad_workspace_bytes(int64_t capacity, int64_t q) {
  if (q < 2 || q > MAXQ || capacity < 0) return 0;
  const Geom g((int)q);
  const int nc = 1024;  // upper bound on the cooperative grid
  fct::Carver c(nullptr);
  for (int a = 0; a < 11; ++a) c.take<double>((size_t)capacity);
  c.take<double>((size_t)nc * g.PE);
  c.take<double>((size_t)g.PE);
  c.take<double>(2 * nc);
  c.take<double>(nc);
  c.take<double>(3 * MAXQ);
  c.take<double>(16);
  return c.off;
}

extern "C" fct_status l1_lad_solve(const double* Z, const int64_t* m, int64_t capacity, int64_t q, int64_t ldz,
                                   int32_t max_iter, double tol, double* x, double* info, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(Z && x && info, FCT_ERR_ARG, "l1_lad_solve: NULL pointer");
  FCT_CHECK_ARG(q >= 2 && q <= MAXQ && ldz >= q && capacity >= 1, FCT_ERR_SHAPE,
                "l1_lad_solve: q=%lld (2..%d) ldz=%lld capacity=%lld", (long long)q, MAXQ, (long long)ldz,
                (long long)capacity);
  FCT_CHECK_ARG(max_iter >= 1 && tol > 0.0, FCT_ERR_ARG, "l1_lad_solve: max_iter=%d tol=%g", max_iter, tol);
  const size_t need = l1_lad_workspace_bytes(capacity, q);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_ARG, "l1_lad_solve: workspace %zu < %zu bytes",
                workspace_bytes, need);
  const int grid = lad_grid();
  FCT_CHECK_ARG(grid >= 1 && grid <= 1024, FCT_ERR_CUDA, "l1_lad_solve: cooperative launch not possible");
  fct::Carver c(workspace);
  const Geom g((int)q);
  Ws w;
  double** rows[11] = {&w.u, &w.v, &w.y, &w.su, &w.sv, &w.th, &w.rho, &w.dya, &w.du, &w.dv, &w.dy};
  for (auto r : rows) *r = c.take<double>((size_t)capacity);
  w.part = c.take<double>((size_t)1024 * g.PE);
  w.red = c.take<double>((size_t)g.PE);
  w.rat = c.take<double>(2 * 1024);
  w.mus = c.take<double>(1024);
  w.x = c.take<double>(3 * MAXQ);
  w.dx = w.x + MAXQ;
  w.dxa = w.x + 2 * MAXQ;
  w.scal = c.take<double>(16);
  cudaStream_t st = (cudaStream_t)stream;
  int qi = (int)q;
  void* args[] = {(void*)&Z, (void*)&ldz, (void*)&m, (void*)&capacity, (void*)&qi, (void*)&max_iter, (void*)&tol,
                  (void*)&w, (void*)&x, (void*)&info};
  FCT_CUDA_RET(cudaLaunchCooperativeKernel((const void*)lad_ipm_kernel, dim3(grid), dim3(NT), args,
                                           lad_smem_bytes((int)q), st));
  FCT_LAUNCHED("l1_lad_solve", st);
  return FCT_OK;
}
