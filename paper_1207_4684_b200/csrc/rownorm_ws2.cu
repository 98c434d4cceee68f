// rownorm_ws2.cu -- K2 v3: l1 row-norm estimate lambda_i = median_j |(A (Rinv Pi2))_ij|
// (Lemma medCauchy; the FastCauchyRegression row norms P:L2921-2938, with
// M = Rinv Pi2 formed first).  Warp-specialised, one persistent CTA per SM:
//   warp 0-3   split: thread r <-> tile row r <-> TMEM lane r.  ||a||_2^2 -> smem, A_lo = A - tf32(A) -> TMEM.
//   warp 4     TMA producer: 128-row tiles of A (SWIZZLE_128B) into NA shared buffers.
//   warp 5     MMA issuer: D = A*M_hi + A*M_lo + A_lo*M_hi (3xTF32, kind::tf32) into a rotating TMEM
//              accumulator (descriptors precomputed), committed to mbarriers.
//   warp 6..   EG epilogue groups of 4 warps (one TMEM lane quadrant each); group g takes tiles g mod EG:
//              tcgen05.ld of D, the certified median for a compile-time k (below), lambda, sum lambda.
// Certified median (K2): with v_j = |D_j| and the rigorous bound |v_j - |Lambda_ij|| <= e_j =
// gam ||a||_2 ||m~_j||_2 (gam covers the 3xTF32 evaluation and the fp32 rounding of M), the order statistic
// t_(m1) >= L = min_{v_j >= v_(m1)} (v_j - e_j) and t_(m2) <= H = max_{v_j <= v_(m2)} (v_j + e_j); entries with
// v_j + e_j < L lie below the middle, entries with v_j - e_j > H above it, and the rest (1-2 per row) are
// evaluated exactly in fp64 from the row kept in shared memory (fp64 M) and ranked.  lambda is the exact
// median up to fp64 rounding, rounded once to fp32.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <type_traits>
#include "common.cuh"
#include "selnet.cuh"
#include "tc.cuh"

namespace {

constexpr int kSplitWarps = 4;
constexpr int kTmaWarp = 4;
constexpr int kMmaWarp = 5;
constexpr int kEpiWarp0 = 6;

struct CSwap2 {
  __device__ __forceinline__ void operator()(float& a, float& b) const {
    const float lo = fminf(a, b), hi = fmaxf(a, b);
    a = lo;
    b = hi;
  }
};

// exact |sum_l a_l M_lj| for two columns j0, j1 in fp64.  Row: KEEP -> row r of the swizzled shared tile, else
// the row in global memory (L2: five 16-B loads in flight per chunk, the next chunk's loads issued before this
// chunk's FMAs).  D = d at compile time (0: runtime d); d % 4 == 0.
template <int KK, int D, bool KEEP>
__device__ __forceinline__ void exact_pair(const float* __restrict__ tile, const float* __restrict__ grow, int r, int d,
                                          const double* __restrict__ M64, int j0, int j1, double& x0, double& x1) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  const int dd = D ? D : d;
  auto step = [&](const float4 a, int l) {
    const double d0 = a.x, d1 = a.y, d2 = a.z, d3 = a.w;
    const double* m = M64 + (size_t)l * KK;
    a0 = fma(d0, m[j0], a0);
    a1 = fma(d1, m[KK + j0], a1);
    a2 = fma(d2, m[2 * KK + j0], a2);
    a3 = fma(d3, m[3 * KK + j0], a3);
    b0 = fma(d0, m[j1], b0);
    b1 = fma(d1, m[KK + j1], b1);
    b2 = fma(d2, m[2 * KK + j1], b2);
    b3 = fma(d3, m[3 * KK + j1], b3);
  };
  if constexpr (!KEEP && D > 0 && D % 20 == 0) {
    float4 q[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) q[t] = __ldg((const float4*)(grow + 4 * t));
#pragma unroll 1
    for (int l0 = 0; l0 < D; l0 += 20) {
      float4 nx[5];
      const int ln = l0 + 20 < D ? l0 + 20 : l0;   // last chunk: harmless reload
#pragma unroll
      for (int t = 0; t < 5; ++t) nx[t] = __ldg((const float4*)(grow + ln + 4 * t));
#pragma unroll
      for (int t = 0; t < 5; ++t) step(q[t], l0 + 4 * t);
#pragma unroll
      for (int t = 0; t < 5; ++t) q[t] = nx[t];
    }
  } else {
#pragma unroll 4
    for (int l = 0; l < dd; l += 4)
      step(KEEP ? *(const float4*)(tile + tcx::sw_off(r, l)) : __ldg((const float4*)(grow + l)), l);
  }
  x0 = fabs((a0 + a1) + (a2 + a3));
  x1 = fabs((b0 + b1) + (b2 + b3));
}

// rare: several candidates -- exact value of each, then rank by counting (ties broken by index); out of line.
// Two candidate columns per pass over the row (ceil(nc/2) passes instead of nc: at the cfg-5 geometry the row comes
// from L2 and 0.55 % of the rows have nc > 2).  The pending-column form keeps the caller free of spills.
template <int KK, int D, bool KEEP>
__device__ __noinline__ void rare_candidates(const float* __restrict__ tile, const float* __restrict__ grow, int r, int d,
                                             const double* __restrict__ M64, unsigned cmask, int q1, int q2, double& x1,
                                             double& x2) {
  double ex[KK];
  x1 = x2 = 0.0;
  int pend = -1;
#pragma unroll 1
  for (unsigned m = cmask; m; m &= m - 1u) {   // candidate columns only (ex[] is read for them only)
    const int j = __ffs(m) - 1;
    if (pend < 0) {
      pend = j;
    } else {
      double c0, c1;
      exact_pair<KK, D, KEEP>(tile, grow, r, d, M64, pend, j, c0, c1);
      ex[pend] = c0;
      ex[j] = c1;
      pend = -1;
    }
  }
  if (pend >= 0) {
    double c0, c1;
    exact_pair<KK, D, KEEP>(tile, grow, r, d, M64, pend, pend, c0, c1);
    ex[pend] = c0;
  }
  // rank among the candidates only (nc^2 comparisons instead of k^2: at cfg 3 the k^2 loop was 17 % of the
  // kernel's instructions)
#pragma unroll 1
  for (unsigned ma = cmask; ma; ma &= ma - 1u) {
    const int a = __ffs(ma) - 1;
    int rank = 0;
#pragma unroll 1
    for (unsigned mb = cmask; mb; mb &= mb - 1u) {
      const int b = __ffs(mb) - 1;
      rank += ex[b] < ex[a] || (ex[b] == ex[a] && b < a);
    }
    if (rank == q1) x1 = ex[a];
    if (rank == q2) x2 = ex[a];
  }
}

// Selection half of the certified median (no fp64 work): returns
//   kSettled  -- never at present (kept for the degenerate cases a caller may settle itself),
//   kResolve  -- 1-2 candidates, desc = j0 | j1 << 5 | q1 << 10 | q2 << 15 | (nc - 1) << 20,
//   kRare     -- nc > 2 candidates (or a degenerate row: all k), rmask = the candidate mask, desc = q1 | q2 << 5.
// Rare rows are not evaluated here: a warp with one of them would stall all 32 lanes on a serial fp64 pass
// over the row; the caller queues them and evaluates 32 at a time, one per lane (rare_candidates).
enum { kSettled = 0, kResolve = 1, kRare = 2 };
template <int KK>
__device__ __forceinline__ int certify(const uint32_t (&dv)[32], float n2, const float* __restrict__ cm, float gam,
                                       uint32_t& desc, uint32_t& rmask) {
  constexpr int m1 = (KK - 1) / 2, m2 = KK / 2;
  float v[KK], srt[KK];
  const float g = gam * __fsqrt_ru(n2);
  bool bad = !(n2 >= 1e-30f) || !(g <= 1e30f);
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    v[j] = fabsf(__uint_as_float(dv[j]));
    srt[j] = v[j];
    bad |= !(v[j] <= 3.0e38f);   // inf / NaN
  }
  selnet<KK>(srt, CSwap2{});
  const float v1 = srt[m1], v2 = srt[m2];
  float La = INFINITY, Lb = INFINITY, Ha = 0.f, Hb = 0.f;
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    const float e = g * cm[j];
    float& Lx = (j & 1) ? Lb : La;
    float& Hx = (j & 1) ? Hb : Ha;
    if (v[j] >= v1) Lx = fminf(Lx, __fsub_rd(v[j], e));
    if (v[j] <= v2) Hx = fmaxf(Hx, __fadd_ru(v[j], e));
  }
  const float L = fminf(La, Lb), H = fmaxf(Ha, Hb);
  int below = 0;
  unsigned cmask = 0u;
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    const float e = g * cm[j];
    if (__fadd_ru(v[j], e) < L) ++below;
    else if (__fsub_rd(v[j], e) <= H) cmask |= 1u << j;
  }
  if (bad) {
    below = 0;
    cmask = KK == 32 ? 0xFFFFFFFFu : ((1u << KK) - 1u);
  }
  const int q1 = m1 - below, q2 = m2 - below;
  const int nc = __popc(cmask);
  if (nc <= 2) {
    const int j0 = __ffs(cmask) - 1, j1 = 31 - __clz(cmask);
    desc = (uint32_t)j0 | ((uint32_t)j1 << 5) | ((uint32_t)q1 << 10) | ((uint32_t)q2 << 15) | ((uint32_t)(nc - 1) << 20);
    return kResolve;
  }
  rmask = cmask;
  desc = (uint32_t)q1 | ((uint32_t)q2 << 5);
  return kRare;
}

// Per-warp queue of rare rows, one entry per lane (row, candidate mask, q1 | q2 << 5).  push() appends the rows
// whose lanes have rare set (flushing first when they do not fit); flush() evaluates every queued row at once, one
// row per lane, exactly in fp64 from global memory, and writes lambda.  The order in which a warp settles its rows
// is fixed, so the warp's share of sum(lambda) is reproducible.
struct RareQueue {
  uint32_t row = 0, mask = 0, q = 0;
  int cnt = 0;
  template <int KK, int D>
  __device__ __forceinline__ void flush(const float* __restrict__ A, int64_t lda, int d, const double* __restrict__ M64,
                                        float* __restrict__ lambda, double& local, int lane) {
    if (lane < cnt) {
      double x1, x2;
      rare_candidates<KK, D, false>(nullptr, A + (int64_t)row * lda, 0, d, M64, mask, (int)(q & 31u),
                                    (int)((q >> 5) & 31u), x1, x2);
      const float lam = (float)(0.5 * (x1 + x2));
      lambda[row] = lam;
      local += (double)lam;
    }
    cnt = 0;
  }
  template <int KK, int D>
  __device__ __forceinline__ void push(bool rare, uint32_t r_row, uint32_t r_mask, uint32_t r_q, const float* __restrict__ A,
                                       int64_t lda, int d, const double* __restrict__ M64, float* __restrict__ lambda,
                                       double& local, int lane) {
    const unsigned rb = __ballot_sync(0xFFFFFFFFu, rare);
    if (!rb) return;
    const int nr = __popc(rb);
    if (cnt + nr > 32) flush<KK, D>(A, lda, d, M64, lambda, local, lane);
    const int k = lane - cnt;
    const bool mine = k >= 0 && k < nr;
    const int src = mine ? (int)__fns(rb, 0u, k + 1) : lane;
    const uint32_t xr = __shfl_sync(0xFFFFFFFFu, r_row, src), xm = __shfl_sync(0xFFFFFFFFu, r_mask, src),
                   xq = __shfl_sync(0xFFFFFFFFu, r_q, src);
    if (mine) {
      row = xr;
      mask = xm;
      q = xq;
    }
    cnt += nr;
  }
};

// fp64 half: exact values of the 1-2 candidates of a descriptor, ranked.  One loop for both cases (the second
// column's loads and FMAs predicated): a warp whose rows mix one- and two-candidate descriptors would otherwise run
// a one-column and a two-column pass back to back (3 columns of conversions, loads and FMAs instead of 2)
template <int KK, int D, bool KEEP>
__device__ __forceinline__ float resolve(uint32_t desc, const float* __restrict__ tile, const float* __restrict__ grow,
                                         int r, int d, const double* __restrict__ M64) {
  const int j0 = desc & 31, q1 = (desc >> 10) & 31, q2 = (desc >> 15) & 31;
  const bool two = (desc >> 20) & 1u;
  const int j1 = two ? (int)((desc >> 5) & 31) : j0;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  const int dd = D ? D : d;
  // odd k: the second column's loads and FMAs run only when some lane of the warp has two candidates (a
  // warp-uniform branch; at cfg 4 about 40 % of the warps have none: 5.80 -> 5.68 ms)
  auto pass = [&](auto two_tag) {
    constexpr bool TWO = decltype(two_tag)::value;
    auto step = [&](const float4 a, int l) {
      const double d0 = a.x, d1 = a.y, d2 = a.z, d3 = a.w;
      const double* m = M64 + (size_t)l * KK;
      a0 = fma(d0, m[j0], a0);
      a1 = fma(d1, m[KK + j0], a1);
      a2 = fma(d2, m[2 * KK + j0], a2);
      a3 = fma(d3, m[3 * KK + j0], a3);
      if (TWO && two) {
        b0 = fma(d0, m[j1], b0);
        b1 = fma(d1, m[KK + j1], b1);
        b2 = fma(d2, m[2 * KK + j1], b2);
        b3 = fma(d3, m[3 * KK + j1], b3);
      }
    };
    if constexpr (!KEEP && D > 0 && D % 20 == 0) {   // row from L2: chunked and prefetched as in exact_pair
      float4 q[5];
#pragma unroll
      for (int t = 0; t < 5; ++t) q[t] = __ldg((const float4*)(grow + 4 * t));
#pragma unroll 1
      for (int l0 = 0; l0 < D; l0 += 20) {
        float4 nx[5];
        const int ln = l0 + 20 < D ? l0 + 20 : l0;
#pragma unroll
        for (int t = 0; t < 5; ++t) nx[t] = __ldg((const float4*)(grow + ln + 4 * t));
#pragma unroll
        for (int t = 0; t < 5; ++t) step(q[t], l0 + 4 * t);
#pragma unroll
        for (int t = 0; t < 5; ++t) q[t] = nx[t];
      }
    } else {
#pragma unroll 4
      for (int l = 0; l < dd; l += 4)
        step(KEEP ? *(const float4*)(tile + tcx::sw_off(r, l)) : __ldg((const float4*)(grow + l)), l);
    }
  };
  if constexpr (KK % 2 == 0) {
    pass(std::true_type{});   // even k: two middle order statistics, nearly every row has two candidates
  } else {
    if (__any_sync(__activemask(), two)) pass(std::true_type{});
    else pass(std::false_type{});
  }
  const double c0 = fabs((a0 + a1) + (a2 + a3));
  if (!two) return (float)c0;
  const double c1 = fabs((b0 + b1) + (b2 + b3));
  const double cmin = fmin(c0, c1), cmax = fmax(c0, c1);
  return (float)(0.5 * ((q1 == 0 ? cmin : cmax) + (q2 == 0 ? cmin : cmax)));
}

struct Smem {   // byte offsets inside the 1024-aligned dynamic shared memory
  int a, b, m64, cm, nrm, cq, bars, total;
};
constexpr int kCQ = 4;   // candidate-descriptor ring (selection -> recompute warps)
// fp64 M for the exact candidate recompute in shared memory (14 KB at d = 64, k = 27).  Reading it through L1
// from global memory instead frees one more tile buffer but measured no faster (2.158 vs 2.169 ms per 2^24 rows,
// profiles/r02_k2_experiments.txt); a runtime choice between the two costs generic (non-LDS) loads
constexpr bool kM64Smem = true;

// FCT_ROWNORM_DIAG bit 3 (diagnostics only): per-warp cycles spent in mbarrier waits and in total, CTA 0
__device__ unsigned long long g_rn_prof[32][2];
__device__ unsigned long long g_rn_cta[1024][2];
// FCT_ROWNORM_DIAG bit 4 (diagnostics only, with kTraceBuild): CTA-0 timeline of the first kTrace tiles, clock64 per event:
// 0 TMA issued, 1 split start, 2 split done, 3 MMA start, 4 MMA committed, 5 epilogue start (max over warps),
// 6 epilogue done (max over warps), 7 selection done (max over warps)
// compiled in only when kTraceBuild is set (rebuild to use it): the runtime check alone costs ~2 % at cfg 4
constexpr bool kTraceBuild = false;
constexpr int kTrace = 256;
__device__ unsigned long long g_rn_trace[kTrace][8];
__device__ __forceinline__ void trace(bool on, int i, int ev) {
  if (kTraceBuild && on && blockIdx.x == 0 && i < kTrace && (threadIdx.x & 31) == 0)
    atomicMax(&g_rn_trace[i][ev], (unsigned long long)clock64());
}   // per-CTA globaltimer at start / end (FCT_ROWNORM_PROF)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct WaitClock {
  bool on;
  unsigned long long waited = 0, t0 = 0;
  __device__ explicit WaitClock(bool o) : on(o) { if (on) t0 = clock64(); }
  template <class F>
  __device__ __forceinline__ void wait(F f) {
    if (!on) { f(); return; }
    const unsigned long long a = clock64();
    f();
    waited += clock64() - a;
  }
  __device__ void flush(int warp) {
    if (on && (threadIdx.x & 31) == 0 && blockIdx.x == 0) {
      g_rn_prof[warp][0] = waited;
      g_rn_prof[warp][1] = clock64() - t0;
    }
  }
};
__host__ __device__ inline Smem layout(int d, int KK, int NA, int ND, bool cq, bool m64s) {
  const int nch = (d + 31) / 32;
  Smem s;
  s.a = 0;
  s.b = s.a + NA * nch * 16384;          // B = [M_hi | M_lo]^T: nch chunks x 64 rows x 128 B
  s.m64 = s.b + nch * 8192;
  s.cm = s.m64 + (m64s ? ((d * KK * 8 + 15) & ~15) : 0);
  s.nrm = s.cm + 32 * 4;
  s.cq = s.nrm + ND * 128 * 4;           // [kCQ][128] descriptors + [kCQ][128] settled lambdas
  s.bars = s.cq + (cq ? kCQ * 128 * 8 : 0);
  s.total = s.bars + 8 * (2 * NA + 4 + 3 * ND + 2 * kCQ);
  return s;
}

// TMEM columns of one A buffer: [A_hi (KP) | A_lo (KP)] when AT (A_hi fed from TMEM), else [A_lo (KP)]
template <bool AT>
__host__ __device__ inline int abuf_cols(int KP) { return AT ? 2 * KP : KP; }

template <int KK, int D, int EG, int RG, bool KEEP, bool AT>   // RG: always 0 (recompute groups were removed)
__global__ void __launch_bounds__(32 * (kEpiWarp0 + 4 * EG + 4 * RG), 1)
rownorm_ws2_kernel(const __grid_constant__ CUtensorMap tmA, const float* __restrict__ A, int64_t n, int d, int64_t lda,
                   const float* __restrict__ M32g, int KP32, const double* __restrict__ M64g,
                   const float* __restrict__ colbg, float gam, int NA, int ND, float* __restrict__ lambda,
                   double* __restrict__ partial, int diag, unsigned whint, unsigned* __restrict__ tctr) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* base = smraw + ((1024u - (tcx::su32(smraw) & 1023u)) & 1023u);
  const int dd = D ? D : d;
  const int nch = (dd + 31) >> 5, KP = nch * 32;
  const int tile_floats = nch * 128 * 32;
  const Smem L = layout(dd, KK, NA, ND, RG > 0, kM64Smem);
  float* sA = (float*)(base + L.a);
  float* sB = (float*)(base + L.b);
  const double* M64 = kM64Smem ? (const double*)(base + L.m64) : M64g;
  float* cm = (float*)(base + L.cm);
  float* norms = (float*)(base + L.nrm);
  uint64_t* tma_full = (uint64_t*)(base + L.bars);   // [NA]  tile landed
  uint64_t* a_free = tma_full + NA;                   // [NA]  tile buffer reusable
  uint64_t* at_full = a_free + NA;                    // [2]   A pieces in TMEM (4 split-warp arrivals)
  uint64_t* at_free = at_full + 2;                    // [2]   TMEM A buffer reusable (MMA done)
  uint64_t* d_full = at_free + 2;                     // [ND]  accumulator ready
  uint64_t* n_full = d_full + ND;                     // [ND]  norms written (4 split-warp arrivals)
  uint64_t* d_free = n_full + ND;                     // [ND]  accumulator + norms drained (4 warp arrivals)
  constexpr int NWARPS = kEpiWarp0 + 4 * EG + 4 * RG;
  __shared__ uint32_t tbase;
  __shared__ int tid_a[8], tid_d[8];   // tile index of each tile buffer / accumulator slot (-1: end marker)
  __shared__ double red[NWARPS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int i = 0; i < NA; ++i) {
      tcx::bar_init(&tma_full[i], 1);
      tcx::bar_init(&a_free[i], KEEP ? 4 : 1);   // KEEP: released by the warps that finish the tile's rows
    }
    for (int i = 0; i < 2; ++i) {
      tcx::bar_init(&at_full[i], 4);
      tcx::bar_init(&at_free[i], 1);
    }
    for (int i = 0; i < ND; ++i) {
      tcx::bar_init(&d_full[i], 1);
      tcx::bar_init(&n_full[i], 4);
      tcx::bar_init(&d_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tcx::su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B operand (N = 64 rows x KP columns, K-major SWIZZLE_128B): rows j < 32 = tf32(M~)^T, rows 32 + j = the
  // remainder M~ - tf32(M~); one MMA yields A*M_hi in D[0:32) and A*M_lo in D[32:64)
  for (int e = tid; e < 64 * KP; e += blockDim.x) {
    const int jj = e / KP, l = e - jj * KP, j = jj & 31;
    const float m = (j < KK && l < dd) ? M32g[l * KP32 + j] : 0.f;
    const float hi = tcx::trunc_tf32(m);
    sB[(l >> 5) * 64 * 32 + jj * 32 + ((((l & 31) >> 2) ^ (jj & 7)) << 2) + (l & 3)] = jj < 32 ? hi : m - hi;
  }
  if (kM64Smem)
    for (int e = tid; e < KK * dd; e += blockDim.x) ((double*)(base + L.m64))[e] = M64g[e];
  for (int e = tid; e < 32; e += blockDim.x) cm[e] = e < KK ? colbg[2 * e] : 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const int acols = abuf_cols<AT>(KP);
  const uint32_t dcol0 = 2u * acols;   // TMEM: [A buf 0][A buf 1][D 0] ... [D ND-1], D = 64 columns
  const bool prof = (diag & 8) != 0;
  const bool trc = (diag & 16) != 0;
  diag &= 7;
  WaitClock wc(prof);
  if (prof && threadIdx.x == 0) g_rn_cta[blockIdx.x][0] = gtimer();
  // Tile schedule: CTA b starts with tile b; with a counter (tctr) the TMA producer takes each further tile from it
  // (dynamic: the CTAs end within a tile of each other; static round robin left a 9 % spread of CTA end times at
  // cfg 4), else tile b + j * gridDim.x.  After its last tile the producer emits EG end markers (-1) through the
  // same rings, one for each epilogue group, so every role leaves its loop without knowing the count in advance.
  const int ntiles = (int)((n + 127) / 128);
  const int t0 = blockIdx.x, tstep = gridDim.x;
  double local = 0.0;

  if (warp < kSplitWarps) {
    // ------------------------------------------------------------------ split: norms, A pieces -> TMEM
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int sa = 0, sd = 0, ends = 0;
    unsigned pa = 0, pd = 0;   // phase parities of the current ring slots
    for (int i = 0;; ++i) {
      const int sl = i & 1;
      wc.wait([&] { tcx::bar_wait(&tma_full[sa], pa); });
      const int tile_id = *(volatile int*)&tid_a[sa];
      if (i >= 2) wc.wait([&] { tcx::bar_wait(&at_free[sl], (unsigned)(((i - 2) >> 1) & 1)); });
      trace(trc, i, 1);
      const float* tile = sA + sa * tile_floats;
      const uint32_t tb = tm + lane_off + (uint32_t)(sl * acols);
      float s2 = 0.f, s2b = 0.f;
#pragma unroll(D ? (D + 31) / 32 : 1)
      for (int q = 0; q < (tile_id >= 0 ? nch : 0); ++q) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *(const float4*)(tile + q * 128 * 32 + tid * 32 + ((c ^ (tid & 7)) << 2));
          s2 = fmaf(v.x, v.x, s2);
          s2b = fmaf(v.y, v.y, s2b);
          s2 = fmaf(v.z, v.z, s2);
          s2b = fmaf(v.w, v.w, s2b);
          const float h0 = tcx::trunc_tf32(v.x), h1 = tcx::trunc_tf32(v.y), h2 = tcx::trunc_tf32(v.z),
                      h3 = tcx::trunc_tf32(v.w);
          hi[c * 4 + 0] = __float_as_uint(h0);
          hi[c * 4 + 1] = __float_as_uint(h1);
          hi[c * 4 + 2] = __float_as_uint(h2);
          hi[c * 4 + 3] = __float_as_uint(h3);
          lo[c * 4 + 0] = __float_as_uint(v.x - h0);
          lo[c * 4 + 1] = __float_as_uint(v.y - h1);
          lo[c * 4 + 2] = __float_as_uint(v.z - h2);
          lo[c * 4 + 3] = __float_as_uint(v.w - h3);
        }
        if (AT) tcx::tmem_st32(tb + (uint32_t)(q * 32), hi);
        tcx::tmem_st32(tb + (uint32_t)((AT ? KP : 0) + q * 32), lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&at_full[sl]);
      trace(trc, i, 2);
      if (i >= ND) wc.wait([&] { tcx::bar_wait(&d_free[sd], pd ^ 1u); });
      norms[sd * 128 + tid] = s2 + s2b;
      if (tid == 0) tid_d[sd] = tile_id;
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&n_full[sd]);
      if (++sa == NA) { sa = 0; pa ^= 1u; }
      if (++sd == ND) { sd = 0; pd ^= 1u; }
      if (tile_id < 0 && ++ends == EG) break;
    }
  } else if (warp == kTmaWarp) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int sa = 0, ends = 0;
      unsigned pa = 0;
      for (int j = 0; ends < EG; ++j) {
        int tile_id = -1;
        if (!ends) {
          tile_id = (j == 0 || !tctr) ? t0 + j * tstep : (int)(tstep + atomicAdd(tctr, 1u));
          if (tile_id >= ntiles) tile_id = -1;
        }
        if (j >= NA) wc.wait([&] { tcx::bar_wait(&a_free[sa], pa ^ 1u); });
        trace(trc, j, 0);
        tid_a[sa] = tile_id;   // published by the arrive below (release) to the split warps and, through them, the MMA
        if (tile_id >= 0) {
          tcx::tma_tile(sA + sa * tile_floats, &tmA, nch, tile_id * 128, &tma_full[sa]);
        } else {
          tcx::bar_arrive(&tma_full[sa]);
          ++ends;
        }
        if (++sa == NA) { sa = 0; pa ^= 1u; }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      // kind::tf32, M = 128, N = 64, K-major A and B, fp32 accumulate
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const int ksteps = (dd + 7) >> 3;
      const uint64_t b00 = tcx::sdesc_sw128(sB), a00 = tcx::sdesc_sw128(sA);
      int sa = 0, sd = 0, ends = 0;
      unsigned pd = 0;
      for (int i = 0;; ++i) {
        const int sl = i & 1;
        wc.wait([&] { tcx::bar_wait(&at_full[sl], (unsigned)((i >> 1) & 1)); });   // implies the TMA tile has landed
        if (i >= ND) wc.wait([&] { tcx::bar_wait(&d_free[sd], pd ^ 1u); });
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        trace(trc, i, 3);
        const uint32_t tD = tm + dcol0 + (uint32_t)(sd * 64);
        const uint32_t tA = tm + (uint32_t)(sl * acols);
        const uint64_t a0 = a00 + (uint64_t)((sa * tile_floats * 4) >> 4);
        const int tile_id = *(volatile int*)&tid_a[sa];
        if (tile_id >= 0 && diag != 3) {
          // D = (A_hi + A_lo) [M_hi | M_lo]: every product of the two-term splits, nothing dropped
#pragma unroll(D ? (D + 7) / 8 : 1)
          for (int ks = 0; ks < ksteps; ++ks) {
            const uint64_t bd = b00 + (uint64_t)(((ks >> 2) * 8192 + (ks & 3) * 32) >> 4);
            if (AT)
              tcx::mma_tf32_ts(tD, tA + (uint32_t)(ks * 8), bd, idesc, ks > 0);
            else
              tcx::mma_tf32_ss(tD, a0 + (uint64_t)(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4), bd, idesc, ks > 0);
          }
        }
#pragma unroll(D ? (D + 7) / 8 : 1)
        for (int ks = 0; ks < (tile_id >= 0 ? ksteps : 0); ++ks) {
          const uint64_t bd = b00 + (uint64_t)(((ks >> 2) * 8192 + (ks & 3) * 32) >> 4);
          tcx::mma_tf32_ts(tD, tA + (uint32_t)((AT ? KP : 0) + ks * 8), bd, idesc, diag != 3 || ks > 0);
        }
        tcx::mma_commit(&d_full[sd]);   // an end marker commits too (arrives once the earlier MMAs are done)
        tcx::mma_commit(&at_free[sl]);
        if (!KEEP) tcx::mma_commit(&a_free[sa]);
        trace(trc, i, 4);
        if (++sa == NA) sa = 0;
        if (++sd == ND) { sd = 0; pd ^= 1u; }
        if (tile_id < 0 && ++ends == EG) break;
      }
    }
  } else if (warp < kEpiWarp0 + 4 * EG) {
    // ------------------------------------------------------------------ selection (epilogue) groups
    const int ew = warp - kEpiWarp0;
    const int g = ew >> 2;
    const int quad = warp & 3;                        // TMEM lane quadrant this warp may access
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int sd = g % ND, sa = g % NA;
    unsigned ph = (unsigned)((g / ND) & 1);
    RareQueue rq;
    for (int i = g;; i += EG) {
      wc.wait([&] {
        tcx::bar_wait_sleep(&d_full[sd], ph, whint);
        tcx::bar_wait_sleep(&n_full[sd], ph, whint);
      });
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      trace(trc, i, 5);
      uint32_t dv[32];
      {
        uint32_t dw[32];
        tcx::tmem_ld32(tm + lane_off + dcol0 + (uint32_t)(sd * 64), dv);
        tcx::tmem_ld32(tm + lane_off + dcol0 + (uint32_t)(sd * 64 + 32), dw);
#pragma unroll
        for (int j = 0; j < 32; ++j) dv[j] = __float_as_uint(__uint_as_float(dv[j]) + __uint_as_float(dw[j]));
      }
      const float n2 = norms[sd * 128 + r];
      const int tile_id = *(volatile int*)&tid_d[sd];
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&d_free[sd]);
      if (tile_id < 0) {   // end marker: release the tile buffer slot as for a tile, then leave
        if (KEEP && lane == 0) tcx::bar_arrive(&a_free[sa]);
        break;
      }
      const int64_t row = (int64_t)tile_id * 128 + r;
      const float* tile = sA + sa * tile_floats;
      float lam = 0.f;
      uint32_t desc = 0u, rmask = 0u;
      int st = kSettled;
      if (row < n) {
        if (diag >= 2) lam = __uint_as_float(dv[0]) + n2;   // diag (profiling only): no epilogue arithmetic
        else st = certify<KK>(dv, n2, cm, gam, desc, rmask);
      }
      trace(trc, i, 7);
      {
        // rare rows: queued and evaluated 32 at a time (cfg 4: 6.50 -> 5.89 ms, cfg-5 shard 10.6 -> 8.7 ms) where
        // the registers allow it; with four groups (80 registers) the queue spills in the loop and the rows are
        // settled in place from the kept tile instead
        constexpr bool kDefer = EG <= 3;
        if (kDefer) {
          rq.push<KK, D>(st == kRare, (uint32_t)row, rmask, desc, A, lda, dd, M64, lambda, local, lane);
        } else if (st == kRare) {
          double x1, x2;
          rare_candidates<KK, D, KEEP>(tile, A + row * lda, r, dd, M64, rmask, (int)(desc & 31u), (int)((desc >> 5) & 31u),
                                       x1, x2);
          lam = (float)(0.5 * (x1 + x2));
          st = kSettled;
        }
        if (row < n && st != kRare) {
          if (st == kResolve) lam = diag == 1 ? 0.f : resolve<KK, D, KEEP>(desc, tile, A + row * lda, r, dd, M64);
          lambda[row] = lam;
          local += (double)lam;
        }
        __syncwarp();
        trace(trc, i, 6);
        if (KEEP && lane == 0) tcx::bar_arrive(&a_free[sa]);
      }
      sa += EG;
      while (sa >= NA) sa -= NA;
      sd += EG;
      if (sd >= ND) { sd -= ND; ph ^= 1u; }
    }
    if (EG <= 3) rq.flush<KK, D>(A, lda, dd, M64, lambda, local, lane);
  }
  wc.flush(warp);
  if (prof && threadIdx.x == 0) g_rn_cta[blockIdx.x][1] = gtimer();
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) red[warp] = local;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < NWARPS; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn2() {
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

constexpr size_t kSmemMax = 232448;   // max dynamic shared memory per block (sm_100)

template <int KK, int D, int EG, int RG>
fct_status launch(const float* A, int64_t n, int d, int64_t lda, const float* M32, int KP32, const double* M64,
                  const float* colb, double* partial, int grid, float* lambda, cudaStream_t st) {
  auto enc = encode_fn2();
  if (!enc) return FCT_ERR_UNSUPPORTED;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(float)};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  FCT_CHECK_ARG(cr == CUDA_SUCCESS, FCT_ERR_CUDA, "l1_rownorm: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  const int nch = (d + 31) / 32, KP = nch * 32;
  // A_hi from TMEM (TS form, default where it fits next to EG + 1 accumulators): with the single-pass candidate
  // recompute measured 2 % faster at cfg 4 (6.59 vs 6.73 ms; before it, SS was 1 % faster: 7.50 vs 7.57).
  // FCT_ROWNORM_SS=1 feeds A_hi from the shared tile (SS form) instead.
  const bool at = 4 * KP + 64 * (EG + 1) <= 512 && !getenv("FCT_ROWNORM_SS");
  const int ND = std::min(8, (512 - 2 * (at ? 2 * KP : KP)) / 64);
  const bool m64s = kM64Smem;
  int NA = 0;
  for (int na = 8; na >= 2; --na)
    if (layout(d, KK, na, ND, RG > 0, m64s).total + 1024 <= (int)kSmemMax - 512) { NA = na; break; }   // static: < 256 B
  if (NA < 2 || ND < EG + 1) return FCT_ERR_UNSUPPORTED;
  // keep the tile until the epilogue is done (exact recompute from shared memory) when enough buffers fit
  const bool keep = NA >= EG + 2 && !getenv("FCT_ROWNORM_NOKEEP");
  if (RG > 0) return FCT_ERR_UNSUPPORTED;   // separate recompute groups were measured slower and removed
  const size_t smem = (size_t)layout(d, KK, NA, ND, RG > 0, m64s).total + 1024;
  const int g = std::max(1, std::min(grid, fct::num_sms()));
  const int threads = 32 * (kEpiWarp0 + 4 * EG + 4 * RG);
  const float gam = 6.103515625e-05f * 1.05f;   // 3xTF32 bound, 2^-14 (measured 1.9e-6) x 1.05 for roundings
  auto kern = keep ? (at ? rownorm_ws2_kernel<KK, D, EG, RG, true, true> : rownorm_ws2_kernel<KK, D, EG, RG, true, false>)
                   : (at ? rownorm_ws2_kernel<KK, D, EG, RG, false, true> : rownorm_ws2_kernel<KK, D, EG, RG, false, false>);
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (fct::debug_sync())
    fprintf(stderr, "[fct] rownorm_ws2<k=%d,D=%d,EG=%d,RG=%d,keep=%d,at=%d>: grid %d NA %d ND %d m64s %d smem %zu\n", KK, D,
            EG, RG, (int)keep, (int)at, g, NA, ND, (int)m64s, smem);
  FCT_CUDA_RET(cudaMemsetAsync(partial, 0, sizeof(double) * grid, st));
  const char* dg = getenv("FCT_ROWNORM_DIAG");
  const int diag = dg ? atoi(dg) : 0;
  if (diag & 16) {
    void* tp = nullptr;
    if (cudaGetSymbolAddress(&tp, g_rn_trace) == cudaSuccess) cudaMemsetAsync(tp, 0, sizeof(unsigned long long) * kTrace * 8, st);
  }
  const char* wh = getenv("FCT_WAIT_HINT");
  // dynamic tile schedule: the counter lives in the last partial slot (g < grid, zeroed above; reset after the
  // kernel so the partial sum is unchanged).  FCT_ROWNORM_STATIC=1 keeps the round-robin schedule.
  const bool dyn = g < grid && !getenv("FCT_ROWNORM_STATIC");
  unsigned* tctr = dyn ? (unsigned*)(partial + grid - 1) : nullptr;
  kern<<<g, threads, smem, st>>>(map, A, n, d, lda, M32, KP32, M64, colb, gam, NA, ND, lambda, partial, diag,
                                 wh ? (unsigned)atoi(wh) : 20000u, tctr);
  FCT_LAUNCHED("rownorm_ws2_kernel", st);
  if (dyn) FCT_CUDA_RET(cudaMemsetAsync(partial + grid - 1, 0, sizeof(double), st));
  fct::set_instance(1, "rownorm_ws2_kernel<%d, %d, %d, %d, %d, %d>", KK, D, EG, RG, keep ? 1 : 0, at ? 1 : 0);
  if (diag & 16) {
    static unsigned long long tr[kTrace][8];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(tr, g_rn_trace, sizeof(tr));
    const unsigned long long z = tr[0][0];
    fprintf(stderr, "[fct trace] tile: tma split0 split1 mma0 mma1 epi0 epi1 (cycles from tile 0's TMA issue)\n");
    for (int i = 0; i < 64; ++i) {
      fprintf(stderr, "[fct trace] %3d:", i);
      for (int e = 0; e < 7; ++e) fprintf(stderr, " %8lld", tr[i][e] ? (long long)(tr[i][e] - z) : -1LL);
      fprintf(stderr, "\n");
    }
    for (int e = 0; e < 7; ++e) {
      if (!tr[200][e] || !tr[100][e]) continue;
      fprintf(stderr, "[fct trace] event %d period %.0f cycles/tile\n", e, (double)(tr[200][e] - tr[100][e]) / 100.0);
    }
    const char* nm[6] = {"tma->split0", "split0->split1", "split1->mma0", "mma0->mma1", "mma1->epi0", "epi0->epi1"};
    for (int e = 0; e < 6; ++e) {
      double acc = 0;
      int cnt = 0;
      for (int i = 100; i < 200; ++i)
        if (tr[i][e] && tr[i][e + 1]) { acc += (double)(long long)(tr[i][e + 1] - tr[i][e]); ++cnt; }
      fprintf(stderr, "[fct trace] %-15s mean %.0f cycles\n", nm[e], cnt ? acc / cnt : -1.0);
    }
    double a5 = 0, a7 = 0;
    int c5 = 0;
    for (int i = 100; i < 200; ++i)
      if (tr[i][5] && tr[i][7] && tr[i][6]) { a5 += (double)(long long)(tr[i][7] - tr[i][5]); a7 += (double)(long long)(tr[i][6] - tr[i][7]); ++c5; }
    if (c5) fprintf(stderr, "[fct trace] epi0->select   mean %.0f cycles, select->epi1 mean %.0f cycles\n", a5 / c5, a7 / c5);
  }
  if (diag & 8) {
    unsigned long long h[32][2];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_rn_prof, sizeof(h));
    unsigned long long c[1024][2];
    cudaMemcpyFromSymbol(c, g_rn_cta, sizeof(c));
    unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
    for (int b = 0; b < g; ++b) {
      s0 = std::min(s0, c[b][0]); s1 = std::max(s1, c[b][0]);
      e0 = std::min(e0, c[b][1]); e1 = std::max(e1, c[b][1]);
    }
    fprintf(stderr, "[fct prof] %d CTAs: start spread %.1f us, first end %.1f us, last end %.1f us\n", g,
            (s1 - s0) * 1e-3, (e0 - s0) * 1e-3, (e1 - s0) * 1e-3);
    for (int b = 0; b < g; b += 16)
      fprintf(stderr, "[fct prof] cta %3d start %8.1f end %8.1f us\n", b, (c[b][0] - s0) * 1e-3, (c[b][1] - s0) * 1e-3);
    const int nw = threads / 32;
    for (int w = 0; w < nw; ++w)
      fprintf(stderr, "[fct prof] warp %2d %-9s waited %5.1f%% of %llu cycles\n", w,
              w < 4 ? "split" : w == 4 ? "tma" : w == 5 ? "mma" : (w < kEpiWarp0 + 4 * EG ? "epilogue" : "recompute"),
              100.0 * h[w][0] / (double)(h[w][1] ? h[w][1] : 1), h[w][1]);
  }
  return FCT_OK;
}

template <int KK, int DC>
fct_status launch_k(const float* A, int64_t n, int d, int64_t lda, const float* M32, int KP32, const double* M64,
                    const float* colb, double* partial, int grid, float* lambda, cudaStream_t st) {
  // variants (FCT_ROWNORM_VAR): 1 = 3 epilogue groups (default), 2 = 2 groups, 3 = 4 groups.  Four groups were
  // faster at d = 32 while rare rows were settled in place (2.06 vs 2.18 ms); with the rare-row queue, which needs
  // the registers of three groups, three are faster there too (cfg 3: 1.06 vs 1.25 ms)
  const char* ve = getenv("FCT_ROWNORM_VAR");
  const int var = ve ? atoi(ve) : (getenv("FCT_ROWNORM_EG2") ? 2 : 1);
#define FCT_RN_LAUNCH(DD)                                                                                  \
  do {                                                                                                     \
    fct_status rc_ = FCT_ERR_UNSUPPORTED;                                                                  \
    if (rc_ != FCT_ERR_UNSUPPORTED) return rc_;                                                            \
    if (var == 2) return launch<KK, DD, 2, 0>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st); \
    if (var == 3) {                                                                                        \
      rc_ = launch<KK, DD, 4, 0>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);           \
      if (rc_ != FCT_ERR_UNSUPPORTED) return rc_;                                                          \
    }                                                                                                      \
    return launch<KK, DD, 3, 0>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);            \
  } while (0)
  if (d == DC) FCT_RN_LAUNCH(DC);
  FCT_RN_LAUNCH(0);
#undef FCT_RN_LAUNCH
}

}  // namespace

// Returns FCT_ERR_UNSUPPORTED (nothing enqueued) when no instance covers (k, d, alignment).
// M32: fp32 M~ row-major [d][KP32]; M64: fp64 M row-major [d][k]; colb[2j] = ||m~_j||_2 rounded up.
// Instances: k of the five BASELINE configurations, each with its config's d unrolled at compile time.
fct_status fct_rownorm_ws2(const float* A, int64_t n, int d, int64_t lda, const float* M32, int KP32,
                           const double* M64, const float* colb, int k, double* partial, int grid, float* lambda,
                           cudaStream_t st) {
  if (getenv("FCT_ROWNORM_WS1") || getenv("FCT_ROWNORM_SIMT")) return FCT_ERR_UNSUPPORTED;
  if (d % 4 || d > 128 || lda % 4 || ((uintptr_t)A & 15) || n >= (1LL << 31)) return FCT_ERR_UNSUPPORTED;
  switch (k) {
    case 16: return launch_k<16, 8>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);
    case 20: return launch_k<20, 16>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);
    case 24: return launch_k<24, 32>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);
    case 27: return launch_k<27, 64>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);
    case 29: return launch_k<29, 100>(A, n, d, lda, M32, KP32, M64, colb, partial, grid, lambda, st);
    default: return FCT_ERR_UNSUPPORTED;
  }
}
