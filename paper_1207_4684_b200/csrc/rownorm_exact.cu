// rownorm_exact.cu -- §8(f) NEXT-1: exact l1 row norms of the well-conditioned basis U = A R^-1,
//     lambda_i = ||U_i||_1 = sum_j |sum_l A_il (R^-1)_lj|,
// which is what the paper's §6.2 experiments use instead of the Cauchy estimate ("we compute the row norms
// of U exactly instead of estimating them"; U = A R^-1 of FastL1Basis).
// A true dense contraction (d x d per row), so it runs on the 5th-generation tensor cores:
//   warps 0-3 split (thread r <-> tile row r <-> TMEM lane r: A_hi = tf32(A), A_lo = A - A_hi -> TMEM),
//   warp 4 TMA producer (128-row SWIZZLE_128B tiles), warp 5 MMA issuer, warps 6.. two epilogue groups.
//   d <= 64 ("stacked"): B = [R~_hi | R~_lo] (N = 2 KP rows), D = (A_hi + A_lo) B -> the two halves of D hold
//                        A R~_hi and A R~_lo; A_hi and A_lo both from TMEM; 2 MMAs per k-step.
//   (d > 64 does not fit [R~_hi | R~_lo] next to the tile buffers: the SIMT kernel below takes it.)
// Every product of the splits is formed (R~ = fp32(R^-1) split hi/lo exactly), so the only errors are the
// rounding of R^-1 to fp32, the tensor core's fp32 accumulation and the fp32 sum over j (DESIGN.md derives
// the tolerance |lambda - exact| <= 2^-14 sum_j sum_l |A_il||R^-1_lj| + 2^-17 lambda from these).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include "common.cuh"
#include "tc.cuh"

namespace {

constexpr int kSplitW = 4, kTmaW = 4, kMmaW = 5, kEpiW0 = 6, kEG = 2;
constexpr int kThreadsX = 32 * (kEpiW0 + 4 * kEG);

struct LayoutX {
  int a, b, bars, total;
};
__host__ __device__ inline LayoutX layout_x(int KP, int NA, int ND) {
  const int nch = KP / 32;
  LayoutX s;
  s.a = 0;
  s.b = NA * nch * 16384;
  const int brows = 2 * KP;   // [hi | lo] rows
  s.bars = s.b + nch * brows * 128;
  s.total = s.bars + 8 * (2 * NA + 4 + 2 * ND);
  return s;
}

__global__ void __launch_bounds__(kThreadsX, 1)
rownorm_exact_kernel(const __grid_constant__ CUtensorMap tmA, int64_t n, int d, const float* __restrict__ R32,
                     int NA, int ND, float* __restrict__ lambda, double* __restrict__ partial) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* base = smraw + ((1024u - (tcx::su32(smraw) & 1023u)) & 1023u);
  const int nch = (d + 31) >> 5, KP = nch * 32;
  const int tile_floats = nch * 128 * 32;
  const LayoutX L = layout_x(KP, NA, ND);
  float* sA = (float*)(base + L.a);
  float* sB = (float*)(base + L.b);
  uint64_t* tma_full = (uint64_t*)(base + L.bars);
  uint64_t* a_free = tma_full + NA;
  uint64_t* at_full = a_free + NA;   // [2]
  uint64_t* at_free = at_full + 2;   // [2]
  uint64_t* d_full = at_free + 2;    // [ND]
  uint64_t* d_free = d_full + ND;    // [ND]
  __shared__ uint32_t tbase;
  __shared__ double red[kThreadsX / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int brows = 2 * KP;          // B rows (N of the stacked MMA, or hi then lo blocks)
  const int acols = 2 * KP;   // TMEM columns per A buffer: [A_hi | A_lo]
  const int dcols = 2 * KP;   // TMEM columns per accumulator: [A R_hi | A R_lo]

  if (tid == 0) {
    for (int i = 0; i < NA; ++i) {
      tcx::bar_init(&tma_full[i], 1);
      tcx::bar_init(&a_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tcx::bar_init(&at_full[i], 4);
      tcx::bar_init(&at_free[i], 1);
    }
    for (int i = 0; i < ND; ++i) {
      tcx::bar_init(&d_full[i], 1);
      tcx::bar_init(&d_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tcx::su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B: row jj < KP = tf32(R~^T)[jj], row KP + jj = remainder; K-major SWIZZLE_128B, K = KP (l)
  for (int e = tid; e < brows * KP; e += blockDim.x) {
    const int jj = e / KP, l = e - jj * KP, j = jj % KP;
    const float m = (j < d && l < d) ? R32[l * d + j] : 0.f;
    const float hi = tcx::trunc_tf32(m);
    sB[(l >> 5) * brows * 32 + jj * 32 + ((((l & 31) >> 2) ^ (jj & 7)) << 2) + (l & 3)] = jj < KP ? hi : m - hi;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t dcol0 = 2u * acols;
  const int ntiles = (int)((n + 127) / 128);
  const int t0 = blockIdx.x, tstep = gridDim.x;
  const int my_tiles = t0 < ntiles ? (ntiles - 1 - t0) / tstep + 1 : 0;
  double local = 0.0;

  if (warp < kSplitW) {
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int sa = 0;
    unsigned pa = 0;
    for (int i = 0; i < my_tiles; ++i) {
      const int sl = i & 1;
      tcx::bar_wait(&tma_full[sa], pa);
      if (i >= 2) tcx::bar_wait(&at_free[sl], (unsigned)(((i - 2) >> 1) & 1));
      const float* tile = sA + sa * tile_floats;
      const uint32_t tb = tm + lane_off + (uint32_t)(sl * acols);
      for (int q = 0; q < nch; ++q) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *(const float4*)(tile + q * 128 * 32 + tid * 32 + ((c ^ (tid & 7)) << 2));
          const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const float h = tcx::trunc_tf32(a[w]);
            hi[c * 4 + w] = __float_as_uint(h);
            lo[c * 4 + w] = __float_as_uint(a[w] - h);
          }
        }
        tcx::tmem_st32(tb + (uint32_t)(q * 32), hi);
        tcx::tmem_st32(tb + (uint32_t)(KP + q * 32), lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&at_full[sl]);
      if (++sa == NA) { sa = 0; pa ^= 1u; }
    }
  } else if (warp == kTmaW) {
    if (lane == 0) {
      int sa = 0;
      unsigned pa = 0;
      for (int j = 0; j < my_tiles; ++j) {
        if (j >= NA) tcx::bar_wait(&a_free[sa], pa ^ 1u);
        tcx::tma_tile(sA + sa * tile_floats, &tmA, nch, (t0 + j * tstep) * 128, &tma_full[sa]);
        if (++sa == NA) { sa = 0; pa ^= 1u; }
      }
    }
  } else if (warp == kMmaW) {
    if (lane == 0) {
      const uint32_t N = 2 * KP;
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const int ksteps = (d + 7) >> 3;
      const uint64_t b00 = tcx::sdesc_sw128(sB);
      int sa = 0, sd = 0;
      unsigned pd = 0;
      for (int i = 0; i < my_tiles; ++i) {
        const int sl = i & 1;
        tcx::bar_wait(&at_full[sl], (unsigned)((i >> 1) & 1));
        if (i >= ND) tcx::bar_wait(&d_free[sd], pd ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tD = tm + dcol0 + (uint32_t)(sd * dcols);
        const uint32_t tA = tm + (uint32_t)(sl * acols);
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint64_t bd = b00 + (uint64_t)(((ks >> 2) * brows * 128 + (ks & 3) * 32) >> 4);
          tcx::mma_tf32_ts(tD, tA + (uint32_t)(ks * 8), bd, idesc, ks > 0);        // A_hi [R_hi | R_lo]
          tcx::mma_tf32_ts(tD, tA + (uint32_t)(KP + ks * 8), bd, idesc, 1);        // A_lo [R_hi | R_lo]
        }
        tcx::mma_commit(&d_full[sd]);
        tcx::mma_commit(&at_free[sl]);
        tcx::mma_commit(&a_free[sa]);
        if (++sa == NA) sa = 0;
        if (++sd == ND) { sd = 0; pd ^= 1u; }
      }
    }
  } else {
    const int ew = warp - kEpiW0;
    const int g = ew >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int sd = g % ND;
    unsigned ph = (unsigned)((g / ND) & 1);
    for (int i = g; i < my_tiles; i += kEG) {
      tcx::bar_wait(&d_full[sd], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tD = tm + lane_off + dcol0 + (uint32_t)(sd * dcols);
      float s0 = 0.f, s1 = 0.f;
      for (int q = 0; q < nch; ++q) {
        uint32_t v[32];
        tcx::tmem_ld32(tD + (uint32_t)(q * 32), v);
        {
          uint32_t w[32];
          tcx::tmem_ld32(tD + (uint32_t)(KP + q * 32), w);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
        }
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          if (q * 32 + j < d) s0 += fabsf(__uint_as_float(v[j]));
          if (q * 32 + j + 1 < d) s1 += fabsf(__uint_as_float(v[j + 1]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&d_free[sd]);
      const int64_t row = (int64_t)(t0 + i * tstep) * 128 + r;
      if (row < n) {
        const float lam = s0 + s1;
        lambda[row] = lam;
        local += (double)lam;
      }
      sd += kEG;
      if (sd >= ND) { sd -= ND; ph ^= 1u; }
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) red[warp] = local;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreadsX / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// SIMT fallback (d > 64, where [R_hi | R_lo] and the tiles do not fit in shared memory together, or
// d % 4 != 0): one row per thread, R~ in shared memory, 16 sequential-FMA accumulators per column chunk.
// fp32 FMA error <= d u / (1 - d u) * sum_l |a_l||R_lj| per column, inside the tensor-core tolerance.
__global__ void __launch_bounds__(256) rownorm_exact_simt(const float* __restrict__ A, int64_t n, int d, int64_t lda,
                                                           const float* __restrict__ R32, float* __restrict__ lambda,
                                                           double* __restrict__ partial) {
  extern __shared__ float sR[];
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) sR[e] = R32[e];
  __syncthreads();
  double local = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float* a = A + i * lda;
    float lam0 = 0.f, lam1 = 0.f;
    for (int j0 = 0; j0 < d; j0 += 16) {
      float acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = 0.f;
      for (int l = 0; l < d; ++l) {
        const float al = __ldg(a + l);
        const float* rr = sR + l * d + j0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (j0 + q < d) acc[q] = fmaf(al, rr[q], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        if (j0 + q < d) lam0 += fabsf(acc[q]);
        if (j0 + q + 1 < d) lam1 += fabsf(acc[q + 1]);
      }
    }
    lambda[i] = lam0 + lam1;
    local += (double)(lam0 + lam1);
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

// R~ = fp32(Rinv) (row-major d x d)
__global__ void rinv32_kernel(const double* __restrict__ Rinv, int d, float* __restrict__ R32) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d * d; e += gridDim.x * blockDim.x) R32[e] = (float)Rinv[e];
}
__global__ void sum_partials_x(const double* __restrict__ partial, int np, double* __restrict__ out, int zero_first) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += partial[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = zero_first ? t : *out + t;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_x() {
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

}  // namespace

extern "C" size_t l1_rownorm_exact_workspace_bytes(int64_t n, int64_t d) {
  (void)n;
  if (d < 1) return 0;
  return fct::align256(sizeof(float) * (size_t)d * d) + fct::align256(sizeof(double) * 1024) +
         fct::align256(sizeof(double));
}

extern "C" fct_status l1_rownorm_exact(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                                       float* lambda, double* lambda_sum, void* workspace, size_t workspace_bytes,
                                       void* stream) {
  FCT_CHECK_ARG(A && Rinv && lambda && lambda_sum, FCT_ERR_ARG, "l1_rownorm_exact: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && d >= 1 && d <= FCT_MAX_D && lda >= d, FCT_ERR_SHAPE,
                "l1_rownorm_exact: bad shape n=%lld d=%lld lda=%lld (d <= %d)", (long long)n, (long long)d,
                (long long)lda, FCT_MAX_D);
  const size_t need = l1_rownorm_exact_workspace_bytes(n, d);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_WORKSPACE, "l1_rownorm_exact: workspace %zu < %zu bytes",
                workspace_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  fct::Carver cv(workspace);
  float* R32 = cv.take<float>((size_t)d * d);
  double* partial = cv.take<double>(1024);
  rinv32_kernel<<<(int)((d * d + 255) / 256), 256, 0, st>>>(Rinv, (int)d, R32);
  FCT_LAUNCHED("rinv32_kernel", st);
  auto enc = encode_x();
  const bool tc = enc && d <= 64 && d % 4 == 0 && lda % 4 == 0 && ((uintptr_t)A & 15) == 0 && n < (1LL << 31) &&
                  !getenv("FCT_ROWNORM_SIMT");
  if (!tc) {
    const int grid = std::min(fct::num_sms() * 4, 1024);
    const size_t smem = sizeof(float) * (size_t)d * d;
    FCT_CUDA_RET(cudaFuncSetAttribute(rownorm_exact_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rownorm_exact_simt<<<grid, 256, smem, st>>>(A, n, (int)d, lda, R32, lambda, partial);
    FCT_LAUNCHED("rownorm_exact_simt", st);
    sum_partials_x<<<1, 256, 0, st>>>(partial, grid, lambda_sum, 1);
    FCT_LAUNCHED("sum_partials_x", st);
    return FCT_OK;
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(float)};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  FCT_CHECK_ARG(cr == CUDA_SUCCESS, FCT_ERR_CUDA, "l1_rownorm_exact: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  const int KP = (int)((d + 31) / 32) * 32;
  const int acols = 2 * KP, dcols = 2 * KP;
  const int ND = std::min(4, (512 - 2 * acols) / dcols);
  int NA = 0;
  for (int na = 6; na >= 2; --na)
    if (layout_x(KP, na, ND).total + 1024 <= 232448 - 2048) { NA = na; break; }
  FCT_CHECK_ARG(NA >= 2 && ND >= 2, FCT_ERR_UNSUPPORTED, "l1_rownorm_exact: no tile configuration for d=%lld",
                (long long)d);
  const size_t smem = (size_t)layout_x(KP, NA, ND).total + 1024;
  const int grid = std::min(fct::num_sms(), 1024);
  FCT_CUDA_RET(cudaFuncSetAttribute(rownorm_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rownorm_exact_kernel<<<grid, kThreadsX, smem, st>>>(map, n, (int)d, R32, NA, ND, lambda, partial);
  FCT_LAUNCHED("rownorm_exact_kernel", st);
  sum_partials_x<<<1, 256, 0, st>>>(partial, grid, lambda_sum, 1);
  FCT_LAUNCHED("sum_partials_x", st);
  return FCT_OK;
}
