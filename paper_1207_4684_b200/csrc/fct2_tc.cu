// fct2_tc.cu -- NEXT-3: the dense Cauchy contraction of FCT2,  W += C Z  (C: r1 x K, Z: K x d, PAPER.md
// P:L2361-2367, time O(n r1 s / t) P:L839-854), on the tcgen05 tensor cores in 3xTF32:
//     C Z ~= C_hi Z_hi + C_hi Z_lo + C_lo Z_hi     (x_hi = tf32(x), x_lo = x - x_hi; C_lo Z_lo ~ 2^-22 dropped)
// One CTA per (128-row tile of C, N-column tile of Z, K range); warp-specialised like K2 (rownorm_ws2.cu):
//   warps 0-3  split: thread r <-> row r of the C tile <-> TMEM lane r: C_lo -> TMEM (A operand of the TS MMA)
//   warp 4     TMA producer: per 32-wide K chunk the C tile (128 x 32, SWIZZLE_128B) and the Z^T_hi, Z^T_lo tiles
//              (N x 32) written transposed by the SRHT kernel, into an NA-deep ring
//   warp 5     MMA issuer: 12 MMAs per chunk (kind::tf32, M = 128, N = 32 or 64) into a TMEM accumulator
//   warps 6-9  epilogue: every FL chunks (FL * 32 = 256 K) the fp32 accumulator is folded into fp64 registers
//              (two TMEM accumulators alternate), at the end added into the fp64 workspace W (atomics)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include "common.cuh"
#include "tc.cuh"

namespace {

constexpr int kNA = 4;      // TMA ring depth
constexpr int kFL = 8;      // chunks per fp32 accumulation window (8 x 32 = 256 K)
constexpr int kThreads = 320;

template <int N>
struct TcSmem {
  static constexpr int ctile = 128 * 128;       // bytes: 128 rows x 32 fp32
  static constexpr int ztile = N * 128;         // bytes: N rows x 32 fp32
  static constexpr int stage = ctile + 2 * ztile;
  static constexpr int bars = kNA * stage;
  static constexpr int total = bars + 8 * (2 * kNA + 4 + 4);
};

template <int N>
__global__ void __launch_bounds__(kThreads, 1)
cz_tc_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmZh,
             const __grid_constant__ CUtensorMap tmZl, int r1, int d, int64_t nchunks_total, int chunks_per_cta,
             double* __restrict__ W) {
  using L = TcSmem<N>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* base = smraw + ((1024u - (tcx::su32(smraw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)(base + L::bars);   // [kNA] TMA landed
  uint64_t* empty = full + kNA;                    // [kNA] stage reusable (MMA done)
  uint64_t* lo_full = empty + kNA;                 // [2]   C_lo in TMEM (4 split-warp arrivals)
  uint64_t* lo_free = lo_full + 2;                 // [2]   C_lo buffer reusable (MMA done)
  uint64_t* d_full = lo_free + 2;                  // [2]   accumulator window complete
  uint64_t* d_free = d_full + 2;                   // [2]   accumulator drained (4 epilogue-warp arrivals)
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * N;
  const int64_t j0 = (int64_t)blockIdx.z * chunks_per_cta;
  const int nch = (int)max((int64_t)0, min((int64_t)chunks_per_cta, nchunks_total - j0));
  const int nwin = (nch + kFL - 1) / kFL;

  if (tid == 0) {
    for (int i = 0; i < kNA; ++i) {
      tcx::bar_init(&full[i], 1);
      tcx::bar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tcx::bar_init(&lo_full[i], 4);
      tcx::bar_init(&lo_free[i], 1);
      tcx::bar_init(&d_full[i], 1);
      tcx::bar_init(&d_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tcx::su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;            // TMEM: [C_lo 0 | C_lo 1] (32 cols each) [D 0 | D 1] (N cols each)
  const uint32_t dcol0 = 64;

  if (warp < 4) {
    // ---------------------------------------------------------------- split: C_lo -> TMEM
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    for (int j = 0; j < nch; ++j) {
      const int sa = j % kNA, sl = j & 1;
      tcx::bar_wait(&full[sa], (unsigned)((j / kNA) & 1));
      if (j >= 2) tcx::bar_wait(&lo_free[sl], (unsigned)(((j - 2) >> 1) & 1));
      const float* ct = (const float*)(base + sa * L::stage);
      uint32_t lo[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 v = *(const float4*)(ct + tid * 32 + ((c ^ (tid & 7)) << 2));
        lo[c * 4 + 0] = __float_as_uint(v.x - tcx::trunc_tf32(v.x));
        lo[c * 4 + 1] = __float_as_uint(v.y - tcx::trunc_tf32(v.y));
        lo[c * 4 + 2] = __float_as_uint(v.z - tcx::trunc_tf32(v.z));
        lo[c * 4 + 3] = __float_as_uint(v.w - tcx::trunc_tf32(v.w));
      }
      tcx::tmem_st32(tm + lane_off + (uint32_t)(sl * 32), lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&lo_full[sl]);
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int j = 0; j < nch; ++j) {
        const int sa = j % kNA;
        if (j >= kNA) tcx::bar_wait(&empty[sa], (unsigned)(((j - kNA) / kNA) & 1));
        unsigned char* st = base + sa * L::stage;
        const int k0 = (int)((j0 + j) * 32);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tcx::su32(&full[sa])),
                     "r"(L::stage) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                tcx::su32(st)), "l"(&tmC), "r"(k0), "r"(m0), "r"(tcx::su32(&full[sa])) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                tcx::su32(st + L::ctile)), "l"(&tmZh), "r"(k0), "r"(n0), "r"(tcx::su32(&full[sa])) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                tcx::su32(st + L::ctile + L::ztile)), "l"(&tmZl), "r"(k0), "r"(n0), "r"(tcx::su32(&full[sa])) : "memory");
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int j = 0; j < nch; ++j) {
        const int sa = j % kNA, sl = j & 1, w = j / kFL, sd = w & 1;
        const bool first = (j % kFL) == 0;
        tcx::bar_wait(&lo_full[sl], (unsigned)((j >> 1) & 1));       // implies the stage has landed
        if (first && w >= 2) tcx::bar_wait(&d_free[sd], (unsigned)(((w - 2) >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        unsigned char* st = base + sa * L::stage;
        const uint64_t ad = tcx::sdesc_sw128(st), bh = tcx::sdesc_sw128(st + L::ctile),
                       bl = tcx::sdesc_sw128(st + L::ctile + L::ztile);
        const uint32_t tD = tm + dcol0 + (uint32_t)(sd * N);
        const uint32_t tA = tm + (uint32_t)(sl * 32);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t o = (uint64_t)((ks * 32) >> 4);
          tcx::mma_tf32_ss(tD, ad + o, bh + o, idesc, (first && ks == 0) ? 0u : 1u);   // C_hi Z_hi
          tcx::mma_tf32_ss(tD, ad + o, bl + o, idesc, 1u);                               // C_hi Z_lo
          tcx::mma_tf32_ts(tD, tA + (uint32_t)(ks * 8), bh + o, idesc, 1u);               // C_lo Z_hi
        }
        tcx::mma_commit(&empty[sa]);
        tcx::mma_commit(&lo_free[sl]);
        if ((j % kFL) == kFL - 1 || j == nch - 1) tcx::mma_commit(&d_full[sd]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue: fold windows into fp64
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    double acc[N];
#pragma unroll
    for (int c = 0; c < N; ++c) acc[c] = 0.0;
    for (int w = 0; w < nwin; ++w) {
      const int sd = w & 1;
      tcx::bar_wait_sleep(&d_full[sd], (unsigned)((w >> 1) & 1), 2000);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int q = 0; q < N / 32; ++q) {
        uint32_t v[32];
        tcx::tmem_ld32(tm + lane_off + dcol0 + (uint32_t)(sd * N + q * 32), v);
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[q * 32 + c] += (double)__uint_as_float(v[c]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tcx::bar_arrive(&d_free[sd]);
    }
    if (m0 + r < r1 && nwin > 0) {
#pragma unroll
      for (int c = 0; c < N; ++c)
        if (n0 + c < d && acc[c] != 0.0) atomicAdd(&W[(int64_t)(m0 + r) * d + n0 + c], acc[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
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

bool make_map(CUtensorMap* map, const float* ptr, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {32, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int N>
fct_status launch_tc(const float* C, int64_t ldc, const float* Zh, const float* Zl, int64_t ldzt, int64_t K, int r1,
                     int d, double* W, cudaStream_t st) {
  CUtensorMap mc, mh, ml;
  if (!make_map(&mc, C, K, r1, ldc, 128) || !make_map(&mh, Zh, K, d, ldzt, N) || !make_map(&ml, Zl, K, d, ldzt, N))
    return FCT_ERR_UNSUPPORTED;
  const int mt = (r1 + 127) / 128, ntl = (d + N - 1) / N;
  const int64_t nchunks = (K + 31) / 32;
  int64_t splits = std::max<int64_t>(1, (int64_t)fct::num_sms() / (mt * ntl));
  int64_t per = (nchunks + splits - 1) / splits;
  per = std::max<int64_t>(per, kFL);
  splits = (nchunks + per - 1) / per;
  if (splits > 65535 || per > (1 << 30)) return FCT_ERR_UNSUPPORTED;
  const size_t smem = (size_t)TcSmem<N>::total + 1024;
  FCT_CUDA_RET(cudaFuncSetAttribute(cz_tc_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cz_tc_kernel<N><<<dim3(mt, ntl, (unsigned)splits), kThreads, smem, st>>>(mc, mh, ml, r1, d, nchunks, (int)per, W);
  FCT_LAUNCHED("fct2 cz_tc_kernel", st);
  return FCT_OK;
}

}  // namespace

// W (r1 x d fp64, pre-zeroed) += C Z with Z given transposed and split: Zh = tf32(Z)^T, Zl = (Z - tf32(Z))^T, both
// d x K fp32 with row stride ldzt.  FCT_ERR_UNSUPPORTED (nothing enqueued) when the TMA constraints fail.
fct_status fct2_cz_tc(const float* C, int64_t ldc, const float* Zh, const float* Zl, int64_t ldzt, int64_t K, int r1,
                      int d, double* W, cudaStream_t st) {
  if ((ldc % 4) || (ldzt % 4) || ((uintptr_t)C & 15) || ((uintptr_t)Zh & 15) || ((uintptr_t)Zl & 15) || K < 1 ||
      K >= (1LL << 31) || r1 < 1 || d < 1)
    return FCT_ERR_UNSUPPORTED;
  if (d <= 32) return launch_tc<32>(C, ldc, Zh, Zl, ldzt, K, r1, d, W, st);
  return launch_tc<64>(C, ldc, Zh, Zl, ldzt, K, r1, d, W, st);
}
