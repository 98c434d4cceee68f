// sketch_v1.cu -- K1 v1: FCT1 sketch with TMA-staged tiles and a register FWHT (Sec. 3.1).
//
// Per CTA: one column slice [c0, c0+DT) of the output, fp32 partial P[r1][DT] in shared memory for the
// CTA's lifetime (flushed once into the fp64 workspace).  The CTA's threads form TILES independent
// "tile groups" (NT threads each, own TMA buffer, own named barrier) that take row blocks round-robin.
// Per block b (S = s rows) and tile group:
//   TMA     tile[S][DT] <- A[bS : bS+S, c0 : c0+DT]            (zero fill past n / past d)
//   phase A thread (c, g) holds rows g + (S/RA) k, k < RA (high row bits in registers):
//           z = sign * a; identity half scatter P[h(2sb+s+r)][c] += 4 c_t z;
//           LA butterfly stages; STS back with an XOR row swizzle
//   phase B thread (c, g') holds rows RB g' + k, k < RB (low row bits): LDS; the buffer is now free
//           -> the next block's TMA is issued; LB butterfly stages; Hadamard half scatter
//           P[h(2sb+r)][c] += (4 c_t / sqrt(s)) (H_s z)_r
// s = 2^(LA+LB).  Scatter-add into P uses shared-memory atomics (exclusive: any two threads may
// hit the same bucket).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include "common.cuh"

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}


// Batched shared-memory float add with ILP: all loads, then all CAS (ATOMS.CAS returns the old
// word), then a retry loop for the (rare) lanes whose word changed in between.  Exact: an update is
// applied only by a successful CAS on the value it read.
template <int N>
__device__ __forceinline__ void smem_add_batch(float* __restrict__ P, const int (&addr)[N], const float (&val)[N]) {
  float old[N];
#pragma unroll
  for (int q = 0; q < N; ++q) old[q] = P[addr[q]];
  unsigned pending = 0u;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const int want = __float_as_int(old[q]);
    const int got = atomicCAS((int*)&P[addr[q]], want, __float_as_int(old[q] + val[q]));
    if (got != want) pending |= 1u << q;
  }
  while (pending) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      if ((pending >> q) & 1u) {
        const float o = P[addr[q]];
        const int want = __float_as_int(o);
        if (atomicCAS((int*)&P[addr[q]], want, __float_as_int(o + val[q])) == want) pending &= ~(1u << q);
      }
    }
  }
}

template <int LA, int LB, int DT, int TILES_>
struct Geo {
  static constexpr int S = 1 << (LA + LB);
  static constexpr int RA = 1 << LA;            // registers per thread in phase A
  static constexpr int RB = 1 << LB;            // registers per thread per group in phase B
  static constexpr int NT = S * DT / RA;        // threads per tile group
  static constexpr int NB = (S / RB) * DT / NT; // phase-B groups per thread
  static constexpr int TILES = TILES_;
  static constexpr int THREADS = NT * TILES;
  static constexpr int G = DT >= 32 ? 1 : 32 / DT;  // rows per warp-instruction
  static constexpr int BOXR = S < 256 ? S : 256;
  static_assert(NT >= 32 && THREADS <= 1024 && TILES <= 15, "tile group size");
  static_assert(NB >= 1 && RB >= G, "phase B layout");
  static constexpr size_t tile_bytes = (size_t)S * DT * sizeof(float);
};

// physical row of logical row r in the exchange layout (conflict-free phase-B reads)
template <int LB, int G>
__device__ __forceinline__ int swz(int r) {
  return G > 1 ? (r ^ ((r >> LB) & (G - 1))) : r;
}

template <int LA, int LB, int DT, int TL>
__global__ void __launch_bounds__(Geo<LA, LB, DT, TL>::THREADS, 1)
sketch_v1_kernel(const __grid_constant__ CUtensorMap tmap, int64_t n, int d, const int8_t* __restrict__ signs,
                 const float* __restrict__ cauchy, const int32_t* __restrict__ hash, int r1, int nslices,
                 int64_t nblocks, float inv_sqrt_s, double* __restrict__ W) {
  using Gm = Geo<LA, LB, DT, TL>;
  constexpr int S = Gm::S, RA = Gm::RA, RB = Gm::RB, NT = Gm::NT, NB = Gm::NB, TILES = Gm::TILES, G = Gm::G;
  extern __shared__ __align__(128) unsigned char smraw[];
  float* tiles = (float*)smraw;                                     // [TILES][S][DT]
  float* P = (float*)(smraw + TILES * Gm::tile_bytes);             // [r1][DT]
  __shared__ __align__(8) uint64_t bars[TILES];

  const int cs = blockIdx.x % nslices;
  const int grp = blockIdx.x / nslices;
  const int ngrp = gridDim.x / nslices;
  const int c0 = cs * DT;
  const int tg = threadIdx.x / NT;        // tile group
  const int lt = threadIdx.x - tg * NT;   // thread within the tile group
  const int c = lt % DT;
  float* tile = tiles + (size_t)tg * S * DT;
  uint64_t* bar = &bars[tg];

  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) P[e] = 0.f;
  if (threadIdx.x < TILES) mbar_init(&bars[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  // blocks of this tile group: b = grp + ngrp * (tg + TILES * t)
  const int64_t bstep = (int64_t)ngrp * TILES;
  int64_t b = grp + (int64_t)ngrp * tg;
  if (lt == 0 && b < nblocks) {
    mbar_expect_tx(bar, (unsigned)Gm::tile_bytes);
#pragma unroll
    for (int q = 0; q < S / Gm::BOXR; ++q)
      tma_load_2d(tile + (size_t)q * Gm::BOXR * DT, &tmap, c0, (int)(b * S + q * Gm::BOXR), bar);
  }
  unsigned phase = 0;
  for (; b < nblocks; b += bstep) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int64_t rowb = b * S;
    const int64_t t0 = 2 * rowb;  // first H~-row of the block
    // ---------------- phase A: rows g + (S/RA) k
    {
      const int g = lt / DT;
      float x[RA];
#pragma unroll
      for (int k = 0; k < RA; ++k) x[k] = tile[(g + (S / RA) * k) * DT + c];
      // aux loads software-pipelined one batch ahead of the shared-memory atomics (which would
      // otherwise serialise them behind the CAS loops)
      constexpr int BA = RA < 8 ? RA : 8;
      int sgv[2][BA], hv[2][BA];
      float cwv[2][BA];
      auto load_a = [&](int buf, int k0) {
#pragma unroll
        for (int q = 0; q < BA; ++q) {
          const int r = g + (S / RA) * (k0 + q);
          const int64_t row = rowb + r;
          const int64_t t = t0 + S + r;
          sgv[buf][q] = row < n ? (int)__ldg(signs + row) : 0;   // converted at use, not at load
          cwv[buf][q] = __ldg(cauchy + t);
          hv[buf][q] = __ldg(hash + t);
        }
      };
      load_a(0, 0);
#pragma unroll
      for (int k0 = 0; k0 < RA; k0 += BA) {
        const int cur = (k0 / BA) & 1;
        if (k0 + BA < RA) load_a(cur ^ 1, k0 + BA);
        int ad[BA];
        float vv[BA];
#pragma unroll
        for (int q = 0; q < BA; ++q) {
          x[k0 + q] *= (float)sgv[cur][q];
          ad[q] = hv[cur][q] * DT + c;
          vv[q] = (4.f * cwv[cur][q]) * x[k0 + q];
        }
        smem_add_batch<BA>(P, ad, vv);
      }
#pragma unroll
      for (int h = 1; h < RA; h <<= 1)
#pragma unroll
        for (int k = 0; k < RA; ++k)
          if (!(k & h)) {
            const float a = x[k], bb = x[k + h];
            x[k] = a + bb;
            x[k + h] = a - bb;
          }
      named_bar(1 + tg, NT);  // everyone has read the TMA tile
#pragma unroll
      for (int k = 0; k < RA; ++k) tile[swz<LB, G>(g + (S / RA) * k) * DT + c] = x[k];
    }
    named_bar(1 + tg, NT);
    // ---------------- phase B: rows RB g' + k
    float y[NB][RB];
#pragma unroll
    for (int gi = 0; gi < NB; ++gi) {
      const int gp = lt / DT + (NT / DT) * gi;
#pragma unroll
      for (int k = 0; k < RB; ++k) y[gi][k] = tile[swz<LB, G>(RB * gp + k) * DT + c];
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    named_bar(1 + tg, NT);  // the buffer is free: prefetch the next block
    const int64_t bn = b + bstep;
    if (lt == 0 && bn < nblocks) {
      mbar_expect_tx(bar, (unsigned)Gm::tile_bytes);
#pragma unroll
      for (int q = 0; q < S / Gm::BOXR; ++q)
        tma_load_2d(tile + (size_t)q * Gm::BOXR * DT, &tmap, c0, (int)(bn * S + q * Gm::BOXR), bar);
    }
#pragma unroll
    for (int gi = 0; gi < NB; ++gi) {
      const int gp = lt / DT + (NT / DT) * gi;
#pragma unroll
      for (int h = 1; h < RB; h <<= 1)
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (!(k & h)) {
            const float a = y[gi][k], bb = y[gi][k + h];
            y[gi][k] = a + bb;
            y[gi][k + h] = a - bb;
          }
      // contiguous rows: 16-byte vector loads of (hash, cauchy), 8 rows per batch, one batch ahead
      const int64_t tb = t0 + RB * gp;
      static_assert(RB % 8 == 0, "phase B batches");
      int4 hq[2][2];
      float4 cq[2][2];
      auto load_b = [&](int buf, int k0) {
        hq[buf][0] = __ldg((const int4*)(hash + tb + k0));
        hq[buf][1] = __ldg((const int4*)(hash + tb + k0 + 4));
        cq[buf][0] = __ldg((const float4*)(cauchy + tb + k0));
        cq[buf][1] = __ldg((const float4*)(cauchy + tb + k0 + 4));
      };
      load_b(0, 0);
      const float sc = 4.f * inv_sqrt_s;
#pragma unroll
      for (int k0 = 0; k0 < RB; k0 += 8) {
        const int cur = (k0 / 8) & 1;
        if (k0 + 8 < RB) load_b(cur ^ 1, k0 + 8);
        const int hv[8] = {hq[cur][0].x, hq[cur][0].y, hq[cur][0].z, hq[cur][0].w,
                           hq[cur][1].x, hq[cur][1].y, hq[cur][1].z, hq[cur][1].w};
        const float cw[8] = {cq[cur][0].x, cq[cur][0].y, cq[cur][0].z, cq[cur][0].w,
                             cq[cur][1].x, cq[cur][1].y, cq[cur][1].z, cq[cur][1].w};
        int ad[8];
        float vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          ad[q] = hv[q] * DT + c;
          vv[q] = (sc * cw[q]) * y[gi][k0 + q];
        }
        smem_add_batch<8>(P, ad, vv);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) {
    const int h = e / DT, cc = e - h * DT;
    const float v = P[e];
    if (c0 + cc < d && v != 0.f) atomicAdd(&W[(size_t)h * d + c0 + cc], (double)v);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

template <int LA, int LB, int DT, int TL>
fct_status launch_v1(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                     const int32_t* hash, int s, int r1, double* W, cudaStream_t st) {
  using Gm = Geo<LA, LB, DT, TL>;
  auto enc = get_encode();
  FCT_CHECK_ARG(enc, FCT_ERR_CUDA, "fct_sketch: cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)DT, (cuuint32_t)Gm::BOXR};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  FCT_CHECK_ARG(cr == CUDA_SUCCESS, FCT_ERR_CUDA, "fct_sketch: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  const int nslices = (int)((d + DT - 1) / DT);
  const int64_t nblocks = (n + s - 1) / s;
  const size_t smem = Gm::TILES * Gm::tile_bytes + (size_t)r1 * DT * sizeof(float);
  auto kern = sketch_v1_kernel<LA, LB, DT, TL>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  FCT_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Gm::THREADS, smem));
  if (occ < 1) occ = 1;
  // CTAs per slice: fill the SMs, and keep <= ~2048 expected terms per bucket per CTA partial
  int64_t ngrp = ((int64_t)fct::num_sms() * occ) / nslices;
  const int64_t min_grp = (2 * nblocks * (int64_t)s + 2048LL * r1 - 1) / (2048LL * r1);
  ngrp = std::max<int64_t>(std::max<int64_t>(ngrp, 1), min_grp);
  ngrp = std::min<int64_t>(ngrp, (nblocks + Gm::TILES - 1) / Gm::TILES);
  if (ngrp < 1) ngrp = 1;
  kern<<<(unsigned)(ngrp * nslices), Gm::THREADS, smem, st>>>(map, n, (int)d, signs, cauchy, hash, r1, nslices,
                                                               nblocks, (float)(1.0 / sqrt((double)s)), W);
  FCT_LAUNCHED("sketch_v1_kernel", st);
  return FCT_OK;
}

constexpr size_t kV1Smem = 220 * 1024;

template <int LA, int LB, int DT, int TL>
bool fits(int r1) {
  using Gm = Geo<LA, LB, DT, TL>;
  return Gm::TILES * Gm::tile_bytes + (size_t)r1 * DT * sizeof(float) <= kV1Smem;
}

}  // namespace

// Returns FCT_ERR_UNSUPPORTED (without enqueueing) when no v1 instance covers (s, d, r1, alignment).
fct_status fct_sketch_v1(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                         const int32_t* hash, int s, int r1, double* W, cudaStream_t st) {
  if (((uintptr_t)A & 15) || ((uintptr_t)cauchy & 15) || ((uintptr_t)hash & 15) || (lda % 4) || n >= (1LL << 31))
    return FCT_ERR_UNSUPPORTED;
#define TRY(LA_, LB_, DT_, TL_)                                                              \
  if (s == (1 << (LA_ + LB_)) && fits<LA_, LB_, DT_, TL_>(r1) && (DT_ <= 8 || d >= DT_))     \
    return launch_v1<LA_, LB_, DT_, TL_>(A, n, d, lda, signs, cauchy, hash, s, r1, W, st);
  // widest column slice that fits first (fewer aux re-reads, fewer bank conflicts), then narrower
  TRY(6, 5, 16, 1) TRY(6, 5, 8, 2) TRY(6, 5, 4, 2) TRY(6, 5, 4, 1)        // s = 2048
  TRY(5, 5, 16, 1) TRY(5, 5, 8, 2) TRY(5, 5, 4, 4) TRY(5, 5, 4, 2)        // s = 1024
  TRY(4, 4, 16, 2) TRY(4, 4, 8, 4) TRY(4, 4, 4, 8)                        // s = 256
  TRY(3, 3, 8, 8) TRY(3, 3, 4, 8)                                         // s = 64
#undef TRY
  return FCT_ERR_UNSUPPORTED;
}
