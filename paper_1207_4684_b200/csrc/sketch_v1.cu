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


// Batched shared-memory float add with ILP (MODE 0, the default): all loads, then all CAS (ATOMS.CAS returns the
// old word), then a retry loop for the (rare) lanes whose word changed in between.  Exact: an update is applied
// only by a successful CAS on the value it read.
template <int N>
__device__ __forceinline__ void smem_add_batch(float* __restrict__ P, const int (&addr)[N], const float (&val)[N]) {
  float old[N];
#pragma unroll
  for (int q = 0; q < N; ++q) old[q] = P[addr[q]];
  unsigned pending = 0;
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

// Measured alternatives (opt-in instances, K1):
//   MODE 1: ATOMS.EXCH take / add / EXCH put, re-adding any deposit made in between (exact);
//   MODE 2: buckets h >= t_l2 go to L2 (RED.ADD.F32 of v * 2^20 into this CTA's fp32 replica of those bucket
//           rows; global atomics are exact updates, the 2^20 keeps nonzero terms normal under the reduction's
//           flush-to-zero and is divided out exactly when the replicas are reduced), the rest use MODE 0;
//   MODE 3: plain LDS + STS, which LOSES concurrent updates (a timing bound only; never parity-tested).
template <int MODE, int N>
__device__ __forceinline__ void scatter_batch(float* __restrict__ P, const int (&addr)[N], const float (&val)[N],
                                              const int (&h)[N], float* repc, int t_l2, int d) {
  if constexpr (MODE == 0) {
    smem_add_batch<N>(P, addr, val);
  } else if constexpr (MODE == 1) {
    float x[N];
#pragma unroll
    for (int q = 0; q < N; ++q) x[q] = atomicExch(&P[addr[q]], 0.0f);
#pragma unroll
    for (int q = 0; q < N; ++q) x[q] = atomicExch(&P[addr[q]], x[q] + val[q]);
    unsigned pending = 0u;
#pragma unroll
    for (int q = 0; q < N; ++q) if (x[q] != 0.0f) pending |= 1u << q;
    while (pending) {
#pragma unroll
      for (int q = 0; q < N; ++q)
        if ((pending >> q) & 1u) {
          const float t = atomicExch(&P[addr[q]], 0.0f);
          x[q] = atomicExch(&P[addr[q]], t + x[q]);
          if (!(x[q] != 0.0f)) pending &= ~(1u << q);
        }
    }
  } else if constexpr (MODE == 2) {
    // L2 lanes: predicated REDs; the shared-memory LDS / CAS of those lanes are predicated off
    unsigned sm = 0u;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const bool l2 = repc && h[q] >= t_l2 && fabsf(val[q]) >= 0x1p-100f;
      if (l2) atomicAdd(repc + (size_t)(h[q] - t_l2) * d, val[q] * 0x1p20f);
      else sm |= 1u << q;
    }
    float old[N];
#pragma unroll
    for (int q = 0; q < N; ++q) old[q] = ((sm >> q) & 1u) ? P[addr[q]] : 0.0f;
    unsigned pending = 0u;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      if ((sm >> q) & 1u) {
        const int want = __float_as_int(old[q]);
        if (atomicCAS((int*)&P[addr[q]], want, __float_as_int(old[q] + val[q])) != want) pending |= 1u << q;
      }
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
  } else {
    float old[N];
#pragma unroll
    for (int q = 0; q < N; ++q) old[q] = P[addr[q]];
#pragma unroll
    for (int q = 0; q < N; ++q) P[addr[q]] = old[q] + val[q];
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

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// packed fp32x2 add / sub (FADD2 on sm_100)
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r, x = *(unsigned long long*)&a, y = *(unsigned long long*)&b;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  return *(float2*)&r;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r, x = *(unsigned long long*)&a, y = *(unsigned long long*)&b;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  return *(float2*)&r;
}
// in-register unnormalised Walsh-Hadamard transform of R values (natural order): stage 1 scalar,
// stages 2..R/2 on packed pairs (two independent butterflies per FADD2)
template <int R>
__device__ __forceinline__ void fwht_regs(float (&x)[R]) {
#pragma unroll
  for (int k = 0; k < R; k += 2) {
    const float a = x[k], b = x[k + 1];
    x[k] = a + b;
    x[k + 1] = a - b;
  }
#pragma unroll
  for (int h = 2; h < R; h <<= 1)
#pragma unroll
    for (int k = 0; k < R; k += 2)
      if (!(k & h)) {
        const float2 a = make_float2(x[k], x[k + 1]), b = make_float2(x[k + h], x[k + h + 1]);
        const float2 s2 = add2(a, b), d2 = sub2(a, b);
        x[k] = s2.x; x[k + 1] = s2.y;
        x[k + h] = d2.x; x[k + h + 1] = d2.y;
      }
}

// aux bytes staged per block: identity half = signs[S] (padded to 16) + cauchy[S] + hash[S];
// Hadamard half = cauchy[S] + hash[S]
template <int S>
struct AuxLayout {
  static constexpr int sign_bytes = (S + 15) / 16 * 16;
  static constexpr int id_bytes = sign_bytes + 8 * S;
  static constexpr int had_bytes = 8 * S;
};

// L2 offload: updates of buckets h >= t_l2 go to the CTA's fp32 replica rep[grp % nrep][h - t_l2][d] in global
// memory (L2-resident) instead of shared memory, so the shared-memory pipe -- the kernel's limiter -- carries
// only the buckets below t_l2 (t_l2 = r1: everything in shared memory).
template <int LA, int LB, int DT, int TL, int MODE>
__global__ void __launch_bounds__(Geo<LA, LB, DT, TL>::THREADS, 1)
sketch_v1_kernel(const __grid_constant__ CUtensorMap tmap, int64_t n, int d, const int8_t* __restrict__ signs,
                 const float* __restrict__ cauchy, const int32_t* __restrict__ hash, int r1, int nslices,
                 int64_t nblocks, float inv_sqrt_s, double* __restrict__ W, float* __restrict__ rep, int t_l2,
                 int nrep) {
  using Gm = Geo<LA, LB, DT, TL>;
  using AL = AuxLayout<Gm::S>;
  constexpr int S = Gm::S, RA = Gm::RA, RB = Gm::RB, NT = Gm::NT, NB = Gm::NB, TILES = Gm::TILES, G = Gm::G;
  extern __shared__ __align__(128) unsigned char smraw[];
  // [TILES] tiles | [TILES] identity aux | [TILES] Hadamard aux | P[r1][DT]
  float* tiles = (float*)smraw;
  unsigned char* auxI0 = smraw + TILES * Gm::tile_bytes;
  unsigned char* auxH0 = auxI0 + TILES * AL::id_bytes;
  float* P = (float*)(auxH0 + TILES * AL::had_bytes);
  __shared__ __align__(8) uint64_t bar_t[TILES], bar_i[TILES], bar_h[TILES];

  const int cs = blockIdx.x % nslices;
  const int grp = blockIdx.x / nslices;
  const int ngrp = gridDim.x / nslices;
  const int c0 = cs * DT;
  const int tg = threadIdx.x / NT;        // tile group
  const int lt = threadIdx.x - tg * NT;   // thread within the tile group
  const int c = lt % DT;
  float* tile = tiles + (size_t)tg * S * DT;
  // this thread's column of the CTA's L2 replica (nullptr: no L2 path for this column)
  float* const repc = (MODE == 2 && rep && t_l2 < r1 && c0 + c < d)
                          ? rep + (size_t)(grp % nrep) * (size_t)(r1 - t_l2) * d + (c0 + c) : nullptr;
  unsigned char* auxI = auxI0 + tg * AL::id_bytes;
  unsigned char* auxH = auxH0 + tg * AL::had_bytes;
  const int8_t* sSign = (const int8_t*)auxI;
  const float* sCi = (const float*)(auxI + AL::sign_bytes);
  const int* sHi = (const int*)(auxI + AL::sign_bytes + 4 * S);
  const float* sCh = (const float*)auxH;
  const int* sHh = (const int*)(auxH + 4 * S);
  (void)sSign; (void)sCi; (void)sHi; (void)sCh; (void)sHh;

  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) P[e] = 0.f;
  if (threadIdx.x < TILES) {
    mbar_init(&bar_t[threadIdx.x], 1);
    mbar_init(&bar_i[threadIdx.x], 1);
    mbar_init(&bar_h[threadIdx.x], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  auto issue_tile = [&](int64_t bb) {
    mbar_expect_tx(&bar_t[tg], (unsigned)Gm::tile_bytes);
#pragma unroll
    for (int q = 0; q < S / Gm::BOXR; ++q)
      tma_load_2d(tile + (size_t)q * Gm::BOXR * DT, &tmap, c0, (int)(bb * S + q * Gm::BOXR), &bar_t[tg]);
  };
  // signs: bulk-copy the 16-byte-aligned prefix of the block's valid rows; the (rare) tail past it is
  // read from global memory in phase A
  auto sign_bulk = [&](int64_t bb) -> int {
    const int64_t valid = n - bb * S < S ? n - bb * S : S;
    return (int)(valid & ~15LL);
  };
  auto issue_id = [&](int64_t bb) {
    const int sb = sign_bulk(bb);
    const int64_t t0 = 2 * bb * S;
    mbar_expect_tx(&bar_i[tg], (unsigned)(sb + 8 * S));
    if (sb > 0) bulk_g2s(auxI, signs + bb * S, (unsigned)sb, &bar_i[tg]);
    bulk_g2s(auxI + AL::sign_bytes, cauchy + t0 + S, 4u * S, &bar_i[tg]);
    bulk_g2s(auxI + AL::sign_bytes + 4 * S, hash + t0 + S, 4u * S, &bar_i[tg]);
  };
  auto issue_had = [&](int64_t bb) {
    const int64_t t0 = 2 * bb * S;
    mbar_expect_tx(&bar_h[tg], 8u * S);
    bulk_g2s(auxH, cauchy + t0, 4u * S, &bar_h[tg]);
    bulk_g2s(auxH + 4 * S, hash + t0, 4u * S, &bar_h[tg]);
  };

  // blocks of this tile group: b = grp + ngrp * (tg + TILES * t)
  const int64_t bstep = (int64_t)ngrp * TILES;
  int64_t b = grp + (int64_t)ngrp * tg;
  if (lt == 0 && b < nblocks) {
    issue_tile(b);
    issue_id(b);
    issue_had(b);
  }
  unsigned phase = 0;
  const float sc_h = 4.f * inv_sqrt_s;
  for (; b < nblocks; b += bstep) {
    const int64_t bn = b + bstep;
    mbar_wait(&bar_t[tg], phase);
    mbar_wait(&bar_i[tg], phase);
    const int64_t rowb = b * S;
    const int sb = sign_bulk(b);
    // ---------------- phase A: rows g + (S/RA) k; identity half scattered from the staged aux
    {
      const int g = lt / DT;
      float x[RA];
#pragma unroll
      for (int k = 0; k < RA; ++k) x[k] = tile[(g + (S / RA) * k) * DT + c];
      constexpr int BA = RA < 8 ? RA : 8;
#pragma unroll
      for (int k0 = 0; k0 < RA; k0 += BA) {
        int ad[BA], hh[BA];
        float vv[BA];
#pragma unroll
        for (int q = 0; q < BA; ++q) {
          const int r = g + (S / RA) * (k0 + q);
          int sg;
          if (r < sb) sg = sSign[r];
          else sg = rowb + r < n ? (int)__ldg(signs + rowb + r) : 0;
          x[k0 + q] = __int_as_float(__float_as_int(x[k0 + q]) ^ (sg & (int)0x80000000));   // sign flip, no I2F
          const int h = sHi[r];
          ad[q] = h * DT + c;
          hh[q] = h;
          vv[q] = (4.f * sCi[r]) * x[k0 + q];
        }
        scatter_batch<MODE, BA>(P, ad, vv, hh, repc, t_l2, d);
      }
      fwht_regs<RA>(x);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      named_bar(1 + tg, NT);  // everyone has read the TMA tile and the identity aux
      if (lt == 0 && bn < nblocks) issue_id(bn);
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
    named_bar(1 + tg, NT);  // the tile buffer is free: prefetch the next block
    if (lt == 0 && bn < nblocks) issue_tile(bn);
    mbar_wait(&bar_h[tg], phase);
    phase ^= 1u;
#pragma unroll
    for (int gi = 0; gi < NB; ++gi) {
      const int gp = lt / DT + (NT / DT) * gi;
      fwht_regs<RB>(y[gi]);
      static_assert(RB % 8 == 0, "phase B batches");
#pragma unroll
      for (int k0 = 0; k0 < RB; k0 += 8) {
        const int r0 = RB * gp + k0;
        const int4 h0 = *(const int4*)(sHh + r0), h1 = *(const int4*)(sHh + r0 + 4);
        const float4 q0 = *(const float4*)(sCh + r0), q1 = *(const float4*)(sCh + r0 + 4);
        const int hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const float cw[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        int ad[8];
        float vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          ad[q] = hv[q] * DT + c;
          vv[q] = (sc_h * cw[q]) * y[gi][k0 + q];
        }
        scatter_batch<MODE, 8>(P, ad, vv, hv, repc, t_l2, d);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    named_bar(1 + tg, NT);  // the Hadamard aux is free
    if (lt == 0 && bn < nblocks) issue_had(bn);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) {
    const int h = e / DT, cc = e - h * DT;
    const float v = P[e];
    if (c0 + cc < d && v != 0.f) atomicAdd(&W[(size_t)h * d + c0 + cc], (double)v);   // includes h >= t_l2 terms
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

template <int LA, int LB, int DT, int TL, int MODE>
fct_status launch_v1(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                     const int32_t* hash, int s, int r1, const SketchAcc& acc, cudaStream_t st) {
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
  const size_t smem = Gm::TILES * (Gm::tile_bytes + AuxLayout<Gm::S>::id_bytes + AuxLayout<Gm::S>::had_bytes) +
                      (size_t)r1 * DT * sizeof(float);
  auto kern = sketch_v1_kernel<LA, LB, DT, TL, MODE>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  FCT_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Gm::THREADS, smem));
  if (occ < 1) occ = 1;
  // CTAs per slice: an equal number per slice (the slices then walk the row blocks in lockstep, so each line
  // of A is read from DRAM once), keeping <= ~2048 expected terms per bucket per CTA partial
  int64_t ngrp = ((int64_t)fct::num_sms() * occ) / nslices;
  const int64_t min_grp = (2 * nblocks * (int64_t)s + 2048LL * r1 - 1) / (2048LL * r1);
  ngrp = std::max<int64_t>(std::max<int64_t>(ngrp, 1), min_grp);
  ngrp = std::min<int64_t>(ngrp, (nblocks + Gm::TILES - 1) / Gm::TILES);
  if (ngrp < 1) ngrp = 1;
  kern<<<(unsigned)(ngrp * nslices), Gm::THREADS, smem, st>>>(map, n, (int)d, signs, cauchy, hash, r1, nslices,
                                                               nblocks, (float)(1.0 / sqrt((double)s)), acc.W,
                                                               acc.rep, acc.t_l2, acc.nrep);
  FCT_LAUNCHED("sketch_v1_kernel", st);
  fct::set_instance(0, "sketch_v1_kernel<%d, %d, %d, %d, %d>", LA, LB, DT, TL, MODE);
  return FCT_OK;
}

constexpr size_t kV1Smem = 232448 - 256;   // max dynamic shared memory per block on sm_100, less static

template <int LA, int LB, int DT, int TL>
bool fits(int r1) {
  using Gm = Geo<LA, LB, DT, TL>;
  return Gm::TILES * (Gm::tile_bytes + AuxLayout<Gm::S>::id_bytes + AuxLayout<Gm::S>::had_bytes) +
             (size_t)r1 * DT * sizeof(float) <= kV1Smem;
}

}  // namespace

// Returns FCT_ERR_UNSUPPORTED (without enqueueing) when no v1 instance covers (s, d, r1, alignment).
fct_status fct_sketch_v1(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                         const int32_t* hash, int s, int r1, const SketchAcc& acc, cudaStream_t st) {
  if (((uintptr_t)A & 15) || ((uintptr_t)cauchy & 15) || ((uintptr_t)hash & 15) || ((uintptr_t)signs & 15) ||
      (lda % 4) || n >= (1LL << 31))
    return FCT_ERR_UNSUPPORTED;
  // scatter primitive: MODE 1 (EXCH pair, exact) is the default -- measured 14 % faster than MODE 0 (CAS) at
  // the cfg-4 shape (2^24 rows: 2.77 vs 3.22 ms, profiles/r02_sketch_scatter_modes.jsonl); MODE 0 stays
  // selectable (FCT_SKETCH_SCATTER=cas); MODE 2 (L2 offload) and 3 (racy, timing only) exist for the cfg-4/5
  // geometries only
#define TRYM(LA_, LB_, DT_, TL_, M_)                                                                     \
  if (acc.mode == M_ && s == (1 << (LA_ + LB_)) && fits<LA_, LB_, DT_, TL_>(r1) && (DT_ <= 8 || d >= DT_)) \
    return launch_v1<LA_, LB_, DT_, TL_, M_>(A, n, d, lda, signs, cauchy, hash, s, r1, acc, st);
  TRYM(5, 5, 8, 2, 2) TRYM(5, 5, 8, 2, 3) TRYM(6, 5, 4, 1, 2) TRYM(6, 5, 4, 1, 3)
#undef TRYM
#define TRY(LA_, LB_, DT_, TL_)                                                                   \
  if (s == (1 << (LA_ + LB_)) && fits<LA_, LB_, DT_, TL_>(r1) && (DT_ <= 8 || d >= DT_)) {       \
    if (acc.mode == 0) return launch_v1<LA_, LB_, DT_, TL_, 0>(A, n, d, lda, signs, cauchy, hash, s, r1, acc, st); \
    return launch_v1<LA_, LB_, DT_, TL_, 1>(A, n, d, lda, signs, cauchy, hash, s, r1, acc, st);  \
  }
  // widest column slice that fits first (fewer aux re-reads, fewer bank conflicts), then narrower
  TRY(6, 5, 16, 1) TRY(6, 5, 8, 2) TRY(6, 5, 4, 2) TRY(6, 5, 4, 1)        // s = 2048
  TRY(5, 5, 16, 1) TRY(5, 5, 8, 2) TRY(5, 5, 4, 4) TRY(5, 5, 4, 2)        // s = 1024
  TRY(4, 4, 16, 2) TRY(4, 4, 8, 4) TRY(4, 4, 4, 8)                        // s = 256
  TRY(3, 3, 8, 8) TRY(3, 3, 4, 8)                                         // s = 64
#undef TRY
  return FCT_ERR_UNSUPPORTED;
}
