// sketch_v5.cu -- K1 v5: the FCT1 sketch Y = 4 B C H~ D A (Sec. 3.1) for the full s-blocks
// of A; the ragged tail block goes to the generic kernel (sketch.cu).
//
// Same skeleton as v1 (one column slice of DT columns per CTA, fp32 partial P[r1][DT] in shared memory for the
// CTA's lifetime, TILES independent tile groups, register FWHT with one shared-memory exchange), with the two
// phases swapped so that the phase with the costlier aux (the identity half: sign, C and B per row) holds
// CONTIGUOUS rows and reads its aux with vector loads:
//   TMA (4-D box) tile[k][g][c] <- A[b S + RA g + k][c0 + c]    (k < RA, g < S/RA; conflict-free phase-A reads)
//   TMA (2-D, SWIZZLE_128B) the block's C and B halves as rows of 32 entries (conflict-free LDS.128 in phase A,
//       one broadcast word per row group in phase B); signs by a bulk copy
//   phase A thread (g, c) holds rows RA g + k (low row bits): z = sign a; identity half scatter
//           P[h(2sb+s+r)][c] += 4 c_t z (aux: LDS.128 of 4 rows); LA butterfly stages; STS with an XOR row
//           swizzle
//   phase B thread (g', c) holds rows g' + RA k (high row bits): LDS; next block's tile TMA; LB butterfly
//           stages; Hadamard half scatter P[h(2sb+r)][c] += (4 c_t / sqrt(s)) (H_s z)_r
// Scatter: ATOMS.EXCH take / add / EXCH put, re-adding any deposit made in between (exact; MODE 1), or the
// LDS + ATOMS.CAS batch (MODE 0).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include "common.cuh"

namespace {

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          su32(dst)),
      "l"(m), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, int x, int y, int z, int w, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
          su32(dst)),
      "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void nbar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
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
// in-register unnormalised Walsh-Hadamard transform of R values (Sylvester order)
template <int R>
__device__ __forceinline__ void fwht(float (&x)[R]) {
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

// exact scatter-add of N updates into the shared partial (see the file header)
template <int MODE, int N>
__device__ __forceinline__ void scatter(float* __restrict__ P, const int (&addr)[N], const float (&val)[N]) {
  if constexpr (MODE == 1) {
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
  } else {
    float old[N];
#pragma unroll
    for (int q = 0; q < N; ++q) old[q] = P[addr[q]];
    unsigned pending = 0u;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const int want = __float_as_int(old[q]);
      if (atomicCAS((int*)&P[addr[q]], want, __float_as_int(old[q] + val[q])) != want) pending |= 1u << q;
    }
    while (pending) {
#pragma unroll
      for (int q = 0; q < N; ++q)
        if ((pending >> q) & 1u) {
          const float o = P[addr[q]];
          const int want = __float_as_int(o);
          if (atomicCAS((int*)&P[addr[q]], want, __float_as_int(o + val[q])) == want) pending &= ~(1u << q);
        }
    }
  }
}

// the 8 updates of a row group go out in two batches of 4: fewer take/put windows open at once, so fewer collide
// and take the re-add loop (cfg 4: 9.52 -> 9.31 ms; batches of 2: 9.81 ms; tools/sk_batch.sh)
constexpr int kScatN = 4;
template <int MODE>
__device__ __forceinline__ void scatter8(float* __restrict__ P, const int (&ad)[8], const float (&vv)[8]) {
#pragma unroll
  for (int h = 0; h < 8; h += kScatN) {
    int a2[kScatN];
    float v2[kScatN];
#pragma unroll
    for (int q = 0; q < kScatN; ++q) {
      a2[q] = ad[h + q];
      v2[q] = vv[h + q];
    }
    scatter<MODE, kScatN>(P, a2, v2);
  }
}

template <int LA, int LB, int DT, int TILES_, bool SA_ = false>
struct Geo5 {
  // SA (shared aux): the identity and Hadamard halves of the aux use ONE pair of buffers in turn (the Hadamard
  // half is loaded after phase A has consumed the identity half) and the signs are read from global memory, so
  // that two tile groups fit next to P at r1 = 8192 (the cfg-5 geometry)
  static constexpr bool SA = SA_;
  static constexpr int S = 1 << (LA + LB);
  static constexpr int RA = 1 << LA;            // contiguous rows per thread, phase A
  static constexpr int RB = 1 << LB;            // strided rows per thread per group, phase B
  static constexpr int NG = S / RA;             // phase-A row groups (= phase-B row stride / ... = RA)
  static constexpr int NT = NG * DT;            // threads per tile group
  static constexpr int NB = RA * DT / NT;       // phase-B groups per thread (RA row offsets x DT columns)
  static constexpr int TILES = TILES_;
  static constexpr int THREADS = NT * TILES;
  static constexpr int G = DT >= 32 ? 1 : 32 / DT;   // rows per warp-instruction
  static_assert(NT >= 32 && THREADS <= 1024, "tile group size");
  static_assert(NB >= 1 && RB % 8 == 0 && RA % 16 == 0 && G <= RA && S >= 256, "layout");
  static constexpr size_t tile_bytes = (size_t)S * DT * sizeof(float);
  static constexpr size_t half_bytes = (size_t)S * 4;              // one aux half (C or B) of a block
  static constexpr size_t sign_bytes = (size_t)(S + 1023) / 1024 * 1024;
  // per tile group: tile | C_id | B_id | C_had | B_had | signs (aux halves 1024-B aligned for SWIZZLE_128B)
  static constexpr size_t group_bytes = tile_bytes + (SA ? 2 * half_bytes : 4 * half_bytes + sign_bytes);
};

// physical row of logical row r in the exchange layout: conflict-free for both phases' access patterns
template <int LA, int G>
__device__ __forceinline__ int xswz(int r) {
  return G > 1 ? (r ^ ((r >> LA) & (G - 1))) : r;
}
// word offset of aux entry e in a SWIZZLE_128B-staged array of 32-entry (128-B) rows
__device__ __forceinline__ int aux_off(int e) { return (e & ~31) | (((((e >> 2) & 7) ^ ((e >> 5) & 7)) << 2) | (e & 3)); }

template <int LA, int LB, int DT, int TL, int MODE, bool SA>
__global__ void __launch_bounds__(Geo5<LA, LB, DT, TL, SA>::THREADS, 1)
sketch_v5_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
                 const __grid_constant__ CUtensorMap tmH, const int8_t* __restrict__ signs, int r1, int d,
                 int nslices, int64_t nblocks, float inv_sqrt_s, double* __restrict__ W, int* __restrict__ pace,
                 int pace_every, int64_t nmain, int nextra) {
  using Gm = Geo5<LA, LB, DT, TL, SA>;
  constexpr int S = Gm::S, RA = Gm::RA, RB = Gm::RB, NG = Gm::NG, NT = Gm::NT, NB = Gm::NB, TILES = Gm::TILES,
                G = Gm::G;
  // SWIZZLE_128B destinations must be 1024-byte aligned: the dynamic region is declared 1024-aligned (the
  // static barriers then occupy the first 1 KB of the CTA's shared memory)
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar_t[TILES], bar_i[TILES], bar_h[TILES];
  // Work split (all SMs busy when the slice count does not divide them): the first ngrp * nslices CTAs form ngrp
  // groups of nslices (one CTA per column slice) over the blocks [0, nmain); the nextra further CTAs (nslices a
  // multiple of nextra) take the blocks [nmain, nblocks) in nslices / nextra passes, slices e, e + nextra, ...,
  // flushing P between passes.  nmain is chosen so that both kinds of CTA do the same number of block-slices.
  const int ngrp = (gridDim.x - nextra) / nslices;
  const bool extra = (int)blockIdx.x >= ngrp * nslices;
  const int eidx = extra ? (int)blockIdx.x - ngrp * nslices : 0;
  const int nseg = extra ? nslices / nextra : 1;
  const int grp = extra ? ngrp : (int)blockIdx.x / nslices;
  int cs = extra ? eidx : (int)blockIdx.x % nslices;
  int c0 = cs * DT;
  const int tg = threadIdx.x / NT;
  const int lt = threadIdx.x - tg * NT;
  const int c = lt % DT;
  unsigned char* gb = smraw + (size_t)tg * Gm::group_bytes;
  float* tile = (float*)gb;
  const float* sCi = (const float*)(gb + Gm::tile_bytes);
  const int* sHi = (const int*)(gb + Gm::tile_bytes + Gm::half_bytes);
  const float* sCh = SA ? sCi : (const float*)(gb + Gm::tile_bytes + 2 * Gm::half_bytes);
  const int* sHh = SA ? sHi : (const int*)(gb + Gm::tile_bytes + 3 * Gm::half_bytes);
  const int8_t* sSg = (const int8_t*)(gb + Gm::tile_bytes + 4 * Gm::half_bytes);   // !SA only
  float* P = (float*)(smraw + (size_t)TILES * Gm::group_bytes);

  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) P[e] = 0.f;
  if (threadIdx.x < TILES) {
    mb_init(&bar_t[threadIdx.x], 1);
    mb_init(&bar_i[threadIdx.x], 1);
    mb_init(&bar_h[threadIdx.x], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  auto issue_tile = [&](int64_t bb) {
    mb_expect(&bar_t[tg], (unsigned)Gm::tile_bytes);
    tma4(tile, &tmA, c0, 0, 0, (int)bb, &bar_t[tg]);
  };
  auto issue_id = [&](int64_t bb) {   // identity-half C and B, and the block's signs (!SA)
    mb_expect(&bar_i[tg], (unsigned)(2 * Gm::half_bytes + (SA ? 0 : S)));
    const int row = (int)((2 * bb * S + S) / 32);
    tma2((void*)sCi, &tmC, 0, row, &bar_i[tg]);
    tma2((void*)sHi, &tmH, 0, row, &bar_i[tg]);
    if (!SA) bulk((void*)sSg, signs + bb * S, (unsigned)S, &bar_i[tg]);
  };
  auto issue_had = [&](int64_t bb) {  // Hadamard-half C and B
    mb_expect(&bar_h[tg], (unsigned)(2 * Gm::half_bytes));
    const int row = (int)(2 * bb * S / 32);
    tma2((void*)sCh, &tmC, 0, row, &bar_h[tg]);
    tma2((void*)sHh, &tmH, 0, row, &bar_h[tg]);
  };

  unsigned phase = 0;
  const float sc_h = 4.f * inv_sqrt_s;
  for (int seg = 0; seg < nseg; ++seg) {
  if (seg > 0) {   // extra CTA: flush this slice's partial, then the next slice
    __syncthreads();
    for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) {
      const int h = e / DT, cc = e - h * DT;
      const float v = P[e];
      if (c0 + cc < d && v != 0.f) atomicAdd(&W[(size_t)h * d + c0 + cc], (double)v);
      P[e] = 0.f;
    }
    cs += nextra;
    c0 = cs * DT;
    __syncthreads();
  }
  const int64_t bstep = extra ? (int64_t)TILES : (int64_t)ngrp * TILES;
  const int64_t bend = extra ? nblocks : nmain;
  int64_t b = extra ? nmain + tg : grp + (int64_t)ngrp * tg;
  const int pidx = extra ? ngrp + seg : grp, parts = extra ? nextra : nslices;
  if (lt == 0 && b < bend) {
    issue_tile(b);
    issue_id(b);
    if (!SA) issue_had(b);
  }
  int it = 0;
  for (; b < bend; b += bstep, ++it) {
    const int64_t bn = b + bstep;
    // pacing: the nslices CTAs of a row-block group meet every pace_every blocks (a counter in global memory), so
    // the column slices stay in lockstep and each line of A / of the aux is still in L2 when the neighbours read it
    if (pace && tg == 0 && lt == 0 && it > 0 && it % pace_every == 0) {
      int* cnt = pace + pidx;
      const int want = parts * (it / pace_every);
      atomicAdd(cnt, 1);
      int v, spins = 0;   // a soft meeting point: the wait is bounded (~0.4 ms), so it can never deadlock
      do {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
        if (v < want) __nanosleep(200);
      } while (v < want && ++spins < 2000);
    }
    mb_wait(&bar_t[tg], phase);
    mb_wait(&bar_i[tg], phase);
    // ---------------- phase A: rows RA g + k (contiguous); identity half scattered
    {
      const int g = lt / DT;
      float x[RA];
#pragma unroll
      for (int k = 0; k < RA; ++k) x[k] = tile[(k * NG + g) * DT + c];
      static_assert(RA % 16 == 0, "phase A sign vectors");
#pragma unroll
      for (int k0 = 0; k0 < RA; k0 += 16) {   // 16 signs per 16-B load
        const int4 sv = SA ? __ldg((const int4*)(signs + b * S + RA * g + k0)) : *(const int4*)(sSg + RA * g + k0);
        const int sw[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int sgb = (sw[q >> 2] << (24 - 8 * (q & 3))) & (int)0x80000000;   // sign bit of byte q
          x[k0 + q] = __int_as_float(__float_as_int(x[k0 + q]) ^ sgb);
        }
      }
#pragma unroll
      for (int k0 = 0; k0 < RA; k0 += 8) {
        const int e0 = RA * g + k0;
        const int4 h0 = *(const int4*)(sHi + aux_off(e0)), h1 = *(const int4*)(sHi + aux_off(e0 + 4));
        const float4 q0 = *(const float4*)(sCi + aux_off(e0)), q1 = *(const float4*)(sCi + aux_off(e0 + 4));
        const int hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const float cw[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        int ad[8];
        float vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          ad[q] = hv[q] * DT + c;
          vv[q] = (4.f * cw[q]) * x[k0 + q];
        }
        scatter8<MODE>(P, ad, vv);
      }
      fwht<RA>(x);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      nbar(1 + tg, NT);   // tile and identity aux consumed
      if (lt == 0) {
        if (SA) issue_had(b);                 // the Hadamard half of THIS block into the same buffers
        else if (bn < bend) issue_id(bn);
      }
#pragma unroll
      for (int k = 0; k < RA; ++k) tile[xswz<LA, G>(RA * g + k) * DT + c] = x[k];
    }
    nbar(1 + tg, NT);
    // ---------------- phase B: rows g' + RA k (strided); Hadamard half scattered
    float y[NB][RB];
#pragma unroll
    for (int gi = 0; gi < NB; ++gi) {
      const int gp = lt / DT + (NT / DT) * gi;
#pragma unroll
      for (int k = 0; k < RB; ++k) y[gi][k] = tile[xswz<LA, G>(gp + RA * k) * DT + c];
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    nbar(1 + tg, NT);   // the tile buffer is free: prefetch the next block
    if (lt == 0 && bn < bend) issue_tile(bn);
    mb_wait(&bar_h[tg], phase);
    phase ^= 1u;
#pragma unroll
    for (int gi = 0; gi < NB; ++gi) {
      const int gp = lt / DT + (NT / DT) * gi;
      fwht<RB>(y[gi]);
#pragma unroll
      for (int k0 = 0; k0 < RB; k0 += 8) {
        int ad[8];
        float vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = gp + RA * (k0 + q);
          ad[q] = sHh[aux_off(e)] * DT + c;
          vv[q] = (sc_h * sCh[aux_off(e)]) * y[gi][k0 + q];
        }
        scatter8<MODE>(P, ad, vv);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    nbar(1 + tg, NT);   // the Hadamard aux is free
    if (lt == 0 && bn < bend) {
      if (SA) issue_id(bn);
      else issue_had(bn);
    }
  }
  }   // segments
  __syncthreads();
  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) {
    const int h = e / DT, cc = e - h * DT;
    const float v = P[e];
    if (c0 + cc < d && v != 0.f) atomicAdd(&W[(size_t)h * d + c0 + cc], (double)v);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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

template <int LA, int LB, int DT, int TL, bool SA = false>
size_t v5_smem(int r1) {
  using Gm = Geo5<LA, LB, DT, TL, SA>;
  return (size_t)TL * Gm::group_bytes + (size_t)r1 * DT * sizeof(float);
}

template <int LA, int LB, int DT, int TL, int MODE, bool SA = false>
fct_status launch_v5(const float* A, int64_t nfull, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                     const int32_t* hash, int s, int r1, double* W, int* pace, cudaStream_t st) {
  using Gm = Geo5<LA, LB, DT, TL, SA>;
  auto enc = encoder();
  FCT_CHECK_ARG(enc, FCT_ERR_CUDA, "fct_sketch: cuTensorMapEncodeTiled unavailable");
  const int64_t nblocks = nfull / s;
  // A as [block][k][g][c] viewed through dims (c, g, k, block): row = block S + RA g + k
  CUtensorMap mA, mC, mH;
  {
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)Gm::NG, (cuuint64_t)Gm::RA, (cuuint64_t)nblocks};
    cuuint64_t strides[3] = {(cuuint64_t)Gm::RA * lda * 4, (cuuint64_t)lda * 4, (cuuint64_t)s * lda * 4};
    cuuint32_t box[4] = {(cuuint32_t)DT, (cuuint32_t)Gm::NG, (cuuint32_t)Gm::RA, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult cr = enc(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)A, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return FCT_ERR_UNSUPPORTED;
  }
  for (int which = 0; which < 2; ++which) {   // C and B as rows of 32 entries, SWIZZLE_128B
    cuuint64_t dims[2] = {32, (cuuint64_t)(2 * nfull / 32)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)(s / 32)};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(which ? &mH : &mC, which ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      which ? (void*)hash : (void*)cauchy, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return FCT_ERR_UNSUPPORTED;
  }
  const int nslices = (int)((d + DT - 1) / DT);
  const size_t smem = v5_smem<LA, LB, DT, TL, SA>(r1);
  auto kern = sketch_v5_kernel<LA, LB, DT, TL, MODE, SA>;
  int pace_every = 16;   // measured: DRAM reads 34.0 -> 22.9 GB at 8 (cfg 4), time within 1 %
  if (const char* e = getenv("FCT_SKETCH_PACE")) pace_every = atoi(e);   // 0: no pacing
  if (pace_every <= 0) pace = nullptr;
  // (pacing also requires the whole grid to be resident: one CTA per SM, grid <= #SMs; checked below)
  if (pace) FCT_CUDA_RET(cudaMemsetAsync(pace, 0, sizeof(int) * 1024, st));
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // an equal number of CTAs per column slice (the slices then walk the row blocks in lockstep, so each line of A
  // is read from DRAM once), keeping <= ~2048 expected terms per bucket per CTA partial
  int64_t ngrp = (int64_t)fct::num_sms() / nslices;
  const int64_t min_grp = (2 * nblocks * (int64_t)s + 2048LL * r1 - 1) / (2048LL * r1);
  ngrp = std::max<int64_t>(std::max<int64_t>(ngrp, 1), min_grp);
  // One wave leaves SMs idle when neither the groups nor the extra CTAs below fill them (cfg 5: 25 slices, 5 groups
  // + 5 extra CTAs = 130 of 148 SMs), and min_grp can force several waves (cfg 5 at 2^26 rows and more). Then run
  // several waves of one CTA per SM, unpaced, with the smallest group count >= max(min_grp, 4 waves' worth) whose
  // last wave is >= 98 % full. Measured (tools/ngrp_sweep.sh, profiles/r02_sketch_ngrp_sweep.jsonl): cfg-5 shard
  // 2^25 rows 11.75 -> 10.18 ms, cfg 5 2^28 rows 87.7 -> 81.6 ms; cfg 4 (one full wave) 9.18 vs 9.13-9.22 ms.
  {
    const int64_t nsm = fct::num_sms();
    int64_t left = nsm - ngrp * nslices, ne = left;
    while (ne > 0 && nslices % ne) --ne;
    const bool one_wave_full = left >= 0 && (ngrp * nslices + ne) * 100 >= nsm * 95;
    if (!one_wave_full && !getenv("FCT_SKETCH_ONEWAVE")) {
      int64_t g = std::max<int64_t>(min_grp, (4 * nsm + nslices - 1) / nslices);
      for (int64_t t = g; t < g + 2 * nsm; ++t) {
        const int64_t ctas = t * nslices, waves = (ctas + nsm - 1) / nsm;
        if (ctas * 100 >= waves * nsm * 98) { g = t; break; }
      }
      ngrp = g;
    }
  }
  if (const char* e = getenv("FCT_SKETCH_NGRP")) ngrp = std::max<int64_t>(min_grp, atoll(e));   // sweep override
  ngrp = std::min<int64_t>(ngrp, (nblocks + TL - 1) / TL);
  if (ngrp < 1) ngrp = 1;
  if (ngrp * nslices > fct::num_sms()) pace = nullptr;
  // SMs left over by the groups (cfg 4: 148 - 18 x 8 = 4) take a tail of the blocks in nslices / nextra passes;
  // the tail is sized so that an extra CTA does as many block-slices as a group CTA (FCT_SKETCH_NOEXTRA=1: off)
  // (nextra = the largest divisor of nslices that the leftover SMs hold: cfg 5 has 148 - 5 x 25 = 23 left, uses 5)
  int nextra = (int)(fct::num_sms() - ngrp * nslices);
  while (nextra > 0 && nslices % nextra) --nextra;
  int64_t nmain = nblocks;
  if (nextra > 0 && pace && !getenv("FCT_SKETCH_NOEXTRA")) {
    const int64_t passes = nslices / nextra;
    const int64_t tail = nblocks / (1 + passes * ngrp);
    if (tail >= 4 * TL) nmain = nblocks - tail;
  }
  if (nmain == nblocks) nextra = 0;
  kern<<<(unsigned)(ngrp * nslices + nextra), Gm::THREADS, smem, st>>>(mA, mC, mH, signs, r1, (int)d, nslices, nblocks,
                                                                       (float)(1.0 / sqrt((double)s)), W, pace, pace_every,
                                                                       nmain, nextra);
  FCT_LAUNCHED("sketch_v5_kernel", st);
  fct::set_instance(0, "sketch_v5_kernel<%d, %d, %d, %d, %d, %d>", LA, LB, DT, TL, MODE, SA ? 1 : 0);   // ncu's spelling
  return FCT_OK;
}

constexpr size_t kV5Smem = 232448 - 1024;   // shared memory per block on sm_100a, less the 1-KB-aligned static part

}  // namespace

// Full s-blocks of A (n / s of them) through v5; returns FCT_ERR_UNSUPPORTED (nothing enqueued) when no instance
// covers (s, d, r1, alignment).  *rows_done = the rows handled (the caller sketches the tail).
fct_status fct_sketch_v5(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                         const int32_t* hash, int s, int r1, int mode, double* W, int* pace, int64_t* rows_done,
                         cudaStream_t st) {
  *rows_done = 0;
  const int64_t nfull = n / s * s;
  if (getenv("FCT_SKETCH_V1") || nfull == 0 || ((uintptr_t)A & 15) || ((uintptr_t)cauchy & 15) ||
      ((uintptr_t)hash & 15) || ((uintptr_t)signs & 15) || (lda % 4) || nfull >= (1LL << 31) || s < 256)
    return FCT_ERR_UNSUPPORTED;
  fct_status rc = FCT_ERR_UNSUPPORTED;
#define TRY5(LA_, LB_, DT_, TL_)                                                                              \
  if (rc == FCT_ERR_UNSUPPORTED && s == (1 << (LA_ + LB_)) && v5_smem<LA_, LB_, DT_, TL_>(r1) <= kV5Smem &&    \
      (DT_ <= 8 || d >= DT_))                                                                                  \
    rc = mode == 0 ? launch_v5<LA_, LB_, DT_, TL_, 0>(A, nfull, d, lda, signs, cauchy, hash, s, r1, W, pace, st)      \
                   : launch_v5<LA_, LB_, DT_, TL_, 1>(A, nfull, d, lda, signs, cauchy, hash, s, r1, W, pace, st);
  if (rc == FCT_ERR_UNSUPPORTED && s == 2048 && v5_smem<6, 5, 8, 2>(r1) > kV5Smem && v5_smem<6, 5, 4, 2>(r1) > kV5Smem &&
      v5_smem<6, 5, 4, 2, true>(r1) <= kV5Smem && !getenv("FCT_SKETCH_NOSA"))   // cfg-5 geometry: two tile groups
    rc = mode == 0 ? launch_v5<6, 5, 4, 2, 0, true>(A, nfull, d, lda, signs, cauchy, hash, s, r1, W, pace, st)
                   : launch_v5<6, 5, 4, 2, 1, true>(A, nfull, d, lda, signs, cauchy, hash, s, r1, W, pace, st);
  TRY5(6, 5, 8, 2) TRY5(6, 5, 4, 2) TRY5(6, 5, 4, 1)     // s = 2048
  TRY5(5, 5, 16, 2) TRY5(5, 5, 16, 1) TRY5(5, 5, 8, 2) TRY5(5, 5, 4, 2)    // s = 1024
  TRY5(4, 4, 16, 2) TRY5(4, 4, 8, 4) TRY5(4, 4, 4, 8)                      // s = 256
#undef TRY5
  if (rc == FCT_OK) *rows_done = nfull;
  return rc;
}
