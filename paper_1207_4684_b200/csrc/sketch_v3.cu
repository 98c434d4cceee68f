// sketch_v3.cu -- K1 v3: FCT1 sketch Y = 4 B C H~ D A (Sec. 3.1, FCT1 construction P:L2221-2294)
// with the phases of the block Walsh-Hadamard transform swapped relative to v1, to cut the per-element
// instruction count and the shared-memory wavefronts spent on the per-row auxiliary data:
//
//   phase 1 (contiguous rows): thread (c, g') holds rows RB g' + k, k < RB, of column c, read from a
//           tile stored as S/RB padded row groups (16-byte cp.async copies with zero fill past n; PAD = DT
//           floats between groups makes the column reads conflict-free -- TMA destinations must be
//           128-byte aligned, which rules out the padding).  The identity half of G_s = [H_s; I_s] is scattered here:
//           its signs, Cauchy weights and hashes for the thread's RB rows are 16-byte vector loads shared
//           by the row's DT column lanes.  D is applied as a sign-bit XOR, the factor 4 folded into it.
//           Then the butterflies over the low LB row bits, and one XOR-swizzled shared-memory exchange.
//   phase 2 (strided rows g + (S/RA) k): the butterflies over the high LA row bits, then the Hadamard half,
//           scaled by c / sqrt(s), scattered with scalar aux loads (broadcast across the DT column lanes).
// The scatter is the batched shared-memory CAS of v1 (any two threads may hit the same bucket; sm_100 has
// no native shared fp32 atomic add).  Each CTA owns a column slice [c0, c0 + DT) and keeps an fp32
// partial P[r1][DT] for its lifetime, flushed once into the fp64 workspace (same as v1).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include "common.cuh"

namespace {

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(su32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
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
// unnormalised in-register Walsh-Hadamard transform of R values (natural / Sylvester order)
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
        x[k] = s2.x;
        x[k + 1] = s2.y;
        x[k + h] = d2.x;
        x[k + h + 1] = d2.y;
      }
}
// batched exact shared-memory float add: loads, CAS (ATOMS.CAS returns the old word), retry the rare misses
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
struct Geo3 {
  static constexpr int S = 1 << (LA + LB);
  static constexpr int RA = 1 << LA;           // phase-2 registers (strided rows)
  static constexpr int RB = 1 << LB;           // phase-1 registers (contiguous rows)
  static constexpr int NT = S * DT / RB;       // threads per tile group (one phase-1 row group per thread)
  static constexpr int NA = (S / RA) * DT / NT;// phase-2 groups per thread
  static constexpr int TILES = TILES_;
  static constexpr int THREADS = NT * TILES;
  static constexpr int G = 32 / DT;            // rows per warp-instruction
  static constexpr int PADF = DT;              // floats between padded row groups
  static constexpr int GROUPF = RB * DT + PADF;
  static constexpr size_t tile_bytes = (size_t)(S / RB) * GROUPF * sizeof(float);
  static constexpr int id_bytes = 8 * S;       // identity-half Cauchy + hash
  static constexpr int had_bytes = 8 * S;      // Hadamard-half Cauchy + hash
  static constexpr size_t smem_bytes(int r1) { return TILES * (tile_bytes + id_bytes + had_bytes) + (size_t)r1 * DT * 4; }
  static_assert(NT >= 32 && THREADS <= 1024 && NA >= 1 && RB % 8 == 0 && RA >= G && (RB * DT) % 32 == 0, "geometry");
};

// exchange layout: physical row of logical row r (conflict-free phase-1 writes and phase-2 reads)
template <int LB, int G>
__device__ __forceinline__ int swz3(int r) {
  return G > 1 ? (r ^ ((r >> LB) & (G - 1))) : r;
}

template <int LA, int LB, int DT, int TL>
__global__ void __launch_bounds__(Geo3<LA, LB, DT, TL>::THREADS, 1)
sketch_v3_kernel(const float* __restrict__ A, int64_t lda, int64_t n, int d, const int8_t* __restrict__ signs,
                 const float* __restrict__ cauchy, const int32_t* __restrict__ hash, int r1, int nslices,
                 int64_t nblocks, float inv_sqrt_s, double* __restrict__ W) {
  using Gm = Geo3<LA, LB, DT, TL>;
  constexpr int S = Gm::S, RA = Gm::RA, RB = Gm::RB, NT = Gm::NT, NA = Gm::NA, TILES = Gm::TILES, G = Gm::G;
  extern __shared__ __align__(128) unsigned char smraw[];
  // [TILES] padded tiles | [TILES] identity aux (c, h) | [TILES] Hadamard aux (c, h) | P[r1][DT]
  float* tiles = (float*)smraw;
  unsigned char* auxI0 = smraw + TILES * Gm::tile_bytes;
  unsigned char* auxH0 = auxI0 + TILES * Gm::id_bytes;
  float* P = (float*)(auxH0 + TILES * Gm::had_bytes);
  __shared__ __align__(8) uint64_t bar_i[TILES], bar_h[TILES];

  const int cs = blockIdx.x % nslices;
  const int grp = blockIdx.x / nslices;
  const int ngrp = gridDim.x / nslices;
  const int c0 = cs * DT;
  const int tg = threadIdx.x / NT;
  const int lt = threadIdx.x - tg * NT;
  const int c = lt % DT;
  float* tile = tiles + (size_t)tg * (Gm::tile_bytes / 4);
  unsigned char* auxI = auxI0 + tg * Gm::id_bytes;
  unsigned char* auxH = auxH0 + tg * Gm::had_bytes;
  const float* sCi = (const float*)auxI;
  const int* sHi = (const int*)(auxI + 4 * S);
  const float* sCh = (const float*)auxH;
  const int* sHh = (const int*)(auxH + 4 * S);

  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) P[e] = 0.f;
  if (threadIdx.x < TILES) {
    mbar_init(&bar_i[threadIdx.x], 1);
    mbar_init(&bar_h[threadIdx.x], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  // the group's block tile: S rows x DT columns in 16-byte pieces, every thread of the group copies its share
  constexpr int PIECES = S * DT / 4, PPR = DT / 4;   // 16-byte pieces per block / per row
  const int dvalid = d - c0;                          // columns of this slice inside the matrix
  auto issue_tile = [&](int64_t bb) {
#pragma unroll
    for (int q = lt; q < PIECES; q += NT) {
      const int r = q / PPR, h = q - r * PPR;
      const int64_t grow = bb * S + r;
      const bool ok = grow < n && 4 * h < dvalid;
      const float* src = A + (ok ? grow * lda + c0 + 4 * h : 0);
      cp_async16(tile + (size_t)(r / RB) * Gm::GROUPF + (r % RB) * DT + 4 * h, src, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto issue_id = [&](int64_t bb) {
    const int64_t t0 = 2 * bb * S;
    mbar_expect_tx(&bar_i[tg], 8u * S);
    bulk_g2s(auxI, cauchy + t0 + S, 4u * S, &bar_i[tg]);
    bulk_g2s(auxI + 4 * S, hash + t0 + S, 4u * S, &bar_i[tg]);
  };
  auto issue_had = [&](int64_t bb) {
    const int64_t t0 = 2 * bb * S;
    mbar_expect_tx(&bar_h[tg], 8u * S);
    bulk_g2s(auxH, cauchy + t0, 4u * S, &bar_h[tg]);
    bulk_g2s(auxH + 4 * S, hash + t0, 4u * S, &bar_h[tg]);
  };

  const int64_t bstep = (int64_t)ngrp * TILES;
  int64_t b = grp + (int64_t)ngrp * tg;
  if (b < nblocks) {
    issue_tile(b);
    if (lt == 0) {
      issue_id(b);
      issue_had(b);
    }
  }
  unsigned phase = 0;
  const float sc_h = 4.f * inv_sqrt_s;
  const int gp = lt / DT;   // phase-1 row group of this thread
  for (; b < nblocks; b += bstep) {
    const int64_t bn = b + bstep;
    const int64_t rowb = b * S;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    named_bar(1 + tg, NT);   // the group's tile copies are visible
    mbar_wait(&bar_i[tg], phase);
    // ---------------- phase 1: rows RB gp + k (contiguous); identity half
    {
      float x[RB];
      const float* src = tile + (size_t)gp * Gm::GROUPF + c;
#pragma unroll
      for (int k = 0; k < RB; ++k) x[k] = src[k * DT];
      // signs of the RB rows: 16-byte vector loads from global (L1/L2), guarded in the ragged last block
      const int r0 = RB * gp;
      const int64_t grow0 = rowb + r0;
      unsigned sw[RB / 4];
      if (grow0 + RB <= n) {
        if constexpr (RB >= 16) {
#pragma unroll
          for (int q = 0; q < RB / 16; ++q) {
            const uint4 v = __ldg((const uint4*)(signs + grow0) + q);
            sw[4 * q + 0] = v.x; sw[4 * q + 1] = v.y; sw[4 * q + 2] = v.z; sw[4 * q + 3] = v.w;
          }
        } else {
          const uint2 v = __ldg((const uint2*)(signs + grow0));
          sw[0] = v.x; sw[1] = v.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < RB / 4; ++q) {
          unsigned w = 0u;
#pragma unroll
          for (int bq = 0; bq < 4; ++bq) {
            const int64_t gr = grow0 + 4 * q + bq;
            const unsigned sb = gr < n ? (unsigned)(uint8_t)__ldg(signs + gr) : 1u;
            w |= sb << (8 * bq);
          }
          sw[q] = w;
        }
      }
#pragma unroll
      for (int k0 = 0; k0 < RB; k0 += 8) {
        const int4 h0 = *(const int4*)(sHi + r0 + k0), h1 = *(const int4*)(sHi + r0 + k0 + 4);
        const float4 q0 = *(const float4*)(sCi + r0 + k0), q1 = *(const float4*)(sCi + r0 + k0 + 4);
        const int hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const float cw[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        int ad[8];
        float vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int k = k0 + q;
          // D_ii = -1 iff the int8 sign is negative: XOR its top bit into 4.0f and into x
          const unsigned sbit = (sw[k >> 2] << (24 - 8 * (k & 3))) & 0x80000000u;
          x[k] = __uint_as_float(__float_as_uint(x[k]) ^ sbit);
          ad[q] = hv[q] * DT + c;
          vv[q] = (4.f * cw[q]) * x[k];
        }
        smem_add_batch<8>(P, ad, vv);
      }
      fwht_regs<RB>(x);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      named_bar(1 + tg, NT);   // everyone has read the TMA tile and the identity aux
      if (lt == 0 && bn < nblocks) issue_id(bn);
#pragma unroll
      for (int k = 0; k < RB; ++k) tile[swz3<LB, G>(r0 + k) * DT + c] = x[k];
    }
    named_bar(1 + tg, NT);
    // ---------------- phase 2: rows g + (S/RA) k (strided); Hadamard half
    float y[NA][RA];
#pragma unroll
    for (int gi = 0; gi < NA; ++gi) {
      const int g = lt / DT + (NT / DT) * gi;
#pragma unroll
      for (int k = 0; k < RA; ++k) y[gi][k] = tile[swz3<LB, G>(g + (S / RA) * k) * DT + c];
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    named_bar(1 + tg, NT);   // the tile buffer is free: prefetch the next block
    if (bn < nblocks) issue_tile(bn);
    mbar_wait(&bar_h[tg], phase);
    phase ^= 1u;
#pragma unroll
    for (int gi = 0; gi < NA; ++gi) {
      const int g = lt / DT + (NT / DT) * gi;
      fwht_regs<RA>(y[gi]);
#pragma unroll
      for (int k0 = 0; k0 < RA; k0 += 8) {
        int ad[8];
        float vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = g + (S / RA) * (k0 + q);
          ad[q] = sHh[r] * DT + c;
          vv[q] = (sc_h * sCh[r]) * y[gi][k0 + q];
        }
        smem_add_batch<8>(P, ad, vv);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    named_bar(1 + tg, NT);   // the Hadamard aux is free
    if (lt == 0 && bn < nblocks) issue_had(bn);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r1 * DT; e += blockDim.x) {
    const int h = e / DT, cc = e - h * DT;
    const float v = P[e];
    if (c0 + cc < d && v != 0.f) atomicAdd(&W[(size_t)h * d + c0 + cc], (double)v);
  }
}

constexpr size_t kSmem3 = 232448 - 256;

template <int LA, int LB, int DT, int TL>
fct_status launch_v3(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                     const int32_t* hash, int s, int r1, double* W, cudaStream_t st) {
  using Gm = Geo3<LA, LB, DT, TL>;
  const int nslices = (int)((d + DT - 1) / DT);
  const int64_t nblocks = (n + s - 1) / s;
  const size_t smem = Gm::smem_bytes(r1);
  auto kern = sketch_v3_kernel<LA, LB, DT, TL>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  FCT_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Gm::THREADS, smem));
  if (occ < 1) occ = 1;
  int64_t ngrp = ((int64_t)fct::num_sms() * occ) / nslices;
  const int64_t min_grp = (2 * nblocks * (int64_t)s + 2048LL * r1 - 1) / (2048LL * r1);
  ngrp = std::max<int64_t>(std::max<int64_t>(ngrp, 1), min_grp);
  ngrp = std::min<int64_t>(ngrp, (nblocks + Gm::TILES - 1) / Gm::TILES);
  if (ngrp < 1) ngrp = 1;
  kern<<<(unsigned)(ngrp * nslices), Gm::THREADS, smem, st>>>(A, lda, n, (int)d, signs, cauchy, hash, r1, nslices,
                                                               nblocks, (float)(1.0 / sqrt((double)s)), W);
  FCT_LAUNCHED("sketch_v3_kernel", st);
  return FCT_OK;
}

template <int LA, int LB, int DT, int TL>
bool fits3(int r1) {
  return Geo3<LA, LB, DT, TL>::smem_bytes(r1) <= kSmem3;
}

}  // namespace

// Returns FCT_ERR_UNSUPPORTED (without enqueueing) when no v3 instance covers (s, d, r1, alignment).
fct_status fct_sketch_v3(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                         const int32_t* hash, int s, int r1, double* W, cudaStream_t st) {
  // opt-in (FCT_SKETCH_V3=1): measured 13.4 ms vs v1's 12.7 ms at cfg 4 (12.4 vs 13.0 ms at cfg 5 shapes)
  if (!getenv("FCT_SKETCH_V3")) return FCT_ERR_UNSUPPORTED;
  if (((uintptr_t)A & 15) || ((uintptr_t)cauchy & 15) || ((uintptr_t)hash & 15) || ((uintptr_t)signs & 15) ||
      (lda % 4) || (d % 4) || n >= (1LL << 31))
    return FCT_ERR_UNSUPPORTED;
#define TRY3(LA_, LB_, DT_, TL_)                                                          \
  if (s == (1 << (LA_ + LB_)) && fits3<LA_, LB_, DT_, TL_>(r1) && (DT_ <= 8 || d >= DT_)) \
    return launch_v3<LA_, LB_, DT_, TL_>(A, n, d, lda, signs, cauchy, hash, s, r1, W, st);
  TRY3(5, 6, 16, 1) TRY3(5, 6, 8, 2) TRY3(5, 6, 4, 2) TRY3(5, 6, 4, 1)   // s = 2048
  TRY3(5, 5, 16, 1) TRY3(5, 5, 8, 2) TRY3(5, 5, 4, 4) TRY3(5, 5, 4, 2)   // s = 1024
  TRY3(4, 4, 16, 2) TRY3(4, 4, 8, 4) TRY3(4, 4, 4, 8)                    // s = 256
  TRY3(3, 3, 8, 8) TRY3(3, 3, 4, 8)                                      // s = 64
#undef TRY3
  return FCT_ERR_UNSUPPORTED;
}
