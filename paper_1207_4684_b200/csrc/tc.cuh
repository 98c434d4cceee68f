// tc.cuh -- small sm_100a building blocks shared by the tcgen05 kernels: shared-memory addresses,
// UMMA shared-memory descriptors (K-major, SWIZZLE_128B), mbarriers, TMA tile loads, TMEM ld/st.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace tcx {

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_128B canonical layout: 8-row x 128-B atoms, stride byte offset 1024 B
__device__ __forceinline__ uint64_t sdesc_sw128(const void* p) {
  const uint64_t a = (su32(p) >> 4) & 0x3FFF;
  return a | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ float trunc_tf32(float x) { return __int_as_float(__float_as_int(x) & 0xFFFFE000); }

__device__ __forceinline__ void bar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// blocking wait on the phase with parity `ph`
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nBW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra BW_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
// the same for warps that may wait long (consumers of a slower stage): the suspend-time hint lets the
// hardware park the warp until the phase completes instead of re-issuing try_wait, which would steal
// issue slots from the producer warps sharing the SM sub-partition
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, unsigned ph, unsigned hint_ns) {
  asm volatile(
      "{\n.reg .pred p;\nBS_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra BS_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph), "r"(hint_ns)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
// 128-row x (32*nchunk) fp32 tile, one 128-B-wide box per 32-column chunk (SWIZZLE_128B)
__device__ __forceinline__ void tma_tile(float* dst, const CUtensorMap* map, int nchunk, int row0, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(nchunk * 16384) : "memory");
  for (int q = 0; q < nchunk; ++q)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst + q * 128 * 32)),
        "l"(map), "r"(q * 32), "r"(row0), "r"(su32(bar))
        : "memory");
}
// element l of row r in a SWIZZLE_128B tile of 128 rows (32-float chunks)
__device__ __forceinline__ int sw_off(int r, int l) {
  return (l >> 5) * 128 * 32 + r * 32 + ((((l & 31) >> 2) ^ (r & 7)) << 2) + (l & 3);
}

#define TCX_R32 \
  "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32}"
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " TCX_R32 ";" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]),
               "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
               "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
               "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// D(tmem) [+]= A(smem desc) * B(smem desc), kind::tf32
__device__ __forceinline__ void mma_tf32_ss(uint32_t tD, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                   tD),
               "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
// D(tmem) [+]= A(tmem) * B(smem desc), kind::tf32
__device__ __forceinline__ void mma_tf32_ts(uint32_t tD, uint32_t ta, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                   tD),
               "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
}

}  // namespace tcx
