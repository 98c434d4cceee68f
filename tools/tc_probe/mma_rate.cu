// mma_rate.cu -- issue/throughput of tcgen05.mma streams on sm_100a (cycles per instruction), for the
// shapes the row-norm contraction can use: kind::tf32 M=128, N in {32..256}, K=8; A from shared memory (SS)
// or TMEM (TS); kind::f16 (bf16) K=16.  Variants: descriptor start offset inside the 128-B swizzle atom,
// number of issuing warps.  Operands are uninitialised (timing only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(const void* p) {
  const uint64_t a = (su32(p) >> 4) & 0x3FFF;
  return a | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// MODE 0 = tf32 SS, 1 = tf32 TS, 2 = bf16 SS.  OFFS: step the K offset inside the swizzle atom per MMA.
template <int MODE, int N, bool OFFS>
__global__ void __launch_bounds__(128) mma_rate(int iters, int nwarps, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 4) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[tid])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (warp < nwarps && lane == 0) {
    constexpr uint32_t fmt = MODE == 2 ? 1u : 2u;
    constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = sdesc(base + warp * 16384), bd = sdesc(base + 65536 + warp * 16384);
    const uint32_t tD = tm + 128 + (uint32_t)(warp * (N < 96 ? N : 96));
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = OFFS ? (uint64_t)((i & 3) * 2) : 0;
      if (MODE == 1)
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n" ::"r"(tD),
                     "r"(tm + (uint32_t)(OFFS ? (i & 3) * 8 : 0)), "l"(bd + off), "r"(idesc));
      else if (MODE == 0)
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(tD), "l"(ad + off), "l"(bd + off),
                     "r"(idesc));
      else
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(tD), "l"(ad + off), "l"(bd + off),
                     "r"(idesc));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar[warp])) : "memory");
    long long t2 = clock64();
    if (warp == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

long long* d_out;
template <int MODE, int N, bool OFFS>
void run(int nwarps) {
  const int smem = 65536 + 65536 + 1024, iters = 4096;
  auto k = mma_rate<MODE, N, OFFS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, 128, smem>>>(iters, nwarps, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[3] = {"tf32 SS", "tf32 TS", "bf16 SS"};
  const double macs = 128.0 * N * (MODE == 2 ? 16 : 8) * nwarps;
  printf("%s N=%3d offs=%d warps=%d: issue %.1f cyc/mma/warp, complete %.1f (%.0f MAC/cyc/SM)\n", names[MODE], N, (int)OFFS,
         nwarps, (double)h[0] / iters, (double)h[1] / iters, macs * iters / h[1]);
}

int main() {
  cudaMalloc(&d_out, 148 * 2 * sizeof(long long));
  run<0, 32, false>(1); run<0, 32, true>(1); run<0, 32, false>(2); run<0, 32, false>(4);
  run<0, 64, false>(1); run<0, 128, false>(1); run<0, 256, false>(1);
  run<1, 32, false>(1); run<1, 32, true>(1); run<1, 32, false>(2);
  run<2, 32, false>(1); run<2, 256, false>(1); run<2, 256, false>(2);
  return 0;
}
