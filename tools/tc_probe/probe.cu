// probe.cu -- standalone check of the tcgen05 3xTF32 contraction used by the row-norm kernel:
// one 128-row tile of A (d = 64) TMA-loaded with SWIZZLE_128B, A_lo = A - trunc_tf32(A) written to
// TMEM, D = A*Mhi + A*Mlo + A_lo*Mhi accumulated in TMEM (M = 128, N = 32, K = 8 per instruction),
// read back with tcgen05.ld and compared with a CPU fp64 product.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int D = 64, N = 32, MT = 128;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(const void* p, int sbo_bytes) {
  uint64_t a = (su32(p) >> 4) & 0x3FFF;
  return a | (1ull << 16) | ((uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ float trunc_tf32(float x) { return __int_as_float(__float_as_int(x) & 0xFFFFE000); }

__global__ void __launch_bounds__(128) probe_kernel(const __grid_constant__ CUtensorMap tmA, const float* __restrict__ Mt,
                                                    float* __restrict__ Dout, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)base;                  // 2 chunks x 128 rows x 128 B = 32 KB
  float* sMhi = (float*)(base + 32768);      // 2 chunks x 32 rows x 128 B = 8 KB
  float* sMlo = (float*)(base + 32768 + 8192);
  __shared__ __align__(8) uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_tma)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Mt: N x D (row j = column j of M), split into hi/lo and stored K-major SW128
  for (int e = tid; e < N * D; e += blockDim.x) {
    const int j = e / D, l = e % D;
    const float m = Mt[e];
    const float hi = trunc_tf32(m), lo = m - hi;
    const int q = l / 32, c = (l % 32) / 4, w = l % 4;
    const int off = q * (32 * 32) + j * 32 + ((c ^ (j & 7)) * 4) + w;  // in floats
    sMhi[off] = hi;
    sMlo[off] = lo;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar_tma)), "r"(32768));
    for (int q = 0; q < 2; ++q)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sA + q * 128 * 32)), "l"(&tmA), "r"(q * 32), "r"(0), "r"(su32(&bar_tma)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}\n" ::"r"(su32(&bar_tma)) : "memory");
  // split: thread = row; A_lo to TMEM columns [0, 64) of lane = row
  {
    const int r = tid;
    uint32_t lo[64];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 v = *(const float4*)(sA + q * 128 * 32 + r * 32 + ((c ^ (r & 7)) * 4));
        const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) lo[q * 32 + c * 4 + w] = __float_as_uint(a[w] - trunc_tf32(a[w]));
      }
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]), "r"(lo[8]),
        "r"(lo[9]), "r"(lo[10]), "r"(lo[11]), "r"(lo[12]), "r"(lo[13]), "r"(lo[14]), "r"(lo[15]), "r"(lo[16]),
        "r"(lo[17]), "r"(lo[18]), "r"(lo[19]), "r"(lo[20]), "r"(lo[21]), "r"(lo[22]), "r"(lo[23]), "r"(lo[24]),
        "r"(lo[25]), "r"(lo[26]), "r"(lo[27]), "r"(lo[28]), "r"(lo[29]), "r"(lo[30]), "r"(lo[31]));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + 32),
        "r"(lo[32]), "r"(lo[33]), "r"(lo[34]), "r"(lo[35]), "r"(lo[36]), "r"(lo[37]), "r"(lo[38]), "r"(lo[39]),
        "r"(lo[40]), "r"(lo[41]), "r"(lo[42]), "r"(lo[43]), "r"(lo[44]), "r"(lo[45]), "r"(lo[46]), "r"(lo[47]),
        "r"(lo[48]), "r"(lo[49]), "r"(lo[50]), "r"(lo[51]), "r"(lo[52]), "r"(lo[53]), "r"(lo[54]), "r"(lo[55]),
        "r"(lo[56]), "r"(lo[57]), "r"(lo[58]), "r"(lo[59]), "r"(lo[60]), "r"(lo[61]), "r"(lo[62]), "r"(lo[63]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tD = tm + 64;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(MT >> 4) << 24);
    int cnt = 0;
    for (int pass = 0; pass < 3; ++pass) {
      if (mode == 1 && pass > 0) break;
      for (int ks = 0; ks < D / 8; ++ks) {
        const int q = ks / 4, kin = ks % 4;    // 128-B chunk, 32-B step inside it
        const float* Bm = (pass == 1) ? sMlo : sMhi;
        const uint64_t bdesc = sdesc((const unsigned char*)(Bm + q * 32 * 32) + kin * 32, 1024);
        const uint32_t acc = cnt > 0 ? 1u : 0u;
        if (pass < 2) {
          const uint64_t adesc = sdesc((const unsigned char*)(sA + q * 128 * 32) + kin * 32, 1024);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tD), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
        } else {
          const uint32_t ta = tm + ks * 8;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tD), "r"(ta), "l"(bdesc), "r"(idesc), "r"(acc));
        }
        ++cnt;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar_mma)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(su32(&bar_mma)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tD + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 32; ++j) Dout[tid * 32 + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
  std::vector<float> A(MT * D), Mt(N * D);
  srand(1);
  for (auto& x : A) x = (float)((rand() / (double)RAND_MAX) * 2 - 1) * (1 + rand() % 3);
  for (auto& x : Mt) x = (float)tan(M_PI * ((rand() + 0.5) / ((double)RAND_MAX + 1) - 0.5));
  float *dA, *dM, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dM, Mt.size() * 4));
  CK(cudaMalloc(&dD, MT * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dM, Mt.data(), Mt.size() * 4, cudaMemcpyHostToDevice));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  CUtensorMap map;
  cuuint64_t dims[2] = {D, MT};
  cuuint64_t str[1] = {D * 4};
  cuuint32_t box[2] = {32, MT};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es,
                                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024));
  for (int mode = 0; mode < 2; ++mode) {
    CK(cudaMemset(dD, 0, MT * N * 4));
    probe_kernel<<<1, 128, 60 * 1024>>>(map, dM, dD, mode);
    CK(cudaDeviceSynchronize());
    std::vector<float> Dh(MT * N);
    CK(cudaMemcpy(Dh.data(), dD, Dh.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0, maxabs_rel_mag = 0;
    for (int i = 0; i < MT; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0, mag = 0;
        for (int l = 0; l < D; ++l) { s += (double)A[i * D + l] * Mt[j * D + l]; mag += fabs((double)A[i * D + l] * Mt[j * D + l]); }
        const double err = fabs(Dh[i * N + j] - s);
        maxabs_rel_mag = fmax(maxabs_rel_mag, err / mag);
        if (i < 2 && j < 3) printf("  D[%d][%d] gpu %.8g ref %.8g\n", i, j, Dh[i * N + j], s);
      }
    printf("mode %d (%s): max |err| / sum|a m| = %.3e\n", mode, mode ? "tf32 only" : "3xTF32", maxabs_rel_mag);
  }
  return 0;
}
