// Microbenchmark 2: vector-width shared scatter-add variants (CAS.128, CAS.64 spin, racy RMW.128)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t mix(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

__device__ __forceinline__ void cas128_add(uint32_t a, float4 v){
  float4 old;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(old.x),"=f"(old.y),"=f"(old.z),"=f"(old.w) : "r"(a) : "memory");
  while (true) {
    float4 nw = make_float4(old.x+v.x, old.y+v.y, old.z+v.z, old.w+v.w);
    unsigned long long e0 = __double_as_longlong(*(double*)&old.x), e1 = *(unsigned long long*)&old.z;
    unsigned long long n0 = *(unsigned long long*)&nw.x, n1 = *(unsigned long long*)&nw.z;
    unsigned long long r0, r1;
    asm volatile("{ .reg .b128 d, e, n;\n mov.b128 e, {%2, %3};\n mov.b128 n, {%4, %5};\n atom.shared.cas.b128 d, [%6], e, n;\n mov.b128 {%0, %1}, d; }"
      : "=l"(r0), "=l"(r1) : "l"(e0), "l"(e1), "l"(n0), "l"(n1), "r"(a) : "memory");
    if (r0==e0 && r1==e1) break;
    *(unsigned long long*)&old.x = r0; *(unsigned long long*)&old.z = r1;
  }
}
__device__ __forceinline__ void cas64_add(uint32_t a, float2 v){
  unsigned long long old;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(old) : "r"(a) : "memory");
  while (true) {
    float2 o = *(float2*)&old; float2 nw = make_float2(o.x+v.x, o.y+v.y);
    unsigned long long n = *(unsigned long long*)&nw, r;
    asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(r) : "r"(a), "l"(old), "l"(n) : "memory");
    if (r==old) break; old = r;
  }
}

// MODE 0: CAS.128 (VW=4); 1: CAS.64 (VW=2); 2: racy RMW .v4 ; 3: racy RMW scalar
template<int MODE, int COLS, int VW>
__global__ void __launch_bounds__(512) scatter_bench(float* out, int iters, int r1){
  extern __shared__ float tab[];
  const int nfl = r1*COLS;
  for (int i=threadIdx.x;i<nfl;i+=blockDim.x) tab[i]=0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  constexpr int LPR = COLS/VW;              // lanes per row
  const int col = (lane % LPR)*VW;
  uint32_t st = mix(threadIdx.x/LPR*7919u + blockIdx.x*104729u);
  float v = 1.0f + lane;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  for (int it=0; it<iters; ++it){
    #pragma unroll 4
    for (int u=0; u<8; ++u){
      st = st*1664525u + 1013904223u;
      uint32_t h = (st >> 8) & (r1-1);
      uint32_t a = base + (h*COLS + col)*4;
      if (MODE==0) cas128_add(a, make_float4(v,v,v,v));
      else if (MODE==1) cas64_add(a, make_float2(v,v));
      else if (MODE==2) { float4 o; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(o.x),"=f"(o.y),"=f"(o.z),"=f"(o.w) : "r"(a) : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" :: "r"(a), "f"(o.x+v),"f"(o.y+v),"f"(o.z+v),"f"(o.w+v) : "memory"); }
      else { float o; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(a) : "memory");
        asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(o+v) : "memory"); }
    }
  }
  __syncthreads();
  float s=0; for (int i=threadIdx.x;i<nfl;i+=blockDim.x) s+=tab[i];
  if (s==12345.f) out[0]=s;
}

template<class K, class... Args>
float timeit(K k, dim3 g, dim3 b, size_t smem, Args... args){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<g,b,smem>>>(args...);
  cudaEventRecord(e0);
  for(int r=0;r<3;r++) k<<<g,b,smem>>>(args...);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1); return ms/3;
}
int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; CK(cudaMalloc(&out, 1024));
  const int iters = 1000;
  #define RUN(MODE, COLS, VW, R1, NT) { auto k = scatter_bench<MODE,COLS,VW>; size_t sm=(size_t)(R1)*(COLS)*4; \
     CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
     float ms = timeit(k, dim3(nsm), dim3(NT), sm, out, iters, R1); CK(cudaGetLastError()); \
     double upd = (double)nsm*NT*iters*8*VW; \
     printf("mode=%d cols=%d vw=%d r1=%d nt=%d: %.3f ms, %.2f updates/clk/SM\n", MODE, COLS, VW, R1, NT, ms, upd/(ms*1e-3)/nsm/(clk*1e3)); }
  RUN(0,8,4,4096,512) RUN(0,8,4,4096,256) RUN(1,8,2,4096,512) RUN(2,8,4,4096,512) RUN(3,8,1,4096,512)
  RUN(0,4,4,8192,512) RUN(1,4,2,8192,512) RUN(2,4,4,8192,512)
  RUN(0,32,4,1024,512) RUN(2,32,4,1024,512) RUN(3,32,1,1024,512)
  RUN(0,16,4,2048,512) RUN(2,16,4,2048,512)
  return 0;
}
