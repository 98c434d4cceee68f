// lat.cu -- dependent-chain latencies on sm_100a (one warp): DFMA, DMUL, fp64 rsqrt(), fp64 division, FFMA,
// float rsqrtf, LDS round trip, __syncthreads with 256 threads.  Prints cycles per link of each chain.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, float* outf, long long* cyc, int n) {
  __shared__ double sh[256];
  const int t = threadIdx.x;
  sh[t] = 1.0 + t * 1e-9;
  __syncthreads();
  double x = 1.0 + t * 1e-12, y = 0.999999;
  float xf = 1.0f + t * 1e-7f;
  long long c0, c1;
  // DFMA chain
  c0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  c1 = clock64();
  if (t == 0) cyc[0] = c1 - c0;
  // DMUL chain
  c0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  c1 = clock64();
  if (t == 0) cyc[1] = c1 - c0;
  // rsqrt(double) chain
  double z = x + 2.0;
  c0 = clock64();
  for (int i = 0; i < n; ++i) z = rsqrt(z) + 1.5;
  c1 = clock64();
  if (t == 0) cyc[2] = c1 - c0;
  // division chain
  double w = x + 3.0;
  c0 = clock64();
  for (int i = 0; i < n; ++i) w = 1.0 / w + 1.25;
  c1 = clock64();
  if (t == 0) cyc[3] = c1 - c0;
  // FFMA chain
  c0 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, 0.9999f, 1e-7f);
  c1 = clock64();
  if (t == 0) cyc[4] = c1 - c0;
  // LDS chain (pointer chase through shared memory)
  int idx = t;
  int* shi = (int*)sh;
  __syncthreads();
  for (int e = t; e < 512; e += blockDim.x) shi[e] = (e + 1) & 255;
  __syncthreads();
  c0 = clock64();
  for (int i = 0; i < n; ++i) idx = shi[idx];
  c1 = clock64();
  if (t == 0) cyc[5] = c1 - c0;
  // __syncthreads chain
  c0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  c1 = clock64();
  if (t == 0) cyc[6] = c1 - c0;
  // F2F.F64.F32 + DADD chain
  double v = x;
  c0 = clock64();
  for (int i = 0; i < n; ++i) v = (double)(float)v + 1e-3;
  c1 = clock64();
  if (t == 0) cyc[7] = c1 - c0;
  // SHFL (double) + DFMA chain
  double q = x;
  c0 = clock64();
  for (int i = 0; i < n; ++i) q = fma(__shfl_sync(0xffffffffu, q, i & 31), 0.999, 1e-3);
  c1 = clock64();
  if (t == 0) cyc[8] = c1 - c0;
  // LDS.64 + DFMA chain (address depends on the previous value's low bit)
  double q2 = x;
  c0 = clock64();
  for (int i = 0; i < n; ++i) q2 = fma(sh[(t + i + (int)(q2 > 5.0)) & 255], 0.999, q2 * 1e-3);
  c1 = clock64();
  if (t == 0) cyc[9] = c1 - c0;
  out[t] = x + z + w + v + idx + q + q2;
  outf[t] = xf;
}

int main() {
  double* o;
  float* of;
  long long* c;
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&of, 256 * 4);
  cudaMalloc(&c, 16 * 8);
  const int n = 4096;
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(o, of, c, n);
    cudaDeviceSynchronize();
    long long h[10];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[10] = {"DFMA", "DMUL", "rsqrt(double)+DADD", "1/x double + DADD", "FFMA", "LDS chase", "__syncthreads",
                          "F2F.F32.F64 + F2F.F64.F32 + DADD", "SHFL(double) + DFMA", "LDS.64 + DFMA"};
    for (int i = 0; i < 10; ++i) printf("threads %3d  %-36s %7.1f cycles per link\n", nt, nm[i], (double)h[i] / n);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
