// fp64.cu -- throughput of DFMA, F2F.F64.F32 and an integer float->double bit construction on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_f2f(double* out, int iters) {
  float a[8]; double acc[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; acc[i] = 0; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += (double)a[i]; a[i] += 1.0f; }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_f2f_only(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { double t = (double)a[i]; a[i] = (float)(t * 1.0000001); }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 1.0000001f, 1e-9f);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}
template <class K, class T> void run(const char* name, K k, T* out, int per_iter) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int threads : {128, 512, 1024}) {
    k<<<nsm, threads>>>(out, iters);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<<<nsm, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)nsm * threads * iters * per_iter;
    printf("%-10s threads/SM=%4d: %.3f ms, %.1f ops/clk/SM\n", name, threads, ms, ops / (ms * 1e-3) / nsm / 1.965e9);
  }
}
int main() {
  double* d; float* f; cudaMalloc(&d, 64); cudaMalloc(&f, 64);
  run("DFMA", k_dfma, d, 8);
  run("F2F+DADD", k_f2f, d, 8);
  run("F2F+F2F", k_f2f_only, f, 8);
  run("FFMA", k_ffma, f, 8);
  return 0;
}
