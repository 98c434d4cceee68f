// common.cuh -- shared helpers of libfct.so (error plumbing, workspace carving, launch checks).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <algorithm>
#include <stdlib.h>

#include "../../include/fct.h"

namespace fct {

// thread-local last-error message (fct_last_error)
void set_error(const char* fmt, ...);
const char* get_error();
bool debug_sync();  // FCT_DEBUG=1
void count_launch();
// record the template instance a hot-path stage launched (slot 0: sketch, 1: row norms)
void set_instance(int slot, const char* fmt, ...);

#define FCT_CHECK_ARG(cond, code, ...)          \
  do {                                          \
    if (!(cond)) {                              \
      ::fct::set_error(__VA_ARGS__);            \
      return (code);                            \
    }                                           \
  } while (0)

#define FCT_CUDA_RET(expr)                                                                  \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::fct::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return FCT_ERR_CUDA;                                                                  \
    }                                                                                       \
  } while (0)

// after a launch: catch configuration errors; in debug mode also synchronise
inline fct_status post_launch(const char* what, cudaStream_t st) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && debug_sync()) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FCT_ERR_CUDA;
  }
  return FCT_OK;
}
#define FCT_LAUNCHED(what, st)                     \
  do {                                             \
    fct_status s_ = ::fct::post_launch(what, st);  \
    if (s_ != FCT_OK) return s_;                   \
  } while (0)

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// sequential carving of a caller workspace into 256-byte aligned pieces
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* p) : base((char*)p) {}
  template <class T> T* take(size_t count) {
    T* p = base ? (T*)(base + off) : nullptr;
    off += align256(count * sizeof(T));
    return p;
  }
};

inline int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

inline bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

}  // namespace fct

// internal entry points used by the pipeline (same validation as the public ones)
fct_status fct2_cz_tc(const float* C, int64_t ldc, const float* Zh, const float* Zl, int64_t ldzt, int64_t K, int r1,
                      int d, double* W, cudaStream_t st);
// FCT1 sketch accumulation state: W (r1 x d fp64) plus the optional fp32 L2 replicas of the buckets >= t_l2
struct SketchAcc {
  double* W = nullptr;
  float* rep = nullptr;   // [nrep][r1 - t_l2][d], values scaled by 2^20 (nullptr: no L2 offload)
  int t_l2 = 0;           // first bucket scattered through L2 (r1: none)
  int nrep = 1;
  int mode = 0;           // scatter: 0 shared-memory CAS, 1 EXCH, 2 CAS + L2 offload, 3 racy (timing only)
  int* pace = nullptr;    // [1024] per-row-block-group pacing counters (v5)
};
// carve W and the replicas from a fct_sketch workspace and zero them on st
fct_status fct_sketch_begin(void* workspace, size_t workspace_bytes, int64_t d, int s, int r1, SketchAcc* acc,
                            cudaStream_t st);
// W (+ replicas) += 4 B C H~ D A for the given rows (row shards / host chunks, s-aligned)
fct_status fct_sketch_accum(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                            const float* cauchy_diag, const int32_t* hash_rows, int s, int r1, const SketchAcc& acc,
                            cudaStream_t st);
// replicas -> W (fixed order, fp64), then Y = (float)(W [+ Y])
fct_status fct_sketch_end(const SketchAcc& acc, int r1, int64_t d, float* Y, int accumulate, cudaStream_t st);
fct_status fct_sketch_v5(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                         const int32_t* hash, int s, int r1, int mode, double* W, int* pace, int64_t* rows_done,
                         cudaStream_t st);
fct_status fct_sketch_v1(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs, const float* cauchy,
                         const int32_t* hash, int s, int r1, const SketchAcc& acc, cudaStream_t st);
fct_status fct_rownorm_impl(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                            const float* Pi2, int32_t k, float* lambda, double* lambda_sum,
                            bool zero_sum, void* ws, size_t wsb, cudaStream_t st);
fct_status fct_rownorm_ws2(const float* A, int64_t n, int d, int64_t lda, const float* M32, int KP32,
                           const double* M64, const float* colb, int k, double* partial, int grid, float* lambda,
                           cudaStream_t st);
