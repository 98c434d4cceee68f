// pipeline.cu -- the whole single-device hot path behind one call, and the
// host-buffer (end-to-end) variant.
#include "common.cuh"

namespace {
struct PipeWS {
  size_t sketch, cond, rown, samp, total;
};
PipeWS pipe_ws(int64_t n, int64_t d, int32_t s, int32_t r1, int32_t k) {
  PipeWS w;
  w.sketch = fct::align256(fct_sketch_workspace_bytes(n, d, s, r1));
  w.cond = fct::align256(fct_condition_workspace_bytes(r1, d));
  w.rown = fct::align256(l1_rownorm_workspace_bytes(n, d, k));
  w.samp = fct::align256(std::max(l1_sample_workspace_bytes(n), l1_probs_sample_workspace_bytes(n)));
  w.total = w.sketch + w.cond + w.rown + w.samp + fct::align256(sizeof(double));
  return w;
}
}  // namespace

extern "C" size_t fct_pipeline_workspace_bytes(int64_t n, int64_t d, int32_t s, int32_t r1, int32_t k) {
  if (n < 1 || d < 1 || s < 1 || r1 < 1 || k < 1) return 0;
  return pipe_ws(n, d, s, r1, k).total;
}

namespace {
// a1-a10 on one device; sketch_ready: Y already holds Pi1 A (the host variant sketches chunk by chunk while A is
// still being copied) and the sketch step is skipped
fct_status pipeline_impl(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                         const float* cauchy_diag, const int32_t* hash_rows, int32_t s, int32_t r1, const float* Pi2,
                         int32_t k, int64_t m, uint64_t seed, float* Y, double* R, double* Rinv, float* lambda,
                         float* p, int64_t* idx, double* weight, int64_t capacity, int64_t* count, int32_t* info,
                         void* workspace, size_t workspace_bytes, void* stream, bool sketch_ready) {
  FCT_CHECK_ARG(n >= 1 && d >= 1 && s >= 1 && r1 >= 1 && k >= 1, FCT_ERR_SHAPE, "fct_pipeline: bad sizes");
  const PipeWS w = pipe_ws(n, d, s, r1, k);
  FCT_CHECK_ARG(workspace && workspace_bytes >= w.total, FCT_ERR_WORKSPACE,
                "fct_pipeline: workspace %zu < %zu bytes", workspace_bytes, w.total);
  FCT_CHECK_ARG(r1 >= d, FCT_ERR_SHAPE, "fct_pipeline: r1=%d < d=%lld", r1, (long long)d);
  char* base = (char*)workspace;
  void* ws_sk = base;
  void* ws_cd = base + w.sketch;
  void* ws_rn = base + w.sketch + w.cond;
  void* ws_sp = base + w.sketch + w.cond + w.rown;
  double* total = (double*)(base + w.sketch + w.cond + w.rown + w.samp);
  cudaStream_t st = (cudaStream_t)stream;
  fct_status rc;
  if (!sketch_ready &&
      (rc = fct_sketch(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, Y, 0, ws_sk, w.sketch, stream)) != FCT_OK)
    return rc;
  if ((rc = fct_condition(Y, r1, d, R, Rinv, info, ws_cd, w.cond, stream)) != FCT_OK) return rc;
  if ((rc = fct_rownorm_impl(A, n, d, lda, Rinv, Pi2, k, lambda, total, true, ws_rn, w.rown, st)) != FCT_OK)
    return rc;
  return l1_probs_sample(lambda, n, total, 0, m, seed, p, idx, weight, capacity, count, ws_sp, w.samp, stream);
}
}  // namespace

extern "C" fct_status fct_pipeline(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                                   const float* cauchy_diag, const int32_t* hash_rows, int32_t s, int32_t r1,
                                   const float* Pi2, int32_t k, int64_t m, uint64_t seed, float* Y, double* R,
                                   double* Rinv, float* lambda, float* p, int64_t* idx, double* weight,
                                   int64_t capacity, int64_t* count, int32_t* info, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  return pipeline_impl(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, Pi2, k, m, seed, Y, R, Rinv, lambda, p,
                       idx, weight, capacity, count, info, workspace, workspace_bytes, stream, false);
}

// ------------------------------------------------------------------------------ host-buffer variant
namespace {
struct AuxLayout {
  size_t signs, cauchy, hash, pi2, total;
};
AuxLayout aux_layout(int64_t n, int64_t d, int32_t s, int32_t k) {
  const int64_t np = (n + s - 1) / s * s;
  AuxLayout a;
  a.signs = 0;
  a.cauchy = a.signs + fct::align256((size_t)np);
  a.hash = a.cauchy + fct::align256(sizeof(float) * 2 * (size_t)np);
  a.pi2 = a.hash + fct::align256(sizeof(int32_t) * 2 * (size_t)np);
  a.total = a.pi2 + fct::align256(sizeof(float) * (size_t)d * k);
  return a;
}
struct HostWS {
  size_t Y, R, Rinv, lam, p, idx, w, cnt, info, sk, pipe, total;
};
HostWS host_ws(int64_t n, int64_t d, int32_t s, int32_t r1, int32_t k, int64_t cap) {
  HostWS h;
  size_t o = 0;
  h.Y = o; o += fct::align256(sizeof(float) * (size_t)r1 * d);
  h.R = o; o += fct::align256(sizeof(double) * (size_t)d * d);
  h.Rinv = o; o += fct::align256(sizeof(double) * (size_t)d * d);
  h.lam = o; o += fct::align256(sizeof(float) * (size_t)n);
  h.p = o; o += fct::align256(sizeof(float) * (size_t)n);
  h.idx = o; o += fct::align256(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  h.w = o; o += fct::align256(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  h.cnt = o; o += fct::align256(sizeof(int64_t));
  h.info = o; o += fct::align256(sizeof(int32_t));
  h.sk = o; o += fct::align256(fct_sketch_workspace_bytes(n, d, s, r1));
  h.pipe = o; o += fct_pipeline_workspace_bytes(n, d, s, r1, k);
  h.total = o;
  return h;
}
}  // namespace

extern "C" size_t fct_pipeline_aux_bytes(int64_t n, int64_t d, int32_t s, int32_t k) {
  if (n < 1 || d < 1 || s < 1 || k < 1) return 0;
  return aux_layout(n, d, s, k).total;
}

extern "C" size_t fct_pipeline_host_workspace_bytes(int64_t n, int64_t d, int32_t s, int32_t r1, int32_t k,
                                                    int64_t capacity) {
  if (n < 1 || d < 1 || s < 1 || r1 < 1 || k < 1 || capacity < 0) return 0;
  return host_ws(n, d, s, r1, k, capacity).total;
}

extern "C" fct_status fct_pipeline_host(const float* A_host, int64_t n, int64_t d, int64_t lda,
                                        const int8_t* signs_host, const float* cauchy_host,
                                        const int32_t* hash_host, int32_t s, int32_t r1, const float* Pi2_host,
                                        int32_t k, int64_t m, uint64_t seed, int64_t* idx_host,
                                        double* weight_host, int64_t capacity, int64_t* count_host, float* dev_A,
                                        void* dev_aux, void* workspace, size_t workspace_bytes, void* stream) {
  FCT_CHECK_ARG(A_host && signs_host && cauchy_host && hash_host && Pi2_host && count_host && dev_A && dev_aux,
                FCT_ERR_ARG, "fct_pipeline_host: NULL pointer");
  FCT_CHECK_ARG(capacity == 0 || (idx_host && weight_host), FCT_ERR_ARG, "fct_pipeline_host: NULL outputs");
  FCT_CHECK_ARG(n >= 1 && d >= 1 && lda >= d && k >= 1 && fct::is_pow2(s) && s <= FCT_MAX_S, FCT_ERR_SHAPE,
                "fct_pipeline_host: bad sizes");
  const HostWS h = host_ws(n, d, s, r1, k, capacity);
  FCT_CHECK_ARG(workspace && workspace_bytes >= h.total, FCT_ERR_WORKSPACE,
                "fct_pipeline_host: workspace %zu < %zu bytes", workspace_bytes, h.total);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t np = (n + s - 1) / s * s;
  const AuxLayout a = aux_layout(n, d, s, k);
  char* aux = (char*)dev_aux;
  int8_t* dsg = (int8_t*)(aux + a.signs);
  float* dc = (float*)(aux + a.cauchy);
  int32_t* dh = (int32_t*)(aux + a.hash);
  float* dpi2 = (float*)(aux + a.pi2);
  // host -> device: the aux arrays first, then A in s-aligned row chunks on the caller's stream; the sketch of
  // each chunk runs on a second stream as soon as the chunk has landed (W accumulates the chunks in fp64), so
  // the sketch overlaps the PCIe copy of the later chunks.  The row norms need all of A and start after it.
  FCT_CUDA_RET(cudaMemcpyAsync(dsg, signs_host, (size_t)n, cudaMemcpyHostToDevice, st));
  FCT_CUDA_RET(cudaMemcpyAsync(dc, cauchy_host, sizeof(float) * 2 * np, cudaMemcpyHostToDevice, st));
  FCT_CUDA_RET(cudaMemcpyAsync(dh, hash_host, sizeof(int32_t) * 2 * np, cudaMemcpyHostToDevice, st));
  FCT_CUDA_RET(cudaMemcpyAsync(dpi2, Pi2_host, sizeof(float) * d * k, cudaMemcpyHostToDevice, st));
  char* w = (char*)workspace;
  int64_t* dcnt = (int64_t*)(w + h.cnt);
  int32_t* dinfo = (int32_t*)(w + h.info);
  float* dY = (float*)(w + h.Y);
  SketchAcc acc;
  fct_status rc = fct_sketch_begin(w + h.sk, h.pipe - h.sk, d, s, r1, &acc, st);
  if (rc != FCT_OK) return rc;
  const size_t row_bytes = sizeof(float) * (size_t)lda;
  const int64_t chunk = std::max<int64_t>(s, (int64_t)((512u << 20) / row_bytes) / s * s);
  const int nchunks = (int)((n + chunk - 1) / chunk);
  cudaStream_t st2 = nullptr;
  FCT_CUDA_RET(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  cudaEvent_t ev_done = nullptr;
  cudaEvent_t* evs = (cudaEvent_t*)calloc((size_t)nchunks + 1, sizeof(cudaEvent_t));
  for (int c = 0; c <= nchunks && rc == FCT_OK; ++c)
    if (cudaEventCreateWithFlags(&evs[c], cudaEventDisableTiming) != cudaSuccess) rc = FCT_ERR_CUDA;
  if (rc == FCT_OK && cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) != cudaSuccess) rc = FCT_ERR_CUDA;
  // chunk 0's event also covers the aux copies and the W reset queued above
  for (int c = 0; c < nchunks && rc == FCT_OK; ++c) {
    const int64_t r0 = (int64_t)c * chunk, nr = std::min(chunk, n - r0);
    if (cudaMemcpyAsync(dev_A + r0 * lda, A_host + r0 * lda, row_bytes * nr, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(evs[c], st) != cudaSuccess || cudaStreamWaitEvent(st2, evs[c], 0) != cudaSuccess) {
      rc = FCT_ERR_CUDA;
      break;
    }
    rc = fct_sketch_accum(dev_A + r0 * lda, nr, d, lda, dsg + r0, dc + 2 * r0, dh + 2 * r0, s, r1, acc, st2);
  }
  if (rc == FCT_OK) rc = fct_sketch_end(acc, r1, d, dY, 0, st2);
  if (rc == FCT_OK && (cudaEventRecord(ev_done, st2) != cudaSuccess || cudaStreamWaitEvent(st, ev_done, 0) != cudaSuccess))
    rc = FCT_ERR_CUDA;
  if (rc != FCT_OK && fct_last_error()[0] == 0) fct::set_error("fct_pipeline_host: chunked copy/sketch failed");
  for (int c = 0; c <= nchunks; ++c)
    if (evs[c]) cudaEventDestroy(evs[c]);
  free(evs);
  if (ev_done) cudaEventDestroy(ev_done);
  cudaStreamDestroy(st2);   // deferred by the runtime until its queued work completes
  if (rc != FCT_OK) return rc;
  rc = pipeline_impl(dev_A, n, d, lda, dsg, dc, dh, s, r1, dpi2, k, m, seed, dY, (double*)(w + h.R),
                     (double*)(w + h.Rinv), (float*)(w + h.lam), (float*)(w + h.p), (int64_t*)(w + h.idx),
                     (double*)(w + h.w), capacity, dcnt, dinfo, w + h.pipe, h.total - h.pipe, stream, true);
  if (rc != FCT_OK) return rc;
  int64_t cnt = 0;
  int32_t inf = 0;
  FCT_CUDA_RET(cudaMemcpyAsync(&cnt, dcnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FCT_CUDA_RET(cudaMemcpyAsync(&inf, dinfo, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FCT_CUDA_RET(cudaStreamSynchronize(st));
  *count_host = cnt;
  FCT_CHECK_ARG(inf <= 0, FCT_ERR_SINGULAR,
                "fct_pipeline_host: Cholesky pivot %d failed even with the shifted fallback (non-finite Pi1 A)", inf);
  const int64_t ncopy = std::min(cnt, capacity);
  if (ncopy > 0) {
    FCT_CUDA_RET(cudaMemcpyAsync(idx_host, w + h.idx, sizeof(int64_t) * ncopy, cudaMemcpyDeviceToHost, st));
    FCT_CUDA_RET(cudaMemcpyAsync(weight_host, w + h.w, sizeof(double) * ncopy, cudaMemcpyDeviceToHost, st));
    FCT_CUDA_RET(cudaStreamSynchronize(st));
  }
  FCT_CHECK_ARG(cnt <= capacity, FCT_ERR_CAPACITY, "fct_pipeline_host: %lld samples > capacity %lld",
                (long long)cnt, (long long)capacity);
  return FCT_OK;
}
