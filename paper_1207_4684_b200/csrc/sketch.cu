// sketch.cu -- K1: the FCT1 sketch Y = 4 B C H~ D A  (Sec. 3.1).
//
// Structure:
//   * the r1 x d output is split into column slices of DT columns; every CTA owns ONE slice and
//     keeps an fp32 partial sketch P[r1][DT] of it in shared memory for the CTA's lifetime;
//   * CTAs of the same slice take row blocks b = grp, grp + ngrp, ...; all slices of a block are
//     in flight at about the same time, so the aux arrays (signs, C, B) are re-read from L2;
//   * per block: z = D_b A_b[:, slice] -> shared tile; identity half of G_s scattered at load;
//     FWHT of length s in place (normalised Sylvester H_s); Hadamard half scattered;
//   * every `flush_every` blocks (<= ~2048 expected terms per bucket) the fp32 partial is added
//     into the fp64 workspace W[r1][d] (hierarchical accumulation);
//   * a final kernel writes Y = (float)(W [+ Y]).
#include <math.h>
#include <string.h>
#include "common.cuh"

namespace {

constexpr int kThreads = 512;

__device__ __forceinline__ void smem_add(float* p, float v) { atomicAdd(p, v); }

template <int DT>
__global__ void __launch_bounds__(kThreads)
sketch_generic_kernel(const float* __restrict__ A, int64_t n, int d, int64_t lda,
                      const int8_t* __restrict__ signs, const float* __restrict__ cauchy,
                      const int32_t* __restrict__ hash, int s, int r1, int nslices,
                      int64_t nblocks, int flush_every, float inv_sqrt_s,
                      double* __restrict__ W) {
  extern __shared__ float smem[];
  float* part = smem;                 // [r1][DT]
  float* tile = smem + (size_t)r1 * DT;  // [s][DT]
  const int cs = blockIdx.x % nslices;
  const int grp = blockIdx.x / nslices;
  const int ngrp = gridDim.x / nslices;
  const int c0 = cs * DT;
  const int nt = blockDim.x;

  for (int e = threadIdx.x; e < r1 * DT; e += nt) part[e] = 0.f;
  __syncthreads();

  int since_flush = 0;
  for (int64_t b = grp; b < nblocks; b += ngrp) {
    const int64_t t0 = 2 * (int64_t)s * b;     // first H~-row of the block
    // load z = D_b A_b (zero-padded) and scatter the identity half: Y[h(t)] += 4 c_t z_r
    for (int e = threadIdx.x; e < s * DT; e += nt) {
      const int r = e / DT, c = e - r * DT;
      const int64_t row = b * s + r;
      const int col = c0 + c;
      float v = 0.f;
      if (row < n && col < d) v = A[row * lda + col] * (float)signs[row];
      tile[e] = v;
      const int64_t t = t0 + s + r;
      smem_add(&part[hash[t] * DT + c], (4.f * cauchy[t]) * v);
    }
    __syncthreads();
    // in-place FWHT over the s rows of every column (unnormalised; 1/sqrt(s) folded below)
    for (int h = 1; h < s; h <<= 1) {
      for (int e = threadIdx.x; e < (s >> 1) * DT; e += nt) {
        const int pidx = e / DT, c = e - pidx * DT;
        const int i = ((pidx & ~(h - 1)) << 1) | (pidx & (h - 1));
        const float a = tile[i * DT + c], bb = tile[(i + h) * DT + c];
        tile[i * DT + c] = a + bb;
        tile[(i + h) * DT + c] = a - bb;
      }
      __syncthreads();
    }
    // Hadamard half: Y[h(t)] += 4 c_t (H z)_r / sqrt(s)
    for (int e = threadIdx.x; e < s * DT; e += nt) {
      const int r = e / DT, c = e - r * DT;
      const int64_t t = t0 + r;
      smem_add(&part[hash[t] * DT + c], (4.f * cauchy[t] * inv_sqrt_s) * tile[e]);
    }
    __syncthreads();
    if (++since_flush == flush_every) {
      since_flush = 0;
      for (int e = threadIdx.x; e < r1 * DT; e += nt) {
        const int h = e / DT, c = e - h * DT;
        if (c0 + c < d && part[e] != 0.f) atomicAdd(&W[(size_t)h * d + c0 + c], (double)part[e]);
        part[e] = 0.f;
      }
      __syncthreads();
    }
  }
  if (since_flush) {
    for (int e = threadIdx.x; e < r1 * DT; e += nt) {
      const int h = e / DT, c = e - h * DT;
      if (c0 + c < d && part[e] != 0.f) atomicAdd(&W[(size_t)h * d + c0 + c], (double)part[e]);
    }
  }
}

__global__ void finalize_kernel(const double* __restrict__ W, float* __restrict__ Y, int64_t cells,
                                int accumulate) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = W[i];
    if (accumulate) v += (double)Y[i];
    Y[i] = (float)v;
  }
}

__global__ void check_hash_kernel(const int32_t* hash, int64_t count, int r1, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (hash[i] < 0 || hash[i] >= r1) atomicAdd(bad, 1);
}

constexpr size_t kSmemBudget = 160 * 1024;

int pick_dt(int64_t d, int s, int r1) {
  int dmax = 1;
  while (dmax < d && dmax < 32) dmax <<= 1;
  for (int dt = dmax; dt >= 1; dt >>= 1)
    if ((size_t)(r1 + s) * dt * sizeof(float) <= kSmemBudget) return dt;
  return 0;
}

template <int DT>
fct_status launch_generic(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                          const float* cauchy, const int32_t* hash, int s, int r1, double* W,
                          cudaStream_t st) {
  const int nslices = (int)((d + DT - 1) / DT);
  const int64_t nblocks = (n + s - 1) / s;
  const size_t smem = (size_t)(r1 + s) * DT * sizeof(float);
  auto kern = sketch_generic_kernel<DT>;
  FCT_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  FCT_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
  if (occ < 1) occ = 1;
  int64_t ngrp = ((int64_t)fct::num_sms() * occ) / nslices;
  if (ngrp < 1) ngrp = 1;
  if (ngrp > nblocks) ngrp = nblocks;
  const int flush_every = (int)std::max<int64_t>(1, (int64_t)1024 * r1 / s);
  const float inv_sqrt_s = (float)(1.0 / sqrt((double)s));
  kern<<<(unsigned)(ngrp * nslices), kThreads, smem, st>>>(A, n, (int)d, lda, signs, cauchy, hash, s, r1,
                                                           nslices, nblocks, flush_every, inv_sqrt_s, W);
  FCT_LAUNCHED("sketch_generic_kernel", st);
  return FCT_OK;
}

__global__ void rep_reduce_kernel(const float* __restrict__ rep, int nrep, int64_t cells, double* __restrict__ W) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nrep; ++r) s += (double)rep[(size_t)r * cells + i];
    W[i] += s * 0x1p-20;   // exact rescale of the replicas' 2^20
  }
}

constexpr int kMaxRep = 16;

// L2 offload fraction of the buckets and scatter primitive (environment overrides; K1)
void sketch_policy(int r1, int s, int64_t d, int* t_l2, int* nrep, int* mode) {
  double frac = 0.0;
  if (const char* e = getenv("FCT_SKETCH_L2")) frac = atof(e);
  frac = frac < 0.0 ? 0.0 : (frac > 1.0 ? 1.0 : frac);
  *t_l2 = r1 - (int)(frac * r1);
  *nrep = kMaxRep;
  if (const char* e = getenv("FCT_SKETCH_NREP")) *nrep = std::max(1, std::min(kMaxRep, atoi(e)));
  *mode = 1;   // EXCH pair (exact); "cas": the round-1 CAS batch; "racy": timing bound only
  if (const char* e = getenv("FCT_SKETCH_SCATTER")) *mode = !strcmp(e, "cas") ? 0 : (!strcmp(e, "racy") ? 3 : 1);
  if (frac > 0.0) *mode = 2;
  (void)s; (void)d;
}

}  // namespace

fct_status fct_sketch_begin(void* workspace, size_t workspace_bytes, int64_t d, int s, int r1, SketchAcc* acc,
                            cudaStream_t st) {
  (void)workspace_bytes;
  fct::Carver cv(workspace);
  acc->W = cv.take<double>((size_t)r1 * d);
  acc->pace = cv.take<int>(1024);
  int t_l2, nrep, mode;
  sketch_policy(r1, s, d, &t_l2, &nrep, &mode);
  acc->t_l2 = t_l2;
  acc->nrep = nrep;
  acc->mode = mode;
  acc->rep = mode == 2 && t_l2 < r1 ? cv.take<float>((size_t)kMaxRep * (r1 - t_l2) * d) : nullptr;
  FCT_CUDA_RET(cudaMemsetAsync(acc->W, 0, sizeof(double) * (size_t)r1 * d, st));
  if (acc->rep) FCT_CUDA_RET(cudaMemsetAsync(acc->rep, 0, sizeof(float) * (size_t)nrep * (r1 - t_l2) * d, st));
  return FCT_OK;
}

fct_status fct_sketch_accum(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                            const float* cauchy_diag, const int32_t* hash_rows, int s, int r1, const SketchAcc& acc,
                            cudaStream_t st) {
  const int dt = pick_dt(d, s, r1);
  FCT_CHECK_ARG(dt >= 1, FCT_ERR_UNSUPPORTED, "fct_sketch: r1 + s = %d too large", r1 + s);
  fct_status rc = FCT_ERR_UNSUPPORTED;
  if (!getenv("FCT_SKETCH_GENERIC") && (acc.mode == 0 || acc.mode == 1)) {
    // v5 takes the full s-blocks; the ragged tail block (if any) continues below through v1 / generic
    int64_t done = 0;
    rc = fct_sketch_v5(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, acc.mode, acc.W, acc.pace, &done, st);
    if (rc != FCT_OK && rc != FCT_ERR_UNSUPPORTED) return rc;
    if (rc == FCT_OK) {
      if (done == n) return FCT_OK;
      A += done * lda;
      signs += done;
      cauchy_diag += 2 * done;
      hash_rows += 2 * done;
      n -= done;
      rc = FCT_ERR_UNSUPPORTED;
    }
  }
  if (!getenv("FCT_SKETCH_GENERIC"))
    rc = fct_sketch_v1(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, acc, st);
  double* W = acc.W;
  if (rc == FCT_ERR_UNSUPPORTED) switch (dt) {   // the generic kernel keeps everything in shared memory / W
    case 32: rc = launch_generic<32>(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, W, st); break;
    case 16: rc = launch_generic<16>(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, W, st); break;
    case 8: rc = launch_generic<8>(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, W, st); break;
    case 4: rc = launch_generic<4>(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, W, st); break;
    case 2: rc = launch_generic<2>(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, W, st); break;
    default: rc = launch_generic<1>(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, W, st); break;
  }
  return rc;
}

fct_status fct_sketch_end(const SketchAcc& acc, int r1, int64_t d, float* Y, int accumulate, cudaStream_t st) {
  if (acc.rep) {
    const int64_t cells = (int64_t)(r1 - acc.t_l2) * d;
    rep_reduce_kernel<<<(unsigned)std::min<int64_t>((cells + 255) / 256, 4096), 256, 0, st>>>(
        acc.rep, acc.nrep, cells, acc.W + (size_t)acc.t_l2 * d);
    FCT_LAUNCHED("rep_reduce_kernel", st);
  }
  const int64_t cells = (int64_t)r1 * d;
  finalize_kernel<<<(unsigned)std::min<int64_t>((cells + 255) / 256, 4096), 256, 0, st>>>(acc.W, Y, cells, accumulate);
  FCT_LAUNCHED("finalize_kernel", st);
  return FCT_OK;
}

extern "C" size_t fct_sketch_workspace_bytes(int64_t n, int64_t d, int32_t s, int32_t r1) {
  (void)n; (void)s;
  if (d < 1 || r1 < 1) return 0;
  return fct::align256((size_t)r1 * (size_t)d * sizeof(double)) + fct::align256(1024 * sizeof(int)) +
         fct::align256((size_t)kMaxRep * r1 * (size_t)d * sizeof(float)) + 256;
}

extern "C" fct_status fct_sketch(const float* A, int64_t n, int64_t d, int64_t lda,
                                 const int8_t* signs, const float* cauchy_diag,
                                 const int32_t* hash_rows, int32_t s, int32_t r1, float* Y,
                                 int accumulate, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  FCT_CHECK_ARG(A && signs && cauchy_diag && hash_rows && Y, FCT_ERR_ARG, "fct_sketch: NULL pointer");
  FCT_CHECK_ARG(n >= 1 && d >= 1 && lda >= d && r1 >= 1, FCT_ERR_SHAPE,
                "fct_sketch: bad shape n=%lld d=%lld lda=%lld r1=%d", (long long)n, (long long)d,
                (long long)lda, r1);
  FCT_CHECK_ARG(fct::is_pow2(s) && s <= FCT_MAX_S, FCT_ERR_ARG,
                "fct_sketch: s=%d must be a power of two in [1, %d]", s, FCT_MAX_S);
  const size_t need = fct_sketch_workspace_bytes(n, d, s, r1);
  FCT_CHECK_ARG(workspace && workspace_bytes >= need, FCT_ERR_WORKSPACE,
                "fct_sketch: workspace %zu < %zu bytes", workspace_bytes, need);
  FCT_CHECK_ARG(pick_dt(d, s, r1) >= 1, FCT_ERR_UNSUPPORTED, "fct_sketch: r1 + s = %d too large", r1 + s);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n_pad = (n + s - 1) / s * s;
  if (fct::debug_sync()) {
    int* bad = (int*)((char*)workspace + need - 256);
    FCT_CUDA_RET(cudaMemsetAsync(bad, 0, sizeof(int), st));
    check_hash_kernel<<<256, 256, 0, st>>>(hash_rows, 2 * n_pad, r1, bad);
    FCT_LAUNCHED("check_hash_kernel", st);
    int hb = 0;
    FCT_CUDA_RET(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    FCT_CUDA_RET(cudaStreamSynchronize(st));
    FCT_CHECK_ARG(hb == 0, FCT_ERR_ARG, "fct_sketch: %d hash_rows entries outside [0, r1)", hb);
  }
  SketchAcc acc;
  fct_status rc = fct_sketch_begin(workspace, workspace_bytes, d, s, r1, &acc, st);
  if (rc == FCT_OK) rc = fct_sketch_accum(A, n, d, lda, signs, cauchy_diag, hash_rows, s, r1, acc, st);
  if (rc == FCT_OK) rc = fct_sketch_end(acc, r1, d, Y, accumulate, st);
  return rc;
}
