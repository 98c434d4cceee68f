/*
 * fct.h -- C ABI of libfct.so: the B200 (sm_100a) hot path of the Fast Cauchy Transform
 * l1-conditioning pipeline of Clarkson, Drineas, Magdon-Ismail, Mahoney, Meng, Woodruff,
 * "The Fast Cauchy Transform and Faster Robust Linear Regression" (arXiv 1207.4684).
 * Citations "P:L<n>" are lines of that paper's text; DESIGN.md lists the readings
 * taken where the paper is silent.
 *
 * Conventions (all entry points):
 *  - Matrices are row-major.  A is n x d with leading dimension lda (>= d), fp32.
 *  - Unless an argument is documented as HOST memory, every pointer is a DEVICE pointer owned
 *    by the caller.  The library allocates no device memory: scratch space is the caller's
 *    `workspace` (size from the matching *_workspace_bytes query, 256-byte aligned).
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream).  All device work is
 *    enqueued asynchronously on it; argument validation is synchronous and happens before
 *    anything is enqueued, so a non-OK return means nothing was enqueued.
 *  - Return value: FCT_OK or a negative fct_status; fct_last_error() gives a message
 *    (thread-local).  Asynchronous device faults surface at the next synchronising call
 *    (CUDA semantics).  No C++ exception crosses this boundary.  Functions are re-entrant;
 *    the library keeps no global state besides the thread-local error string and a
 *    per-device cache of kernel attributes.
 *  - Setting the environment variable FCT_DEBUG=1 synchronises after every launch and
 *    range-checks hash_rows (slow; for debugging).
 */
#ifndef FCT_H_
#define FCT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int fct_status;
enum {
  FCT_OK = 0,
  FCT_ERR_ARG = -1,         /* bad scalar argument or NULL pointer                           */
  FCT_ERR_SHAPE = -2,       /* inconsistent sizes (n < 1, d < 1, lda < d, r1 < 1, r1 < d ...) */
  FCT_ERR_CUDA = -3,        /* a CUDA launch/runtime error                                   */
  FCT_ERR_CAPACITY = -4,    /* a host-side result does not fit the caller's buffer           */
  FCT_ERR_SINGULAR = -5,    /* Cholesky of Y^T Y broke down (host-synchronous entry points)  */
  FCT_ERR_UNSUPPORTED = -6, /* no kernel instance for these sizes                            */
  FCT_ERR_WORKSPACE = -7    /* workspace NULL or smaller than the *_workspace_bytes query    */
};

/* Message of the last failing call on this thread ("" if none). */
const char* fct_last_error(void);
/* Library version string, e.g. "fct-b200 0.1 sm_100a". */
const char* fct_version(void);
/* Number of kernels this library has launched in this process (all threads, all devices). */
uint64_t fct_launch_count(void);
/* The kernel template instance the last call of a hot-path stage launched (stage 0: the FCT1 sketch's main
 * kernel, 1: the row-norm kernel), e.g. "sketch_v5_kernel<5, 5, 8, 2, 1>", copied NUL-terminated into buf
 * (len bytes, host memory).  Returns 0, or -1 for a bad stage / buffer.  Used to match ncu captures. */
int fct_last_instance(int32_t stage, char* buf, size_t len);

/* Limits of this build. */
#define FCT_MAX_S 4096   /* Hadamard block size s: power of two in [1, FCT_MAX_S]          */
#define FCT_MAX_D 128    /* columns handled by fct_condition / l1_rownorm                  */
#define FCT_MAX_K 32     /* r2 = k, the number of Cauchy columns of Pi2                    */

/* ------------------------------------------------------------------------------------------
 * FCT1 sketch (Sec. 3.1; Thm FCT1):
 *     Y (r1 x d, ld = d, fp32)  :=  [accumulate ? Y : 0]  +  4 * B * C * H~ * D * A_pad
 * with A_pad = A zero-padded to n' = s*ceil(n/s) rows (P:L2255-2256 assumes s | n).
 *   signs[n]        D, the Rademacher diagonal (+1/-1), int8 (north_star addition; D = I gives
 *                   the paper's Pi1 = 4 B C H~ exactly).
 *   cauchy_diag[2n'] diag(C), i.i.d. standard Cauchy, fp32, indexed by H~-row.
 *   hash_rows[2n']  B: column t of B is e_{hash_rows[t]}, values in [0, r1).
 *   H~ row layout: block b occupies H~-rows [2sb, 2sb+2s); row 2sb+r (r < s) is row r of the
 *   normalised Hadamard H_s = H/sqrt(s) (Sylvester order) applied to block b,
 *   row 2sb+s+r is row r of I_s (G_s = [H_s; I_s]).
 * s must be a power of two in [1, FCT_MAX_S].
 * Row shards: call with A + row0*lda, signs + row0, cauchy_diag + 2*row0, hash_rows + 2*row0
 * (row0 % s == 0) and accumulate = 1 to add the shard's contribution (Pi1 A = sum of shards).
 * Accuracy: each CTA keeps an fp32 partial of its column slice in shared memory for its lifetime (about
 * 2048 expected terms per bucket cell for uniform hashes: the launch sizes the grid for it) and adds it once
 * into an fp64 accumulator; Y is that fp64 sum rounded to fp32.  The error of an fp32 cell of N terms is
 * below N u sum|terms| (u = 2^-24) in the worst case and ~sqrt(N) u sum|terms| typically, so the bound
 * |Y - exact| <= 1e-5 * (4|B||C||H~||D||A|) entrywise is an EXPECTED property, not a worst-case guarantee:
 * measured at full size on the real cfg-3 / cfg-4 data at <= 2.1e-6 of the bound, and on adversarial
 * hashes (most H~-rows in a few buckets) in tests/test_gpu_parity.py.
 * Y may be written by any order of floating-point additions (run-to-run bitwise variation).
 */
size_t fct_sketch_workspace_bytes(int64_t n, int64_t d, int32_t s, int32_t r1);
fct_status fct_sketch(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                      const float* cauchy_diag, const int32_t* hash_rows, int32_t s, int32_t r1,
                      float* Y, int accumulate, void* workspace, size_t workspace_bytes,
                      void* stream);

/* ------------------------------------------------------------------------------------------
 * Conditioning (FastL1Basis: "construct Pi1 A and an R such that Pi1 A = QR"):
 * R with Y = Q R, Q orthonormal columns, diag(R) > 0 (unique; reading R19), and Rinv = R^-1
 * (O(r1 d^2) + O(d^3)).  Y: r1 x d fp32 (the sketch); R, Rinv: d x d fp64 row-major
 * (upper triangular).  Computed by CholeskyQR2 in fp64 (one cooperative kernel, nothing returns to the host);
 * when a Cholesky pivot is not positive/finite or the second Gram is far from I (cond(Y) > ~1e8), the device
 * restarts with the shifted CholeskyQR3 of Fukaya et al. (sigma = 11 (r1 d + d(d+1)) u ||Y||_F^2 on the first
 * Gram, three passes), which is stable up to cond(Y) ~ 1/u.
 * info (device int32): 0 = success (CholeskyQR2), -1 = success via the shifted CholeskyQR3 fallback,
 * j > 0 = the j-th pivot failed even with the shift (non-finite Y); R and Rinv are then all NaN so that no
 * downstream result can look valid.  Deterministic (fixed summation orders).
 * Requires 1 <= d <= FCT_MAX_D and r1 >= d; a device that supports cooperative launches.
 */
size_t fct_condition_workspace_bytes(int32_t r1, int64_t d);
fct_status fct_condition(const float* Y, int32_t r1, int64_t d, double* R, double* Rinv,
                         int32_t* info, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * l1 row-norm estimation (Lemma medCauchy, cost P:L2168-2175):
 *     M = Rinv * Pi2 (formed first, fp64);  Lambda = A M;
 *     lambda[i] = median_j |Lambda_ij|   (even k: mean of the two middle order statistics)
 *     *lambda_sum += sum_i lambda[i]      (fp64 device scalar)
 * lambda is deterministic (each entry is the exact median rounded once).  lambda_sum is a sum of per-CTA fp64
 * partials; the tensor-core kernel hands tiles to CTAs dynamically, so its summation order (and the last bits of
 * lambda_sum) may vary run to run, as Y does (R20); FCT_ROWNORM_STATIC=1 fixes the order.
 * Rinv: d x d fp64; Pi2: d x k fp32 (i.i.d. Cauchy); lambda: n fp32.
 * Accuracy: |lambda - exact| <= 1e-5 * exact per row.  Rows whose fp32 evaluation cannot be
 * certified to that bound (cancellation) are recomputed in fp64 inside the kernel.
 * Requires 1 <= d <= FCT_MAX_D, 1 <= k <= FCT_MAX_K.
 */
size_t l1_rownorm_workspace_bytes(int64_t n, int64_t d, int32_t k);
fct_status l1_rownorm(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                      const float* Pi2, int32_t k, float* lambda, double* lambda_sum,
                      void* workspace, size_t workspace_bytes, void* stream);
/* NEXT-1: exact l1 row norms of the well-conditioned basis U = A R^-1,
 *     lambda[i] = sum_j |sum_l A[i][l] Rinv[l][j]|      (Sec. 6.2: the paper's
 * experiments "compute the row norms of U exactly instead of estimating them"; U of FastL1Basis
 * P:L2771-2796).  *lambda_sum = sum_i lambda[i] (fp64, overwritten).  A: n x d fp32 row-major (lda),
 * Rinv: d x d fp64 row-major (device).  The contraction runs on the tensor cores with every product of
 * two-term fp32 splits formed; accuracy: |lambda - exact| <= 2^-14 sum_j sum_l |A_il||Rinv_lj| + 2^-17
 * lambda.  d <= 64 with d % 4 == 0, lda % 4 == 0, 16-byte aligned A and n < 2^31 takes the
 * tensor-core kernel; other shapes (d <= FCT_MAX_D) a SIMT fp32 kernel with the same tolerance.
 * workspace: l1_rownorm_exact_workspace_bytes(n, d) device bytes.
 */
size_t l1_rownorm_exact_workspace_bytes(int64_t n, int64_t d);
fct_status l1_rownorm_exact(const float* A, int64_t n, int64_t d, int64_t lda, const double* Rinv,
                            float* lambda, double* lambda_sum, void* workspace,
                            size_t workspace_bytes, void* stream);
/* p[i] = (float)((double)lambda[i] / *lambda_total)   (t_i of P:L2028-2033). */
fct_status l1_probs(const float* lambda, int64_t n, const double* lambda_total, float* p,
                    void* stream);
/* Single-device convenience: l1_rownorm (with a zeroed local sum) followed by l1_probs.
 * lambda_sum (device fp64, may be NULL) receives the total. */
fct_status l1_rownorm_probs(const float* A, int64_t n, int64_t d, int64_t lda,
                            const double* Rinv, const float* Pi2, int32_t k, float* lambda,
                            float* p, double* lambda_sum, void* workspace,
                            size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * Bernoulli l1 sampling (l1 sampling lemma P:L1258-1268 with s := m):
 *     phat_i = min(1, m * (double)p[i])   (exact in fp64 for m <= 2^29)
 *     keep row i  iff  u_i < phat_i,  u_i = u53(rng_u64(seed, 9, row_base + i))
 *     idx[]    = kept GLOBAL row indices row_base + i, strictly increasing (int64)
 *     weight[] = 1.0 / phat_i (fp64, IEEE division)        -- D_ii = 1/phat_i
 *     *count   = number kept (device int64; may exceed capacity: only the first `capacity`
 *                entries are written -- compare on the host).
 * rng_u64(seed, stream, i) = mix64(mix64(seed + G(stream+1)) + G(i+1)), G = 0x9E3779B97F4A7C15,
 * mix64 = SplitMix64 finaliser; u53(x) = (x >> 11) * 2^-53.  Recommended capacity: 2m + 64
 * (S <= 2s w.p. >= 1 - e^{-3s/8}).  Bit-exact given p and the uniforms.
 */
size_t l1_sample_workspace_bytes(int64_t n);
fct_status l1_sample(const float* p, int64_t n, int64_t row_base, int64_t m, uint64_t seed,
                     int64_t* idx, double* weight, int64_t capacity, int64_t* count,
                     void* workspace, size_t workspace_bytes, void* stream);
/* Same with explicit uniforms u[n] in [0,1) (device fp64) instead of the generator. */
fct_status l1_sample_u(const float* p, const double* u, int64_t n, int64_t row_base,
                       int64_t m, int64_t* idx, double* weight, int64_t capacity,
                       int64_t* count, void* workspace, size_t workspace_bytes, void* stream);

/* NEXT-4: multinomial sampling -- exactly m i.i.d. row draws with probability
 * proportional to p (the "sample m rows with probabilities p_i" reading of P:L1258-1268 / P:L2178-2188,
 * drawn with replacement), from an exact fixed-point CDF so that the result is bit-exact:
 *   F = 62 - ceil(log2 n) - e with max_i p_i < 2^e;  W_i = floor(p_i 2^F) (uint64; p_i <= 0 or NaN -> 0);
 *   CDF_i = sum_{t<=i} W_t;  T = CDF_{n-1} (< 2^62)  -> *total (device uint64; 0: no positive p,
 *   then idx[] = -1, weight[] = 0);  X_j = rng_u64(seed, 10, j) >> 11;  target_j = (X_j T) >> 53;
 *   idx[j] = row_base + min{i : CDF_i > target_j};  weight[j] = (double)T / ((double)m (double)W_idx)
 *   (= 1/(m phat_i), the Horvitz-Thompson weight).  idx/weight: m entries each (device).
 * workspace: l1_sample_multinomial_workspace_bytes(n) device bytes.
 */
size_t l1_sample_multinomial_workspace_bytes(int64_t n);
fct_status l1_sample_multinomial(const float* p, int64_t n, int64_t m, uint64_t seed, int64_t row_base,
                                 int64_t* idx, double* weight, uint64_t* total, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * NEXT-2: the coreset l1 regression of FastCauchyRegression, steps 6-8
 * (Thm P:L2955-2980: x_hat minimises ||D(Ax - b)||_1).  X = [A, -b]
 * (P:L2915-2917): n x q fp32 row-major (ldx), the last column is -b.
 *
 * l1_coreset_gather: Z[j, :] = weight[j] * (double)X[idx[j] - row_base, :] for j < min(*count,
 *   capacity) -- the rows of D X, so that sum_j |Z_j . [x; 1]| = ||D(Ax - b)||_1 over the sample.
 *   idx/weight as written by l1_sample / l1_probs_sample / l1_sample_multinomial (device);
 *   idx == NULL: rows 0..m-1; weight == NULL: 1; count == NULL: m = capacity (device int64 else).
 *   Z: capacity x q fp64, row stride ldz >= q (device, caller-owned).  An index outside
 *   [row_base, row_base + n) yields a NaN row (the solve then reports status 2).  Asynchronous.
 * l1_lad_solve: x[0..q-2] = argmin_x sum_{j < m} |Z_j . [x; 1]| (m = *m, device int64, clamped to
 *   capacity; m == NULL: capacity).  Primal-dual interior-point method (Mehrotra predictor-corrector)
 *   on the LP  min 1'(u + v) s.t. Z[:, :q-1] x + u - v = -Z[:, q-1], u, v >= 0  and its dual
 *   max b'y s.t. A'y = 0, |y| <= 1, in fp64; one cooperative kernel, nothing returns to the host.
 *   Stops when f(x) - sum_j y_j rho_j(x) <= tol * max(f(x), 1e-5 f(0)) (f = the l1 objective at x,
 *   rho = -Z.[x;1]) or
 *   after max_iter iterations.  info (device, 8 doubles): [0] f(x), [1] sum y rho (dual value),
 *   [2] relative gap, [3] iterations, [4] max |A'y|, [5] status (0 converged, 1 max_iter,
 *   2 non-finite / breakdown), [6] m, [7] collapsed Cholesky pivots (rank-deficient coreset).
 *   2 <= q <= 128.  workspace: l1_lad_workspace_bytes(capacity, q) device bytes.
 */
fct_status l1_coreset_gather(const float* X, int64_t n, int64_t q, int64_t ldx, const int64_t* idx,
                             const double* weight, const int64_t* count, int64_t row_base,
                             int64_t capacity, double* Z, int64_t ldz, void* stream);
size_t l1_lad_workspace_bytes(int64_t capacity, int64_t q);
fct_status l1_lad_solve(const double* Z, const int64_t* m, int64_t capacity, int64_t q, int64_t ldz,
                        int32_t max_iter, double tol, double* x, double* info, void* workspace,
                        size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * NEXT-3: the FCT2 sketch (Sec. 3.2)
 *   Y = Pi1 A,  Pi1 = (8 / r1) sqrt(pi t / (2 s)) * C * H~,  H~ = blockdiag(G, ..., G) over t-row blocks of A
 *   (zero-padded to nb = ceil(n / t) blocks), G = sqrt(t / s) * R * (H_t / sqrt t) * D_t the SRHT the paper
 *   uses as its FJLT, the SAME G in every block.
 * signs_t: int8[t] (+-1) = D_t; sel: int32[s] distinct rows of H_t kept by R (in [0, t), not validated);
 * C: r1 x (nb s) fp32 i.i.d. standard Cauchy, row-major with row stride ldc >= nb s (device, caller-owned).
 * Y: r1 x d fp32 (overwritten).  t a power of two <= 32768, 1 <= s <= t, nb <= 65535.
 * workspace: fct2_workspace_bytes(n, d, t, s, r1) device bytes (Z = H~ A in fp32 and an fp64 r1 x d
 * accumulator).  Asynchronous on `stream`; argument errors are reported before anything is enqueued.
 */
size_t fct2_workspace_bytes(int64_t n, int64_t d, int32_t t, int32_t s, int32_t r1);
fct_status fct2_sketch(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs_t,
                       const int32_t* sel, const float* C, int64_t ldc, int32_t t, int32_t s, int32_t r1,
                       float* Y, void* workspace, size_t workspace_bytes, void* stream);

/* Fused a9 + a10 (what the pipeline runs): p[i] = (float)((double)lambda[i] / *lambda_total)
 * exactly as l1_probs, then the Bernoulli sampling of l1_sample on that p, in ONE pass over
 * lambda (single-pass decoupled look-back compaction).  Outputs (p, idx, weight, count) are
 * bit-identical to l1_probs followed by l1_sample.  workspace: l1_probs_sample_workspace_bytes(n)
 * device bytes (zeroed by the call, on `stream`).  Errors as l1_sample.
 */
size_t l1_probs_sample_workspace_bytes(int64_t n);
fct_status l1_probs_sample(const float* lambda, int64_t n, const double* lambda_total,
                           int64_t row_base, int64_t m, uint64_t seed, float* p, int64_t* idx,
                           double* weight, int64_t capacity, int64_t* count, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * Whole single-device hot path: sketch -> condition -> row-norm ->
 * probabilities -> sample, all enqueued on `stream` (device pointers).  Y (r1 x d fp32),
 * R, Rinv (d x d fp64), lambda, p (n fp32), idx/weight (capacity), count, info are outputs.
 */
size_t fct_pipeline_workspace_bytes(int64_t n, int64_t d, int32_t s, int32_t r1, int32_t k);
fct_status fct_pipeline(const float* A, int64_t n, int64_t d, int64_t lda, const int8_t* signs,
                        const float* cauchy_diag, const int32_t* hash_rows, int32_t s,
                        int32_t r1, const float* Pi2, int32_t k, int64_t m, uint64_t seed,
                        float* Y, double* R, double* Rinv, float* lambda, float* p,
                        int64_t* idx, double* weight, int64_t capacity, int64_t* count,
                        int32_t* info, void* workspace, size_t workspace_bytes, void* stream);

/* The same pipeline from HOST buffers (end-to-end entry point).  A_host, signs_host,
 * cauchy_host, hash_host, Pi2_host are HOST pointers (pinned memory recommended); the inputs
 * are copied to the device on `stream` (the aux arrays first, then A in s-aligned chunks of
 * ~512 MiB); the sketch of each chunk runs on an internal second stream as soon as that chunk
 * has landed (accumulated in fp64), so the sketch overlaps the copy of the later chunks; the
 * row norms, which need all of A, start after the last chunk.
 * dev_A (n x lda fp32), dev_aux (fct_pipeline_aux_bytes) are caller-owned device buffers
 * that receive the inputs.  Outputs idx_host/weight_host (capacity), *count_host are HOST
 * memory; the call returns after they are valid (it synchronises `stream`).  Device copies of
 * Y, R, Rinv, lambda, p live in the workspace-derived buffers of fct_pipeline and are
 * discarded.  Returns FCT_ERR_CAPACITY if count > capacity (count still written),
 * FCT_ERR_SINGULAR if the conditioning failed even with its shifted fallback (info > 0).
 */
size_t fct_pipeline_aux_bytes(int64_t n, int64_t d, int32_t s, int32_t k);
size_t fct_pipeline_host_workspace_bytes(int64_t n, int64_t d, int32_t s, int32_t r1, int32_t k,
                                         int64_t capacity);
fct_status fct_pipeline_host(const float* A_host, int64_t n, int64_t d, int64_t lda,
                             const int8_t* signs_host, const float* cauchy_host,
                             const int32_t* hash_host, int32_t s, int32_t r1,
                             const float* Pi2_host, int32_t k, int64_t m, uint64_t seed,
                             int64_t* idx_host, double* weight_host, int64_t capacity,
                             int64_t* count_host, float* dev_A, void* dev_aux,
                             void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FCT_H_ */
