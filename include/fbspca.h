/*
 * fbspca.h -- C ABI of the B200 (sm_100a) Fast Fourier-Bessel steerable PCA hot path.
 *
 * Method: Zhao, Shkolnisky, Singer, "Fast Steerable Principal Component Analysis"
 * (arXiv 1412.0781).  "P:n" cites line n of that paper's text.
 *
 *   Algorithm 1  fbspca_expand      images -> FB coefficients a_{k,q}
 *   Algorithm 2  fbspca_covariance  C^(k) = Re(A_k A_k^*)/n, mean at k=0 only
 *                            fbspca_eig         C^(k) = U_k diag(lambda^(k)) U_k^T
 *                            fbspca_svd         the same eigenpairs from the SVD of A_k (n < p_k)
 *                            fbspca_radial_eigenfunctions  f^{k,l}(xi_j) (Alg. 2 line 5)
 *   NEXT-1 (denoising)       fbspca_backproject  a_k = U_k c_k (+ mean): filtered steerable coefficients -> FB
 *                            fbspca_synthesize   FB coefficients -> pixel images (Eq. (IFT_FB))
 *   NEXT-2 (parameters)      fbspca_estimate_params  sigma^2, R, c from a stack
 *                            fbspca_project     c^i_{k,l} = sum_q a^i_{k,q} u_l^(k)(q) (+ filter)
 *
 * Conventions (all fixed):
 *   - images: n x L x L, row-major, axis 0 = i1 (multiplies xi_1 = xi cos theta),
 *     pixel a <-> i = a - floor(L/2)  (reading Q3).
 *   - Fourier sum with unit prefactor: F(I)(xi) = sum_i I(i) e^{-2 pi i xi.i}  (Eq. (nufft), reading Q1).
 *   - coefficients ("coefficient layout"): complex, k-major.  Block k (k = 0..k_max) is a p_k x ld matrix
 *     starting at complex element coef_off[k]*ld, row q (q = 0..p_k-1, the paper's q-1), column = image,
 *     images contiguous, re/im interleaved.  ld = the number of images of the call (n or n_local).
 *     k = 0 has Im = 0 (reading Q8).  Only k >= 0 is stored: a_{-k,q} = conj(a_{k,q}).
 *   - covariance blocks ("packed layout", fp64): for each k the upper triangle of C^(k), row-major over
 *     q <= q', starting at blk_off[k]; total blk_off[k_max+1].
 *   - eigenpairs (fp64): evals at coef_off[k] + l (descending per k), evecs U_k row-major p_k x p_k at
 *     evec_off[k] (element [q][l] = u_l^(k)(q)); sign: largest-|u| entry positive (reading Q10).
 *
 * Ownership: every pointer argument except the plan is owned by the caller.  "d_" pointers are device
 * pointers on the plan's device; all calls are asynchronous on the given stream unless stated, and a plan
 * must not be used concurrently from two streams.  The plan owns its tables and a workspace sized by
 * max_batch.  The hot-path calls (fbspca_expand, fbspca_covariance*, fbspca_eig, fbspca_project, fbspca_step
 * after its first call with given arguments) allocate no device memory.  The exceptions, each stated at its
 * declaration: the first fbspca_covariance / fbspca_step with a given communicator (NCCL-registered partial
 * buffer), the first fbspca_synthesize (radial tables), fbspca_svd (stream-ordered workspace) and
 * fbspca_estimate_params (not a plan call).
 *
 * Errors: every call returns fbspca_status; fbspca_last_error() returns a thread-local message.
 */
#ifndef FBSPCA_H
#define FBSPCA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fbspca_plan_s* fbspca_plan_t;   /* opaque */
typedef void* fbspca_stream_t;                 /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  FBSPCA_OK = 0,
  FBSPCA_ERR_ARG = 1,      /* null/misaligned pointer, n < 1, n_total < n_local, bad mode        */
  FBSPCA_ERR_CONFIG = 2,   /* c not in (0, 1/2], R < 2 or cR < 1, R > L/2, eps out of range, ...   */
  FBSPCA_ERR_CUDA = 3,     /* a CUDA runtime error (message carries cudaGetErrorString)           */
  FBSPCA_ERR_NCCL = 4,     /* NCCL missing or failed                                             */
  FBSPCA_ERR_NUMERIC = 5   /* Jacobi did not converge (message names k)                           */
} fbspca_status;

typedef enum { FBSPCA_F32 = 0, FBSPCA_F64 = 1 } fbspca_dtype;

/* Build a plan (Alg. 1 lines 1-2): census R_{k,q+1} <= 2 pi c R (Eq. (criterion1)),
 * n_xi = ceil(4cR), n_theta = ceil(16cR), Gauss-Legendre nodes on [0,c], the radial
 * table N_{k,q} J_k(R_{k,q} xi_j/c) xi_j w_j (2 pi/n_theta) (Eq. (a) P:195 with the 1/n_theta of
 * Eq. (1DFFT) P:189 folded in), and the NUFFT window (width from eps) and deapodisation.
 *   L        image side (>= 4).  c band limit in (0, 1/2].  R support radius, 2 <= R <= L/2, cR >= 1.
 *            2L and n_theta must factor into 2, 3, 5, 7, 11, 13 and n_theta must be even, else FBSPCA_ERR_CONFIG.
 *   eps      NUFFT accuracy target, [1e-14, 1e-3]; <= 0 picks the default (1e-5 for F32, 1e-12 for F64).
 *            F32 rejects eps < 1e-6.  The window gets w = ceil(log10(1/eps)) + 1 taps per axis at oversampling ~2
 *            (F32: clamped to [5, 7]; F64: 13), which holds the per-image coefficient
 *            relative l2 error against the exact Fourier sum (reading Q12) to <= max(4 eps, 4e-6) for F32
 *            (measured at L = 128: 6.0e-5 at eps = 1e-4 / w = 5, 5.8e-6 at the default 1e-5 / w = 6, 1.3e-6 at
 *            1e-6 / w = 7; tests/test_gpu_parity_full.py) and <= 1e-9 for F64.
 *   dt       FBSPCA_F32: images float, coefficients complex64.  FBSPCA_F64: double / complex128.
 *   device   CUDA device ordinal, or -1 for a host-only plan (census/tables only; every compute call
 *            on it returns FBSPCA_ERR_ARG).  Synchronous.
 *   max_batch  images per internal batch (workspace size); <= 0 picks 4096. */
fbspca_status fbspca_plan(int L, double c, double R, double eps, fbspca_dtype dt, int device,
                          int64_t max_batch, fbspca_plan_t* out);

/* Read-only views into the plan (valid until fbspca_destroy).  Any output pointer may be NULL.
 *   p_k[k_max+1]; coef_off[k_max+2] (coef_off[k_max+1] = sum p_k); blk_off[k_max+2] (packed fp64
 *   covariance; blk_off[k_max+1] = total); evec_off[k_max+2]. */
fbspca_status fbspca_plan_info(fbspca_plan_t plan, int* n_xi, int* n_theta, int* k_max,
                               const int** p_k, const int64_t** coef_off, const int64_t** blk_off,
                               const int64_t** evec_off);

/* Extra plan facts: NUFFT oversampled grid M, window width w, kernel shape beta, number of column
 * phases of the fused polar kernel, its dynamic shared memory bytes, and the census zeros R_{k,q}
 * (host array, q = 1..p_k, laid out like coef_off) and GL nodes/weights (host, n_xi each). */
fbspca_status fbspca_plan_detail(fbspca_plan_t plan, int* M, int* w, double* beta, int* n_phase,
                                 int* smem_bytes, const double** zeros, const double** xi,
                                 const double** wq);

/* Host-side plan query (no device work): the angular sampling of each ring and K4's first ring per k.
 *   ring_stride  n_xi ints (caller-owned, may be NULL): s_j -- ring j is sampled at theta_l = 2 pi l / n_theta for
 *                l = 0, s_j, 2 s_j, .. (n_theta / s_j angles).  s_j > 1 only for the M = 256 fp32 kernel, where
 *                n_theta / s_j >= kneed(j) + kc(j) keeps every coefficient the ring feeds free of angular aliases
 *                (kc: the Bessel band limit of the image's angular content on the ring, reading Q21 of DESIGN.md);
 *                the paper's grid (Eq. (1DFFT)) is s_j = 1.
 *   k_first_ring k_max + 1 ints (caller-owned, may be NULL): kj0[k], the first ring of Eq. (a)'s sum K4 reads for
 *                block k (rings below carry |T_k| < 1e-9 max |T_k|; 0 for fp64 plans).
 * Errors: FBSPCA_ERR_ARG for a null plan. */
fbspca_status fbspca_plan_rings(fbspca_plan_t plan, int* ring_stride, int* k_first_ring);

/* Alg. 1 lines 3-4: a = T* I for n images.  NUFFT (K1 pad+deapodise+2-D FFT, K2 window gather
 * to the half-plane polar nodes), K3 angular FFT (Eq. (1DFFT)), K4 radial quadrature (Eq. (a)).
 *   d_images  n x L x L (float or double per dt), device.   d_coeffs  sum_k p_k x n complex (coefficient
 *   layout, ld = n), device.  Streams any n in batches of max_batch. */
fbspca_status fbspca_expand(fbspca_plan_t plan, const void* d_images, int64_t n, void* d_coeffs,
                            fbspca_stream_t stream);

/* Alg. 2 lines 1-4, data-parallel form: K5 accumulates, over this rank's n_local
 * coefficient columns, S_k = sum_i Re(a_k a_k^*) (packed), s_0 = sum_i a_{0,i} and the count; then, if
 * nccl_comm != NULL, ONE in-place ncclAllReduce(sum, fp64) of that buffer across ranks; then finalises
 *   C^(0) = S_0/n - s_0 s_0^T / n^2   (= (1/n) sum (a_0 - m)(a_0 - m)^T, Eq. (ck_0) P:348 after P:394),
 *   C^(k) = S_k / n                   (Eq. (ck)),     m = s_0 / n,
 * with n the all-reduced count (= n_total).  d_coeffs: coefficient layout with ld = n_local.
 * d_blocks: blk_off[k_max+1] doubles (packed, finalised).  d_mean: p_0 doubles.  nccl_comm: an ncclComm_t
 * from fbspca_comm_init, or NULL for one GPU. */
fbspca_status fbspca_covariance(fbspca_plan_t plan, const void* d_coeffs, int64_t n_local,
                                int64_t n_total, void* nccl_comm, double* d_blocks, double* d_mean,
                                fbspca_stream_t stream);
/* With a communicator, the partial buffer is the plan's NCCL buffer for that communicator (ncclMemAlloc +
 * ncclCommRegister, NCCL >= 2.19; allocated synchronously on the first call with that communicator and
 * released by fbspca_destroy or fbspca_comm_destroy): K5's reduction writes into it and the all-reduce runs in
 * place on it.  After enqueueing the all-reduce the call polls ncclCommGetAsyncError; an asynchronous NCCL
 * failure is reported as FBSPCA_ERR_NCCL. */

/* One pipeline step (the bench's timed unit): fbspca_expand of n_local images into d_coeffs, then
 * fbspca_covariance (K5, the all-reduce when nccl_comm != NULL, finalise).  use_graph != 0: the first call
 * with a given argument set runs eagerly, the second captures the same launches (both streams of K5, the
 * all-reduce) into one CUDA graph, and every later call with those arguments replays it with one
 * cudaGraphLaunch; stream must then not be the legacy default stream.  Arguments as fbspca_expand and
 * fbspca_covariance. */
fbspca_status fbspca_step(fbspca_plan_t plan, const void* d_images, int64_t n_local, int64_t n_total,
                          void* nccl_comm, void* d_coeffs, double* d_blocks, double* d_mean, int use_graph,
                          fbspca_stream_t stream);

/* Same as fbspca_covariance but stops before the all-reduce: writes the un-finalised partial buffer
 * (packed S_k, then s_0 (p_0 doubles), then the count) to d_partial (blk_off[k_max+1] + p_0 + 1 doubles).
 * fbspca_covariance_finalize turns a (reduced) partial buffer into blocks and mean. */
fbspca_status fbspca_covariance_partial(fbspca_plan_t plan, const void* d_coeffs, int64_t n_local,
                                        double* d_partial, fbspca_stream_t stream);
fbspca_status fbspca_covariance_finalize(fbspca_plan_t plan, const double* d_partial, double* d_blocks,
                                         double* d_mean, fbspca_stream_t stream);

/* Streaming form: like fbspca_covariance_partial but ADDS this call's n_local columns into an existing
 * partial buffer (zero it once with cudaMemset or a first fbspca_covariance_partial).  Lets a caller
 * expand and accumulate a stack chunk by chunk (e.g. overlapping host->device copies with compute). */
fbspca_status fbspca_covariance_accumulate(fbspca_plan_t plan, const void* d_coeffs, int64_t n_local,
                                           double* d_partial, fbspca_stream_t stream);

/* In-place ncclAllReduce(sum, fp64) of a partial buffer over nccl_comm (no-op when nccl_comm == NULL). */
fbspca_status fbspca_allreduce_partial(fbspca_plan_t plan, double* d_partial, void* nccl_comm,
                                       fbspca_stream_t stream);

/* Alg. 2 line 4: batched cyclic (parallel-ordered) Jacobi in fp64, one block per CTA.
 * d_blocks packed (input), d_evals (coef_off[k_max+1] doubles), d_evecs (evec_off[k_max+1] doubles).
 * Synchronises the stream to check convergence (<= 30 sweeps); FBSPCA_ERR_NUMERIC names the block. */
fbspca_status fbspca_eig(fbspca_plan_t plan, const double* d_blocks, double* d_evals, double* d_evecs,
                         fbspca_stream_t stream);

/* Alg. 2 line 4, SVD form ("or perform SVD of A^(k) and take the left singular vectors";
 * the route for n < p_k), fp64, one CTA per block: the left singular vectors and squared singular values of
 * the real p_k x 2n matrix [Re A_k, Im A_k] / sqrt(n) (k = 0: A_0 - mean 1^T, Im taken as 0), i.e. the eigenpairs
 * of C^(k) = Re(A_k A_k^*)/n without forming C^(k), by one-sided (Hestenes) Jacobi.  Output in fbspca_eig's
 * layout, order and sign convention; U_k is complete (orthonormal p_k x p_k) when rank < p_k, with the zero
 * singular values last.
 *   d_coeffs  coefficient layout, ld = n (all the images: the route is single-device).  n >= 1.
 *   d_mean    p_0 doubles receiving the k = 0 mean, or NULL.
 *   Cost O(sweeps p_k^2 (n + p_k)) per block; workspace (2 n sum_k p_k + sum_k p_k^2 doubles) is allocated
 *   and freed stream-ordered inside the call.  Synchronises the stream to check convergence (<= 40 sweeps;
 *   FBSPCA_ERR_NUMERIC names the block).  For large n use fbspca_covariance + fbspca_eig. */
fbspca_status fbspca_svd(fbspca_plan_t plan, const void* d_coeffs, int64_t n, double* d_mean, double* d_evals,
                         double* d_evecs, fbspca_stream_t stream);

/* Alg. 2 line 5, Eq. (sPCArad): the radial eigenfunctions at the plan's GL nodes xi_j,
 *   f^{k,l}(xi_j) = sum_q u_l^(k)(q) N_{k,q} J_k(R_{k,q} xi_j / c),   fp64.
 * d_evecs: eigenvectors as written by fbspca_eig (evec_off layout).  d_f: coef_off[k_max+1] x n_xi doubles,
 * row coef_off[k] + l (l = 0..p_k-1), column j (xi_j from fbspca_plan_detail).  Asynchronous. */
fbspca_status fbspca_radial_eigenfunctions(fbspca_plan_t plan, const double* d_evecs, double* d_f,
                                           fbspca_stream_t stream);

/* Alg. 2 line 6 (Eq. (sPCAcoeff)) with optional filtering:
 *   out_k[l][i] = h^(k)_l sum_q u_l^(k)(q) (a^i_{k,q} - [k=0] m_q)
 *   mode 0: h = 1.   mode 1: Eq. (compselect) lambda > sigma2 (1 + sqrt(gamma_k))^2 (gamma_0 = p_0/n_total,
 *   gamma_k = p_k/(2 n_total)), then h = l/(l + sigma2), l = (lambda - sigma2)_+ (reading Q13), else 0.
 *   mode 2: as 1 with the spiked-model l.
 * d_coeffs / d_out: coefficient layout with ld = n (d_out may not alias d_coeffs). */
fbspca_status fbspca_project(fbspca_plan_t plan, const void* d_coeffs, int64_t n, const double* d_mean,
                             const double* d_evals, const double* d_evecs, double sigma2, int mode,
                             int64_t n_total, void* d_out, fbspca_stream_t stream);

/* NEXT-1: a_k = U_k c_k, plus m at k = 0 (Im kept 0) -- inverts Eq. (sPCAcoeff) P:364 for orthogonal U_k and undoes
 * the centring of Alg. 2 line 1.  With d_c = fbspca_project(mode 1 or 2) output these are the FB coefficients of
 * the denoised images.  d_c, d_coeffs_out: coefficient layout, ld = n (may not alias); d_mean p_0
 * doubles, d_evecs as from fbspca_eig.  Asynchronous. */
fbspca_status fbspca_backproject(fbspca_plan_t plan, const void* d_c, int64_t n, const double* d_mean,
                                 const double* d_evecs, void* d_coeffs_out, fbspca_stream_t stream);

/* NEXT-1: images from FB coefficients on the L x L pixel grid, Eq. (IFT_FB) P:108 read with i^{+k} in the
 * numerator (reading Q2): I(x) = sum_q a_{0,q} rho_{0,q}(r) + 2 Re sum_{k>=1,q} a_{k,q} rho_{k,q}(r) i^k e^{ik phi},
 * rho_{k,q}(r) = 2 c sqrt(pi) (-1)^q R_{k,q} J_k(2 pi c r) / ((2 pi c r)^2 - R_{k,q}^2) (q = 1..p_k), for pixels with
 * r <= R (zero elsewhere, the compact support P:115); axis 0 = i1 (Q3).  fp64 arithmetic.  d_coeffs: coefficient
 * layout, ld = n.  d_images: n x L x L (float or double per dt), n <= 65535 per call.  The first call builds
 * the plan's radial tables on the host and uploads them (cudaMalloc + synchronous copies: the one allocating
 * call of the synthesis path).  Asynchronous otherwise. */
fbspca_status fbspca_synthesize(fbspca_plan_t plan, const void* d_coeffs, int64_t n, void* d_images,
                                fbspca_stream_t stream);

/* NEXT-2 (Fig. 5): noise variance, support radius and band limit of an image stack, as the paper
 * picks R = 98 and c = 0.196 for its ribosome images.  Per-pixel mean and variance (one streaming pass) and the
 * mean power spectrum of the mean-subtracted images, |DFT2|^2 / L^2 (white noise of variance s^2 sits at s^2), are
 * formed on the GPU (fp64 accumulation); radial averages in bins b = floor(r + 1/2) (pixel offsets a - floor(L/2),
 * integer frequencies) are formed on the host, then
 *   sigma2 = mean variance over radius bins ceil(0.45 L) <= b < floor(L/2)   (the outer 10 % of radii below L/2),
 *   R      = smallest b with sum_{b' <= b} max(var_b' - sigma2, 0) b'  >= fraction x its total over b < floor(L/2),
 *   c      = b / L for the smallest frequency bin 1 <= b <= floor(L/2) with the same rule on the power spectrum.
 * d_images: n x L x L (float or double per dt) on `device`; L must be 2^a 3^b 5^c 7^d 11^e 13^f; n >= 2; 0 < fraction <= 1
 * (the paper uses 0.999).  Synchronous; allocates and frees its own scratch (this is not a plan call).
 * FBSPCA_ERR_NUMERIC when no variance / power exceeds the noise level (pure noise). */
fbspca_status fbspca_estimate_params(int L, fbspca_dtype dt, int device, const void* d_images, int64_t n,
                                     double fraction, double* sigma2, double* R, double* c);

/* NCCL plumbing (libnccl.so.2 is dlopen'ed on first use).  unique_id: 128 bytes.  fbspca_comm_destroy first
 * releases the plans' registered buffers for that communicator. */
fbspca_status fbspca_nccl_unique_id(void* unique_id_out);
fbspca_status fbspca_comm_init(const void* unique_id, int nranks, int rank, void** nccl_comm_out);
fbspca_status fbspca_comm_destroy(void* nccl_comm);

/* Failure detection: wait for `stream` while polling ncclCommGetAsyncError every 100 us.
 * Returns FBSPCA_OK when the stream's work is done; on an asynchronous NCCL error, or when timeout_s > 0
 * seconds pass first (a hung peer), aborts the communicator (ncclCommAbort) and returns FBSPCA_ERR_NCCL
 * naming the cause.  Synchronous. */
fbspca_status fbspca_comm_wait(void* nccl_comm, fbspca_stream_t stream, double timeout_s);

/* Per-kernel-family device times when timing is on (CUDA events recorded around each launch on the
 * call's stream; off by default).  fbspca_get_timing synchronises those events, returns *count family
 * names, ms[0..count) = summed milliseconds and ms[count..2*count) = number of timed launch regions since
 * the previous fbspca_get_timing, then resets the accumulators. */
fbspca_status fbspca_set_timing(fbspca_plan_t plan, int enabled);
fbspca_status fbspca_get_timing(fbspca_plan_t plan, int* count, const char* const** names,
                                const float** ms);

void fbspca_destroy(fbspca_plan_t plan);
const char* fbspca_last_error(void);
const char* fbspca_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FBSPCA_H */
