// kernels_linalg.cu -- K4 radial quadrature, K5 covariance accumulation + finalise, K6 batched Jacobi,
// K7 projection / filtering.  SIMT versions (fp32 FFMA with fp64 accumulation across batches).
#include <cuda_runtime.h>

#include <algorithm>

#include "fft_device.cuh"
#include "internal.h"

namespace fbspca {

// ---------------------------------------------------------------- K4: Eq. (a)
// For block k:  D[row][q] = sum_j ghat[k][row][j] * T[coef_off[k] + q][j],  row = 2 b + part (re/im),
// written to coeffs (real view) at [(coef_off[k] + q) * 2 ld + 2 i0 + row].  Im of k = 0 set to 0 (Q8).
template <typename T>
__global__ void __launch_bounds__(256)
radial_kernel(const T* __restrict__ ghat, const T* __restrict__ table, const int* __restrict__ p,
              const int64_t* __restrict__ coef_off, const int* __restrict__ kj0, int nb, int n_xi, int64_t kstride,
              int64_t i0, int64_t ld, T* __restrict__ out) {
  constexpr int BM = 64, BN = 64, BK = 32;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int k = blockIdx.y;
  const int pk = p[k];
  const int q0 = blockIdx.z * BN;
  if (q0 >= pk) return;
  const int rows = 2 * nb;
  const int r0 = blockIdx.x * BM;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const T* A = ghat + (int64_t)k * kstride;
  const T* B = table + coef_off[k] * n_xi;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  const int jlo = kj0[k];                    // rings below carry structural zeros of T_k (plan.cpp) and no ghat
  for (int j0 = jlo; j0 < n_xi; j0 += BK) {
    for (int e = tid; e < BM * BK; e += 256) {
      const int rr = e / BK, jj = e - rr * BK;
      const int r = r0 + rr, j = j0 + jj;
      As[jj][rr] = (r < rows && j < n_xi) ? A[(int64_t)r * n_xi + j] : T(0);
      const int q = q0 + rr;
      Bs[jj][rr] = (q < pk && j < n_xi) ? B[(int64_t)q * n_xi + j] : T(0);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][tx + 16 * i]; b[i] = Bs[kk][ty + 16 * i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
  const int64_t base = coef_off[k];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int q = q0 + ty + 16 * j;
    if (q >= pk) continue;
    T* o = out + (base + q) * 2 * ld + 2 * i0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + tx + 16 * i;
      if (r < rows) o[r] = (k == 0 && (r & 1)) ? T(0) : acc[i][j];
    }
  }
}

cudaError_t launch_radial(const Plan& P, int64_t nb, int64_t i0, int64_t ld, void* d_coeffs, cudaStream_t s) {
  int pmax = P.p[0];
  dim3 grid((unsigned)((2 * nb + 63) / 64), (unsigned)(P.k_max + 1), (unsigned)((pmax + 63) / 64));
  if (P.dt == FBSPCA_F32)
    radial_kernel<float><<<grid, 256, 0, s>>>((const float*)P.d_ghat, (const float*)P.d_table, P.d_p, P.d_coef_off,
                                              P.d_kj0, (int)nb, P.n_xi, P.pp.ghat_kstride, i0, ld, (float*)d_coeffs);
  else
    radial_kernel<double><<<grid, 256, 0, s>>>((const double*)P.d_ghat, (const double*)P.d_table, P.d_p,
                                               P.d_coef_off, P.d_kj0, (int)nb, P.n_xi, P.pp.ghat_kstride, i0, ld,
                                               (double*)d_coeffs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K5: Eqs. (ck), (ck_0)
// partial[blk_off[k] + packed(q, q')] += sum_{c in batch} A_k[q][c] A_k[q'][c]   (q <= q')
// where A_k is the real view (re/im interleaved along images) of block k: sum over re and im gives
// Re(a a^*).  k = 0 accumulates in fp64 (reading F9) and also s_0 and the count.
__device__ __forceinline__ int64_t packed_idx(int q, int qq, int p) {
  return (int64_t)q * p - (int64_t)q * (q - 1) / 2 + (qq - q);
}

template <typename T, typename Acc>
__device__ void cov_tile(const T* __restrict__ Ak, int pk, int64_t ld2, int64_t c0, int64_t ncol, int tq, int tqq,
                         double* __restrict__ dst, T (*S1)[64 + 1], T (*S2)[64 + 1]) {
  constexpr int BK = 32;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int qa = tq * 64, qb = tqq * 64;
  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = Acc(0);
  for (int64_t cb = 0; cb < ncol; cb += BK) {
    for (int e = tid; e < 64 * BK; e += 256) {
      const int rr = e / BK, cc = e - rr * BK;
      const int64_t c = cb + cc;
      const int q1 = qa + rr, q2 = qb + rr;
      S1[cc][rr] = (q1 < pk && c < ncol) ? Ak[(int64_t)q1 * ld2 + c0 + c] : T(0);
      S2[cc][rr] = (q2 < pk && c < ncol) ? Ak[(int64_t)q2 * ld2 + c0 + c] : T(0);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      Acc a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = Acc(S1[kk][tx + 16 * i]); b[i] = Acc(S2[kk][ty + 16 * i]); }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = qa + tx + 16 * i, qq = qb + ty + 16 * j;
      if (q < pk && qq < pk && q <= qq) dst[packed_idx(q, qq, pk)] = double(acc[i][j]);
    }
}

// Split-K: CTA (k, tile pair, chunk) sums its kCovChunk images of the batch and STORES the chunk's partial
// (fp64) into scratch[chunk][.]; cov_reduce_kernel then adds the chunks in fixed order -> deterministic.
template <typename T>
__global__ void __launch_bounds__(256)
cov_accum_kernel(const T* __restrict__ coeffs, const int* __restrict__ p, const int64_t* __restrict__ coef_off,
                 const int64_t* __restrict__ blk_off, int64_t ld, int64_t i0, int64_t nb, int k_max,
                 double* __restrict__ scratch, int64_t scratch_stride) {
  __shared__ T S1[32][64 + 1];
  __shared__ T S2[32][64 + 1];
  const int k = blockIdx.x;
  const int pk = p[k];
  const int nt = (pk + 63) / 64;
  int pair = blockIdx.y, tq = 0;
  while (tq < nt && pair >= nt - tq) { pair -= nt - tq; ++tq; }
  if (tq >= nt) return;
  const int tqq = tq + pair;
  const int64_t c_img0 = i0 + (int64_t)blockIdx.z * kCovChunk;
  const int64_t c_nb = min((int64_t)kCovChunk, i0 + nb - c_img0);
  const T* Ak = coeffs + coef_off[k] * 2 * ld;
  double* dst = scratch + (int64_t)blockIdx.z * scratch_stride + blk_off[k];
  if (k == 0)
    cov_tile<T, double>(Ak, pk, 2 * ld, 2 * c_img0, 2 * c_nb, tq, tqq, dst, S1, S2);
  else
    cov_tile<T, T>(Ak, pk, 2 * ld, 2 * c_img0, 2 * c_nb, tq, tqq, dst, S1, S2);
  if (k == 0 && blockIdx.y == 0) {
    double* s0 = scratch + (int64_t)blockIdx.z * scratch_stride + blk_off[k_max + 1];
    for (int q = threadIdx.x; q < pk; q += blockDim.x) {
      double s = 0;
      const T* row = Ak + (int64_t)q * 2 * ld + 2 * c_img0;
      for (int64_t c = 0; c < c_nb; ++c) s += double(row[2 * c]);
      s0[q] = s;
    }
    if (threadIdx.x == 0) s0[pk] = double(c_nb);
  }
}

// partial[i] += sum over chunks (fixed order).  nsub0 > 0: the k = 0 block [0, blk1) and s_0/count [s0_at, total)
// come from scratch0 (nsub0 sub-chunks of stride0 = blk1 + p_0 + 1, s_0 at blk1) instead of scratch.
__global__ void cov_reduce_kernel(const double* __restrict__ scratch, int64_t stride, int nchunk, int64_t total,
                                  const double* __restrict__ scratch0, int nsub0, int64_t blk1, int64_t s0_at,
                                  double* __restrict__ partial) {
  const int64_t stride0 = blk1 + (total - s0_at);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double s = partial[i];
    // loads in groups of 8 issued before the (fixed-order) adds: memory-level parallelism, same rounding
    const bool k0 = nsub0 > 0 && (i < blk1 || i >= s0_at);
    const double* src = k0 ? scratch0 + (i < blk1 ? i : blk1 + (i - s0_at)) : scratch + i;
    const int64_t st = k0 ? stride0 : stride;
    const int nc = k0 ? nsub0 : nchunk;
    int c = 0;
    for (; c + 8 <= nc; c += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[(int64_t)(c + u) * st];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; c < nc; ++c) s += src[(int64_t)c * st];
    partial[i] = s;
  }
}

bool cov_uses_tc(const Plan& P, int64_t ld) {
  return P.dt == FBSPCA_F32 && P.use_tc && P.k_max >= 1 && ((P.p[1] + 15) & ~15) <= 256 && (ld % 2) == 0;
}

cudaError_t launch_cov_accum(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb,
                             double* d_partial, cudaStream_t s) {
  const int nt = (P.p[0] + 63) / 64;
  const bool tc_ok = cov_uses_tc(P, ld);
  // images per split-K chunk: kCovChunk (SIMT), cov_tma_chunk() (tensor path)
  const int chunk = tc_ok ? cov_tma_chunk() : kCovChunk;
  const int nchunk = (int)((nb + chunk - 1) / chunk);
  if (nchunk > kCovMaxChunks) return cudaErrorInvalidValue;
  const int64_t total = P.blk_off[P.k_max + 1] + P.p[0] + 1;
  dim3 grid((unsigned)(P.k_max + 1), (unsigned)(nt * (nt + 1) / 2), (unsigned)nchunk);
  // k >= 1 on tcgen05 for p_1 <= 256 (p_k > 128: the big-block kernel, kernels_tma.cu)
  const bool tc = tc_ok;
  if (tc) {
    // k >= 1 on the tensor cores (TMA-fed, persistent); k = 0 (uncentred, mean^2/var ~ 10: F9) in fp64 on the
    // CUDA cores, forked onto the plan's side stream so the two overlap
    cudaError_t e = cudaEventRecord(P.ev_fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(P.side, P.ev_fork, 0);
    if (e == cudaSuccess) e = launch_cov_k0(P, d_coeffs, ld, i0, nb, P.side);
    if (e == cudaSuccess) e = cudaEventRecord(P.ev_join, P.side);
    if (e == cudaSuccess) e = launch_cov_tma(P, d_coeffs, ld, i0, nb, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, P.ev_join, 0);
    if (e != cudaSuccess) return e;
  } else if (P.dt == FBSPCA_F32)
    cov_accum_kernel<float><<<grid, 256, 0, s>>>((const float*)d_coeffs, P.d_p, P.d_coef_off, P.d_blk_off, ld, i0, nb,
                                                 P.k_max, P.d_cov_scratch, total);
  else
    cov_accum_kernel<double><<<grid, 256, 0, s>>>((const double*)d_coeffs, P.d_p, P.d_coef_off, P.d_blk_off, ld, i0,
                                                  nb, P.k_max, P.d_cov_scratch, total);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4 * 148);
  cov_reduce_kernel<<<blocks, 256, 0, s>>>(P.d_cov_scratch, total, nchunk, total, P.d_cov_scratch0,
                                           tc ? (int)((nb + kCovChunk0 - 1) / kCovChunk0) : 0, P.blk_off[1],
                                           P.blk_off[P.k_max + 1], d_partial);
  return cudaGetLastError();
}

// C^(0) = S_0/n - s0 s0^T/n^2, C^(k) = S_k/n, mean = s0/n   (n = all-reduced count)
__global__ void cov_finalize_kernel(const double* __restrict__ partial, const int* __restrict__ p,
                                    const int64_t* __restrict__ blk_off, int k_max, double* __restrict__ blocks,
                                    double* __restrict__ mean) {
  const int k = blockIdx.y;
  const int pk = p[k];
  const int64_t tot = blk_off[k_max + 1];
  const double* s0 = partial + tot;
  const double n = s0[p[0]];
  const int64_t npk = (int64_t)pk * (pk + 1) / 2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < npk; idx += (int64_t)gridDim.x * blockDim.x) {
    double v = partial[blk_off[k] + idx] / n;
    if (k == 0) {
      int q = 0;
      while (q + 1 < pk && packed_idx(q + 1, q + 1, pk) <= idx) ++q;
      const int qq = q + int(idx - packed_idx(q, q, pk));
      v -= (s0[q] / n) * (s0[qq] / n);
    }
    blocks[blk_off[k] + idx] = v;
  }
  if (k == 0 && blockIdx.x == 0)
    for (int q = threadIdx.x; q < pk; q += blockDim.x) mean[q] = s0[q] / n;
}

cudaError_t launch_cov_finalize(const Plan& P, const double* d_partial, double* d_blocks, double* d_mean,
                                cudaStream_t s) {
  const int64_t maxp = (int64_t)P.p[0] * (P.p[0] + 1) / 2;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((maxp + 255) / 256, 64)), (unsigned)(P.k_max + 1));
  cov_finalize_kernel<<<grid, 256, 0, s>>>(d_partial, P.d_p, P.d_blk_off, P.k_max, d_blocks, d_mean);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K6: batched parallel-order Jacobi
// One CTA per block.  Round-robin pairing (p' = p rounded up to even; p'/2 disjoint pairs per round,
// p'-1 rounds per sweep); rotations from Golub-Van Loan sym.schur2, applied as A <- J^T A J, V <- V J.
constexpr int kEigMaxSmemA = 144 * 144;   // doubles of A kept in shared memory

__global__ void __launch_bounds__(256)
eig_kernel(const double* __restrict__ blocks, const int* __restrict__ p, const int64_t* __restrict__ blk_off,
           const int64_t* __restrict__ coef_off, const int64_t* __restrict__ evec_off, double* __restrict__ evals,
           double* __restrict__ evecs, double* __restrict__ work, int* __restrict__ sweeps_out) {
  extern __shared__ double sh[];
  const int k = blockIdx.x;
  const int n = p[k];
  const int tid = threadIdx.x, nthr = blockDim.x;
  double* cs_c = sh;                 // pairs
  double* cs_s = sh + 128;
  int* pi = reinterpret_cast<int*>(sh + 256);
  int* qi = pi + 128;
  double* red = sh + 384;            // reduction scratch (nthr)
  double* A = (n * n <= kEigMaxSmemA) ? (sh + 384 + 256) : (work + 2 * evec_off[k]);
  double* V = work + 2 * evec_off[k] + (int64_t)n * n;
  const double* Bk = blocks + blk_off[k];
  for (int idx = tid; idx < n * n; idx += nthr) {
    const int r = idx / n, c = idx - r * n;
    const int q = min(r, c), qq = max(r, c);
    A[idx] = Bk[packed_idx(q, qq, n)];
    V[idx] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int np = n + (n & 1), npairs = np / 2;
  int sweep = 0;
  for (; sweep < 30 && n > 1; ++sweep) {
    double off = 0, dg = 0;
    for (int idx = tid; idx < n * n; idx += nthr) {
      const int r = idx / n, c = idx - r * n;
      const double v = A[idx] * A[idx];
      if (r == c) dg += v; else off += v;
    }
    red[tid] = off; __syncthreads();
    for (int st = nthr / 2; st > 0; st >>= 1) { if (tid < st) red[tid] += red[tid + st]; __syncthreads(); }
    off = red[0]; __syncthreads();
    red[tid] = dg; __syncthreads();
    for (int st = nthr / 2; st > 0; st >>= 1) { if (tid < st) red[tid] += red[tid + st]; __syncthreads(); }
    dg = red[0]; __syncthreads();
    if (off <= 1e-26 * dg || off == 0.0) break;         // off-diagonal Frobenius <= 1e-13 of the diagonal
    for (int round = 0; round < np - 1; ++round) {
      for (int i = tid; i < npairs; i += nthr) {
        auto pos = [&](int t) { return t == 0 ? 0 : 1 + (t - 1 + round) % (np - 1); };
        int a = pos(i), b = pos(np - 1 - i);
        int pp = min(a, b), qq = max(a, b);
        double c = 1, s = 0;
        if (qq < n) {
          const double apq = A[pp * n + qq];
          const double app = A[pp * n + pp], aqq = A[qq * n + qq];
          if (fabs(apq) > 1e-300 && fabs(apq) > 1e-18 * sqrt(fabs(app * aqq))) {
            const double tau = (aqq - app) / (2 * apq);
            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1 + tau * tau));
            c = 1 / sqrt(1 + t * t); s = t * c;
          }
        } else { pp = -1; }
        pi[i] = pp; qi[i] = qq; cs_c[i] = c; cs_s[i] = s;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int idx = tid; idx < npairs * n; idx += nthr) {
        const int i = idx / n, r = idx - i * n;
        const int pp = pi[i];
        if (pp < 0 || cs_s[i] == 0.0) continue;
        const int qq = qi[i];
        const double c = cs_c[i], s = cs_s[i];
        double x = A[r * n + pp], y = A[r * n + qq];
        A[r * n + pp] = c * x - s * y; A[r * n + qq] = s * x + c * y;
        x = V[r * n + pp]; y = V[r * n + qq];
        V[r * n + pp] = c * x - s * y; V[r * n + qq] = s * x + c * y;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int idx = tid; idx < npairs * n; idx += nthr) {
        const int i = idx / n, col = idx - i * n;
        const int pp = pi[i];
        if (pp < 0 || cs_s[i] == 0.0) continue;
        const int qq = qi[i];
        const double c = cs_c[i], s = cs_s[i];
        const double x = A[pp * n + col], y = A[qq * n + col];
        A[pp * n + col] = c * x - s * y; A[qq * n + col] = s * x + c * y;
      }
      __syncthreads();
    }
  }
  if (tid == 0) sweeps_out[k] = (n > 1) ? sweep : 0;
  // sort descending (ties: lower index first) and normalise signs (largest |u| positive, ties lowest q)
  for (int i = tid; i < n; i += nthr) {
    const double li = A[i * n + i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = A[j * n + j];
      rank += (lj > li) || (lj == li && j < i);
    }
    evals[coef_off[k] + rank] = li;
    int arg = 0; double best = -1;
    for (int r = 0; r < n; ++r) { const double a = fabs(V[r * n + i]); if (a > best) { best = a; arg = r; } }
    const double sg = V[arg * n + i] < 0 ? -1.0 : 1.0;
    double* U = evecs + evec_off[k];
    for (int r = 0; r < n; ++r) U[r * n + rank] = sg * V[r * n + i];
  }
}

cudaError_t launch_eig(const Plan& P, const double* d_blocks, double* d_evals, double* d_evecs, cudaStream_t s) {
  const int pmax = P.p[0];
  const int an = std::min(pmax * pmax, kEigMaxSmemA);
  const size_t smem = (384 + 256 + an) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  eig_kernel<<<P.k_max + 1, 256, smem, s>>>(d_blocks, P.d_p, P.d_blk_off, P.d_coef_off, P.d_evec_off, d_evals,
                                            d_evecs, P.d_eig_work, P.d_eig_sweeps);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Alg. 2 line 4, SVD form
// "or perform SVD of A^(k) and take the left singular vectors" -- the route for n < p_k.  Per block k the real
// p_k x m matrix W = [Re A_k, Im A_k] / sqrt(n) (m = 2n; k = 0: A_0 - mean 1^T with Im = 0, reading Q8) has
// W W^T = C^(k), so its left singular vectors / squared singular values are the eigenpairs of C^(k).  One-sided
// (Hestenes) Jacobi on the ROWS of W: rotate row pairs (p, q) until mutually orthogonal, accumulating U <- U J;
// then W = U diag(sigma) V^T with sigma_l^2 = |w_l|^2.  U is a product of rotations, so it is a complete
// orthonormal basis even when rank W = min(p_k, m) < p_k (the zero singular values).  One CTA per block, one warp
// per row pair of a round-robin round (the pairs of a round are disjoint), each pair's dot products reduced in a
// fixed order by one warp (deterministic).  The coefficient rows are contiguous (re, im interleaved): a column
// permutation of W, which leaves every row dot product unchanged.  W and U live in a per-call global workspace
// (L2-resident at the sizes this route is for).
template <typename T>
__global__ void __launch_bounds__(256)
svd_kernel(const T* __restrict__ coeffs, int64_t n, const int* __restrict__ p, const int64_t* __restrict__ coef_off,
           const int64_t* __restrict__ evec_off, double* __restrict__ work, double* __restrict__ mean_out,
           double* __restrict__ evals, double* __restrict__ evecs, int* __restrict__ sweeps_out) {
  __shared__ double smean[kSvdMaxP];
  __shared__ int rotated;
  const int k = blockIdx.x, pk = p[k];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t m = 2 * n;
  double* W = work + 2 * n * coef_off[k] + evec_off[k];     // p_k x m, then U (p_k x p_k)
  double* U = W + (int64_t)pk * m;
  const T* A = coeffs + 2 * n * coef_off[k];
  const double isn = 1.0 / sqrt(double(n));
  if (k == 0) {
    for (int q = warp; q < pk; q += nw) {
      double sacc = 0.0;
      for (int64_t i = lane; i < n; i += 32) sacc += double(A[(int64_t)q * m + 2 * i]);
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_down_sync(0xffffffffu, sacc, o);
      if (lane == 0) { smean[q] = sacc / double(n); if (mean_out) mean_out[q] = sacc / double(n); }
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < (int64_t)pk * m; e += blockDim.x) {
    const int q = int(e / m);
    const int64_t j = e - (int64_t)q * m;
    double v = double(A[e]);
    if (k == 0) v = (j & 1) ? 0.0 : v - smean[q];
    W[e] = v * isn;
  }
  for (int e = tid; e < pk * pk; e += blockDim.x) U[e] = (e / pk == e % pk) ? 1.0 : 0.0;
  // trace(W W^T) (rotation invariant): pairs with |w_p . w_q| <= 1e-28 tr are taken as orthogonal, so rows in
  // the numerical null space (|w|^2 ~ eps^2 tr when rank < p_k) stop rotating
  if (warp == 0) {
    double acc = 0;
    for (int64_t e = lane; e < (int64_t)pk * m; e += 32) acc = fma(W[e], W[e], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) smean[kSvdMaxP - 1] = acc;
  }
  __syncthreads();
  const double floor_g = 1e-28 * smean[kSvdMaxP - 1];
  const int np = pk + (pk & 1);
  int sweep = 0;
  for (; sweep < kSvdMaxSweeps && pk > 1; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < np - 1; ++round) {
      for (int i = warp; i < np / 2; i += nw) {
        auto pos = [&](int t) { return t == 0 ? 0 : 1 + (t - 1 + round) % (np - 1); };
        const int a = pos(i), b = pos(np - 1 - i);
        const int pp = min(a, b), qq = max(a, b);
        if (qq >= pk) continue;
        double* wp = W + (int64_t)pp * m;
        double* wq = W + (int64_t)qq * m;
        double al = 0, be = 0, ga = 0;
        for (int64_t j = lane; j < m; j += 32) {
          const double x = wp[j], y = wq[j];
          al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_down_sync(0xffffffffu, al, o);
          be += __shfl_down_sync(0xffffffffu, be, o);
          ga += __shfl_down_sync(0xffffffffu, ga, o);
        }
        al = __shfl_sync(0xffffffffu, al, 0); be = __shfl_sync(0xffffffffu, be, 0); ga = __shfl_sync(0xffffffffu, ga, 0);
        if (!(fabs(ga) > 1e-15 * sqrt(al * be)) || !(fabs(ga) > floor_g) || fabs(ga) < 1e-300) continue;
        const double zeta = (be - al) / (2 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        const double c = 1 / sqrt(1 + t * t), s = t * c;
        for (int64_t j = lane; j < m; j += 32) {
          const double x = wp[j], y = wq[j];
          wp[j] = c * x - s * y; wq[j] = s * x + c * y;
        }
        for (int r = lane; r < pk; r += 32) {
          const double x = U[r * pk + pp], y = U[r * pk + qq];
          U[r * pk + pp] = c * x - s * y; U[r * pk + qq] = s * x + c * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  if (tid == 0) sweeps_out[k] = (pk > 1) ? sweep : 0;
  // sigma_l^2 = |w_l|^2 (smean reused as scratch), then sort / sign as fbspca_eig (reading Q10)
  for (int q = warp; q < pk; q += nw) {
    const double* wq = W + (int64_t)q * m;
    double acc = 0;
    for (int64_t j = lane; j < m; j += 32) acc = fma(wq[j], wq[j], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) smean[q] = acc;
  }
  __syncthreads();
  for (int i = tid; i < pk; i += blockDim.x) {
    const double li = smean[i];
    int rank = 0;
    for (int j = 0; j < pk; ++j) {
      const double lj = smean[j];
      rank += (lj > li) || (lj == li && j < i);
    }
    evals[coef_off[k] + rank] = li;
    int arg = 0; double best = -1;
    for (int r = 0; r < pk; ++r) { const double a = fabs(U[r * pk + i]); if (a > best) { best = a; arg = r; } }
    const double sg = U[arg * pk + i] < 0 ? -1.0 : 1.0;
    double* Uo = evecs + evec_off[k];
    for (int r = 0; r < pk; ++r) Uo[r * pk + rank] = sg * U[r * pk + i];
  }
}

cudaError_t launch_svd(const Plan& P, const void* d_coeffs, int64_t n, double* d_work, double* d_mean,
                       double* d_evals, double* d_evecs, cudaStream_t s) {
  if (P.dt == FBSPCA_F32)
    svd_kernel<float><<<P.k_max + 1, 256, 0, s>>>(static_cast<const float*>(d_coeffs), n, P.d_p, P.d_coef_off,
                                                   P.d_evec_off, d_work, d_mean, d_evals, d_evecs, P.d_eig_sweeps);
  else
    svd_kernel<double><<<P.k_max + 1, 256, 0, s>>>(static_cast<const double*>(d_coeffs), n, P.d_p, P.d_coef_off,
                                                    P.d_evec_off, d_work, d_mean, d_evals, d_evecs, P.d_eig_sweeps);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- Alg. 2 line 5: Eq. (sPCArad)
// f^{k,l}(xi_j) = sum_q u_l^(k)(q) N_{k,q} J_k(R_{k,q} xi_j / c)  (fp64), one CTA per k (U_k and the basis read
// through L1/L2: p_k^2 <= 179^2 doubles does not always fit shared memory; the step is O(sum p_k^2 n_xi), tiny).
// Output row (coef_off[k] + l), column j (n_xi per row).
__global__ void __launch_bounds__(256)
radial_eigfun_kernel(const double* __restrict__ evecs, const double* __restrict__ rbasis, const int* __restrict__ p,
                     const int64_t* __restrict__ coef_off, const int64_t* __restrict__ evec_off, int n_xi,
                     double* __restrict__ f) {
  const int k = blockIdx.x, pk = p[k];
  const double* Uk = evecs + evec_off[k];
  const double* Bk = rbasis + coef_off[k] * n_xi;
  double* Fk = f + coef_off[k] * n_xi;
  for (int e = threadIdx.x; e < pk * n_xi; e += blockDim.x) {
    const int l = e / n_xi, j = e - l * n_xi;
    double s = 0.0;
    for (int q = 0; q < pk; ++q) s = fma(__ldg(Uk + q * pk + l), __ldg(Bk + (int64_t)q * n_xi + j), s);
    Fk[e] = s;
  }
}

cudaError_t launch_radial_eigfun(const Plan& P, const double* d_evecs, double* d_f, cudaStream_t s) {
  radial_eigfun_kernel<<<P.k_max + 1, 256, 0, s>>>(d_evecs, P.d_rbasis, P.d_p, P.d_coef_off, P.d_evec_off, P.n_xi, d_f);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K7: Eq. (sPCAcoeff) P:364 + filter P:689-699
// K7, Eq. (sPCAcoeff) P:364 + the filter of P:689-699 (modes: include/fbspca.h), and (BACK) the back-projection
// a_k = U_k c_k + m of NEXT-1.  One CTA per (k, slice of images): W (= U_k, or U_k^T when BACK; fp64 -> T, row stride
// padded to 4 for 16-B broadcast loads), the weights h_k and U_k^T m (k = 0) are staged once per CTA; thread = image,
// its (re, im) pair accumulated together (one packed FMA per W entry) over LC outputs at a time, the input column
// read 4 rows per batch of independent loads; the CTA strides over 256-image tiles.
//   out[l][i] = h_l (sum_q W[q][l] in[q][i] - [k = 0] (U^T m)_l)      (project; Im = 0 at k = 0)
//   out[q][i] = sum_l W[l][q] in[l][i] + [k = 0] m_q                  (BACK; Im = 0 at k = 0)
template <typename T, bool BACK>
__global__ void __launch_bounds__(256)
project_kernel(const T* __restrict__ coeffs, int64_t n, const double* __restrict__ mean,
               const double* __restrict__ evals, const double* __restrict__ evecs, const int* __restrict__ p,
               const int64_t* __restrict__ coef_off, const int64_t* __restrict__ evec_off, double sigma2, int mode,
               int64_t n_total, T* __restrict__ out) {
  using T2 = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int k = blockIdx.y;
  const int pk = p[k];
  const int up = (pk + 3) & ~3;                    // padded row stride of W in shared memory
  T* W = reinterpret_cast<T*>(sm_raw);             // pk x up
  T* h = W + pk * up;                              // pk
  T* um = h + up;                                  // pk: U^T mean (k = 0, project) or the mean (k = 0, BACK)
  const double* Uk = evecs + evec_off[k];
  for (int i = threadIdx.x; i < pk * up; i += blockDim.x) {
    const int r = i / up, c = i - r * up;          // W[r][c] = U[r][c] (project) or U[c][r] (BACK)
    W[i] = c < pk ? T(BACK ? Uk[c * pk + r] : Uk[r * pk + c]) : T(0);
  }
  for (int l = threadIdx.x; l < pk; l += blockDim.x) {
    if constexpr (BACK) {
      h[l] = T(1);
      um[l] = k == 0 ? T(mean[l]) : T(0);
    } else {
      const double lam = evals[coef_off[k] + l];
      double hv = 1.0;
      if (mode != 0) {
        const double g = (k == 0) ? double(pk) / double(n_total) : double(pk) / (2.0 * double(n_total));
        const double edge = sigma2 * (1 + sqrt(g)) * (1 + sqrt(g));
        double ell;
        if (mode == 1) ell = fmax(lam - sigma2, 0.0);
        else {
          const double t = lam - sigma2 * (1 + g);
          ell = 0.5 * (t + sqrt(fmax(t * t - 4 * g * sigma2 * sigma2, 0.0)));
        }
        hv = (lam > edge) ? (sigma2 > 0 ? ell / (ell + sigma2) : 1.0) : 0.0;
      }
      h[l] = T(hv);
      double s = 0;
      if (k == 0) for (int q = 0; q < pk; ++q) s += Uk[q * pk + l] * mean[q];
      um[l] = T(s);
    }
  }
  __syncthreads();
  const T2* a0 = reinterpret_cast<const T2*>(coeffs) + coef_off[k] * n;
  T2* o0 = reinterpret_cast<T2*>(out) + coef_off[k] * n;
  constexpr int LC = 32;
  auto fma_row = [&](T2 (&acc)[LC], const T* wr, int l0, T2 v) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int t = 0; t < LC; t += 4) {
        if (l0 + t < up) {
          const float4 w = *reinterpret_cast<const float4*>(wr + t);
          acc[t] = rfma(w.x, v, acc[t]); acc[t + 1] = rfma(w.y, v, acc[t + 1]);
          acc[t + 2] = rfma(w.z, v, acc[t + 2]); acc[t + 3] = rfma(w.w, v, acc[t + 3]);
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < LC; ++t) if (l0 + t < pk) acc[t] = rfma(wr[t], v, acc[t]);
    }
  };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - threadIdx.x < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i >= n) continue;
    const T2* a = a0 + i;
    for (int l0 = 0; l0 < pk; l0 += LC) {
      T2 acc[LC];
#pragma unroll
      for (int t = 0; t < LC; ++t) acc[t] = T2{T(0), T(0)};
      int q = 0;
      for (; q + 4 <= pk; q += 4) {                  // four independent loads in flight, then their FMAs
        const T2 v0 = a[(int64_t)q * n], v1 = a[(int64_t)(q + 1) * n];
        const T2 v2 = a[(int64_t)(q + 2) * n], v3 = a[(int64_t)(q + 3) * n];
        fma_row(acc, W + q * up + l0, l0, v0);
        fma_row(acc, W + (q + 1) * up + l0, l0, v1);
        fma_row(acc, W + (q + 2) * up + l0, l0, v2);
        fma_row(acc, W + (q + 3) * up + l0, l0, v3);
      }
      for (; q < pk; ++q) fma_row(acc, W + q * up + l0, l0, a[(int64_t)q * n]);
#pragma unroll
      for (int t = 0; t < LC; ++t) {
        const int l = l0 + t;
        if (l < pk) {
          T2 v = acc[t];
          if (BACK) { if (k == 0) v = T2{v.x + um[l], T(0)}; }
          else {
            if (k == 0) v = T2{v.x - um[l], T(0)};
            v = T2{h[l] * v.x, h[l] * v.y};
          }
          o0[(int64_t)l * n + i] = v;
        }
      }
    }
  }
}

template <bool BACK>
static cudaError_t launch_transform(const Plan& P, const void* d_coeffs, int64_t n, const double* d_mean,
                                    const double* d_evals, const double* d_evecs, double sigma2, int mode,
                                    int64_t n_total, void* d_out, cudaStream_t s) {
  const int pmax = P.p[0], upmax = (pmax + 3) & ~3;
  // about 8 CTAs per SM in total over the k blocks; each strides over 256-image tiles
  const int64_t tiles = (n + 255) / 256;
  const int per_k = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (8LL * P.num_sms + P.k_max) / (P.k_max + 1)));
  dim3 grid((unsigned)per_k, (unsigned)(P.k_max + 1));
  if (P.dt == FBSPCA_F32) {
    const int smem = (int)((size_t)(pmax * upmax + 2 * upmax) * sizeof(float));
    cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(project_kernel<float, BACK>), smem);
    if (e != cudaSuccess) return e;
    project_kernel<float, BACK><<<grid, 256, smem, s>>>((const float*)d_coeffs, n, d_mean, d_evals, d_evecs, P.d_p,
                                                        P.d_coef_off, P.d_evec_off, sigma2, mode, n_total, (float*)d_out);
  } else {
    const int smem = (int)((size_t)(pmax * upmax + 2 * upmax) * sizeof(double));
    cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(project_kernel<double, BACK>), smem);
    if (e != cudaSuccess) return e;
    project_kernel<double, BACK><<<grid, 256, smem, s>>>((const double*)d_coeffs, n, d_mean, d_evals, d_evecs, P.d_p,
                                                         P.d_coef_off, P.d_evec_off, sigma2, mode, n_total,
                                                         (double*)d_out);
  }
  return cudaGetLastError();
}

cudaError_t launch_project(const Plan& P, const void* d_coeffs, int64_t n, const double* d_mean,
                           const double* d_evals, const double* d_evecs, double sigma2, int mode, int64_t n_total,
                           void* d_out, cudaStream_t s) {
  return launch_transform<false>(P, d_coeffs, n, d_mean, d_evals, d_evecs, sigma2, mode, n_total, d_out, s);
}

cudaError_t launch_backproject(const Plan& P, const void* d_c, int64_t n, const double* d_mean, const double* d_evecs,
                               void* d_out, cudaStream_t s) {
  return launch_transform<true>(P, d_c, n, d_mean, nullptr, d_evecs, 0.0, 0, n, d_out, s);
}

}  // namespace fbspca
