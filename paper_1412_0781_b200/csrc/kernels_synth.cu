// kernels_synth.cu -- NEXT-1: from coefficients back to pixels.
//
//   fbspca_backproject: a_k = U_k c_k (+ the mean at k = 0): steerable-basis coefficients (e.g. the Wiener-filtered
//                       output of fbspca_project) back to Fourier-Bessel coefficients (Eq. (sPCAcoeff)
//                       P:364 inverted, U_k orthogonal).
//   fbspca_synthesize:  I(x) = sum_q a_{0,q} F^-1 psi^{0,q}(x) + 2 Re sum_{k>=1,q} a_{k,q} F^-1 psi^{k,q}(x) on the
//                       L x L grid (r <= R), Eq. (IFT_FB) P:108 with reading Q2 (i^{+k} in the numerator):
//                       F^-1 psi^{k,q}(r, phi) = rho_{k,q}(r) i^k e^{ik phi},
//                       rho_{k,q}(r) = 2 c sqrt(pi) (-1)^q R_{k,q} J_k(2 pi c r) / ((2 pi c r)^2 - R_{k,q}^2).
// The basis is separable in polar coordinates, so per image and k the radial sums s_k(r) = sum_q a_{k,q} rho_{k,q}(r)
// are formed once per distinct pixel radius and then spread over the pixels at that radius with e^{ik phi}
// (advanced by one complex multiply per k).  fp64 throughout (not on the timed path).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace fbspca {

constexpr int kSynthGroup = 2048;      // pixels per CTA (sorted by radius)

template <typename T>
__global__ void __launch_bounds__(256)
synth_kernel(const T* __restrict__ coeffs, int64_t ld, const int* __restrict__ p, const int64_t* __restrict__ coef_off,
             int k_max, const double* __restrict__ rho, int n_r, const int* __restrict__ pix_idx,
             const int* __restrict__ pix_ir, const double2* __restrict__ pix_cs, const int* __restrict__ grp,
             int64_t img_elems, T* __restrict__ out) {
  extern __shared__ double sm[];
  const int g = blockIdx.x, i = blockIdx.y;
  const int p0 = grp[g], p1 = grp[g + 1], np = p1 - p0;
  const int ir0 = pix_ir[p0], nr = pix_ir[p1 - 1] - ir0 + 1;
  double* acc = sm;                                // np
  double2* ph = reinterpret_cast<double2*>(acc + kSynthGroup);   // np: i^k e^{ik phi}
  double2* s = ph + kSynthGroup;                   // nr
  for (int t = threadIdx.x; t < np; t += blockDim.x) { acc[t] = 0.0; ph[t] = make_double2(1.0, 0.0); }
  for (int k = 0; k <= k_max; ++k) {
    const int pk = p[k];
    const T* A = coeffs + coef_off[k] * 2 * ld + 2 * (int64_t)i;
    const double* Rk = rho + coef_off[k] * (int64_t)n_r + ir0;
    __syncthreads();
    for (int t = threadIdx.x; t < nr; t += blockDim.x) {
      double sr = 0.0, si = 0.0;
      for (int q = 0; q < pk; ++q) {
        const double r = __ldg(Rk + (int64_t)q * n_r + t);
        sr = fma(double(A[(int64_t)q * 2 * ld]), r, sr);
        si = fma(double(A[(int64_t)q * 2 * ld + 1]), r, si);
      }
      s[t] = make_double2(sr, si);
    }
    __syncthreads();
    const double w = k == 0 ? 1.0 : 2.0;
    for (int t = threadIdx.x; t < np; t += blockDim.x) {
      double2 e = ph[t];
      if (k > 0) {                                  // e <- e * i e^{i phi}
        const double2 cs = __ldg(pix_cs + p0 + t);
        const double er = e.x * cs.x - e.y * cs.y, ei = e.x * cs.y + e.y * cs.x;
        e = make_double2(-ei, er);
        ph[t] = e;
      }
      const double2 v = s[pix_ir[p0 + t] - ir0];
      acc[t] += w * (v.x * e.x - v.y * e.y);        // Re(a-sum * i^k e^{ik phi})
    }
  }
  __syncthreads();
  T* o = out + (int64_t)i * img_elems;
  for (int t = threadIdx.x; t < np; t += blockDim.x) o[pix_idx[p0 + t]] = T(acc[t]);
}

// a_k = U_k c_k (+ mean at k = 0): launch_backproject in kernels_linalg.cu (shares the K7 kernel)

// ---------------------------------------------------------------- host
static void build_synth_tables(Plan& P, std::vector<int>& pidx, std::vector<int>& pir, std::vector<double>& pcs,
                               std::vector<int>& grp, std::vector<double>& rho, int& n_r) {
  const int L = P.L;
  const double R2 = P.R * P.R;
  std::vector<std::pair<int, int>> pix;            // (r^2, linear index)
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      const int i1 = a - L / 2, i2 = b - L / 2, r2 = i1 * i1 + i2 * i2;
      if (double(r2) <= R2) pix.push_back({r2, a * L + b});
    }
  std::sort(pix.begin(), pix.end());
  std::vector<int> r2s;
  for (auto& e : pix) if (r2s.empty() || r2s.back() != e.first) r2s.push_back(e.first);
  n_r = int(r2s.size());
  pidx.resize(pix.size()); pir.resize(pix.size()); pcs.resize(2 * pix.size());
  for (size_t t = 0, ir = 0; t < pix.size(); ++t) {
    while (r2s[ir] != pix[t].first) ++ir;
    pidx[t] = pix[t].second; pir[t] = int(ir);
    const int a = pix[t].second / L, b = pix[t].second % L;
    const double i1 = a - L / 2, i2 = b - L / 2, r = std::sqrt(i1 * i1 + i2 * i2);
    pcs[2 * t] = r > 0 ? i1 / r : 1.0;             // cos phi, sin phi (phi = atan2(i2, i1), Q3); phi(0) = 0
    pcs[2 * t + 1] = r > 0 ? i2 / r : 0.0;
  }
  grp.clear();
  for (size_t t = 0; t < pix.size(); t += kSynthGroup) grp.push_back(int(t));
  grp.push_back(int(pix.size()));
  const int nk = P.k_max + 1;
  const double c = P.c, pref = 2 * c * std::sqrt(M_PI);
  rho.assign(size_t(P.coef_off[nk]) * n_r, 0.0);
  std::vector<double> jk(n_r);
  for (int k = 0; k < nk; ++k) {
    for (int ir = 0; ir < n_r; ++ir) jk[ir] = jn(k, 2 * M_PI * c * std::sqrt(double(r2s[ir])));
    for (int q = 0; q < P.p[k]; ++q) {
      const int64_t row = P.coef_off[k] + q;
      const double Rq = P.zeros[row], sg = (q % 2 == 0) ? -1.0 : 1.0;      // (-1)^q, paper q = q + 1
      for (int ir = 0; ir < n_r; ++ir) {
        const double x = 2 * M_PI * c * std::sqrt(double(r2s[ir]));
        double v;
        if (std::fabs(x - Rq) < 1e-8) v = c * std::sqrt(M_PI) * (-sg) * jn(k + 1, Rq);   // removable singularity
        else v = pref * sg * Rq * jk[ir] / (x * x - Rq * Rq);
        rho[size_t(row) * n_r + ir] = v;
      }
    }
  }
}

cudaError_t synth_prepare(Plan& P) {
  if (P.d_synth_rho) return cudaSuccess;
  std::vector<int> pidx, pir, grp;
  std::vector<double> pcs, rho;
  int n_r = 0;
  build_synth_tables(P, pidx, pir, pcs, grp, rho, n_r);
  cudaError_t e;
  auto up = [&](void** d, const void* h, size_t bytes) {
    cudaError_t r = cudaMalloc(d, bytes + 16);
    if (r == cudaSuccess) r = cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice);
    return r;
  };
  if ((e = up((void**)&P.d_synth_rho, rho.data(), rho.size() * sizeof(double))) != cudaSuccess) return e;
  if ((e = up((void**)&P.d_synth_pidx, pidx.data(), pidx.size() * sizeof(int))) != cudaSuccess) return e;
  if ((e = up((void**)&P.d_synth_pir, pir.data(), pir.size() * sizeof(int))) != cudaSuccess) return e;
  if ((e = up((void**)&P.d_synth_pcs, pcs.data(), pcs.size() * sizeof(double))) != cudaSuccess) return e;
  if ((e = up((void**)&P.d_synth_grp, grp.data(), grp.size() * sizeof(int))) != cudaSuccess) return e;
  P.synth_nr = n_r;
  P.synth_ngroups = int(grp.size()) - 1;
  return cudaSuccess;
}

cudaError_t launch_synthesize(Plan& P, const void* d_coeffs, int64_t n, void* d_images, cudaStream_t s) {
  cudaError_t e = synth_prepare(P);
  if (e != cudaSuccess) return e;
  const size_t rsz = P.dt == FBSPCA_F32 ? 4 : 8;
  const int64_t elems = (int64_t)P.L * P.L;
  if ((e = cudaMemsetAsync(d_images, 0, size_t(n * elems) * rsz, s)) != cudaSuccess) return e;
  // groups of 2048 sorted pixels span at most 2048 radii
  const size_t smem = kSynthGroup * (sizeof(double) + sizeof(double2)) + kSynthGroup * sizeof(double2);
  dim3 grid((unsigned)P.synth_ngroups, (unsigned)n);
  if (P.dt == FBSPCA_F32) {
    if ((e = cudaFuncSetAttribute(synth_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
    synth_kernel<float><<<grid, 256, smem, s>>>((const float*)d_coeffs, n, P.d_p, P.d_coef_off, P.k_max, P.d_synth_rho,
                                                P.synth_nr, P.d_synth_pidx, P.d_synth_pir,
                                                reinterpret_cast<const double2*>(P.d_synth_pcs), P.d_synth_grp, elems,
                                                (float*)d_images);
  } else {
    if ((e = cudaFuncSetAttribute(synth_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
    synth_kernel<double><<<grid, 256, smem, s>>>((const double*)d_coeffs, n, P.d_p, P.d_coef_off, P.k_max, P.d_synth_rho,
                                                 P.synth_nr, P.d_synth_pidx, P.d_synth_pir,
                                                 reinterpret_cast<const double2*>(P.d_synth_pcs), P.d_synth_grp, elems,
                                                 (double*)d_images);
  }
  return cudaGetLastError();
}

}  // namespace fbspca
