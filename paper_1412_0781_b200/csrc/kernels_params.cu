// kernels_params.cu -- NEXT-2: noise variance, support radius and band limit from the data, the way
// the paper chooses R = 98 and c = 0.196 for its ribosome set (Fig. 5; SPEC estimate_noise_variance /
// estimate_support / estimate_bandlimit):
//   * per-pixel mean m and variance v of the stack (one streaming pass, fp64 sums);           [pixstats_kernel]
//   * mean power spectrum P = (1/n) sum_i |DFT2(I_i)|^2 / L^2 - |DFT2(m)|^2 / L^2 (= the power of the
//     mean-subtracted images; the 1/L^2 puts white noise of variance s^2 at level s^2);       [powspec_kernel]
//   * radial averages, noise level from the outer 10 % of radii, cumulative (r dr / xi dxi) fraction points (host).
// Definitions (readings Q18-Q20): pixel / frequency offsets i = a - floor(L/2), f = fftfreq(L) L; radial
// bin b = floor(r + 1/2); sigma^2 = mean of the variance profile over bins ceil(0.45 L) <= b < floor(L/2);
// R = the smallest bin b with sum_{b' <= b} max(prof - sigma^2, 0) b' >= fraction x the total over b < floor(L/2);
// c = b / L for the smallest frequency bin 1 <= b <= floor(L/2) reaching the fraction of the power excess.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "fft_device.cuh"
#include "internal.h"

namespace fbspca {

constexpr int kPixTile = 1024;       // pixels per CTA (4 per thread)
constexpr int kPixChunk = 2048;      // images per CTA

// partial[chunk][0..P) = sum x, partial[chunk][P..2P) = sum x^2 over the chunk's images, for the CTA's pixel tile
template <typename T>
__global__ void __launch_bounds__(256)
pixstats_kernel(const T* __restrict__ img, int64_t n, int P, double* __restrict__ partial) {
  const int p0 = blockIdx.x * kPixTile;
  const int64_t i0 = (int64_t)blockIdx.y * kPixChunk, i1 = min(n, i0 + kPixChunk);
  double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
  for (int64_t i = i0; i < i1; ++i) {
    const T* row = img + i * P;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + threadIdx.x + 256 * u;
      if (p < P) { const double x = double(__ldg(row + p)); s[u] += x; q[u] = fma(x, x, q[u]); }
    }
  }
  double* out = partial + (int64_t)blockIdx.y * 2 * P;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int p = p0 + threadIdx.x + 256 * u;
    if (p < P) { out[p] = s[u]; out[P + p] = q[u]; }
  }
}

// fixed-order sum over chunks: out[j] = sum_c partial[c][j], j < len
__global__ void sum_chunks_kernel(const double* __restrict__ partial, int nchunk, int64_t len, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < len; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0;
    for (int c = 0; c < nchunk; ++c) s += partial[(int64_t)c * len + j];
    out[j] = s;
  }
}

// Power spectrum accumulation.  CTA b owns images b, b + grid, ...; per image: row FFTs of pairs of real rows
// (half spectra f2 = 0..L/2 into the CTA's scratch S[a][f2]), then column FFTs of S[:, f2] whose |.|^2 / L^2 are
// added into the CTA's fp64 accumulator Acc[f1][f2] (owned by the CTA: no atomics; reduced afterwards in fixed
// order).  Runtime mixed-radix FFT (5-smooth L); per-warp ping-pong in shared memory.
template <typename T>
__global__ void __launch_bounds__(256)
powspec_kernel(const T* __restrict__ img, int64_t n, int L, FftPlan fp, const double* __restrict__ twg,
               typename Cx<T>::t* __restrict__ scratch, double* __restrict__ acc) {
  using T2 = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int H = L / 2 + 1;
  T2* tw = reinterpret_cast<T2*>(smraw);
  for (int i = tid; i < L; i += blockDim.x) tw[i] = T2{T(twg[2 * i]), T(twg[2 * i + 1])};
  T2* A = tw + L + (size_t)warp * 2 * L;
  T2* B = A + L;
  T2* res = ((fp.nstages - 1) & 1) ? B : A;                 // buffer the last stage does not read
  __syncthreads();
  T2* S = scratch + (int64_t)blockIdx.x * L * H;            // S[a][f2]
  double* Acc = acc + (int64_t)blockIdx.x * L * H;           // Acc[f1][f2]
  const double inv = 1.0 / (double(L) * double(L));
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const T* I = img + i * (int64_t)L * L;
    for (int pr = warp; 2 * pr < L; pr += nw) {               // rows 2 pr, 2 pr + 1 as re / im
      const int a0 = 2 * pr, a1 = a0 + 1;
      const bool has1 = a1 < L;
      auto ld = [&](int t) -> T2 { return T2{__ldg(I + (int64_t)a0 * L + t), has1 ? __ldg(I + (int64_t)a1 * L + t) : T(0)}; };
      auto st = [&](int t, T2 v) { res[t] = v; };
      fft_rt<T2>(fp, ld, st, A, B, tw, lane);
      for (int f = lane; f < H; f += 32) {
        const T2 zm = res[f];
        T2 zc = res[(L - f) % L];
        zc.y = -zc.y;                                         // conj Z(-f)
        S[(int64_t)a0 * H + f] = T2{T(0.5) * (zm.x + zc.x), T(0.5) * (zm.y + zc.y)};
        if (has1) S[(int64_t)a1 * H + f] = T2{T(0.5) * (zm.y - zc.y), T(-0.5) * (zm.x - zc.x)};
      }
      __syncwarp();
    }
    __syncthreads();
    for (int f2 = warp; f2 < H; f2 += nw) {                   // column f2 (owned by this warp)
      auto ld = [&](int t) -> T2 { return S[(int64_t)t * H + f2]; };
      auto st = [&](int t, T2 v) {
        double* a = Acc + (int64_t)t * H + f2;
        *a += (double(v.x) * double(v.x) + double(v.y) * double(v.y)) * inv;
      };
      fft_rt<T2>(fp, ld, st, A, B, tw, lane);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host
namespace {

int round_bin(double r) { return int(std::floor(r + 0.5)); }

// cumulative fraction point: smallest b in [b0, b1] with sum_{b0 <= b' <= b} w[b'] >= frac * sum w
int frac_point(const std::vector<double>& w, int b0, int b1, double frac, double& total) {
  total = 0;
  for (int b = b0; b <= b1; ++b) total += w[b];
  if (!(total > 0)) return -1;
  double cum = 0;
  for (int b = b0; b <= b1; ++b) {
    cum += w[b];
    if (cum >= frac * total) return b;
  }
  return b1;
}

}  // namespace

template <typename T>
static fbspca_status estimate_t(int L, int device, const T* d_img, int64_t n, double fraction, double* out3) {
  const int P = L * L, H = L / 2 + 1;
  FftPlan fp;
  {   // radix plan (same rules as the polar kernel's runtime FFT)
    int m = L;
    fp.n = L; fp.nstages = 0;
    auto push = [&](int r) { fp.radix[fp.nstages++] = r; m /= r; };
    while (m % 8 == 0 && fp.nstages < kMaxRadixStages) push(8);
    while (m % 4 == 0 && fp.nstages < kMaxRadixStages) push(4);
    while (m % 2 == 0 && fp.nstages < kMaxRadixStages) push(2);
    while (m % 5 == 0 && fp.nstages < kMaxRadixStages) push(5);
    while (m % 3 == 0 && fp.nstages < kMaxRadixStages) push(3);
    for (int r : {7, 11, 13})
      while (m % r == 0 && fp.nstages < kMaxRadixStages) push(r);
    if (m != 1) { set_error("estimate_params: L must be 2^a 3^b 5^c 7^d 11^e 13^f"); return FBSPCA_ERR_CONFIG; }
  }
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const int nchunk = int((n + kPixChunk - 1) / kPixChunk);
  const int grid_ps = int(std::min<int64_t>(n, 2 * nsm));
  std::vector<double> tw(2 * L);
  for (int i = 0; i < L; ++i) { tw[2 * i] = std::cos(-2 * M_PI * i / L); tw[2 * i + 1] = std::sin(-2 * M_PI * i / L); }
  double *d_part = nullptr, *d_stats = nullptr, *d_acc = nullptr, *d_spec = nullptr, *d_tw = nullptr, *d_mean = nullptr,
         *d_acc_m = nullptr;
  void* d_scr = nullptr;
  const size_t csz = 2 * sizeof(T);
  auto cleanup = [&]() {
    for (void* p : {(void*)d_part, (void*)d_stats, (void*)d_acc, (void*)d_spec, (void*)d_tw, (void*)d_mean,
                    (void*)d_acc_m, d_scr}) if (p) cudaFree(p);
  };
#define PC(call, what) do { cudaError_t _e = (call); if (_e != cudaSuccess) { cleanup(); \
    set_error(std::string("estimate_params: ") + what + ": " + cudaGetErrorString(_e)); return FBSPCA_ERR_CUDA; } } while (0)
  PC(cudaMalloc(&d_part, size_t(nchunk) * 2 * P * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_stats, size_t(2) * P * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_acc, size_t(grid_ps) * L * H * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_acc_m, size_t(L) * H * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_spec, size_t(L) * H * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_tw, 2 * L * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_mean, size_t(P) * sizeof(double)), "alloc");
  PC(cudaMalloc(&d_scr, size_t(grid_ps) * L * H * std::max(csz, 2 * sizeof(double))), "alloc");
  PC(cudaMemcpy(d_tw, tw.data(), 2 * L * sizeof(double), cudaMemcpyHostToDevice), "copy");
  PC(cudaMemset(d_acc, 0, size_t(grid_ps) * L * H * sizeof(double)), "memset");
  PC(cudaMemset(d_acc_m, 0, size_t(L) * H * sizeof(double)), "memset");
  // pass 1: per-pixel sums
  pixstats_kernel<T><<<dim3((P + kPixTile - 1) / kPixTile, nchunk), 256>>>(d_img, n, P, d_part);
  sum_chunks_kernel<<<std::max(1, std::min(4 * nsm, (2 * P + 255) / 256)), 256>>>(d_part, nchunk, 2 * (int64_t)P, d_stats);
  // pass 2: power spectra of the images and of the mean image
  const size_t smem = (size_t(L) + 8 * 2 * size_t(L)) * csz;
  const size_t smem_d = (size_t(L) + 8 * 2 * size_t(L)) * 2 * sizeof(double);
  PC(cudaFuncSetAttribute(powspec_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
  PC(cudaFuncSetAttribute(powspec_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d), "attr");
  powspec_kernel<T><<<grid_ps, 256, smem>>>(d_img, n, L, fp, d_tw, reinterpret_cast<typename Cx<T>::t*>(d_scr), d_acc);
  PC(cudaGetLastError(), "powspec kernel");
  std::vector<double> stats(2 * size_t(P));
  PC(cudaMemcpy(stats.data(), d_stats, stats.size() * sizeof(double), cudaMemcpyDeviceToHost), "copy");
  std::vector<double> mean(P), var(P);
  for (int p = 0; p < P; ++p) {
    mean[p] = stats[p] / double(n);
    var[p] = std::max(stats[P + p] / double(n) - mean[p] * mean[p], 0.0);
  }
  PC(cudaMemcpy(d_mean, mean.data(), P * sizeof(double), cudaMemcpyHostToDevice), "copy");
  sum_chunks_kernel<<<std::max(1, std::min(4 * nsm, (L * H + 255) / 256)), 256>>>(d_acc, grid_ps, (int64_t)L * H, d_spec);
  powspec_kernel<double><<<1, 256, smem_d>>>(d_mean, 1, L, fp, d_tw, reinterpret_cast<double2*>(d_scr), d_acc_m);
  PC(cudaGetLastError(), "powspec kernel (mean)");
  std::vector<double> spec(size_t(L) * H), specm(size_t(L) * H);
  PC(cudaMemcpy(spec.data(), d_spec, spec.size() * sizeof(double), cudaMemcpyDeviceToHost), "copy");
  PC(cudaMemcpy(specm.data(), d_acc_m, specm.size() * sizeof(double), cudaMemcpyDeviceToHost), "copy");
  cleanup();
#undef PC
  // ---- radial profiles (host, fp64)
  const int nb = L / 2;                                      // bins b < floor(L/2) (real space), b <= floor(L/2) (freq.)
  std::vector<double> vs(nb + 1, 0.0), vc(nb + 1, 0.0);
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      const double i1 = a - L / 2, i2 = b - L / 2;
      const int bin = round_bin(std::sqrt(i1 * i1 + i2 * i2));
      if (bin < nb) { vs[bin] += var[a * L + b]; vc[bin] += 1; }
    }
  std::vector<double> prof(nb, 0.0);
  for (int b = 0; b < nb; ++b) prof[b] = vc[b] > 0 ? vs[b] / vc[b] : 0.0;
  const int blo = int(std::ceil(0.45 * L - 1e-12));
  double s2 = 0; int cnt = 0;
  for (int b = blo; b < nb; ++b) if (vc[b] > 0) { s2 += prof[b]; ++cnt; }
  s2 = cnt ? s2 / cnt : 0.0;
  std::vector<double> wr(nb, 0.0);
  for (int b = 0; b < nb; ++b) wr[b] = std::max(prof[b] - s2, 0.0) * double(b);
  double tot_r = 0;
  const int Rb = frac_point(wr, 0, nb - 1, fraction, tot_r);
  // frequency profile over the half plane f2 = 0..L/2 (weight 2 where the mirror -f is a different column)
  std::vector<double> ps(nb + 1, 0.0), pc(nb + 1, 0.0);
  for (int r1 = 0; r1 < L; ++r1) {
    const int f1 = r1 < (L + 1) / 2 ? r1 : r1 - L;
    for (int f2 = 0; f2 < H; ++f2) {
      const bool self_mirror = (f2 == 0) || (L % 2 == 0 && f2 == L / 2);
      const double wgt = self_mirror ? 1.0 : 2.0;
      const int bin = round_bin(std::sqrt(double(f1) * f1 + double(f2) * f2));
      if (bin >= 1 && bin <= nb) {
        const double pv = spec[size_t(r1) * H + f2] / double(n) - specm[size_t(r1) * H + f2];
        ps[bin] += wgt * pv; pc[bin] += wgt;
      }
    }
  }
  std::vector<double> wf(nb + 1, 0.0);
  for (int b = 1; b <= nb; ++b) wf[b] = std::max((pc[b] > 0 ? ps[b] / pc[b] : 0.0) - s2, 0.0) * double(b);
  double tot_f = 0;
  const int Cb = frac_point(wf, 1, nb, fraction, tot_f);
  out3[0] = s2;
  out3[1] = Rb >= 0 ? double(Rb) : NAN;
  out3[2] = Cb >= 0 ? double(Cb) / double(L) : NAN;
  if (Rb < 0 || Cb < 0) { set_error("estimate_params: no signal variance above the noise level"); return FBSPCA_ERR_NUMERIC; }
  return FBSPCA_OK;
}

fbspca_status estimate_params(int L, fbspca_dtype dt, int device, const void* d_images, int64_t n, double fraction,
                              double* out3) {
  return dt == FBSPCA_F32 ? estimate_t<float>(L, device, (const float*)d_images, n, fraction, out3)
                          : estimate_t<double>(L, device, (const double*)d_images, n, fraction, out3);
}

}  // namespace fbspca
