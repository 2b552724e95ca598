// kernels_polar.cu -- fused K1 (deapodise + zero-pad + oversampled 2-D FFT), K2 (window gather to the
// half-plane polar nodes) and K3 (angular FFT per ring), one persistent CTA per SM, one image at a time.
//
//   K1+K2 = type-2 NUFFT of Eq. (nufft) (unit prefactor): F(xi) ~= sum_m phi(M xi - m) G[m],
//           G = DFT_M( I(i) / Phi(i/M) placed at i mod M ).  Only theta in [0, pi) is computed:
//           F(-xi) = conj F(xi) for real I.
//   K3    = Eq. (1DFFT) on each ring j, from the full ring F(l + n/2) = conj F(l); the 2 pi/n_theta
//           weight is folded into the radial table.  Output ghat[k][b][re|im][j], k = 0..k_max.
//
// The oversampled half spectrum of one image does not fit in shared memory at L >= 128, so the column
// range m2 it needs ([col_lo, col_lo + ncols_x)) is processed in phases of S columns: the row FFTs are
// done once per image into an L2-resident per-CTA scratch X[i1][m2], each phase loads its columns,
// runs the column FFTs in place in shared memory and gathers the nodes whose window lies in the phase.
// Polar samples go to a per-CTA L2-resident scratch and are read back by the angular pass.
#include <cuda_runtime.h>

#include "internal.h"

namespace fbspca {

template <typename T> struct Cx;
template <> struct Cx<float> { using t = float2; };
template <> struct Cx<double> { using t = double2; };

template <typename T2> __device__ __forceinline__ T2 cadd(T2 a, T2 b) { return {a.x + b.x, a.y + b.y}; }
template <typename T2> __device__ __forceinline__ T2 csub(T2 a, T2 b) { return {a.x - b.x, a.y - b.y}; }
template <typename T2> __device__ __forceinline__ T2 cmul(T2 a, T2 b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T2> __device__ __forceinline__ T2 mul_mi(T2 a) { return {a.y, -a.x}; }   // -i * a

// ---------------------------------------------------------------- small forward DFTs (e^{-2 pi i})
template <typename T2, int R> struct Dft;
template <typename T2> struct Dft<T2, 2> {
  __device__ __forceinline__ static void run(T2* v) { T2 a = v[0]; v[0] = cadd(a, v[1]); v[1] = csub(a, v[1]); }
};
template <typename T2> struct Dft<T2, 4> {
  __device__ __forceinline__ static void run(T2* v) {
    T2 s0 = cadd(v[0], v[2]), d0 = csub(v[0], v[2]);
    T2 s1 = cadd(v[1], v[3]), d1 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(s0, s1); v[2] = csub(s0, s1);
    v[1] = cadd(d0, d1); v[3] = csub(d0, d1);
  }
};
template <typename T2> struct Dft<T2, 8> {
  __device__ __forceinline__ static void run(T2* v) {
    using T = decltype(v[0].x);
    const T h = T(0.70710678118654752440);
    T2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    Dft<T2, 4>::run(e); Dft<T2, 4>::run(o);
    // twiddles e^{-2 pi i k / 8}, k = 0..3
    T2 t1 = {h * (o[1].x + o[1].y), h * (o[1].y - o[1].x)};
    T2 t2 = mul_mi(o[2]);
    T2 t3 = {h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y)};
    v[0] = cadd(e[0], o[0]); v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], t1);   v[5] = csub(e[1], t1);
    v[2] = cadd(e[2], t2);   v[6] = csub(e[2], t2);
    v[3] = cadd(e[3], t3);   v[7] = csub(e[3], t3);
  }
};
template <typename T2> struct Dft<T2, 3> {
  __device__ __forceinline__ static void run(T2* v) {
    using T = decltype(v[0].x);
    const T c1 = T(-0.5), s1 = T(-0.86602540378443864676);   // e^{-2 pi i/3}
    T2 s = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    T2 a = {v[0].x + c1 * s.x, v[0].y + c1 * s.y};
    T2 b = {-s1 * d.y, s1 * d.x};                                // i s1 d
    v[0] = cadd(v[0], s);
    v[1] = cadd(a, b);
    v[2] = csub(a, b);
  }
};
template <typename T2> struct Dft<T2, 5> {
  __device__ __forceinline__ static void run(T2* v) {
    using T = decltype(v[0].x);
    const T c1 = T(0.30901699437494742410), c2 = T(-0.80901699437494742410);
    const T s1 = T(-0.95105651629515357212), s2 = T(-0.58778525229247312917);   // sin(-2pi k/5)
    T2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    T2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    T2 x0 = v[0];
    v[0] = cadd(x0, cadd(a1, a2));
    T2 r1 = {x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y};
    T2 r2 = {x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y};
    // i * (s1 b1 + s2 b2) and i * (s2 b1 - s1 b2)
    T2 i1 = {-(s1 * b1.y + s2 * b2.y), s1 * b1.x + s2 * b2.x};
    T2 i2 = {-(s2 * b1.y - s1 * b2.y), s2 * b1.x - s1 * b2.x};
    v[1] = cadd(r1, i1); v[4] = csub(r1, i1);
    v[2] = cadd(r2, i2); v[3] = csub(r2, i2);
  }
};

// One out-of-place Stockham stage of radix R (src -> dst, strided), executed by one warp, one
// butterfly per lane at a time (registers: R complex values).
template <typename T2, int R>
__device__ __forceinline__ void fft_stage(const T2* src, int sst, T2* dst, int dstr, int N, int Ns,
                                          const T2* __restrict__ tw, int lane) {
  const int NB = N / R;
  const int step = N / (Ns * R);
  for (int j = lane; j < NB; j += 32) {
    T2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[(j + r * NB) * sst];
    const int jm = j % Ns;
    const int base = jm * step;
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[base * r]);
    Dft<T2, R>::run(v);
    const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[(idxD + r * Ns) * dstr] = v[r];
  }
  __syncwarp();
}

template <typename T2>
__device__ __forceinline__ void fft_stage_any(int R, const T2* src, int sst, T2* dst, int dstr, int N, int Ns,
                                              const T2* tw, int lane) {
  switch (R) {
    case 8: fft_stage<T2, 8>(src, sst, dst, dstr, N, Ns, tw, lane); break;
    case 4: fft_stage<T2, 4>(src, sst, dst, dstr, N, Ns, tw, lane); break;
    case 2: fft_stage<T2, 2>(src, sst, dst, dstr, N, Ns, tw, lane); break;
    case 5: fft_stage<T2, 5>(src, sst, dst, dstr, N, Ns, tw, lane); break;
    default: fft_stage<T2, 3>(src, sst, dst, dstr, N, Ns, tw, lane); break;
  }
}

// Length-N forward FFT by one warp with ping-pong buffers A, B (stride 1, N complex each).
// out == nullptr: the input must be in A; the result is left in A or B and its pointer returned.
// out != nullptr: input `in` (stride ist) -> output `out` (stride ost); needs >= 2 stages.
template <typename T2>
__device__ T2* warp_fft(const T2* in, int ist, T2* out, int ost, T2* A, T2* B, const FftPlan& f, const T2* tw,
                        int lane) {
  int Ns = 1;
  const int last = f.nstages - 1;
  if (out == nullptr) {
    for (int s = 0; s <= last; ++s) {
      const T2* src = (s & 1) ? B : A;
      T2* dst = (s & 1) ? A : B;
      fft_stage_any<T2>(f.radix[s], src, 1, dst, 1, f.n, Ns, tw, lane);
      Ns *= f.radix[s];
    }
    return (f.nstages & 1) ? B : A;
  }
  for (int s = 0; s <= last; ++s) {
    const T2* src = (s == 0) ? in : ((s - 1) & 1 ? B : A);
    const int sst = (s == 0) ? ist : 1;
    T2* dst = (s == last) ? out : ((s & 1) ? B : A);
    const int dstr = (s == last) ? ost : 1;
    fft_stage_any<T2>(f.radix[s], src, sst, dst, dstr, f.n, Ns, tw, lane);
    Ns *= f.radix[s];
  }
  return out;
}

template <typename T> __device__ __forceinline__ T es_weight(T d, T inv_hw, T beta);
template <> __device__ __forceinline__ float es_weight<float>(float d, float inv_hw, float beta) {
  float z = d * inv_hw;
  float s = sqrtf(fmaxf(0.f, 1.f - z * z));
  return __expf(beta * (s - 1.f));
}
template <> __device__ __forceinline__ double es_weight<double>(double d, double inv_hw, double beta) {
  double z = d * inv_hw;
  double s = sqrt(fmax(0.0, 1.0 - z * z));
  return exp(beta * (s - 1.0));
}

template <typename T, int W>
__global__ void __launch_bounds__(512, 1)
polar_kernel(const PolarParams* __restrict__ ppg, const T* __restrict__ images, int64_t n_img, int64_t img_stride,
             T* __restrict__ ghat) {
  using T2 = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PolarParams& pp = *reinterpret_cast<PolarParams*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nwarps = nthr >> 5;
  {
    const int* src = reinterpret_cast<const int*>(ppg);
    int* dst = reinterpret_cast<int*>(smem_raw);
    for (int i = tid; i < (int)(sizeof(PolarParams) / 4); i += nthr) dst[i] = src[i];
  }
  __syncthreads();
  const int M = pp.M, L = pp.L, nt = pp.n_theta, half = pp.half, n_xi = pp.n_xi;
  unsigned char* base = smem_raw + ((sizeof(PolarParams) + 15) / 16) * 16;
  T2* twM = reinterpret_cast<T2*>(base);
  T2* twT = twM + M;
  T* dap = reinterpret_cast<T*>(twT + nt);
  T2* wscr = reinterpret_cast<T2*>(base + (((size_t)(M + nt) * sizeof(T2) + (size_t)L * sizeof(T) + 15) / 16) * 16);
  T2* region = wscr + (size_t)nwarps * 2 * M;
  T2* myA = wscr + (size_t)warp * 2 * M;          // row / column FFT ping-pong
  T2* myB = myA + M;
  T2* angA = region + (size_t)warp * 2 * nt;      // angular FFT ping-pong (region is free then)
  T2* angB = angA + nt;

  {
    const T2* gtM = reinterpret_cast<const T2*>(pp.tw_M);
    const T2* gtT = reinterpret_cast<const T2*>(pp.tw_theta);
    const T* gd = reinterpret_cast<const T*>(pp.deapod);
    for (int i = tid; i < M; i += nthr) twM[i] = gtM[i];
    for (int i = tid; i < nt; i += nthr) twT[i] = gtT[i];
    for (int i = tid; i < L; i += nthr) dap[i] = gd[i];
  }
  __syncthreads();

  T2* X = reinterpret_cast<T2*>(pp.xscratch) + (int64_t)blockIdx.x * pp.xscratch_stride;
  T2* Pol = reinterpret_cast<T2*>(pp.pscratch) + (int64_t)blockIdx.x * pp.pscratch_stride;
  const int ncx = pp.ncols_x, col_lo = pp.col_lo, S = pp.S;
  const int kk = (pp.k_max + 1) | 1;
  const T hw = T(pp.half_w), inv_hw = T(1) / hw, beta = T(pp.beta);

  for (int64_t img = blockIdx.x; img < n_img; img += gridDim.x) {
    const T* I = images + img * img_stride;
    // ---------------- K1a: row FFTs (pairs of real rows packed as one complex sequence) ----------------
    for (int pr = warp; pr < (L + 1) / 2; pr += nwarps) {
      T2* sc = myA;
      for (int t = lane; t < M; t += 32) sc[t] = T2{T(0), T(0)};
      __syncwarp();
      const int a0 = 2 * pr, a1 = a0 + 1;
      const bool has1 = a1 < L;
      const T d0 = dap[a0], d1 = has1 ? dap[a1] : T(0);
      for (int b = lane; b < L; b += 32) {
        int pos = b - L / 2; if (pos < 0) pos += M;
        T v0 = I[(int64_t)a0 * L + b] * d0 * dap[b];
        T v1 = has1 ? I[(int64_t)a1 * L + b] * d1 * dap[b] : T(0);
        sc[pos] = T2{v0, v1};
      }
      __syncwarp();
      sc = warp_fft<T2>(myA, 1, nullptr, 1, myA, myB, pp.fft_M, twM, lane);
      for (int cc = lane; cc < ncx; cc += 32) {
        int m = (col_lo + cc) % M; if (m < 0) m += M;
        int mm = M - m; if (mm == M) mm = 0;
        T2 zm = sc[m], zc = sc[mm];
        zc.y = -zc.y;                                          // conj Z(-m)
        T2 xa = {T(0.5) * (zm.x + zc.x), T(0.5) * (zm.y + zc.y)};
        T2 dd = csub(zm, zc);
        T2 xb = {T(0.5) * dd.y, T(-0.5) * dd.x};               // (Z(m) - conj Z(-m)) / (2i)
        X[(int64_t)a0 * ncx + cc] = xa;
        if (has1) X[(int64_t)a1 * ncx + cc] = xb;
      }
      __syncwarp();
    }
    __syncthreads();

    // ---------------- per phase: K1b column FFTs in shared memory, K2 gather ----------------
    for (int ph = 0; ph < pp.n_phase; ++ph) {
      const int lo = pp.phase_lo[ph];
      int ncols = col_lo + ncx - lo; if (ncols > S) ncols = S;
      T2* Gc = region;
      for (int idx = tid; idx < M * ncols; idx += nthr) {
        const int row = idx / ncols, cc = idx - row * ncols;
        const int i1 = row < M / 2 ? row : row - M;
        const int a = i1 + L / 2;
        T2 v = T2{T(0), T(0)};
        if (a >= 0 && a < L) v = X[(int64_t)a * ncx + (lo - col_lo) + cc];
        Gc[row * S + cc] = v;
      }
      __syncthreads();
      for (int cc = warp; cc < ncols; cc += nwarps) warp_fft<T2>(Gc + cc, S, Gc + cc, S, myA, myB, pp.fft_M, twM, lane);
      __syncthreads();
      const int nb = pp.phase_node_begin[ph], ne = pp.phase_node_begin[ph + 1];
      for (int t = nb + tid; t < ne; t += nthr) {
        const uint32_t nd = __ldg(pp.nodes + t);
        const int j = int(nd >> 16), l = int(nd & 0xffffu);
        const double r = __ldg(pp.rho + j);
        const double k1 = r * __ldg(pp.cs + 2 * l), k2 = r * __ldg(pp.cs + 2 * l + 1);
        const double f1 = ceil(k1 - pp.half_w), f2 = ceil(k2 - pp.half_w);
        const int b1 = int(f1), b2 = int(f2);
        const T t1 = T(k1 - f1), t2 = T(k2 - f2);
        T wx[W], wy[W];
#pragma unroll
        for (int q = 0; q < W; ++q) {
          wx[q] = es_weight<T>(t1 - T(q), inv_hw, beta);
          wy[q] = es_weight<T>(t2 - T(q), inv_hw, beta);
        }
        T2 acc = T2{T(0), T(0)};
        const T2* gcol = Gc + (b2 - lo);
#pragma unroll
        for (int q = 0; q < W; ++q) {
          int row = b1 + q;
          row = row < 0 ? row + M : (row >= M ? row - M : row);
          const T2* gp = gcol + row * S;
          T2 s = T2{T(0), T(0)};
#pragma unroll
          for (int c = 0; c < W; ++c) {
            const T2 g = gp[c];
            s.x += wy[c] * g.x; s.y += wy[c] * g.y;
          }
          acc.x += wx[q] * s.x; acc.y += wx[q] * s.y;
        }
        Pol[(int64_t)j * half + l] = acc;
      }
      __syncthreads();
    }

    // ---------------- K3: angular FFT per ring, staged, written k-major ----------------
    const int G = pp.ring_group;
    for (int j0 = 0; j0 < n_xi; j0 += G) {
      const int g = min(G, n_xi - j0);
      T2* stg = region + (size_t)nwarps * 2 * nt;
      for (int jj = warp; jj < g; jj += nwarps) {
        T2* sc = angA;
        const T2* src = Pol + (int64_t)(j0 + jj) * half;
        for (int l = lane; l < half; l += 32) {
          T2 v = src[l];
          sc[l] = v;
          sc[l + half] = T2{v.x, -v.y};
        }
        __syncwarp();
        sc = warp_fft<T2>(angA, 1, nullptr, 1, angA, angB, pp.fft_theta, twT, lane);
        for (int k = lane; k <= pp.k_max; k += 32) stg[jj * kk + k] = sc[k];
        __syncwarp();
      }
      __syncthreads();
      const int tot = (pp.k_max + 1) * 2 * g;
      for (int idx = tid; idx < tot; idx += nthr) {
        const int jj = idx % g, rest = idx / g, part = rest & 1, k = rest >> 1;
        const T2 v = stg[jj * kk + k];
        ghat[(((int64_t)k * n_img + img) * 2 + part) * n_xi + j0 + jj] = part ? v.y : v.x;
      }
      __syncthreads();
    }
  }
}

int polar_max_smem() { return 227 * 1024; }

int polar_fixed_smem(int M, int n_theta, int L, int csz, int nwarps) {
  return (int)(((sizeof(PolarParams) + 15) / 16) * 16) + (int)((((M + n_theta) * csz + L * (csz / 2)) + 15) / 16) * 16 +
         nwarps * 2 * M * csz;
}

template <typename T, int W>
static cudaError_t launch_polar_t(const Plan& P, const void* d_images, int64_t n_img, int64_t stride,
                                  cudaStream_t s) {
  auto kern = polar_kernel<T, W>;
  static int configured = 0;
  if (configured < P.polar_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P.polar_smem);
    if (e != cudaSuccess) return e;
    configured = P.polar_smem;
  }
  int grid = (int)std::min<int64_t>(P.polar_grid, n_img);
  kern<<<grid, P.pp.nwarps * 32, P.polar_smem, s>>>(P.d_pp, reinterpret_cast<const T*>(d_images), n_img, stride,
                                                    reinterpret_cast<T*>(P.d_ghat));
  return cudaGetLastError();
}

cudaError_t launch_polar(const Plan& P, const void* d_images, int64_t n_img, int64_t stride, cudaStream_t s) {
  if (P.dt == FBSPCA_F64) {
    if (P.w != 13) return cudaErrorInvalidValue;
    return launch_polar_t<double, 13>(P, d_images, n_img, stride, s);
  }
  switch (P.w) {
    case 6: return launch_polar_t<float, 6>(P, d_images, n_img, stride, s);
    case 7: return launch_polar_t<float, 7>(P, d_images, n_img, stride, s);
    case 8: return launch_polar_t<float, 8>(P, d_images, n_img, stride, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fbspca
