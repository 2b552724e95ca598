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

#include "fft_device.cuh"
#include "internal.h"

namespace fbspca {

// ---------------------------------------------------------------- cp.async (LDGSTS): many loads in flight
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Drop dead scratch lines from L2 without a write-back (the per-CTA X / Pol scratch is consumed once).
__device__ __forceinline__ void l2_discard(const void* base, size_t bytes, int tid, int nthr) {
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(base) + 127) & ~uintptr_t(127);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(base) + bytes) & ~uintptr_t(127);
  for (uintptr_t a = a0 + uintptr_t(tid) * 128; a < a1; a += uintptr_t(nthr) * 128)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

// ---------------------------------------------------------------- TMEM as scratch (tcgen05.st / ld, 32x32b: each lane its row)
__device__ __forceinline__ void tm_st4(uint32_t taddr, float a, float b, float c, float d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
               ::"r"(taddr), "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)),
                 "r"(__float_as_uint(d)) : "memory");
}
__device__ __forceinline__ float4 tm_ld4(uint32_t taddr) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return make_float4(__uint_as_float(r0), __uint_as_float(r1), __uint_as_float(r2), __uint_as_float(r3));
}

// ---------------------------------------------------------------- ES window weights
// phi(d) = exp(beta (sqrt(1 - (d/hw)^2) - 1)), |d| <= hw.  fp32: MUFU sqrt.approx / ex2.approx
// (relative error ~1e-7, far below the 1e-5 NUFFT budget); fp64: exact.
__device__ __forceinline__ float sqrt_approx(float x) { float y; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2_approx(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <typename T> struct Es;
template <> struct Es<float> {
  float inv_hw, bl;                       // bl = beta * log2(e)
  __device__ Es(double hw, double beta) : inv_hw(float(1.0 / hw)), bl(float(beta * 1.4426950408889634)) {}
  __device__ __forceinline__ float operator()(float d) const {
    const float z = d * inv_hw;
    const float s = sqrt_approx(fmaxf(fmaf(-z, z, 1.f), 0.f));
    return ex2_approx(fmaf(s, bl, -bl));
  }
  // phi(ta - q), phi(tb - q) with packed f32x2 arithmetic: d = t - q, r = hw^2 - d^2 = (q - t) d + hw^2 (FADD2, FADD2,
  // FFMA2), e = ex2(bl s / hw - bl), s = sqrt|r| (the |.| only absorbs rounding at |d| = hw; FFMA2), 4 MUFU
  __device__ __forceinline__ void pair(float ta, float tb, float q, float& pa, float& pb) const {
    const float hw = 1.f / inv_hw, hw2 = hw * hw, blh = bl * inv_hw;
    unsigned long long t, qq, d, dn, r, e, c2, h2, b2;
    asm("mov.b64 %0, {%1, %2};" : "=l"(t) : "f"(ta), "f"(tb));
    asm("mov.b64 %0, {%1, %1};" : "=l"(qq) : "f"(q));
    asm("mov.b64 %0, {%1, %1};" : "=l"(h2) : "f"(hw2));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(t), "l"(qq));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dn) : "l"(qq), "l"(t));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(dn), "l"(d), "l"(h2));
    float ra, rb;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(ra), "=f"(rb) : "l"(r));
    const float sa = sqrt_approx(fabsf(ra)), sb = sqrt_approx(fabsf(rb));
    asm("mov.b64 %0, {%1, %2};" : "=l"(e) : "f"(sa), "f"(sb));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c2) : "f"(blh));
    asm("mov.b64 %0, {%1, %1};" : "=l"(b2) : "f"(-bl));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(e), "l"(c2), "l"(b2));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(ra), "=f"(rb) : "l"(r));
    pa = ex2_approx(ra);
    pb = ex2_approx(rb);
  }
};
template <> struct Es<double> {
  double inv_hw, beta;
  __device__ Es(double hw, double b) : inv_hw(1.0 / hw), beta(b) {}
  __device__ __forceinline__ double operator()(double d) const {
    const double z = d * inv_hw;
    return exp(beta * (sqrt(fmax(1.0 - z * z, 0.0)) - 1.0));
  }
};

// ---------------------------------------------------------------- optional stage profiler (debug builds only)
#ifdef FBSPCA_PHASE_PROF
static __device__ unsigned long long g_phase_prof[1024 * 8];
#define PROF_INIT() unsigned long long _pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long _pt = clock64();
#define PROF_MARK(i) do { if (threadIdx.x == 0) { long long _n = clock64(); _pacc[i] += _n - _pt; _pt = _n; } } while (0)
#define PROF_STORE() do { if (threadIdx.x == 0) for (int _i = 0; _i < 8; ++_i) g_phase_prof[blockIdx.x * 8 + _i] = _pacc[_i]; } while (0)
#else
#define PROF_INIT()
#define PROF_MARK(i)
#define PROF_STORE()
#endif

// ---------------------------------------------------------------- the fused polar kernel
// MC: compile-time M (0 = runtime plan); when MC > 0 the ring FFT length is 2 MC.
template <typename T, int W, int MC>
__global__ void __launch_bounds__(512, 1)
polar_kernel(const PolarParams* __restrict__ ppg, const T* __restrict__ images, int64_t n_img, int64_t img_stride,
             T* __restrict__ ghat) {
  using T2 = typename Cx<T>::t;
  constexpr int NC = MC > 0 ? 2 * MC : 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PolarParams& pp = *reinterpret_cast<PolarParams*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nwarps = nthr >> 5;
  {
    const int* src = reinterpret_cast<const int*>(ppg);
    int* dst = reinterpret_cast<int*>(smem_raw);
    for (int i = tid; i < (int)(sizeof(PolarParams) / 4); i += nthr) dst[i] = src[i];
  }
  __syncthreads();
  const int M = MC > 0 ? MC : pp.M;
  const int L = pp.L, nt = MC > 0 ? NC : pp.n_theta, half = nt / 2, n_xi = pp.n_xi;
  unsigned char* base = smem_raw + ((sizeof(PolarParams) + 15) / 16) * 16;
  T2* twM = reinterpret_cast<T2*>(base);
  T2* twT = twM + M;
  T* dap = reinterpret_cast<T*>(twT + nt);
  int* skj0 = reinterpret_cast<int*>(dap + L);     // kj0[k] (K4's first ring per k) for the ghat write-out
  T2* wscr = reinterpret_cast<T2*>(base + (((size_t)(M + nt) * sizeof(T2) + (size_t)L * sizeof(T) +
                                            (size_t)(pp.k_max + 1) * sizeof(int) + 15) / 16) * 16);
  const int MP = (M + 15) & ~15, NTP = (nt + 15) & ~15;   // ping-pong lengths: padi permutes within 16-blocks
  // HW: M = 256 fp32 -- every FFT (rows, columns, rings) is the half-warp radix-16 x 16 fft256_hw, two per warp
  constexpr bool HW = (MC == 256) && sizeof(T) == 4;
  static_assert(!HW || W <= 16, "fft256_hw column stores assume PADR <= 16 wrapped rows");
  const int WS = polar_warp_scratch(M, HW);
  T2* region = wscr + (size_t)pp.fft_warps * WS;
  // FFT groups: one warp (FG = 32) or, for M = 512 / 600 / 720 (8 ping-pong pairs fit, not 16), a warp pair (FG = 64)
  // on named barrier 1 + grp, so all 16 warps run the row / column / ring FFTs
  constexpr int FG = (MC == 512 || MC == 600 || MC == 720) ? 64 : 32;
  const int grp = warp / (FG / 32), glane = tid & (FG - 1), gbar = 1 + grp;
  T2* myA = wscr + (size_t)grp * WS;             // row / column FFT ping-pong
  T2* myB = myA + MP;
  T2* angA = region + (size_t)warp * 2 * NTP;     // angular FFT ping-pong (region is free then)
  T2* angB = angA + NTP;
  {
    const T2* gtM = reinterpret_cast<const T2*>(pp.tw_M);
    const T2* gtT = reinterpret_cast<const T2*>(pp.tw_theta);
    const T* gd = reinterpret_cast<const T*>(pp.deapod);
    if constexpr (HW) {                                          // tw2[k1 16 + t2] = w256^(k1 t2)
      for (int i = tid; i < 256; i += nthr) twM[i] = gtM[((i >> 4) * (i & 15)) & 255];
      for (int i = tid; i < NC / 2; i += nthr) twT[i] = gtT[i];
    } else if constexpr (MC > 0) {
      build_stage_tw<T2, MC>(twM, gtM, tid, nthr);             // per-stage tables (<= M entries)
      for (int i = tid; i < NC / 2; i += nthr) twT[i] = gtT[i];   // ring pairs: e^{-2 pi i t / n_theta}, t < n/2
    } else {
      for (int i = tid; i < M; i += nthr) twM[i] = gtM[i];
      for (int i = tid; i < nt; i += nthr) twT[i] = gtT[i];
    }
    for (int i = tid; i < L; i += nthr) dap[i] = gd[i];
    for (int i = tid; i <= pp.k_max; i += nthr) skj0[i] = pp.kj0[i];
  }
  __syncthreads();

  // TMEM parking (pp.tmem_x, M = 256): warp w keeps its row pairs' second-phase columns in TMEM lanes 32 (w % 4) ..,
  // columns 64 (w / 4) .. -- written by the row pass, read back by the same warp as the phase-1 fill (no L2 round trip)
  __shared__ uint32_t tmem_slot;
  uint32_t tmem_base = 0;
  const bool use_tmem = (MC == 256) && pp.tmem_x;
  if (use_tmem) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;"
                   ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_slot))));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    tmem_base = tmem_slot;
  }
  const uint32_t tmem_mine = tmem_base + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(64 * (warp >> 2));
  T2* X = reinterpret_cast<T2*>(pp.xscratch) + (int64_t)blockIdx.x * pp.xscratch_stride;
  T2* Pol = reinterpret_cast<T2*>(pp.pscratch) + (int64_t)blockIdx.x * pp.pscratch_stride;
  const int ncx = pp.ncols_x, col_lo = pp.col_lo, S = pp.S;
  const int PADR = W;                              // wrapped duplicate rows on each side
  const int row0 = M / 2 + PADR;                   // physical row of m1 = 0
  const Es<T> phi(pp.half_w, pp.beta);
  const int G = pp.ring_group;

  // The image is staged in shared memory behind the phase-0 grid rows.  Its load is issued with cp.async right
  // after the previous image's gather (the angular pass only touches the staging rows in front of it), so it
  // overlaps the ring FFTs and the write-out.
  T* simg = reinterpret_cast<T*>(region + (pp.img_off >= 0 ? pp.img_off : 0));
  const int nel = L * L;
  auto issue_image = [&](int64_t im) {
    const T* src = images + im * img_stride;
    if ((nel * (int)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      for (int i = tid; i < nel * (int)sizeof(T) / 16; i += nthr)
        cp_async16(reinterpret_cast<int4*>(simg) + i, reinterpret_cast<const int4*>(src) + i);
    } else {
      for (int i = tid; i < nel; i += nthr) simg[i] = __ldg(src + i);
    }
  };
  bool prefetched = false;
  PROF_INIT();
  for (int64_t img = blockIdx.x; img < n_img; img += gridDim.x) {
    const T* I = images + img * img_stride;
    const T* Isrc = I;
    if (pp.img_off >= 0) {
      if (!prefetched) issue_image(img);
      cp_async_wait_all();
      __syncthreads();
      Isrc = simg;
    }
    // ---------------- K1a: row FFTs, two real rows per complex sequence, deapodised + zero-padded on load
    if constexpr (HW) {
      // half-warp h of warp w transforms row pair pr = base + h FW + w (FW = fft_warps = 16: the TMEM slot of pr is
      // pr >> 4 as in the warp-per-pair path), then the whole warp splits and writes both results
      const int q = lane & 15, h = lane >> 4, FW = pp.fft_warps, nrp = (L + 1) / 2;
      T2* hb = wscr + (size_t)grp * 2 * kHwBuf;
      T2* mybuf = hb + h * kHwBuf;
      const int lo0 = pp.phase_lo[0], hi0 = lo0 + (S < col_lo + ncx - lo0 ? S : col_lo + ncx - lo0);
      const int lo1 = pp.n_phase > 1 ? pp.phase_lo[1] : (1 << 30);
      for (int base = 0; grp < FW && base < nrp; base += 2 * FW) {
        {
          const int pr = base + h * FW + grp;
          const bool okp = pr < nrp;
          const int a0 = okp ? 2 * pr : 0, a1 = a0 + 1;
          const bool has1 = okp && a1 < L;
          const T* r0 = Isrc + (int64_t)a0 * L;
          const T* r1 = Isrc + (int64_t)(has1 ? a1 : a0) * L;
          const T d0 = okp ? dap[a0] : T(0), d1 = has1 ? dap[a1] : T(0);
          float2 v[16];
#pragma unroll
          for (int t1 = 0; t1 < 16; ++t1) {
            if (t1 >= 4 && t1 < 12) { v[t1] = float2{0.f, 0.f}; continue; }      // zero padding (HZ)
            const int t = 16 * t1 + q;
            const int b = (t < 128 ? t : t - 256) + L / 2;
            if (b < 0 || b >= L) { v[t1] = float2{0.f, 0.f}; continue; }
            const T db = dap[b];
            v[t1] = float2{r0[b] * d0 * db, r1[b] * d1 * db};
          }
          fft256_hw<true>(v, mybuf, twM, q);
          hw_store_natural(v, mybuf, q);
        }
        __syncwarp();
        for (int hh = 0; hh < 2; ++hh) {               // warp-uniform: the TMEM stores are warp-collective
          const int pr = base + hh * FW + grp;
          if (pr >= nrp) continue;
          const T2* res = hb + hh * kHwBuf;
          const int a0 = 2 * pr, a1 = a0 + 1;
          const bool has1 = a1 < L;
          for (int cc0 = 0; cc0 < ncx; cc0 += 32) {
            const int cc = cc0 + lane;
            const bool ok = cc < ncx;
            int m = (col_lo + (ok ? cc : 0)) % M; if (m < 0) m += M;
            int mm = M - m; if (mm == M) mm = 0;
            T2 zm = res[hw_idx(m)], zc = res[hw_idx(mm)];
            zc.y = -zc.y;                                            // conj Z(-m)
            const T2 xa = {T(0.5) * (zm.x + zc.x), T(0.5) * (zm.y + zc.y)};
            const T2 dd = csub(zm, zc);
            const T2 xb = {T(0.5) * dd.y, T(-0.5) * dd.x};           // (Z(m) - conj Z(-m)) / (2i)
            const int m2 = col_lo + cc;
            if (use_tmem) {
              const int gi = cc0 / 32 - pp.tmem_g0;
              if (gi >= 0 && gi < pp.tmem_ng)
                tm_st4(tmem_mine + uint32_t(((pr >> 4) * pp.tmem_ng + gi) * 4), float(xa.x), float(xa.y),
                       float(xb.x), float(xb.y));
            } else if (ok && m2 >= lo1) {
              X[(int64_t)a0 * ncx + cc] = xa;
              if (has1) X[(int64_t)a1 * ncx + cc] = xb;
            }
            if (ok && m2 < hi0) {
              region[(size_t)a0 * S + (m2 - lo0)] = xa;
              if (has1) region[(size_t)a1 * S + (m2 - lo0)] = xb;
            }
          }
        }
        __syncwarp();
      }
    } else if (grp < pp.fft_warps) {
      for (int pr = grp; pr < (L + 1) / 2; pr += pp.fft_warps) {
        const int a0 = 2 * pr, a1 = a0 + 1;
        const bool has1 = a1 < L;
        const T* r0 = Isrc + (int64_t)a0 * L;
        const T* r1 = Isrc + (int64_t)(has1 ? a1 : a0) * L;
        const T d0 = dap[a0], d1 = has1 ? dap[a1] : T(0);
        auto ld = [&](int t) -> T2 {
          const int b = (t < M / 2 ? t : t - M) + L / 2;          // pixel column of FFT position t
          if (b < 0 || b >= L) return T2{T(0), T(0)};
          const T db = dap[b];
          return T2{r0[b] * d0 * db, r1[b] * d1 * db};
        };
        // pow2: the result stays in the warp's (swizzled) ping-pong buffer and phase-0 columns go straight
        // into the shared grid (rows = image rows); only columns of later phases go through X.
        // runtime sizes: the result goes to a per-warp slice of the (still free) phase region.
        T2* res = (MC > 0) ? (fft_result_in_A<MC>() ? myA : myB) : region + (size_t)warp * M;
        auto st = [res](int i, T2 v) { res[MC > 0 ? padi(i) : i] = v; };
        fft_any<T2, MC, true, FG>(pp.fft_M, ld, st, myA, myB, twM, glane, gbar);
        const int lo0 = pp.phase_lo[0], hi0 = lo0 + (S < col_lo + ncx - lo0 ? S : col_lo + ncx - lo0);
        const int lo1 = pp.n_phase > 1 ? pp.phase_lo[1] : (1 << 30);
        // (warp-uniform trip count: the TMEM stores are warp-collective)
        for (int cc0 = 0; cc0 < ncx; cc0 += FG) {
          const int cc = cc0 + glane;
          const bool ok = cc < ncx;
          int m = (col_lo + (ok ? cc : 0)) % M; if (m < 0) m += M;
          int mm = M - m; if (mm == M) mm = 0;
          T2 zm = res[MC > 0 ? padi(m) : m], zc = res[MC > 0 ? padi(mm) : mm];
          zc.y = -zc.y;                                              // conj Z(-m)
          const T2 xa = {T(0.5) * (zm.x + zc.x), T(0.5) * (zm.y + zc.y)};
          const T2 dd = csub(zm, zc);
          const T2 xb = {T(0.5) * dd.y, T(-0.5) * dd.x};             // (Z(m) - conj Z(-m)) / (2i)
          const int m2 = col_lo + cc;
          if (use_tmem) {
            const int gi = cc0 / 32 - pp.tmem_g0;
            if (gi >= 0 && gi < pp.tmem_ng)
              tm_st4(tmem_mine + uint32_t(((pr >> 4) * pp.tmem_ng + gi) * 4), float(xa.x), float(xa.y), float(xb.x),
                     float(xb.y));
          } else if (ok && (MC == 0 || m2 >= lo1)) {
            X[(int64_t)a0 * ncx + cc] = xa;
            if (has1) X[(int64_t)a1 * ncx + cc] = xb;
          }
          if (ok && MC > 0 && m2 < hi0) {
            region[(size_t)a0 * S + (m2 - lo0)] = xa;
            if (has1) region[(size_t)a1 * S + (m2 - lo0)] = xb;
          }
        }
        gsync<FG>(gbar);
      }
    }
    if (use_tmem) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();
    PROF_MARK(0);

    // ---------------- per phase: K1b column FFTs (input rows 0..L-1 = image rows, output fftshifted with
    // PADR wrapped duplicate rows), then K2 gather of node pairs (theta, pi - theta)
    for (int ph = 0; ph < pp.n_phase; ++ph) {
      const int lo = pp.phase_lo[ph];
      int ncols = col_lo + ncx - lo; if (ncols > S) ncols = S;
      T2* Gc = region;
      if (use_tmem && ph == 1) {                    // phase 1 from TMEM: each warp reads back its own row pairs
        for (int pr = warp; pr < (L + 1) / 2; pr += 16) {
          const int a0 = 2 * pr, a1 = a0 + 1;
          for (int gi = 0; gi < pp.tmem_ng; ++gi) {
            const float4 v = tm_ld4(tmem_mine + uint32_t(((pr >> 4) * pp.tmem_ng + gi) * 4));
            const int m2 = col_lo + 32 * (pp.tmem_g0 + gi) + lane;
            if (m2 >= lo && m2 < lo + ncols && m2 - col_lo < ncx) {
              Gc[(size_t)a0 * S + (m2 - lo)] = T2{v.x, v.y};
              if (a1 < L) Gc[(size_t)a1 * S + (m2 - lo)] = T2{v.z, v.w};
            }
          }
        }
        __syncthreads();
      } else if (MC == 0 || ph > 0) {               // pow2 phase 0 was written by the row pass directly
        for (int a = warp; a < L; a += nwarps) {
          const T2* src = X + (int64_t)a * ncx + (lo - col_lo);
          T2* dst = Gc + (size_t)a * S;
          for (int cc = lane; cc < ncols; cc += 32) {
            if constexpr (sizeof(T2) == 8) cp_async8(dst + cc, src + cc);
            else dst[cc] = src[cc];
          }
        }
        cp_async_wait_all();
        __syncthreads();
        if (ph == pp.n_phase - 1) l2_discard(X, (size_t)L * ncx * sizeof(T2), tid, nthr);
      }
      PROF_MARK(1);
      if constexpr (HW) {
        // half-warp h of warp w: column cc = base + 2 w + h, in place (all inputs are in registers before the first
        // store: fft256_hw's transpose sync), output fftshifted with PADR wrapped duplicate rows
        const int q = lane & 15, h = lane >> 4, FW = pp.fft_warps;
        T2* mybuf = wscr + (size_t)grp * 2 * kHwBuf + h * kHwBuf;
        for (int base = 0; grp < FW && base + 2 * grp < ncols; base += 2 * FW) {      // warp-uniform bound
          const int cc = base + 2 * grp + h;
          const bool okc = cc < ncols;
          T2* col = Gc + (okc ? cc : 0);
          float2 v[16];
#pragma unroll
          for (int t1 = 0; t1 < 16; ++t1) {
            if (t1 >= 4 && t1 < 12) { v[t1] = float2{0.f, 0.f}; continue; }
            const int t = 16 * t1 + q;
            const int a = (t < 128 ? t : t - 256) + L / 2;
            v[t1] = (okc && a >= 0 && a < L) ? col[(size_t)a * S] : float2{0.f, 0.f};
          }
          fft256_hw<true>(v, mybuf, twM, q);
          if (okc) {
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) {
              const int m1 = k2 < 8 ? q + 16 * k2 : q + 16 * k2 - 256;
              col[(size_t)(m1 + row0) * S] = v[k2];
              if (k2 == 8 && m1 < -128 + PADR) col[(size_t)(m1 + 256 + row0) * S] = v[k2];
              if (k2 == 7 && m1 >= 128 - PADR) col[(size_t)(m1 - 256 + row0) * S] = v[k2];
            }
          }
        }
      } else if (grp < pp.fft_warps) {
        for (int cc = grp; cc < ncols; cc += pp.fft_warps) {
          T2* col = Gc + cc;
          auto ld = [&](int t) -> T2 {
            const int a = (t < M / 2 ? t : t - M) + L / 2;
            return (a >= 0 && a < L) ? col[(size_t)a * S] : T2{T(0), T(0)};
          };
          auto st = [&](int t, T2 v) {
            const int m1 = t < M / 2 ? t : t - M;
            col[(size_t)(m1 + row0) * S] = v;
            if (m1 < -M / 2 + PADR) col[(size_t)(m1 + M + row0) * S] = v;
            if (m1 >= M / 2 - PADR) col[(size_t)(m1 - M + row0) * S] = v;
          };
          fft_any<T2, MC, true, FG>(pp.fft_M, ld, st, myA, myB, twM, glane, gbar);
        }
      }
      __syncthreads();
      PROF_MARK(2);
      if constexpr (sizeof(T) == 4 && (W == 5 || W == 6) && MC > 0) {
        constexpr int W1 = W + 1;                     // the shared (W + 1) x (W + 1) window
        // double entries: nodes a, b of one ring (+ their mirrors) over one shared (W + 1) x (W + 1) window at U
        const int db = pp.phase_dbl_begin[ph], de = pp.phase_dbl_begin[ph + 1];
        // records are loaded one iteration ahead (an L2 round trip per entry was the loop's top stall)
        int4 n0 = make_int4(0, 0, 0, 0), n1 = n0;
        if (db + tid < de) { n0 = __ldg(pp.dnoderec + 2 * (db + tid)); n1 = __ldg(pp.dnoderec + 2 * (db + tid) + 1); }
        for (int t = db + tid; t < de; t += nthr) {
          const int4 r0 = n0, r1 = n1;
          if (t + nthr < de) { n0 = __ldg(pp.dnoderec + 2 * (t + nthr)); n1 = __ldg(pp.dnoderec + 2 * (t + nthr) + 1); }
          const int u1 = int(short(r0.x & 0xFFFF)), u2 = r0.x >> 16, of = r0.w;
          const float t1a = __int_as_float(r0.y), t2a = __int_as_float(r0.z);
          const float t1b = __int_as_float(r1.y), t2b = __int_as_float(r1.z);
          float xa[W1], ya[W1], xb[W1], yb[W1];
          {
            float wa[W], va[W], wb[W], vb[W];
#pragma unroll
            for (int q = 0; q < W; ++q) {               // nodes a and b in one f32x2 pair per direction
              phi.pair(t1a, t1b, float(q), wa[q], wb[q]);
              phi.pair(t2a, t2b, float(q), va[q], vb[q]);
            }
            const bool o1a = of & 1, o2a = of & 2, o1b = of & 4, o2b = of & 8;
#pragma unroll
            for (int r = 0; r < W1; ++r) {
              xa[r] = o1a ? (r ? wa[r - 1] : 0.f) : (r < W ? wa[r] : 0.f);
              ya[r] = o2a ? (r ? va[r - 1] : 0.f) : (r < W ? va[r] : 0.f);
              xb[r] = o1b ? (r ? wb[r - 1] : 0.f) : (r < W ? wb[r] : 0.f);
              yb[r] = o2b ? (r ? vb[r - 1] : 0.f) : (r < W ? vb[r] : 0.f);
            }
          }
          const T2* gcol = Gc + (u2 - lo);
          T2 aa = T2{0.f, 0.f}, ab = aa, ma = aa, mb = aa;      // (node a, node b) x (direct, mirrored)
#pragma unroll
          for (int r = 0; r < W1; ++r) {
            const T2* ga = gcol + (size_t)(u1 + r + row0) * S;
            const T2* gm = gcol + (size_t)(row0 - u1 - r) * S;
            T2 sa = T2{0.f, 0.f}, sb = sa, na = sa, nb2 = sa;
#pragma unroll
            for (int c = 0; c < W1; ++c) {
              const T2 g = ga[c];
              sa = rfma(ya[c], g, sa); sb = rfma(yb[c], g, sb);
            }
#pragma unroll
            for (int c = 0; c < W1; ++c) {
              const T2 g = gm[c];
              na = rfma(ya[c], g, na); nb2 = rfma(yb[c], g, nb2);
            }
            aa = rfma(xa[r], sa, aa); ab = rfma(xb[r], sb, ab);
            ma = rfma(xa[r], na, ma); mb = rfma(xb[r], nb2, mb);
          }
          // Pol slots (plan.cpp pol_slot): ring j holds its samples contiguously, mirror of slot l at half_j - l
          const int ja = (r1.x >> 16) & 0xFFF, la = r1.x & 0xFFFF, ha = half >> ((uint32_t(r1.x) >> 28) & 3);
          const int jb = (r1.w >> 16) & 0xFFF, lb = r1.w & 0xFFFF, hb = half >> ((uint32_t(r1.w) >> 28) & 3);
          // nodes a, b are (ja, la), (jb, lb); their mirrors (ja, half_a - la), (jb, half_b - lb).  Ring neighbours
          // (jb = ja, lb = la + 1) with an even half_j: exactly one of the two adjacent slot pairs starts 16-byte
          // aligned and is one 16-byte store.  Otherwise (cross-ring pairs, odd half_j): four 8-byte stores.
          T2* prow = Pol + (int64_t)ja * half;
          if (jb != ja || lb != la + 1 || (ha & 1)) {     // (odd half_j, e.g. 600 / 8: no aligned pair guaranteed)
            T2* prowb = Pol + (int64_t)jb * half;
            prow[la] = aa;
            prowb[lb] = ab;
            prow[ha - la] = ma;
            prowb[hb - lb] = mb;
          } else if (la & 1) {
            prow[la] = aa;
            prow[la + 1] = ab;
            *reinterpret_cast<float4*>(prow + (ha - la - 1)) = make_float4(mb.x, mb.y, ma.x, ma.y);
          } else {
            *reinterpret_cast<float4*>(prow + la) = make_float4(aa.x, aa.y, ab.x, ab.y);
            prow[ha - la] = ma;
            prow[ha - la - 1] = mb;
          }
        }
      }
      const int nb = pp.phase_node_begin[ph], ne = pp.phase_node_begin[ph + 1];
      // singles are dealt from the last thread down: the threads the double entries' ragged last round left idle
      // take them first (C3 phase 1: 2072 doubles = 4 x 512 + 24, 272 singles -- no thread does both a fifth
      // double and a single).  A reversed 16-aligned half-warp is the same half-warp: the bank packing holds.
#ifdef FBSPCA_SINGLES_FWD
      const int rtid = tid;                           // A/B: the forward deal
#else
      const int rtid = nthr - 1 - tid;
#endif
      int4 rec_next = make_int4(0, 0, 0, 0);          // fp32: next entry's record loaded one iteration ahead
      if (sizeof(T) == 4 && nb + rtid < ne) rec_next = __ldg(pp.noderec + nb + rtid);
      for (int t = nb + rtid; t < ne; t += nthr) {
        int j, l, b1, b2, hj = half;
        T t1, t2;
        if constexpr (sizeof(T) == 4) {             // fp32: precomputed record (one 16-B load)
          const int4 rec = rec_next;
          if (t + nthr < ne) rec_next = __ldg(pp.noderec + t + nthr);
          b1 = int(short(rec.x & 0xFFFF)); b2 = rec.x >> 16;
          t1 = __int_as_float(rec.y); t2 = __int_as_float(rec.z);
          j = (rec.w >> 16) & 0xFFF; l = rec.w & 0xFFFF; hj = half >> ((uint32_t(rec.w) >> 28) & 3);   // Pol slot
        } else {                                    // fp64: node coordinates in fp64 on the fly
          const uint32_t nd = __ldg(pp.nodes + t);
          j = int(nd >> 16); l = int(nd & 0xffffu);
          const double r = __ldg(pp.rho + j);
          const double k1 = r * __ldg(pp.cs + 2 * l), k2 = r * __ldg(pp.cs + 2 * l + 1);
          const double f1 = ceil(k1 - pp.half_w), f2 = ceil(k2 - pp.half_w);
          b1 = int(f1); b2 = int(f2);
          t1 = T(k1 - f1); t2 = T(k2 - f2);
        }
        const bool pair = (l != 0) && (2 * l != hj);
        T wx[W], wy[W];
#pragma unroll
        for (int q = 0; q < W; ++q) { wx[q] = phi(t1 - T(q)); wy[q] = phi(t2 - T(q)); }
        const T2* gcol = Gc + (b2 - lo);
        T2 accA = T2{T(0), T(0)}, accB = T2{T(0), T(0)};
#pragma unroll
        for (int q = 0; q < W; ++q) {
          const T2* ga = gcol + (size_t)(b1 + q + row0) * S;        // node (k1, k2)
          const T2* gb = gcol + (size_t)(row0 - b1 - q) * S;        // node (-k1, k2), mirrored taps
          T2 sa = T2{T(0), T(0)}, sb = T2{T(0), T(0)};
#pragma unroll
          for (int c = 0; c < W; ++c) sa = rfma(wy[c], ga[c], sa);
          if (pair) {
#pragma unroll
            for (int c = 0; c < W; ++c) sb = rfma(wy[c], gb[c], sb);
          }
          accA = rfma(wx[q], sa, accA);
          accB = rfma(wx[q], sb, accB);
        }
        Pol[(int64_t)j * half + l] = accA;
        if (pair) Pol[(int64_t)j * half + (hj - l)] = accB;
      }
      __syncthreads();
      PROF_MARK(3);
    }
    // the next image's load is issued after the first ring group's FFTs (so it does not queue in front of the
    // polar-sample loads of group 0)
    prefetched = false;
    const bool want_prefetch = pp.img_prefetch && img + gridDim.x < n_img;

    // ---------------- K3: ring FFTs, staged [k][jj], written k-major.
    // pow2 plans: ring pairs (j, j+1) per warp as two half-length (N = n_theta/2) FFTs.  With f the half ring and
    // w = e^{-2 pi i / n_theta}, ghat(k) = sum_{l<N} [f_l + (-1)^k conj f_l] w^{kl}, so
    //   even k = 2m: U = DFT_N(Re f_j + i Re f_j'),          ghat_j = U(m) + conj U(-m),   ghat_j' = -i (U(m) - conj U(-m))
    //   odd k = 2m+1: V = DFT_N((Im f_j + i Im f_j') w^l),   ghat_j = i (V(m) + conj V(N-1-m)), ghat_j' = V(m) - conj V(N-1-m)
    // (the real-input pair trick on each parity; w^l shifts the odd frequencies onto the N-point grid).
    // Runtime sizes: one full n_theta-point FFT per ring rebuilt from the half ring.
    T2* stg = (MC > 0 || pp.ring_pairs) ? region : region + (size_t)pp.ang_warps * 2 * NTP;
    const int GS = (G + 1) | 1;                      // odd staging stride >= G + 1 (bank spread, spare slot)
    // staging index of (k, ring jj): row k at k GS, shifted by one slot for k mod 32 >= 16, so that the writers' even
    // (or odd) k of a half-warp (k = 2m, m = 0..15) and the write-out's four consecutive k of a half-warp land in
    // distinct 8-byte bank pairs (no 2-way conflicts; GS odd, <= 33 rings per row + 1 spare slot)
    auto sidx = [GS](int k, int jj) { return (size_t)k * GS + jj + ((k >> 4) & 1); };
    // MC = 256 (HW: one ring pair per warp per group): half-warp 0 transforms U = DFT(Re f_j + i Re f_j'), half-warp 1
    // V = DFT((Im f_j + i Im f_j') w^t) at the same time.  Each lane's 16 inputs f[16 t1 + q] of both rings (its
    // half's component) are loaded into registers one group ahead (the loads of group j0 + G fly during group j0's
    // FFTs and write-out) -- one L2 read of the polar samples, latency hidden.
    constexpr bool REGPF = HW;
    float pfa[REGPF ? 16 : 1], pfb[REGPF ? 16 : 1];
    const bool regpf = REGPF && G <= 2 * pp.fft_warps;
    auto load_pair = [&](int jg) {
      if constexpr (REGPF) {
        const int jj = 2 * warp, gg = min(G, n_xi - jg);
        if (jg < n_xi && warp < pp.fft_warps && jj < gg) {
          const float* fa = reinterpret_cast<const float*>(Pol + (int64_t)(jg + jj) * half) + (lane >> 4);
          const bool two = jj + 1 < gg;
          const float* fb = two ? fa + 2 * half : fa;
          const int q = lane & 15;
          // ring j sampled at every s_j-th angle (plan.cpp): the unsampled positions of the half ring are zeros of
          // the stuffed sequence, never written by the gather and not loaded here
          const int sa = __ldg(pp.ring_s + jg + jj), sb = two ? __ldg(pp.ring_s + jg + jj + 1) : 1;
          const int ma = sa - 1, mb = sb - 1, la2 = 31 - __clz(sa), lb2 = 31 - __clz(sb);
          // volatile: issued here (not sunk to the use a group later), completion tracked by the scoreboard.
          // Sample t of the stuffed ring is slot t / s of the ring's contiguous samples (plan.cpp pol_slot)
#pragma unroll
          for (int t1 = 0; t1 < 16; ++t1) {
            const int t = 16 * t1 + q;
            pfa[t1] = 0.f;
            pfb[t1] = 0.f;
            // predicated loads (no branches): @p ld, the register keeps its 0 otherwise
            asm volatile("{ .reg .pred p; setp.eq.s32 p, %2, 0; @p ld.global.f32 %0, [%1]; }"
                         : "+f"(pfa[t1]) : "l"(fa + 2 * (t >> la2)), "r"(t & ma));
            asm volatile("{ .reg .pred p; setp.eq.s32 p, %2, 0; @p ld.global.f32 %0, [%1]; }"
                         : "+f"(pfb[t1]) : "l"(fb + 2 * (t >> lb2)), "r"(two ? (t & mb) : 1));
          }
        }
      }
    };
    if (regpf) load_pair(0);
    for (int j0 = 0; j0 < n_xi; j0 += G) {
      const int g = min(G, n_xi - j0);
      bool done_reg = false;
      if constexpr (REGPF) if (regpf) {
        done_reg = true;
        const int kmx = pp.k_max;
        const int jj = 2 * warp, q = lane & 15, h = lane >> 4;
        T2* mybuf = wscr + (size_t)warp * 2 * kHwBuf + h * kHwBuf;
        if (warp < pp.fft_warps && jj < g) {
          const bool two = jj + 1 < g;
          float2 v[16];
#pragma unroll
          for (int t1 = 0; t1 < 16; ++t1) {             // V (h = 1): times w^t; U: times 1 (selects, no branch)
            // volatile shared load: loop-invariant, but hoisting 16 twiddles out of the group loop would pin 32
            // registers for the whole angular pass (spills)
            T2 tw;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(tw.x), "=f"(tw.y)
                         : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(twT + 16 * t1 + q))));
            v[t1] = cmul(float2{pfa[t1], pfb[t1]}, float2{h ? tw.x : 1.f, h ? tw.y : 0.f});
          }
          fft256_hw<false>(v, mybuf, twM, q);
          hw_store_natural(v, mybuf, q);
          __syncwarp();
          // even k = 2m from U (h = 0): ghat_j = U(m) + conj U(-m), ghat_j' = -i (U(m) - conj U(-m));
          // odd k = 2m + 1 from V (h = 1): ghat_j = i (V(m) + conj V(N-1-m)), ghat_j' = V(m) - conj V(N-1-m)
          for (int m = q; 2 * m + h <= kmx; m += 16) {
            const T2 u = mybuf[hw_idx(m)];
            T2 uc = mybuf[hw_idx((256 - m - h) & 255)];
            uc.y = -uc.y;
            const T2 sp = cadd(u, uc), dm = csub(u, uc);
            stg[sidx(2 * m + h, jj)] = h ? T2{-sp.y, sp.x} : sp;
            if (two) stg[sidx(2 * m + h, jj + 1)] = h ? dm : T2{dm.y, -dm.x};
          }
          // next group's inputs, consumed one iteration later: issued after this group's FFT (the 32 prefetch
          // registers are not live across it), in flight during the write-out
          load_pair(j0 + G);
          __syncwarp();
          PROF_MARK(6);
        }
      }
      if (done_reg) {
      } else if constexpr (MC > 0) {
        const int kmx = pp.k_max;
        T2* res = fft_result_in_A<MC>() ? myA : myB;
        auto stR = [res](int i, T2 v) { res[padi(i)] = v; };
        for (int pr = grp; grp < pp.fft_warps && 2 * pr < g; pr += pp.fft_warps) {
          const int jj = 2 * pr;
          const bool two = jj + 1 < g;
          const T2* fa = Pol + (int64_t)(j0 + jj) * half;
          const T2* fb = two ? fa + half : fa;
          // rings sampled at every s_j-th angle (reading Q21): the other positions are zeros of the stuffed ring
          // (sample t of the stuffed ring = slot t / s of the ring's contiguous samples, plan.cpp pol_slot)
          const int sa = __ldg(pp.ring_s + j0 + jj), sb = two ? __ldg(pp.ring_s + j0 + jj + 1) : 1;
          const int ma = sa - 1, mb = sb - 1, la2 = 31 - __clz(sa), lb2 = 31 - __clz(sb);
          auto ring_a = [&](int t) -> T2 { return (t & ma) ? T2{T(0), T(0)} : fa[t >> la2]; };
          auto ring_b = [&](int t) -> T2 { return (two && !(t & mb)) ? fb[t >> lb2] : T2{T(0), T(0)}; };
          auto ldu = [&](int t) -> T2 { return T2{ring_a(t).x, ring_b(t).x}; };
          fft_ct<T2, MC, false, FG>(ldu, stR, myA, myB, twM, glane, gbar);
          gsync<FG>(gbar);
          for (int m = glane; 2 * m <= kmx; m += FG) {
            const T2 u = res[padi(m)];
            T2 uc = res[padi(m == 0 ? 0 : MC - m)];
            uc.y = -uc.y;
            const T2 sp = cadd(u, uc), dm = csub(u, uc);
            stg[sidx(2 * m, jj)] = sp;
            if (two) stg[sidx(2 * m, jj + 1)] = T2{dm.y, -dm.x};
          }
          gsync<FG>(gbar);
          auto ldv = [&](int t) -> T2 { return cmul(T2{ring_a(t).y, ring_b(t).y}, twT[t]); };
          fft_ct<T2, MC, false, FG>(ldv, stR, myA, myB, twM, glane, gbar);
          gsync<FG>(gbar);
          for (int m = glane; 2 * m + 1 <= kmx; m += FG) {
            const T2 v = res[padi(m)];
            T2 vc = res[padi(MC - 1 - m)];
            vc.y = -vc.y;
            const T2 sp = cadd(v, vc), dm = csub(v, vc);
            stg[sidx(2 * m + 1, jj)] = T2{-sp.y, sp.x};
            if (two) stg[sidx(2 * m + 1, jj + 1)] = dm;
          }
          gsync<FG>(gbar);
        }
      } else if (pp.ring_pairs) {
        // runtime sizes with n_theta = 2 M: the same ring-pair scheme as above on M-point mixed-radix FFTs
        const int kmx = pp.k_max, Mr = pp.fft_M.n;
        T2* res = ((pp.fft_M.nstages - 1) & 1) ? myB : myA;
        auto stR = [res](int i, T2 v) { res[padi(i)] = v; };
        for (int pr = warp; warp < pp.fft_warps && 2 * pr < g; pr += pp.fft_warps) {
          const int jj = 2 * pr;
          const bool two = jj + 1 < g;
          const T2* fa = Pol + (int64_t)(j0 + jj) * half;
          const T2* fb = two ? fa + half : fa;
          auto ldu = [&](int t) -> T2 { const T2 a = fa[t], b = fb[t]; return T2{a.x, two ? b.x : T(0)}; };
          fft_rt<T2>(pp.fft_M, ldu, stR, myA, myB, twM, lane);
          __syncwarp();
          for (int m = lane; 2 * m <= kmx; m += 32) {
            const T2 u = res[padi(m)];
            T2 uc = res[padi(m == 0 ? 0 : Mr - m)];
            uc.y = -uc.y;
            const T2 sp = cadd(u, uc), dm = csub(u, uc);
            stg[sidx(2 * m, jj)] = sp;
            if (two) stg[sidx(2 * m, jj + 1)] = T2{dm.y, -dm.x};
          }
          __syncwarp();
          auto ldv = [&](int t) -> T2 {
            const T2 a = fa[t], b = fb[t];
            return cmul(T2{a.y, two ? b.y : T(0)}, twT[t]);
          };
          fft_rt<T2>(pp.fft_M, ldv, stR, myA, myB, twM, lane);
          __syncwarp();
          for (int m = lane; 2 * m + 1 <= kmx; m += 32) {
            const T2 v = res[padi(m)];
            T2 vc = res[padi(Mr - 1 - m)];
            vc.y = -vc.y;
            const T2 sp = cadd(v, vc), dm = csub(v, vc);
            stg[sidx(2 * m + 1, jj)] = T2{-sp.y, sp.x};
            if (two) stg[sidx(2 * m + 1, jj + 1)] = dm;
          }
          __syncwarp();
        }
      } else if (warp < pp.ang_warps) {
        for (int jj = warp; jj < g; jj += pp.ang_warps) {
          const T2* src = Pol + (int64_t)(j0 + jj) * half;
          auto ld = [&](int t) -> T2 {
            if (t < half) return src[t];
            const T2 v = src[t - half];
            return T2{v.x, -v.y};
          };
          const int kmx = pp.k_max;
          auto st = [&](int t, T2 v) { if (t <= kmx) stg[sidx(t, jj)] = v; };
          if constexpr (NC > 0) fft_ct<T2, NC>(ld, st, angA, angB, twT, lane);
          else fft_rt<T2, sizeof(T) == 4>(pp.fft_theta, ld, st, angA, angB, twT, lane);
        }
      }
      if (j0 == 0 && want_prefetch) { issue_image(img + gridDim.x); prefetched = true; }
      __syncthreads();
      l2_discard(Pol + (int64_t)j0 * half, (size_t)g * half * sizeof(T2), tid, nthr);   // rings j0.. consumed
      PROF_MARK(4);
      {
        const int64_t kstride = pp.ghat_kstride;
        const int kmx4 = pp.k_max;
        if (sizeof(T) == 4 && g == 32 && (n_xi & 3) == 0) {
          // full fp32 group: lane = (k of 8, quad of 4 rings) over two halves of 16 rings; 16-byte stores of the re
          // and im rows.  A half-warp reads 4 consecutive k x 4 quads: distinct bank pairs under sidx.
          const int kk = lane >> 2, qd = lane & 3;
          for (int hh = 0; hh < 2; ++hh) {
            const int jr = 16 * hh + 4 * qd;
            T* base = ghat + img * 2 * (int64_t)n_xi + j0 + jr;
            for (int k = warp * 8 + kk; k <= kmx4; k += nwarps * 8) {
              if (j0 + jr < skj0[k]) continue;        // below K4's first ring for k: never read (plan.cpp)
              const T2* sp = stg + sidx(k, jr);
              const T2 v0 = sp[0], v1 = sp[1], v2 = sp[2], v3 = sp[3];
              T* d = base + (int64_t)k * kstride;
              __stcs(reinterpret_cast<float4*>(d), make_float4(v0.x, v1.x, v2.x, v3.x));        // streamed: read
              __stcs(reinterpret_cast<float4*>(d + n_xi), make_float4(v0.y, v1.y, v2.y, v3.y)); // back by K4 only
            }
          }
        } else {
        // warp per k: lanes write rings j0 + lane (re row then im row), 128-B coalesced stores
        // g <= 16: each half-warp writes one k (two k per warp instruction); else a warp per k
        const int per = g <= 16 ? 2 : 1;
        const int sub = per == 2 ? (lane >> 4) : 0, ln = per == 2 ? (lane & 15) : lane, lstep = per == 2 ? 16 : 32;
        const int k0 = warp * per + sub, kstep = nwarps * per;
        T* dst = ghat + img * 2 * (int64_t)n_xi + j0 + (int64_t)k0 * kstride;
        const int kmx = pp.k_max;
        (void)lstep;                                  // g <= G <= 32: one element per lane and k
        const bool act = ln < g;
        // 4 k per iteration: all shared loads first, then the global stores (independent -> ILP)
        for (int k = k0; k <= kmx; k += 4 * kstep) {
          T2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool ok = act && (k + u * kstep <= kmx) && (j0 + ln >= skj0[k + u * kstep]);
            v[u] = ok ? stg[sidx(k + u * kstep, ln)] : T2{T(0), T(0)};
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (act && (k + u * kstep <= kmx) && (j0 + ln >= skj0[k + u * kstep])) {
              T* d = dst + (int64_t)u * kstep * kstride;
              d[ln] = v[u].x;
              d[ln + n_xi] = v[u].y;
            }
          }
          dst += 4 * (int64_t)kstep * kstride;
        }
        }
      }
      __syncthreads();
      PROF_MARK(5);
    }
  }
  PROF_STORE();
  if (use_tmem) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
  }
}

template <typename T, int W, int MC>
cudaError_t launch_polar_t(const Plan& P, const void* d_images, int64_t n_img, int64_t stride,
                                  cudaStream_t s) {
  auto kern = polar_kernel<T, W, MC>;
  cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(kern), P.polar_smem);
  if (e != cudaSuccess) return e;
  int grid = (int)std::min<int64_t>(P.polar_grid, n_img);
  kern<<<grid, P.pp.nwarps * 32, P.polar_smem, s>>>(P.d_pp, reinterpret_cast<const T*>(d_images), n_img, stride,
                                                    reinterpret_cast<T*>(P.d_ghat));
  return cudaGetLastError();
}

// The instantiations compile in parallel: build.py compiles this file once per part (FBSPCA_POLAR_PART = 1..6
// via csrc/polar_part*.cu, each one heavy kernel or two) and once as the dispatcher (part 0).  Phase-profiling
// builds (a __device__ counter array) define FBSPCA_POLAR_SINGLE_TU and instantiate everything in part 0.
#ifndef FBSPCA_POLAR_PART
#define FBSPCA_POLAR_PART 0
#endif
#ifdef FBSPCA_POLAR_SINGLE_TU
#define FBSPCA_POLAR_HERE(part) (FBSPCA_POLAR_PART == 0)
#else
#define FBSPCA_POLAR_HERE(part) (FBSPCA_POLAR_PART == (part))
#endif
#define FBSPCA_POLAR_INST(T, W, MC) \
  template cudaError_t launch_polar_t<T, W, MC>(const Plan&, const void*, int64_t, int64_t, cudaStream_t);
#define FBSPCA_POLAR_EXTERN(T, W, MC) \
  extern template cudaError_t launch_polar_t<T, W, MC>(const Plan&, const void*, int64_t, int64_t, cudaStream_t);
#define FBSPCA_POLAR_LIST(X, P1, P2, P3, P4, P5, P6) \
  P1(X(float, 6, 256)) P4(X(float, 5, 256)) P2(X(float, 6, 512)) P2(X(float, 6, 128)) P3(X(float, 6, 0)) P3(X(float, 5, 512)) P6(X(float, 5, 0)) P4(X(float, 7, 0)) \
  P4(X(float, 5, 128)) P5(X(double, 13, 0)) P5(X(double, 13, 64)) P5(X(float, 5, 600)) P6(X(float, 6, 600)) P6(X(float, 6, 720)) P1(X(float, 5, 720))
#define FBSPCA_ON(x) x
#define FBSPCA_OFF(x)
#if FBSPCA_POLAR_HERE(1)
FBSPCA_POLAR_LIST(FBSPCA_POLAR_INST, FBSPCA_ON, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF)
#endif
#if FBSPCA_POLAR_HERE(2)
FBSPCA_POLAR_LIST(FBSPCA_POLAR_INST, FBSPCA_OFF, FBSPCA_ON, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF)
#endif
#if FBSPCA_POLAR_HERE(3)
FBSPCA_POLAR_LIST(FBSPCA_POLAR_INST, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_ON, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF)
#endif
#if FBSPCA_POLAR_HERE(4)
FBSPCA_POLAR_LIST(FBSPCA_POLAR_INST, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_ON, FBSPCA_OFF, FBSPCA_OFF)
#endif
#if FBSPCA_POLAR_HERE(5)
FBSPCA_POLAR_LIST(FBSPCA_POLAR_INST, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_ON, FBSPCA_OFF)
#endif

#if FBSPCA_POLAR_HERE(6)
FBSPCA_POLAR_LIST(FBSPCA_POLAR_INST, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_OFF, FBSPCA_ON)
#endif

#if FBSPCA_POLAR_PART == 0
#ifndef FBSPCA_POLAR_SINGLE_TU
FBSPCA_POLAR_LIST(FBSPCA_POLAR_EXTERN, FBSPCA_ON, FBSPCA_ON, FBSPCA_ON, FBSPCA_ON, FBSPCA_ON, FBSPCA_ON)
#endif
int polar_max_smem() { return 227 * 1024; }

#ifdef FBSPCA_PHASE_PROF
extern "C" int fbspca_debug_phase_prof(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_phase_prof, sizeof(unsigned long long) * n);
}
#endif

int polar_fixed_smem(int M, int n_theta, int L, int csz, int nwarps, int nk, bool hw) {
  return (int)(((sizeof(PolarParams) + 15) / 16) * 16) +
         (int)((((M + n_theta) * csz + L * (csz / 2) + nk * (int)sizeof(int)) + 15) / 16) * 16 +
         nwarps * polar_warp_scratch(M, hw) * csz;
}

cudaError_t launch_polar(const Plan& P, const void* d_images, int64_t n_img, int64_t stride, cudaStream_t s) {
  if (P.dt == FBSPCA_F64) {
    if (P.w != 13) return cudaErrorInvalidValue;
    if (P.n_theta == 2 * P.M && P.M == 64) return launch_polar_t<double, 13, 64>(P, d_images, n_img, stride, s);
    return launch_polar_t<double, 13, 0>(P, d_images, n_img, stride, s);
  }
  if (polar_f32_ct_kernel(P.M, P.n_theta)) {       // compile-time FFT kernels: w = 5 (eps >= 1e-4) or 6
#define FBSPCA_CT_CASE(MC) \
    case MC: return P.w == 5 ? launch_polar_t<float, 5, MC>(P, d_images, n_img, stride, s) \
                             : launch_polar_t<float, 6, MC>(P, d_images, n_img, stride, s);
    if (P.w == 5 || P.w == 6) switch (P.M) {
      FBSPCA_CT_CASE(128) FBSPCA_CT_CASE(256) FBSPCA_CT_CASE(512) FBSPCA_CT_CASE(600) FBSPCA_CT_CASE(720)
      default: break;
    }
#undef FBSPCA_CT_CASE
  }
  switch (P.w) {
    case 5: return launch_polar_t<float, 5, 0>(P, d_images, n_img, stride, s);   // eps >= 1e-4
    case 6: return launch_polar_t<float, 6, 0>(P, d_images, n_img, stride, s);
    case 7: return launch_polar_t<float, 7, 0>(P, d_images, n_img, stride, s);   // eps = 1e-6 (the fp32 floor)
    default: return cudaErrorInvalidValue;
  }
}

#endif  // FBSPCA_POLAR_PART == 0

}  // namespace fbspca
