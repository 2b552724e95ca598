// fft_device.cuh -- warp-level FFT building blocks shared by the polar kernel (K1, K3) and the parameter estimator
// (NEXT-2): complex helpers, small forward DFTs (e^{-2 pi i}), Stockham stages with load/store functors,
// compile-time power-of-two FFTs and the runtime mixed-radix (2, 3, 4, 5, 8) FFT.
#pragma once
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

// acc + w g for a real weight w: one packed FFMA2 (fma.rn.f32x2, w broadcast) in fp32, two FMAs in fp64
__device__ __forceinline__ float2 rfma(float w, float2 g, float2 acc) {
  unsigned long long r, gg, aa, ww;
  asm("mov.b64 %0, {%1, %2};" : "=l"(gg) : "f"(g.x), "f"(g.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(acc.x), "f"(acc.y));
  asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(ww), "l"(gg), "l"(aa));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ double2 rfma(double w, double2 g, double2 acc) {
  return {fma(w, g.x, acc.x), fma(w, g.y, acc.y)};
}

// packed fp32 complex add / subtract (add.rn.f32x2 / sub.rn.f32x2 = SASS FADD2: one instruction per complex op)
__device__ __forceinline__ float2 padd(float2 a, float2 b) {
  unsigned long long r, x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 psub(float2 a, float2 b) {
  unsigned long long r, x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}

// ---------------------------------------------------------------- small forward DFTs (e^{-2 pi i})
template <typename T2, int R> struct Dft;
// fp32 radix-4 / radix-8 butterflies with packed adds (the FFT phases are issue-bound)
template <> struct Dft<float2, 4> {
  __device__ __forceinline__ static void run(float2* v) {
    const float2 s0 = padd(v[0], v[2]), d0 = psub(v[0], v[2]);
    const float2 s1 = padd(v[1], v[3]), d1 = mul_mi(psub(v[1], v[3]));
    v[0] = padd(s0, s1); v[2] = psub(s0, s1);
    v[1] = padd(d0, d1); v[3] = psub(d0, d1);
  }
};
template <> struct Dft<float2, 8> {
  __device__ __forceinline__ static void run(float2* v) {
    const float h = 0.70710678118654752440f;
    float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    Dft<float2, 4>::run(e); Dft<float2, 4>::run(o);
    const float2 t1 = {h * (o[1].x + o[1].y), h * (o[1].y - o[1].x)};
    const float2 t2 = mul_mi(o[2]);
    const float2 t3 = {h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y)};
    v[0] = padd(e[0], o[0]); v[4] = psub(e[0], o[0]);
    v[1] = padd(e[1], t1);   v[5] = psub(e[1], t1);
    v[2] = padd(e[2], t2);   v[6] = psub(e[2], t2);
    v[3] = padd(e[3], t3);   v[7] = psub(e[3], t3);
  }
};
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

// ---------------------------------------------------------------- warp FFTs with load/store functors
// Stockham (autosort) stage of radix R: butterfly j reads ld(j + r NB), twiddles by w^(r (j mod Ns)),
// DFT_R, writes st((j / Ns) Ns R + (j mod Ns) + r Ns).  Out of place; one warp; R values in registers.
// Twiddles come from a per-stage table tws[TOFF + (r - 1) Ns + (j mod Ns)] (contiguous in j: no bank
// conflicts), built once per CTA by build_stage_tw<N>.
// HZ (first stage only): inputs t in [N/4, 3N/4) are known zeros -- the zero-padded rows / columns of K1
// (pixel index L/2 <= M/4 away from 0 on both sides) -- so those butterfly legs are constant zeros.
// GS: lanes per FFT (32 = one warp; 64 = a warp pair synchronised on named barrier `bar`, for sizes whose two
// ping-pong buffers per warp do not fit 16 warps -- the pair shares one buffer set, so all 16 warps work).
template <int GS> __device__ __forceinline__ void gsync(int bar) {
  if constexpr (GS == 32) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(GS) : "memory");
}

// fp32 stage twiddles from one table load + products (fewer shared loads, more FP instructions) or R - 1 table loads;
// measured on B200 (tools/ab_bench.sh, same box ABAB): products 54.5 ms vs table 55.5 ms polar at C3 -> products
#ifndef FBSPCA_TW_RECURRENCE
#define FBSPCA_TW_RECURRENCE 1
#endif
// w[r] = w[1]^r, r = 2..R-1, from w[1] by at most three multiplications deep
template <typename T2, int R>
__device__ __forceinline__ void twiddle_powers(T2* w) {
  if constexpr (R > 2) w[2] = cmul(w[1], w[1]);
  if constexpr (R > 3) w[3] = cmul(w[1], w[2]);
  if constexpr (R > 4) w[4] = cmul(w[2], w[2]);
  if constexpr (R > 5) w[5] = cmul(w[1], w[4]);
  if constexpr (R > 6) w[6] = cmul(w[2], w[4]);
  if constexpr (R > 7) w[7] = cmul(w[3], w[4]);
}

template <typename T2, int N, int R, int Ns, int TOFF, bool HZ = false, int GS = 32, class Ld, class St>
__device__ __forceinline__ void cstage(Ld ld, St st, const T2* __restrict__ tws, int lane, int bar = 0) {
  constexpr int NB = N / R;
#pragma unroll
  for (int j0 = 0; j0 < NB; j0 += GS) {
    const int j = j0 + lane;
    if (NB % GS == 0 || j < NB) {
      T2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (HZ && R >= 4 && r >= R / 4 && r < 3 * R / 4) v[r] = T2{0, 0};
        else v[r] = ld(j + r * NB);
      }
      const int jm = j % Ns;                      // compile-time Ns: a mask for powers of two
      if constexpr (Ns > 1 && sizeof(v[0].x) == 4 && R >= 3 && FBSPCA_TW_RECURRENCE) {
        // fp32: one table load per butterfly; w^r for r >= 2 by products of w (depth <= 3 multiplications,
        // relative error <= ~4e-7, below the fp32 FFT's own ~log2(N) u).  Saves R - 2 shared loads.
        T2 w[R];
        w[1] = tws[TOFF + jm];
        twiddle_powers<T2, R>(w);
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
      } else if constexpr (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tws[TOFF + (r - 1) * Ns + jm]);
      }
      Dft<T2, R>::run(v);
      const int idxD = (j - jm) * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) st(idxD + r * Ns, v[r]);
    }
  }
  gsync<GS>(bar);
}

// Ping-pong scratch index swizzle: XOR the low 4 bits with 3 (i >> 4).  64-bit shared accesses resolve per
// half-warp; this mapping keeps every load/store pattern of the stages below at 1.03x the ideal wavefronts
// (unswizzled: 2.1x).
__device__ __forceinline__ int padi(int i) { return i ^ ((3 * (i >> 4)) & 15); }

// which ping-pong buffer the last stage of fft_ct<N> does NOT read (so the result may be stored there)
// (odd stage count: 128, 256, 512 = 3 stages, 720 = 5; even: 64, 1024, 600)
template <int N> __host__ __device__ constexpr bool fft_result_in_A() { return N == 128 || N == 256 || N == 512 || N == 720; }

// stage list per size: (R, Ns) ... ; table offsets TOFF accumulate (R - 1) Ns over stages with Ns > 1
template <typename T2, int R, int Ns>
__device__ __forceinline__ void fill_stage_tw(T2* dst, const T2* __restrict__ lin, int N, int tid, int nthr) {
  const int step = N / (Ns * R);
  for (int e = tid; e < (R - 1) * Ns; e += nthr) {
    const int r = 1 + e / Ns, jm = e % Ns;
    dst[e] = lin[jm * step * r];
  }
}
template <int N> constexpr int stage_tw_len() {
  return N == 64 ? 56 : N == 128 ? 120 : N == 256 ? 248 : N == 512 ? 504 : N == 1024 ? 1016 : N;
}
template <typename T2, int N>
__device__ void build_stage_tw(T2* dst, const T2* __restrict__ lin, int tid, int nthr) {
  if constexpr (N == 64) {
    fill_stage_tw<T2, 8, 8>(dst, lin, N, tid, nthr);
  } else if constexpr (N == 128) {
    fill_stage_tw<T2, 4, 8>(dst, lin, N, tid, nthr); fill_stage_tw<T2, 4, 32>(dst + 24, lin, N, tid, nthr);
  } else if constexpr (N == 256) {
    fill_stage_tw<T2, 8, 8>(dst, lin, N, tid, nthr); fill_stage_tw<T2, 4, 64>(dst + 56, lin, N, tid, nthr);
  } else if constexpr (N == 512) {
    fill_stage_tw<T2, 8, 8>(dst, lin, N, tid, nthr); fill_stage_tw<T2, 8, 64>(dst + 56, lin, N, tid, nthr);
  } else if constexpr (N == 1024) {
    fill_stage_tw<T2, 8, 8>(dst, lin, N, tid, nthr); fill_stage_tw<T2, 4, 64>(dst + 56, lin, N, tid, nthr);
    fill_stage_tw<T2, 4, 256>(dst + 248, lin, N, tid, nthr);
  } else if constexpr (N == 600) {
    fill_stage_tw<T2, 5, 8>(dst, lin, N, tid, nthr); fill_stage_tw<T2, 5, 40>(dst + 32, lin, N, tid, nthr);
    fill_stage_tw<T2, 3, 200>(dst + 192, lin, N, tid, nthr);
  } else if constexpr (N == 720) {
    fill_stage_tw<T2, 5, 8>(dst, lin, N, tid, nthr); fill_stage_tw<T2, 3, 40>(dst + 32, lin, N, tid, nthr);
    fill_stage_tw<T2, 3, 120>(dst + 112, lin, N, tid, nthr); fill_stage_tw<T2, 2, 360>(dst + 352, lin, N, tid, nthr);
  } else {
    for (int i = tid; i < N; i += nthr) dst[i] = lin[i];     // runtime path: linear table
  }
}

// Compile-time FFT (powers of two 64..1024, and 600 / 720): first stage reads ld(), last stage writes st(),
// ping-pong in A, B.
template <typename T2, int N, bool HZ = false, int GS = 32, class Ld, class St>
__device__ __forceinline__ void fft_ct(Ld ld, St st, T2* A, T2* B, const T2* tw, int lane, int bar = 0) {
  auto lA = [A](int i) { return A[padi(i)]; };
  auto lB = [B](int i) { return B[padi(i)]; };
  auto sA = [A](int i, T2 v) { A[padi(i)] = v; };
  auto sB = [B](int i, T2 v) { B[padi(i)] = v; };
  if constexpr (N == 64) {
    cstage<T2, 64, 8, 1, 0, HZ>(ld, sA, tw, lane); cstage<T2, 64, 8, 8, 0>(lA, st, tw, lane);
  } else if constexpr (N == 128) {
    cstage<T2, 128, 8, 1, 0, HZ>(ld, sA, tw, lane); cstage<T2, 128, 4, 8, 0>(lA, sB, tw, lane);
    cstage<T2, 128, 4, 32, 24>(lB, st, tw, lane);
  } else if constexpr (N == 256) {
    cstage<T2, 256, 8, 1, 0, HZ>(ld, sA, tw, lane); cstage<T2, 256, 8, 8, 0>(lA, sB, tw, lane);
    cstage<T2, 256, 4, 64, 56>(lB, st, tw, lane);
  } else if constexpr (N == 512) {
    cstage<T2, 512, 8, 1, 0, HZ, GS>(ld, sA, tw, lane, bar); cstage<T2, 512, 8, 8, 0, false, GS>(lA, sB, tw, lane, bar);
    cstage<T2, 512, 8, 64, 56, false, GS>(lB, st, tw, lane, bar);
  } else if constexpr (N == 1024) {
    cstage<T2, 1024, 8, 1, 0, HZ>(ld, sA, tw, lane); cstage<T2, 1024, 8, 8, 0>(lA, sB, tw, lane);
    cstage<T2, 1024, 4, 64, 56>(lB, sA, tw, lane); cstage<T2, 1024, 4, 256, 248>(lA, st, tw, lane);
  } else if constexpr (N == 600) {          // 8 5 5 3 (the paper's Table III images, L = 300)
    cstage<T2, 600, 8, 1, 0, HZ, GS>(ld, sA, tw, lane, bar); cstage<T2, 600, 5, 8, 0, false, GS>(lA, sB, tw, lane, bar);
    cstage<T2, 600, 5, 40, 32, false, GS>(lB, sA, tw, lane, bar);
    cstage<T2, 600, 3, 200, 192, false, GS>(lA, st, tw, lane, bar);
  } else if constexpr (N == 720) {          // 8 5 3 3 2 (C5, L = 360)
    cstage<T2, 720, 8, 1, 0, HZ, GS>(ld, sA, tw, lane, bar); cstage<T2, 720, 5, 8, 0, false, GS>(lA, sB, tw, lane, bar);
    cstage<T2, 720, 3, 40, 32, false, GS>(lB, sA, tw, lane, bar);
    cstage<T2, 720, 3, 120, 112, false, GS>(lA, sB, tw, lane, bar);
    cstage<T2, 720, 2, 360, 352, false, GS>(lB, st, tw, lane, bar);
  } else {
    static_assert(N == 64, "unsupported compile-time FFT size");
  }
}

// Runtime mixed-radix (2,3,4,5,8) version for sizes without a compile-time path (e.g. 720, 1440).
template <typename T2, int R, class Ld, class St>
__device__ __forceinline__ void rstage(Ld ld, St st, int N, int Ns, const T2* __restrict__ tw, int lane) {
  const int NB = N / R, step = N / (Ns * R);
  for (int j = lane; j < NB; j += 32) {
    T2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = ld(j + r * NB);
    const int jm = j % Ns;
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[jm * step * r]);
    if constexpr (R == 7 || R == 11) {
      // unrolled prime DFT, w_R^m = tw[m N / R] (only the angular FFT instantiates these: see fft_rt PRIMES)
      T2 o[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        T2 acc = v[0];
#pragma unroll
        for (int r = 1; r < R; ++r) acc = cadd(acc, cmul(v[r], tw[((q * r) % R) * NB]));
        o[q] = acc;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = o[r];
    } else {
      Dft<T2, R>::run(v);
    }
    const int idxD = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) st(idxD + r * Ns, v[r]);
  }
  __syncwarp();
}

// Other prime radices (awkward n_theta = ceil(16 c R), e.g. 308 = 4 7 11, or 2L with such a factor): a direct
// R-point DFT per butterfly, out[q] = sum_r in[r] w^(jm step r) w_R^(q r) with both factors from the same linear
// table (w_R^m = tw[m N / R]), loops not unrolled -- O(R) loads per output, kept compact because these sizes are rare.
template <typename T2, class Ld, class St>
__device__ void rstage_prime(int R, Ld ld, St st, int N, int Ns, const T2* __restrict__ tw, int lane) {
  const int NB = N / R, step = N / (Ns * R);
  for (int j = lane; j < NB; j += 32) {
    const int jm = j % Ns, idxD = (j - jm) * R + jm;
#pragma unroll 1
    for (int q = 0; q < R; ++q) {
      T2 acc = ld(j);
#pragma unroll 1
      for (int r = 1; r < R; ++r) acc = cadd(acc, cmul(ld(j + r * NB), tw[(jm * step * r + ((q * r) % R) * NB) % N]));
      st(idxD + q * Ns, acc);
    }
  }
  __syncwarp();
}

template <typename T2, bool PRIMES = false, class Ld, class St>
__device__ __forceinline__ void rstage_any(int R, Ld ld, St st, int N, int Ns, const T2* tw, int lane) {
  switch (R) {
    case 8: rstage<T2, 8>(ld, st, N, Ns, tw, lane); break;
    case 4: rstage<T2, 4>(ld, st, N, Ns, tw, lane); break;
    case 2: rstage<T2, 2>(ld, st, N, Ns, tw, lane); break;
    case 5: rstage<T2, 5>(ld, st, N, Ns, tw, lane); break;
    case 7:
      if constexpr (PRIMES) rstage<T2, 7>(ld, st, N, Ns, tw, lane); else rstage_prime<T2>(R, ld, st, N, Ns, tw, lane);
      break;
    case 11:
      if constexpr (PRIMES) rstage<T2, 11>(ld, st, N, Ns, tw, lane); else rstage_prime<T2>(R, ld, st, N, Ns, tw, lane);
      break;
    case 13: rstage_prime<T2>(R, ld, st, N, Ns, tw, lane); break;
    default: rstage<T2, 3>(ld, st, N, Ns, tw, lane); break;
  }
}

// PRIMES: radix-7/11 stages unrolled (the angular FFT, where n_theta = ceil(16 c R) brings such factors); other
// call sites use the compact rstage_prime, which keeps their code (and the build) small.
template <typename T2, bool PRIMES = false, class Ld, class St>
__device__ void fft_rt(const FftPlan& f, Ld ld, St st, T2* A, T2* B, const T2* tw, int lane) {
  auto lA = [A](int i) { return A[padi(i)]; };
  auto lB = [B](int i) { return B[padi(i)]; };
  auto sA = [A](int i, T2 v) { A[padi(i)] = v; };
  auto sB = [B](int i, T2 v) { B[padi(i)] = v; };
  const int last = f.nstages - 1;
  int Ns = 1;
  for (int s = 0; s <= last; ++s) {
    const int R = f.radix[s];
    const bool in_A = (s & 1);          // stage s >= 1 reads the buffer written by stage s-1
    if (s == 0 && s == last) rstage_any<T2, PRIMES>(R, ld, st, f.n, Ns, tw, lane);
    else if (s == 0) rstage_any<T2, PRIMES>(R, ld, sA, f.n, Ns, tw, lane);
    else if (s == last) { if (in_A) rstage_any<T2, PRIMES>(R, lA, st, f.n, Ns, tw, lane); else rstage_any<T2, PRIMES>(R, lB, st, f.n, Ns, tw, lane); }
    else { if (in_A) rstage_any<T2, PRIMES>(R, lA, sB, f.n, Ns, tw, lane); else rstage_any<T2, PRIMES>(R, lB, sA, f.n, Ns, tw, lane); }
    Ns *= R;
  }
}

// ---------------------------------------------------------------- 256-point FFT on a half-warp (radix 16 x 16)
// M = 256 (C3) kernels: each half-warp transforms its own 256-point sequence with 16 values per lane, so a warp
// runs two FFTs at once.  t = 16 t1 + t2, k = k1 + 16 k2:
//   X[k1 + 16 k2] = sum_t2 w16^(t2 k2) [ w256^(t2 k1) sum_t1 x[16 t1 + t2] w16^(t1 k1) ]
// Lane q = t2 does the inner 16-point DFT over t1 in registers, twiddles, and writes row k1 of a 16 x 17 padded
// transpose buffer; lane q = k1 reads row q back and does the outer DFT over t2.  One shared-memory round trip
// per point (the Stockham 8-8-4 path: two), no index swizzle arithmetic (the padding keeps both the row writes and
// the row reads conflict-free: bank pair (k1 + t2) mod 16), and two FFTs per warp instruction stream.
__host__ __device__ __forceinline__ float2 hadd(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
  return padd(a, b);
#else
  return {a.x + b.x, a.y + b.y};
#endif
}
__host__ __device__ __forceinline__ float2 hsub(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
  return psub(a, b);
#else
  return {a.x - b.x, a.y - b.y};
#endif
}
// forward 4-point DFT in place: (a, b, c, d) <- (X0, X1, X2, X3)
__host__ __device__ __forceinline__ void dft4f(float2& a, float2& b, float2& c, float2& d) {
  const float2 s0 = hadd(a, c), d0 = hsub(a, c), s1 = hadd(b, d), t = hsub(b, d);
  const float2 d1 = {t.y, -t.x};                                     // -i (b - d)
  a = hadd(s0, s1); c = hsub(s0, s1);
  b = hadd(d0, d1); d = hsub(d0, d1);
}
// forward 16-point DFT in place, natural order in and out (4 x 4: t = 4 a + b, k = k0 + 4 k1).
// HZ: inputs t in [4, 12) are known zeros (zero-padded rows / columns of K1) and are not read.
template <bool HZ>
__host__ __device__ __forceinline__ void dft16(float2 (&v)[16]) {
  constexpr float C = 0.92387953251128675613f, S = 0.38268343236508977173f, H = 0.70710678118654752440f;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if constexpr (HZ) {            // x[b], x[12 + b] only: Y[k0] = x0 + i^k0 x3
      const float2 x0 = v[b], x3 = v[12 + b];
      v[b] = hadd(x0, x3);
      v[8 + b] = hsub(x0, x3);
      v[4 + b] = float2{x0.x - x3.y, x0.y + x3.x};
      v[12 + b] = float2{x0.x + x3.y, x0.y - x3.x};
    } else {
      dft4f(v[b], v[4 + b], v[8 + b], v[12 + b]);
    }
  }
  // twiddles w16^(b k0) on v[b + 4 k0]
  auto mulc = [](float2 x, float wr, float wi) { return float2{x.x * wr - x.y * wi, x.x * wi + x.y * wr}; };
  v[5] = mulc(v[5], C, -S);                                              // w^1
  v[9] = float2{(v[9].x + v[9].y) * H, (v[9].y - v[9].x) * H};           // w^2
  v[13] = mulc(v[13], S, -C);                                            // w^3
  v[6] = float2{(v[6].x + v[6].y) * H, (v[6].y - v[6].x) * H};           // w^2
  v[10] = float2{v[10].y, -v[10].x};                                     // w^4 = -i
  v[14] = float2{(v[14].y - v[14].x) * H, -(v[14].x + v[14].y) * H};     // w^6
  v[7] = mulc(v[7], S, -C);                                              // w^3
  v[11] = float2{(v[11].y - v[11].x) * H, -(v[11].x + v[11].y) * H};     // w^6
  v[15] = mulc(v[15], -C, S);                                            // w^9
#pragma unroll
  for (int k0 = 0; k0 < 4; ++k0) dft4f(v[4 * k0], v[4 * k0 + 1], v[4 * k0 + 2], v[4 * k0 + 3]);
  // v[4 k0 + k1] = X[k0 + 4 k1]  ->  natural order (a compile-time register renaming)
  float2 o[16];
#pragma unroll
  for (int k0 = 0; k0 < 4; ++k0)
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) o[k0 + 4 * k1] = v[4 * k0 + k1];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = o[i];
}
__host__ __device__ __forceinline__ constexpr int hw_idx(int k) { return (k >> 4) * 17 + (k & 15); }   // natural order

#ifndef FBSPCA_HW_TW_VOLATILE
#define FBSPCA_HW_TW_VOLATILE 1
#endif
#ifdef __CUDACC__
// v[t1] = x[16 t1 + q] in, v[k2] = X[q + 16 k2] out (q = lane & 15).  buf: the half-warp's kHwBuf-element buffer;
// tw2[k1 * 16 + t2] = w256^(k1 t2).  Warp-collective (both half-warps call it together).
template <bool HZ>
__device__ __forceinline__ void fft256_hw(float2 (&v)[16], float2* buf, const float2* __restrict__ tw2, int q) {
  dft16<HZ>(v);
  // volatile shared loads: the twiddles depend only on the lane, and hoisting them out of the callers' loops would
  // pin 30 registers across whole passes (spills in the 128-register kernel)
#if FBSPCA_HW_TW_VOLATILE
  const uint32_t twa = static_cast<uint32_t>(__cvta_generic_to_shared(tw2 + q));
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
    float2 w;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(w.x), "=f"(w.y) : "r"(twa + k1 * 16 * 8));
    v[k1] = cmul(v[k1], w);
  }
#else
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw2[k1 * 16 + q]);
#endif
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 17 + q] = v[k1];
  __syncwarp();
#pragma unroll
  for (int t2 = 0; t2 < 16; ++t2) v[t2] = buf[q * 17 + t2];
  __syncwarp();
  dft16<false>(v);
}
// the result in natural order in buf (hw_idx) for readers that need X[k] and X[N - k] together
__device__ __forceinline__ void hw_store_natural(const float2 (&v)[16], float2* buf, int q) {
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) buf[k2 * 17 + q] = v[k2];
}
#endif

template <typename T2, int NC, bool HZ = false, int GS = 32, class Ld, class St>
__device__ __forceinline__ void fft_any(const FftPlan& f, Ld ld, St st, T2* A, T2* B, const T2* tw, int lane,
                                        int bar = 0) {
  if constexpr (NC > 0) fft_ct<T2, NC, HZ, GS>(ld, st, A, B, tw, lane, bar);
  else fft_rt<T2>(f, ld, st, A, B, tw, lane);
}

}  // namespace fbspca
