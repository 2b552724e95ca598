// plan.cpp -- host-side precomputation (Alg. 1 lines 1-2).  Untimed, fp64.
//
// Independent of oracle/: Bessel values come from libm jn(), roots by sign scan + bisection +
// Newton, Gauss-Legendre by Newton on the Legendre recurrence, and the NUFFT window/deapodisation
// are product-only (the oracle uses a direct Fourier sum).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"

namespace fbspca {

namespace {

double bessel_j(int k, double x) { return jn(k, x); }

// All positive zeros of J_k up to xmax, plus the first above (P:87 R_{k,q}).  A sign scan of step
// 0.25 (< pi, below the spacing of consecutive zeros) brackets each root; J_k has no zero below k.
std::vector<double> bessel_zeros_upto(int k, double xmax) {
  std::vector<double> roots;
  const double step = 0.25;
  double x = std::max(double(k), 0.05);
  double fx = bessel_j(k, x);
  while (true) {
    double x2 = x + step;
    double f2 = bessel_j(k, x2);
    if ((fx < 0 && f2 > 0) || (fx > 0 && f2 < 0)) {
      double a = x, b = x2, fa = fx;
      for (int it = 0; it < 200 && b - a > 1e-15 * b; ++it) {     // bisection
        double m = 0.5 * (a + b), fm = bessel_j(k, m);
        if ((fa < 0) == (fm < 0)) { a = m; fa = fm; } else { b = m; }
      }
      double r = 0.5 * (a + b);
      for (int it = 0; it < 3; ++it) {                            // Newton polish, J_k' = (J_{k-1}-J_{k+1})/2
        double d = 0.5 * (bessel_j(k - 1, r) - bessel_j(k + 1, r));
        if (d == 0) break;
        double nr = r - bessel_j(k, r) / d;
        if (!(std::fabs(nr - r) < 0.5)) break;
        r = nr;
      }
      roots.push_back(r);
      if (r > xmax) break;
    }
    x = x2; fx = f2;
  }
  return roots;
}

// n-point Gauss-Legendre on [a,b]: Newton on P_n from cos(pi (i - 1/4)/(n + 1/2)).
void gauss_legendre(int n, double a, double b, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0); w.assign(n, 0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), pp = 0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1, p2 = 0;
      for (int j = 1; j <= n; ++j) { double p3 = p2; p2 = p1; p1 = ((2 * j - 1) * z * p2 - (j - 1) * p3) / j; }
      pp = n * (z * p1 - p2) / (z * z - 1);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-16) break;
    }
    {   // final derivative at the converged root
      double p1 = 1, p2 = 0;
      for (int j = 1; j <= n; ++j) { double p3 = p2; p2 = p1; p1 = ((2 * j - 1) * z * p2 - (j - 1) * p3) / j; }
      pp = n * (z * p1 - p2) / (z * z - 1);
    }
    double wi = 2.0 / ((1 - z * z) * pp * pp);
    // node -z (ascending order from a), +z mirrored
    x[i] = a + (b - a) * (1 - z) / 2;       x[n - 1 - i] = a + (b - a) * (1 + z) / 2;
    w[i] = wi * (b - a) / 2;                w[n - 1 - i] = wi * (b - a) / 2;
  }
}

// Exponential-of-semicircle window phi(y) = exp(beta (sqrt(1 - (2y/w)^2) - 1)), |y| <= w/2 (grid units),
// and its Fourier transform Phi(t) = int phi(y) e^{-2 pi i y t} dy, via y = (w/2) sin u (smooth in u).
double es_Phi(double t, int w, double beta) {
  static thread_local std::vector<double> gx, gw;
  if (gx.empty()) gauss_legendre(256, 0.0, M_PI / 2, gx, gw);
  double s = 0, hw = 0.5 * w;
  for (size_t i = 0; i < gx.size(); ++i) {
    double y = hw * std::sin(gx[i]);
    s += gw[i] * std::exp(beta * (std::cos(gx[i]) - 1.0)) * std::cos(2 * M_PI * y * t) * hw * std::cos(gx[i]);
  }
  return 2 * s;
}

bool smooth5(int n) { for (int f : {2, 3, 5}) while (n % f == 0) n /= f; return n == 1; }

FftPlan make_fft(int n) {
  FftPlan f; f.n = n;
  int m = n;
  auto push = [&](int r) { f.radix[f.nstages++] = r; m /= r; };
  while (m % 8 == 0 && f.nstages < kMaxRadixStages) push(8);
  while (m % 4 == 0 && f.nstages < kMaxRadixStages) push(4);
  while (m % 2 == 0 && f.nstages < kMaxRadixStages) push(2);
  while (m % 5 == 0 && f.nstages < kMaxRadixStages) push(5);
  while (m % 3 == 0 && f.nstages < kMaxRadixStages) push(3);
  for (int r : {7, 11, 13})
    while (m % r == 0 && f.nstages < kMaxRadixStages) push(r);
  if (m != 1) f.nstages = -1;
  return f;
}

int ceil_guard(double x) { return int(std::ceil(x - 1e-9)); }   // reading Q4

// Warp packing of the gather's node pairs (shared-memory bank model of K2's 6 x 6 tap loads).
// Lane i of a warp reads grid words (b1_i + q + row0) S + b2_i + c (node A) and (row0 - b1_i - q) S + b2_i + c
// (mirrored node B) for every tap (q, c): 64-bit words, 16 word-wide bank pairs, served per half-warp.  The tap
// offset is common to all lanes, so a half-warp's load costs max over bank pairs of the number of DISTINCT
// anchors in that pair, for classes cA = (b1 S + b2) mod 16 and cB = (b2 - b1 S) mod 16 -- 1 wavefront when the
// 16 lanes' distinct anchors fall in distinct pairs (equal anchors broadcast).  This model reproduces ncu's
// count for the plain (b1, b2) order at C3 (106.7k vs 102k wavefronts/image measured).  Greedy: walk anchors in
// (b1, b2) order, put an anchor into the open half-warp if neither class is at the cap (equal anchors are
// free), skip it otherwise; the cap doubles only when nothing left in the window fits.  Groups are emitted
// full (16) except the phase's last.

// Model cost (wavefronts per tap, summed over warps) of a node order under the bank model above.
std::vector<uint32_t> pack_gather_items(const std::vector<std::array<int, 3>>& items, int S);

long gather_bank_cost(const std::vector<uint32_t>& ord, const std::vector<double>& rho, const std::vector<double>& cs,
                      double hw, int S, int half, int group = 32) {
  long tot = 0;
  for (size_t w0 = 0; w0 < ord.size(); w0 += group) {
    std::vector<std::pair<int, int>> a, b;
    for (size_t i = w0; i < std::min(ord.size(), w0 + group); ++i) {
      const int j = int(ord[i] >> 16), l = int(ord[i] & 0xffffu);
      const int b1 = int(std::ceil(rho[j] * cs[2 * l] - hw)), b2 = int(std::ceil(rho[j] * cs[2 * l + 1] - hw));
      a.push_back({b1, b2});
      if (l != 0 && 2 * l != half) b.push_back({b1, b2});
    }
    for (int sg = 1; sg >= -1; sg -= 2) {
      auto& v = sg == 1 ? a : b;
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      int cnt[16] = {0}, m = 0;
      for (auto& e : v) m = std::max(m, ++cnt[(((sg * e.first * S + e.second) % 16) + 16) % 16]);
      tot += m;
    }
  }
  return tot;
}

std::vector<uint32_t> pack_gather_items(const std::vector<std::array<int, 3>>& items, int S) {
  struct Anc { int b1, b2; std::vector<uint32_t> ids; };
  std::vector<Anc> anc;
  {
    std::vector<std::array<int, 3>> keyed = items;
    std::sort(keyed.begin(), keyed.end());
    for (auto& e : keyed) {
      if (anc.empty() || anc.back().b1 != e[0] || anc.back().b2 != e[1]) anc.push_back({e[0], e[1], {}});
      anc.back().ids.push_back(uint32_t(e[2]));
    }
  }
  auto cls = [&](int b1, int b2, int sgn) { return (((sgn * b1 * S + b2) % 16) + 16) % 16; };
  std::vector<uint32_t> out;
  out.reserve(items.size());
  std::vector<char> used(anc.size(), 0);
  std::vector<size_t> done_ids(anc.size(), 0);
  size_t next = 0, left = anc.size();
  while (left > 0) {
    int cntA[16] = {0}, cntB[16] = {0}, slots = 16;
    for (int cap = 1; slots > 0 && left > 0 && cap <= 16; cap *= 2) {
      size_t scanned = 0;
      for (size_t a = next; a < anc.size() && slots > 0 && scanned < 4096; ++a) {
        if (used[a]) continue;
        ++scanned;
        const int ca = cls(anc[a].b1, anc[a].b2, 1), cb = cls(anc[a].b1, anc[a].b2, -1);
        if (cntA[ca] >= cap || cntB[cb] >= cap) continue;
        ++cntA[ca]; ++cntB[cb];
        const size_t take = std::min<size_t>(anc[a].ids.size() - done_ids[a], size_t(slots));
        for (size_t t = 0; t < take; ++t) out.push_back(anc[a].ids[done_ids[a] + t]);
        done_ids[a] += take;
        slots -= int(take);
        if (done_ids[a] == anc[a].ids.size()) { used[a] = 1; --left; }
      }
      while (next < anc.size() && used[next]) ++next;
    }
  }
  return out;
}

}  // namespace

int fft_values_per_lane(const FftPlan& f) {
  int v = 0;
  for (int s = 0; s < f.nstages; ++s) {
    int nb = f.n / f.radix[s];
    v = std::max(v, ((nb + 31) / 32) * f.radix[s]);
  }
  return v;
}

fbspca_status build_host_plan(Plan& P) {
  const double c = P.c, R = P.R;
  const int L = P.L;
  if (!(c > 0 && c <= 0.5)) { set_error("c must be in (0, 1/2] (P:78)"); return FBSPCA_ERR_CONFIG; }
  if (L < 4) { set_error("L must be >= 4"); return FBSPCA_ERR_CONFIG; }
  if (!(R >= 2) || c * R < 1) { set_error("R >= 2 and cR >= 1 required (empty basis otherwise)"); return FBSPCA_ERR_CONFIG; }
  if (R > 0.5 * L) { set_error("R must be <= L/2"); return FBSPCA_ERR_CONFIG; }
  if (!(P.eps >= 1e-14 && P.eps <= 1e-3)) { set_error("eps must be in [1e-14, 1e-3]"); return FBSPCA_ERR_CONFIG; }
  if (P.dt == FBSPCA_F32 && P.eps < 1e-6) { set_error("eps below the fp32 floor 1e-6"); return FBSPCA_ERR_CONFIG; }

  // ---- census (Eq. (criterion1)) ----
  const double X = 2 * M_PI * c * R;
  P.p.clear(); P.zeros.clear(); P.norm.clear();
  for (int k = 0;; ++k) {
    std::vector<double> z = bessel_zeros_upto(k, X);
    int pk = 0;
    for (size_t q = 1; q < z.size(); ++q) if (z[q] <= X) ++pk;
    if (pk == 0) break;
    P.p.push_back(pk);
    for (int q = 0; q < pk; ++q) {
      P.zeros.push_back(z[q]);
      P.norm.push_back(1.0 / (c * std::sqrt(M_PI) * std::fabs(bessel_j(k + 1, z[q]))));   // N_{k,q}
    }
  }
  P.k_max = int(P.p.size()) - 1;
  const int nk = P.k_max + 1;
  P.coef_off.assign(nk + 1, 0); P.blk_off.assign(nk + 1, 0); P.evec_off.assign(nk + 1, 0);
  for (int k = 0; k < nk; ++k) {
    P.coef_off[k + 1] = P.coef_off[k] + P.p[k];
    P.blk_off[k + 1] = P.blk_off[k] + int64_t(P.p[k]) * (P.p[k] + 1) / 2;
    P.evec_off[k + 1] = P.evec_off[k] + int64_t(P.p[k]) * P.p[k];
  }

  // ---- quadrature grid and radial table ----
  P.n_xi = ceil_guard(4 * c * R);
  P.n_theta = ceil_guard(16 * c * R);
  if (P.n_theta % 2) { set_error("n_theta = ceil(16cR) must be even (half-plane symmetry)"); return FBSPCA_ERR_CONFIG; }
  if (2 * P.k_max >= P.n_theta) { set_error("k_max >= n_theta/2"); return FBSPCA_ERR_CONFIG; }
  gauss_legendre(P.n_xi, 0.0, c, P.xi, P.wq);
  const int64_t ncoef = P.coef_off[nk];
  P.table.assign(size_t(ncoef) * P.n_xi, 0.0);
  P.rbasis.assign(size_t(ncoef) * P.n_xi, 0.0);
  const double ang = 2 * M_PI / P.n_theta;        // Eq. (1DFFT) weight, folded into the table
  for (int k = 0; k < nk; ++k)
    for (int q = 0; q < P.p[k]; ++q) {
      int64_t row = P.coef_off[k] + q;
      double Rq = P.zeros[row], N = P.norm[row];
      for (int j = 0; j < P.n_xi; ++j)
      {
        const double b = N * bessel_j(k, Rq * P.xi[j] / c);            // N_{k,q} J_k(R_{k,q} xi_j / c)
        P.rbasis[row * P.n_xi + j] = b;
        P.table[row * P.n_xi + j] = b * P.xi[j] * P.wq[j] * ang;
      }
    }
  // Structural zeros of the table: J_k(x) decays like (e x / 2k)^k below its turning point x ~ k, so for large k
  // the inner rings (small xi_j) carry |T_k[q][j]| below 1e-9 max|T_k| -- 1/60 of an fp32 ulp of any partial sum of
  // Eq. (a).  fp32 plans start K4's sum for block k at kj0[k], the first such j rounded down to a multiple of 8
  // (the tf32 MMA's K step); the polar kernel does not store ghat below it.  fp64 plans sum every ring.
  P.kj0.assign(nk, 0);
  if (P.dt == FBSPCA_F32)
    for (int k = 0; k < nk; ++k) {
      double mx = 0;
      const int64_t r0 = P.coef_off[k] * P.n_xi, r1 = P.coef_off[k + 1] * P.n_xi;
      for (int64_t i = r0; i < r1; ++i) mx = std::max(mx, std::fabs(P.table[i]));
      int j0 = P.n_xi;
      for (int64_t row = P.coef_off[k]; row < P.coef_off[k + 1]; ++row)
        for (int j = 0; j < j0; ++j)
          if (std::fabs(P.table[row * P.n_xi + j]) > 1e-9 * mx) { j0 = j; break; }
      P.kj0[k] = (j0 / 8) * 8;
    }

  // ---- NUFFT: oversampled grid, window, deapodisation ----
  int M = 2 * L;
  while (!smooth5(M) || M % 2) ++M;
  P.M = M;
  int w = int(std::ceil(-std::log10(P.eps) - 1e-9)) + 1;         // error ~ 10^{-(w-1)} at sigma = 2
  // fp32: eps >= 1e-6 (the fp32 floor) -> w <= 7; eps >= 1e-4 -> w = 5 (every fp32 polar kernel has W = 5, 6 instances;
  // W = 7 runs the runtime-radix kernel)
  if (P.dt == FBSPCA_F32) w = std::max(getenv("FBSPCA_NO_W5") ? 6 : 5, std::min(w, 7));
  else { w = std::max(w, 13); if (w > 13) w = 13; }
  P.w = w;
  P.beta = 2.30 * w;
  if (P.dt == FBSPCA_F32) P.beta = double(float(P.beta));   // the fp32 kernel evaluates phi with a float beta
  P.deapod.assign(L, 0.0);
  for (int a = 0; a < L; ++a) {
    int i = a - L / 2;
    P.deapod[a] = 1.0 / es_Phi(double(i) / M, w, P.beta);
  }

  // ---- polar nodes (half plane, theta in [0, pi)), column phases ----
  const int half = P.n_theta / 2;
  const double hw = 0.5 * w;
  std::vector<double> rho(P.n_xi), cs(2 * half);
  for (int j = 0; j < P.n_xi; ++j) rho[j] = P.xi[j] * M;
  for (int l = 0; l < half; ++l) {
    double th = 2 * M_PI * l / P.n_theta;
    cs[2 * l] = std::cos(th); cs[2 * l + 1] = std::sin(th);
  }
  std::vector<int> b2(size_t(P.n_xi) * half);
  int b2min = 1 << 30, b2max = -(1 << 30);
  for (int j = 0; j < P.n_xi; ++j)
    for (int l = 0; l < half; ++l) {
      double k2 = rho[j] * cs[2 * l + 1];
      int b = int(std::ceil(k2 - hw));
      b2[size_t(j) * half + l] = b;
      b2min = std::min(b2min, b); b2max = std::max(b2max, b);
    }
  PolarParams& pp = P.pp;
  pp = PolarParams{};
  pp.L = L; pp.M = M; pp.w = w; pp.n_xi = P.n_xi; pp.n_theta = P.n_theta; pp.half = half; pp.k_max = P.k_max;
  pp.col_lo = b2min; pp.ncols_x = b2max + w - b2min;
  pp.beta = P.beta; pp.half_w = hw;
  pp.fft_M = make_fft(M); pp.fft_theta = make_fft(P.n_theta);
  if (pp.fft_M.nstages < 0 || pp.fft_theta.nstages < 0) { set_error("FFT sizes must be 2^a 3^b 5^c 7^d 11^e 13^f"); return FBSPCA_ERR_CONFIG; }
  pp.nwarps = 16;
  const int csz = (P.dt == FBSPCA_F32) ? 8 : 16;       // sizeof complex
  const int cap = polar_max_smem();
  pp.fft_warps = 16;
  // ring-pair plans (n_theta = 2 M) run K3 in the per-warp FFT scratch too, so more of the budget goes there
  const int fft_share = (P.n_theta == 2 * M) ? 2 : 3;
  while (pp.fft_warps > 2 && pp.fft_warps * 2 * M * csz > cap / fft_share) pp.fft_warps /= 2;
  if (const char* e = getenv("FBSPCA_FFT_WARPS")) pp.fft_warps = std::max(1, std::min(16, atoi(e)));
  // the compile-time M = 256 fp32 kernel runs every FFT as half-warp radix-16 x 16 transforms (two per warp) with
  // its own per-warp scratch, on all 16 warps (one ring pair per warp per 32-ring group)
  const bool hw16 = P.dt == FBSPCA_F32 && (w == 5 || w == 6) && M == 256 && P.n_theta == 2 * M;
  if (hw16) pp.fft_warps = 16;
  const int fixed = polar_fixed_smem(M, P.n_theta, L, csz, pp.fft_warps, P.k_max + 1, hw16);
  const int budget = cap - fixed;
  const int kk = (P.k_max + 1) | 1;                    // staging row stride (odd)
  const int ntp = (P.n_theta + 15) & ~15;               // ping-pong length (swizzle permutes 16-blocks)
  // angular pass: (warps running ring FFTs, rings staged per group); prefer all 16 warps busy
  const int cand[][2] = {{16, 16}, {8, 32}, {8, 16}, {4, 16}, {4, 8}, {2, 8}, {1, 4}, {1, 1}};
  pp.ang_warps = 0;
  int Gsel = 1;
  for (auto& c : cand) {
    const int g = std::min(c[1], P.n_xi);
    if (c[0] * 2 * ntp * csz + ((g + 1) | 1) * kk * csz <= budget) { pp.ang_warps = c[0]; Gsel = g; break; }
  }
  if (pp.ang_warps < 1 || budget < M * 11 * csz) {
    set_error("image too large for the fused polar kernel's shared memory"); return FBSPCA_ERR_CONFIG;
  }
  const int ang_scr = pp.ang_warps * 2 * ntp * csz;
  const int rows_g = M + 2 * w;                          // Gc rows incl. wrapped duplicates (PADR = w)
  int S = budget / (rows_g * csz);
  if (S % 2 == 0) --S;                                   // odd row stride (bank spread)
  if (S > pp.ncols_x) S = pp.ncols_x | 1;
  pp.S = S;
  // pow2 plans (n_theta = 2 M, M in {64..512}) run the ring FFTs as pairs of half-length FFTs in the per-warp
  // FFT scratch (kernels_polar.cu K3): the staging [k][ring] for 32 rings is all the region holds then
  // fp32 compile-time FFT kernels (launch_polar's dispatch).  Only they read double entries and ring strides: an fp32
  // plan with M = 64, or with one of these M but n_theta != 2 M (c < 1/2), runs the runtime-radix kernel on singles.
  const bool pow2_kernel = polar_f32_ct_kernel(M, P.n_theta);
  const bool ring_pairs = P.n_theta == 2 * M && !getenv("FBSPCA_NO_RT_PAIRS");
  pp.ring_pairs = ring_pairs ? 1 : 0;
  if (ring_pairs) {
    Gsel = std::min(32, P.n_xi);
    while (Gsel > 2 && ((Gsel + 1) | 1) * kk * csz > std::max(rows_g * S * csz, pp.fft_warps * M * csz)) Gsel /= 2;
  }
  const int G = Gsel;
  pp.ring_group = G;
  if (hw16 && G > 2 * pp.fft_warps) { set_error("internal: M = 256 ring groups exceed one ring pair per warp"); return FBSPCA_ERR_CONFIG; }
  const int region = std::max(std::max(rows_g * S * csz, pp.fft_warps * M * csz),
                              (ring_pairs ? 0 : ang_scr) + ((G + 1) | 1) * kk * csz);
  pp.smem_region_bytes = region;
  {   // image staged behind the phase-0 grid rows (pow2) or the per-warp row results (runtime sizes)
    const int used = std::max(L * S, pp.fft_warps * M);            // complex elements
    const int need = used + (L * L * (csz / 2) + csz - 1) / csz + 2;
    pp.img_off = (need * csz <= region) ? ((used + 1) & ~1) : -1;    // 16-B aligned start
    // the angular pass uses the region below img_off only (staging [k][ring], + ping-pongs on runtime sizes)
    const int ang_use = (ring_pairs ? 0 : ang_scr) + ((G + 1) | 1) * kk * csz;
    pp.img_prefetch = (pp.img_off >= 0 && ang_use <= pp.img_off * csz) ? 1 : 0;
  }
  P.polar_smem = fixed + region;
  // phases over columns: phase p holds m2 in [lo_p, lo_p + S) and owns single entries with b2 in
  // [lo_p, lo_p + S - w] and double entries with union anchor U2 in [lo_p, lo_p + S - w - 1].
  //
  // Double entries (fp32 W = 6 pow2 kernels): two pair leaders (j, l), (j, l + 1) of one ring whose anchors differ
  // by at most 1 in each direction share a (w + 1) x (w + 1) window at U = min(b): 49 + 49 grid loads for four
  // nodes instead of 4 x 36 (the mirrored pair members (j, half - l), (j, half - l - 1) share it mirrored).
  auto anchor = [&](int j, int l) {
    return std::make_pair(int(std::ceil(rho[j] * cs[2 * l] - hw)), int(std::ceil(rho[j] * cs[2 * l + 1] - hw)));
  };
  std::vector<int> phase_lo;
  for (int lo = b2min; lo <= b2max; lo += S - w + 1) phase_lo.push_back(lo);
  if ((int)phase_lo.size() > kMaxPhases) { set_error("too many column phases"); return FBSPCA_ERR_CONFIG; }
  auto phase_of_single = [&](int b2) { return std::min<int>((b2 - b2min) / (S - w + 1), (int)phase_lo.size() - 1); };
  auto phase_of_double = [&](int u2) {     // all w + 1 columns must be valid grid columns of the phase
    const int p = (u2 - b2min) / (S - w + 1);
    if (p >= (int)phase_lo.size()) return -1;
    const int last = std::min(phase_lo[p] + S - 1, b2max + w - 1);
    return (u2 + w <= last) ? p : -1;
  };
  const bool doubles = P.dt == FBSPCA_F32 && (w == 5 || w == 6) && pow2_kernel && !getenv("FBSPCA_NO_DOUBLES");
  std::vector<std::vector<std::array<int, 3>>> ph_single(phase_lo.size()), ph_double(phase_lo.size());
  std::vector<uint32_t> singles;
  std::vector<std::array<uint32_t, 2>> dbl;
  // Angular stride per ring (fp32 compile-time ring-pair kernels: M in {64, 128, 256, 512, 600, 720}).  Ring j only feeds K4 blocks k <= kneed(j) = max{k : kj0[k] <= j},
  // and F restricted to the ring has no angular content beyond kc(j): by Jacobi-Anger its k-th angular Fourier
  // coefficient is sum_x I(x) (-i)^k J_k(2 pi xi_j |x|) e^{-i k phi_x}, and |J_k(z)| < 1e-10 for k >= kc(z) past the
  // turning point, with |x| <= r_c = sqrt(2) ceil(L/2) over the square (no disk mask, reading Q7).  Sampling the ring
  // at n_theta / s_j angles theta_{l s_j} keeps every needed k free of aliases as long as n_theta / s_j >= kneed + kc
  // (the nearest alias of k <= kneed is k - n_theta / s_j).  The ring FFT runs on the zero-stuffed ring (the
  // n_theta-point DFT of the stuffed sequence IS the (n_theta / s_j)-point DFT, exactly), and the quadrature weight
  // 2 pi s_j / n_theta is the table's 2 pi / n_theta times the power of two s_j (capi.cu upload).  Inner rings need
  // far fewer angles: C3 gathers 0.70 of the nodes.  FBSPCA_NO_RING_STRIDE=1 samples every ring at all n_theta angles.
  P.ring_s.assign(P.n_xi, 1);
  const bool ring_stride_kernel = P.dt == FBSPCA_F32 && (w == 5 || w == 6) && pow2_kernel && P.n_theta == 2 * M;
  if (ring_stride_kernel && !getenv("FBSPCA_NO_RING_STRIDE")) {
    const double rc = std::sqrt(2.0) * std::ceil(0.5 * L);
    for (int j = 0; j < P.n_xi; ++j) {
      int kneed = 0;
      for (int k = 0; k < nk; ++k)
        if (P.kj0[k] <= j) kneed = k;
      const double z = 2 * M_PI * P.xi[j] * rc;
      int kc = int(std::floor(z));
      while (std::fabs(bessel_j(kc, z)) > 1e-10 || std::fabs(bessel_j(kc + 1, z)) > 1e-10) ++kc;
      const int need = kneed + kc + 1;
      int sj = 1;
      while (sj < 8 && P.n_theta / (2 * sj) >= need && half % (2 * sj) == 0) sj *= 2;
      P.ring_s[j] = sj;
    }
  }
  auto pol_slot = [&](uint32_t nd) {
    const int j = int(nd >> 16), l = int(nd & 0xffffu), sj = P.ring_s[j];
    const int ls = sj == 8 ? 3 : sj == 4 ? 2 : sj == 2 ? 1 : 0;
    return (uint32_t(j) << 16) | uint32_t(l >> ls) | (uint32_t(ls) << 28);
  };
  if (P.n_xi >= 4096) { set_error("n_xi >= 4096: polar node records hold 12-bit ring indices"); return FBSPCA_ERR_CONFIG; }
  for (int j = 0; j < P.n_xi; ++j) {
    const int sj = P.ring_s[j];               // ring j's angles theta_l, l = 0, sj, 2 sj, .. (sj | half/2)
    for (int l = 0; 2 * l <= half; l += sj) {
      const auto a = anchor(j, l);
      if (doubles && l >= 1 && 2 * (l + sj) < half) {
        const auto b = anchor(j, l + sj);
        const int u1 = std::min(a.first, b.first), u2 = std::min(a.second, b.second);
        const int p = phase_of_double(u2);
        if (std::abs(a.first - b.first) <= 1 && std::abs(a.second - b.second) <= 1 && p >= 0) {
          ph_double[p].push_back({u1, u2, int(dbl.size())});
          dbl.push_back({(uint32_t(j) << 16) | uint32_t(l), (uint32_t(j) << 16) | uint32_t(l + sj)});
          l += sj;
          continue;
        }
      }
      singles.push_back((uint32_t(j) << 16) | uint32_t(l));
    }
  }
  // Leftover pair leaders (no ring neighbour within reach) are paired across rings: any two whose anchors differ by
  // at most 1 in each direction share a 7 x 7 window just as ring neighbours do (the double-entry kernel takes each
  // node's ring from its record).  A single costs 36 grid loads per node, a double 24.5.
  if (doubles) {
    std::vector<char> paired(singles.size(), 0);
    std::vector<std::pair<std::pair<int, int>, int>> by_anchor;       // (anchor, index) of mirrored leaders
    for (size_t i = 0; i < singles.size(); ++i) {
      const int j = int(singles[i] >> 16), l = int(singles[i] & 0xffffu);
      if (l >= 1 && 2 * l < half) by_anchor.push_back({anchor(j, l), int(i)});
    }
    std::sort(by_anchor.begin(), by_anchor.end());
    auto find = [&](std::pair<int, int> an) {
      auto it = std::lower_bound(by_anchor.begin(), by_anchor.end(), std::make_pair(an, -1));
      for (; it != by_anchor.end() && it->first == an; ++it)
        if (!paired[it->second]) return it->second;
      return -1;
    };
    for (auto& e : by_anchor) {
      const int i = e.second;
      if (paired[i]) continue;
      paired[i] = 1;
      int mate = -1;
      for (int d1 = -1; d1 <= 1 && mate < 0; ++d1)
        for (int d2 = -1; d2 <= 1 && mate < 0; ++d2) {
          const int m = find({e.first.first + d1, e.first.second + d2});
          if (m < 0) continue;
          const int u2 = std::min(e.first.second, e.first.second + d2);
          if (phase_of_double(u2) >= 0) mate = m;
        }
      if (mate < 0) { paired[i] = 0; continue; }
      paired[mate] = 1;
      const int j = int(singles[mate] >> 16), l = int(singles[mate] & 0xffffu);
      const auto b = anchor(j, l);
      const int u1 = std::min(e.first.first, b.first), u2 = std::min(e.first.second, b.second);
      ph_double[phase_of_double(u2)].push_back({u1, u2, int(dbl.size())});
      dbl.push_back({singles[i], singles[mate]});
    }
    std::vector<uint32_t> rest;
    for (size_t i = 0; i < singles.size(); ++i)
      if (!paired[i]) rest.push_back(singles[i]);
    singles.swap(rest);
  }
  for (size_t i = 0; i < singles.size(); ++i) {
    const auto a = anchor(int(singles[i] >> 16), int(singles[i] & 0xffffu));
    ph_single[phase_of_single(a.second)].push_back({a.first, a.second, int(i)});
  }
  P.nodes.clear();
  P.dnoderec.clear();
  int np = 0;
  for (size_t p = 0; p < phase_lo.size(); ++p) {
    pp.phase_lo[np] = phase_lo[p];
    pp.phase_node_begin[np] = int(P.nodes.size());
    pp.phase_dbl_begin[np] = int(P.dnoderec.size() / 8);
    for (uint32_t id : pack_gather_items(ph_single[p], S)) P.nodes.push_back(singles[id]);
    for (uint32_t id : pack_gather_items(ph_double[p], S)) {
      // {U1 | U2 << 16, t1a, t2a, offsets}, {node a, t1b, t2b, node b}; t = k - b of each node's own anchor
      int32_t rec[8];
      const uint32_t na = dbl[id][0], nb = dbl[id][1];
      const int ja = int(na >> 16), la = int(na & 0xffffu), jb = int(nb >> 16), lb = int(nb & 0xffffu);
      const auto aa = anchor(ja, la), ab = anchor(jb, lb);
      const int u1 = std::min(aa.first, ab.first), u2 = std::min(aa.second, ab.second);
      const float t1a = float(rho[ja] * cs[2 * la] - aa.first), t2a = float(rho[ja] * cs[2 * la + 1] - aa.second);
      const float t1b = float(rho[jb] * cs[2 * lb] - ab.first), t2b = float(rho[jb] * cs[2 * lb + 1] - ab.second);
      rec[0] = int32_t((uint32_t(u1) & 0xFFFFu) | (uint32_t(u2) << 16));
      std::memcpy(&rec[1], &t1a, 4); std::memcpy(&rec[2], &t2a, 4);
      rec[3] = (aa.first - u1) | ((aa.second - u2) << 1) | ((ab.first - u1) << 2) | ((ab.second - u2) << 3);
      rec[4] = int32_t(pol_slot(na));
      std::memcpy(&rec[5], &t1b, 4); std::memcpy(&rec[6], &t2b, 4);
      rec[7] = int32_t(pol_slot(nb));
      P.dnoderec.insert(P.dnoderec.end(), rec, rec + 8);
    }
    if (getenv("FBSPCA_DEBUG_PLAN"))
      fprintf(stderr, "phase %d: lo %d, %zu single pair-leaders, %zu doubles\n", np, phase_lo[p],
              ph_single[p].size(), ph_double[p].size());
    ++np;
  }
  pp.n_phase = np;
  // TMEM parking of the second phase's columns (kernels_polar.cu): M = 256 compile-time kernel with 16 FFT warps and two
  // phases; the warp's four row pairs x ng 32-column groups x 4 floats fit 64 TMEM columns (4 warps per lane quarter)
  pp.tmem_x = 0;
  if (M == 256 && P.n_theta == 2 * M && P.dt == FBSPCA_F32 && (w == 5 || w == 6) && pp.fft_warps == 16 && np == 2 &&
      (L + 1) / 2 <= 4 * 16 && !getenv("FBSPCA_NO_TMEM_X")) {
    const int c1 = pp.phase_lo[1] - pp.col_lo;               // first row-pass column index of phase 1
    pp.tmem_g0 = c1 / 32;
    pp.tmem_ng = (pp.ncols_x - 1) / 32 - pp.tmem_g0 + 1;
    if (pp.tmem_ng >= 1 && pp.tmem_ng <= 4) pp.tmem_x = 1;
  }
  pp.phase_node_begin[np] = int(P.nodes.size());
  pp.phase_dbl_begin[np] = int(P.dnoderec.size() / 8);
  P.rho = rho;
  P.cs = cs;
  // per-entry record for the fp32 gather: {b1 | b2 << 16, t1, t2, (j << 16) | l}, the same fp64 arithmetic
  // the fp64 kernel path performs on the fly (k = rho_j (cos, sin) theta_l, b = ceil(k - w/2), t = k - b)
  // Pol slot of a node: ring j keeps its n_theta / s_j samples contiguous (sample l at l / s_j, mirrors at
  // half_j - l / s_j, half_j = half / s_j), so the gather writes whole 32-byte sectors of the per-CTA polar scratch
  // (partially written sectors made every ring load an L2 miss filled from DRAM).  Encoded (j << 16) | (l / s_j) |
  // (log2 s_j << 28) in the fp32 records; j < 4096.
  P.noderec.resize(4 * P.nodes.size());
  for (size_t e = 0; e < P.nodes.size(); ++e) {
    const uint32_t nd = P.nodes[e];
    const int j = int(nd >> 16), l = int(nd & 0xffffu);
    const double k1 = rho[j] * cs[2 * l], k2 = rho[j] * cs[2 * l + 1];
    const double f1 = std::ceil(k1 - hw), f2 = std::ceil(k2 - hw);
    const float t1 = float(k1 - f1), t2 = float(k2 - f2);
    const int b1 = int(f1), b2 = int(f2);
    int32_t rec[4];
    rec[0] = int32_t((uint32_t(b1) & 0xFFFFu) | (uint32_t(b2) << 16));
    std::memcpy(&rec[1], &t1, 4);
    std::memcpy(&rec[2], &t2, 4);
    rec[3] = int32_t(pol_slot(nd));
    std::memcpy(&P.noderec[4 * e], rec, 16);
  }
  return FBSPCA_OK;
}

}  // namespace fbspca
