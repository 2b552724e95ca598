// internal.h -- plan structure shared by the host plan builder, the C-ABI layer and the kernels.
// Nothing here is visible through include/fbspca.h.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fbspca.h"

namespace fbspca {

constexpr int kMaxRadixStages = 16;
constexpr int kMaxPhases = 64;
constexpr int kCovChunk = 1024;         // images per SIMT covariance split-K chunk (bounds fp32 accumulation length)
constexpr int kCovBatch = 16384;        // images per SIMT covariance launch
constexpr int kCovChunkTc = 4096;       // images per tensor-core split-K chunk (cov_tma_chunk() <= this)
#ifndef FBSPCA_COV_SLOTS
#define FBSPCA_COV_SLOTS 32
#endif
constexpr int kCovMaxChunks = FBSPCA_COV_SLOTS;              // split-K scratch slots (SIMT: kCovBatch / kCovChunk = 16)
static_assert(kCovBatch / kCovChunk <= kCovMaxChunks, "covariance scratch slots");
constexpr int kCovBatchTc = kCovChunkTc * kCovMaxChunks;     // images per tensor-core covariance launch: 131,072, so a
                                        // C3 step (100,000 images) is one launch (16,384 -> 65,536 took the C3 K5 from
                                        // 2.03 to 1.85 ms: more items per persistent CTA, fewer launch tails)
constexpr int kCovChunk0 = 128;         // images per k = 0 fp64 CTA (tensor-core path: its own scratch, more CTAs)
constexpr int kCovMaxSub0 = kCovBatchTc / kCovChunk0;

// Per-warp FFT scratch of the polar kernel (complex elements): two ping-pong buffers of M (padded to 16), or for the
// M = 256 fp32 kernel (hw: half-warp radix-16 x 16 FFTs, fft_device.cuh) two half-warp buffers of 16 rows x 17.
constexpr int kHwBuf = 272;
__host__ __device__ constexpr int polar_warp_scratch(int M, bool hw) { return hw ? 2 * kHwBuf : 2 * ((M + 15) & ~15); }

// Stockham radix plan for a length-N FFT (N = prod radices; radices in {2,3,4,5,8}).
struct FftPlan {
  int n = 0;
  int nstages = 0;
  int radix[kMaxRadixStages] = {0};
};

// Everything a polar-kernel launch needs, passed by value (fits the 32 KB param space).
struct PolarParams {
  int L, M, w, n_xi, n_theta, half, k_max;
  int col_lo, ncols_x;            // X scratch columns cover m2 in [col_lo, col_lo + ncols_x)
  int S;                          // phase chunk width (columns) and its padded row stride
  int n_phase;
  int phase_lo[kMaxPhases];       // first column (m2) of phase p
  int phase_node_begin[kMaxPhases + 1];
  int phase_dbl_begin[kMaxPhases + 1];       // double entries (2 int4 each) of phase p: [begin[p], begin[p+1])
  double beta;
  double half_w;                  // w/2
  int nwarps;                     // warps per CTA (gather, fills)
  int fft_warps;                  // warps owning row/column FFT scratch
  int ang_warps;                  // warps running ring FFTs
  int ring_group;                 // rings staged together in the angular pass
  int smem_region_bytes;          // bytes of the shared work region (complex units * sizeof)
  int img_off;                    // complex-element offset of the staged image in the region (-1: read global)
  int img_prefetch;               // 1: the next image is loaded (cp.async) during the angular pass
  int ring_pairs;                 // 1: n_theta = 2 M, rings transformed in pairs of M-point FFTs (K3)
  int tmem_x;                     // 1: the second column phase's row-FFT columns are parked in TMEM, not in X (M = 256)
  int tmem_g0, tmem_ng;           //    32-column groups g0 .. g0 + ng - 1 of the row pass hold them
  FftPlan fft_M, fft_theta;
  // device pointers (plan-owned)
  const void* deapod;             // L values (T): d(i) = 1/Phi(i/M), i = a - floor(L/2)
  const void* tw_M;               // M complex (T2): e^{-2 pi i t / M}
  const void* tw_theta;           // n_theta complex (T2)
  const double* rho;              // n_xi: xi_j * M
  const double* cs;               // half x 2: cos(theta_l), sin(theta_l)
  const uint32_t* nodes;          // (j << 16) | l, grouped by phase
  const int* kj0;                 // per k: first ring j K4 reads (rings below carry |T_k| < 1e-9 max|T_k|; plan.cpp)
  const int* ring_s;              // per ring j: angular stride s_j (ring sampled at theta_l, l = 0, s_j, 2 s_j, ..; plan.cpp)
  const int4* noderec;            // per entry {b1 | b2 << 16, t1, t2, (j << 16) | l} (fp32 path)
  const int4* dnoderec;           // per double entry 2 int4 (plan.cpp "Double entries")
  void* xscratch;                 // per resident CTA: L x ncols_x complex
  void* pscratch;                 // per resident CTA: n_xi x half complex
  int64_t ghat_kstride;           // ghat elements (T) per k: 2 max_batch n_xi (fixed, so one TMA map serves all batches)
  int64_t xscratch_stride, pscratch_stride;   // complex elements per CTA
};

struct Plan {
  // configuration
  int L = 0;
  double c = 0, R = 0, eps = 0;
  fbspca_dtype dt = FBSPCA_F32;
  int device = -1;
  int64_t max_batch = 0;
  // census
  int k_max = -1;
  std::vector<int> p;                    // p_k
  std::vector<int64_t> coef_off;         // k_max+2
  std::vector<int64_t> blk_off;          // k_max+2 (packed upper triangles)
  std::vector<int64_t> evec_off;         // k_max+2 (p_k^2)
  std::vector<double> zeros;             // R_{k,q}, coef_off layout
  std::vector<double> norm;              // N_{k,q}
  // quadrature grid
  int n_xi = 0, n_theta = 0;
  std::vector<double> xi, wq;
  std::vector<double> table;             // [coef row][j]: N J_k(R xi_j/c) xi_j w_j (2 pi / n_theta)
  std::vector<double> rbasis;            // [coef row][j]: N J_k(R xi_j/c)  (Eq. (sPCArad))
  std::vector<int> kj0;                  // per k: first ring j of K4's sum (multiple of 8; 0 for fp64 plans)
  int* d_kj0 = nullptr;
  std::vector<int> ring_s;               // per ring j: angular stride s_j (n_theta / s_j samples; 1 = every theta_l)
  int* d_ring_s = nullptr;
  // NUFFT
  int M = 0, w = 0;
  double beta = 0;
  std::vector<double> deapod;            // L
  std::vector<double> rho, cs;           // xi_j M; (cos, sin)(theta_l), l < n_theta/2
  PolarParams pp{};                      // host copy (device pointers filled at upload)
  std::vector<uint32_t> nodes;
  std::vector<int32_t> noderec;          // 4 per node entry
  std::vector<int32_t> dnoderec;         // 8 per double entry
  int polar_smem = 0;
  int polar_grid = 0;                    // resident CTAs of the polar kernel
  // device buffers
  void* d_table = nullptr;               // T (float or double), coef rows x n_xi
  double* d_rbasis = nullptr;            // rbasis (fp64), coef rows x n_xi
  float* d_table_lo = nullptr;           // fp32 plans: T - tf32(T)  (3xTF32 tensor-core K4)
  float* d_table_hi = nullptr;           // fp32 plans: tf32_rna(T)
  bool use_tc = true;                    // K4 on tcgen05 (fp32 plans)
  void* d_deapod = nullptr;
  void* d_tw_M = nullptr;
  void* d_tw_theta = nullptr;
  double* d_rho = nullptr;
  double* d_cs = nullptr;
  uint32_t* d_nodes = nullptr;
  int32_t* d_noderec = nullptr;
  int32_t* d_dnoderec = nullptr;
  PolarParams* d_pp = nullptr;           // device copy of pp
  void* d_xscratch = nullptr;
  void* d_pscratch = nullptr;
  void* d_ghat = nullptr;                // (k_max+1) x max_batch x 2 x n_xi  (T), k stride 2 max_batch n_xi
  double* d_partial = nullptr;           // blk_off[k_max+1] + p_0 + 1
  double* d_cov_scratch = nullptr;       // kCovMaxChunks x (blk_off[k_max+1] + p_0 + 1)
  double* d_cov_scratch0 = nullptr;      // kCovMaxSub0 x (blk_off[1] + p_0 + 1): k = 0 block, s_0, count
  int* d_coef_k = nullptr;               // row -> k lookup (coef rows)
  int* d_p = nullptr;
  int64_t* d_coef_off = nullptr;
  int64_t* d_blk_off = nullptr;
  int64_t* d_evec_off = nullptr;
  double* d_eig_work = nullptr;          // 2 * evec_off[k_max+1]
  int* d_eig_sweeps = nullptr;           // k_max+1
  // timing
  bool timing = false;
  std::vector<std::string> tnames;
  std::vector<const char*> tname_ptrs;
  std::vector<float> tms;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> tevents;
  std::vector<cudaEvent_t> event_pool;   // timing events, created once and reused
  // fbspca_step CUDA graphs: one instantiated graph per argument set (pointers, counts, communicator, stream)
  struct GraphEntry {
    const void* images; int64_t n_local, n_total; void* comm; void* coeffs; double* blocks; double* mean;
    cudaStream_t stream; int uses; cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  int num_sms = 0;
  // NEXT-1 synthesis tables (built on the first fbspca_synthesize)
  double* d_synth_rho = nullptr;         // [coef row][radius]: rho_{k,q}(r)
  int* d_synth_pidx = nullptr;           // disk pixels sorted by radius: linear index, radius index, (cos, sin) phi
  int* d_synth_pir = nullptr;
  double* d_synth_pcs = nullptr;
  int* d_synth_grp = nullptr;            // pixel groups of <= 2048 (CTA work units)
  int synth_nr = 0, synth_ngroups = 0;
  cudaStream_t side = nullptr;           // K5: the k = 0 fp64 CTAs run here, forked from / joined to the caller's stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

// per-(kernel, device) dynamic shared-memory opt-in, thread-safe (capi.cu)
cudaError_t ensure_smem_optin(const void* func, int bytes);

// ---- host plan construction (plan.cpp) ----
fbspca_status build_host_plan(Plan& P);           // census, grid, table, NUFFT, phases (no CUDA)
void set_error(const std::string& msg);

// ---- launchers (kernels_*.cu) ----
cudaError_t launch_polar(const Plan& P, const void* d_images, int64_t n_img, int64_t img_stride_elems,
                         cudaStream_t s);
cudaError_t launch_radial(const Plan& P, int64_t nb, int64_t i0, int64_t ld, void* d_coeffs,
                          cudaStream_t s);
cudaError_t launch_cov_accum(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb,
                             double* d_partial, cudaStream_t s);
cudaError_t launch_cov_finalize(const Plan& P, const double* d_partial, double* d_blocks, double* d_mean,
                                cudaStream_t s);
constexpr int kSvdMaxP = 1024;          // p_k bound of the SVD route's shared mean / norm scratch
constexpr int kSvdMaxSweeps = 40;
cudaError_t launch_svd(const Plan& P, const void* d_coeffs, int64_t n, double* d_work, double* d_mean,
                       double* d_evals, double* d_evecs, cudaStream_t s);
cudaError_t launch_eig(const Plan& P, const double* d_blocks, double* d_evals, double* d_evecs,
                       cudaStream_t s);
cudaError_t launch_radial_eigfun(const Plan& P, const double* d_evecs, double* d_f, cudaStream_t s);
cudaError_t launch_synthesize(Plan& P, const void* d_coeffs, int64_t n, void* d_images, cudaStream_t s);
cudaError_t launch_backproject(const Plan& P, const void* d_c, int64_t n, const double* d_mean, const double* d_evecs,
                               void* d_out, cudaStream_t s);
fbspca_status estimate_params(int L, fbspca_dtype dt, int device, const void* d_images, int64_t n, double fraction,
                              double* out3);
cudaError_t launch_project(const Plan& P, const void* d_coeffs, int64_t n, const double* d_mean,
                           const double* d_evals, const double* d_evecs, double sigma2, int mode,
                           int64_t n_total, void* d_out, cudaStream_t s);
// fp32 plans served by a compile-time-FFT polar kernel (launch_polar's dispatch; the plan emits double entries and
// ring strides only for these -- the runtime-radix kernel gathers single entries on full rings).  Window widths
// w = 5 (eps >= 1e-4) and w = 6 are compiled for every such M and for the runtime-radix kernel; w = 7 only for the latter.
inline bool polar_f32_ct_kernel(int M, int n_theta) {
  return n_theta == 2 * M && (M == 128 || M == 256 || M == 512 || M == 600 || M == 720);
}
int polar_max_smem();
cudaError_t launch_radial_tma(const Plan& P, int64_t nb, int64_t i0, int64_t ld, void* d_coeffs, cudaStream_t s);
cudaError_t launch_cov_tma(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb, cudaStream_t s);
cudaError_t launch_cov_k0(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb, cudaStream_t s);
int cov_tma_chunk();                    // images per split-K chunk of the tensor-core K5 (a multiple of kCovChunk)
bool cov_uses_tc(const Plan& P, int64_t ld);   // K5 for k >= 1 on tcgen05 for this plan and leading dimension
int fft_values_per_lane(const FftPlan& f);
int polar_fixed_smem(int M, int n_theta, int L, int csz, int nwarps, int nk, bool hw);

}  // namespace fbspca
