// capi.cu -- the extern "C" boundary declared in include/fbspca.h.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace fbspca {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: remember what was set per (kernel, device)
// under a mutex so a plan on a second device (or another thread) gets its own opt-in.
cudaError_t ensure_smem_optin(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

fbspca_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return FBSPCA_ERR_CUDA;
}

#define FB_CUDA(call, where)                        \
  do {                                              \
    cudaError_t _e = (call);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

template <typename T>
cudaError_t upload(void** dst, const T* src, size_t count) {
  cudaError_t e = cudaMalloc(dst, count * sizeof(T) + 16);
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

template <typename T>
std::vector<T> cast_vec(const std::vector<double>& v) { return std::vector<T>(v.begin(), v.end()); }

template <typename T2, typename T>
std::vector<T2> twiddles(int n) {
  std::vector<T2> t(n);
  for (int i = 0; i < n; ++i) {
    double a = -2.0 * M_PI * double(i) / double(n);
    t[i].x = T(std::cos(a)); t[i].y = T(std::sin(a));
  }
  return t;
}

enum TimingKind { T_POLAR = 0, T_RADIAL, T_COV, T_ALLREDUCE, T_FINALIZE, T_EIG, T_PROJECT, T_NKINDS };
const char* kTimingNames[T_NKINDS] = {"polar_K1K2K3", "radial_K4", "cov_K5", "allreduce", "finalize", "eig_K6",
                                      "project_K7"};

// Events come from a per-plan pool (created once, reused after every fbspca_get_timing), so a timed region costs
// two cudaEventRecord calls and no event creation.  Regions inside a stream capture are not timed.
struct TimedRegion {
  Plan& P; int kind; cudaStream_t s; bool on = false; cudaEvent_t e0 = nullptr, e1 = nullptr;
  TimedRegion(Plan& p, int kd, cudaStream_t st) : P(p), kind(kd), s(st) {
    if (!P.timing) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    const size_t need = 2 * (P.tevents.size() + 1);
    while (P.event_pool.size() < need) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      P.event_pool.push_back(e);
    }
    e0 = P.event_pool[need - 2]; e1 = P.event_pool[need - 1];
    on = cudaEventRecord(e0, s) == cudaSuccess;
  }
  ~TimedRegion() {
    if (on && cudaEventRecord(e1, s) == cudaSuccess) P.tevents.push_back({kind, {e0, e1}});
  }
};

// ---------------------------------------------------------------- NCCL via dlopen
struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (NCCL >= 2.19): NCCL-allocated, communicator-registered buffers; async error query / abort
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommRegister)(ncclComm_t, void*, size_t, void**) = nullptr;
  ncclResult_t (*CommDeregister)(ncclComm_t, void*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};
Nccl g_nccl;

bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { set_error(std::string("dlopen libnccl.so.2 failed: ") + dlerror()); return false; }
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.MemAlloc = (decltype(g_nccl.MemAlloc))dlsym(h, "ncclMemAlloc");
  g_nccl.MemFree = (decltype(g_nccl.MemFree))dlsym(h, "ncclMemFree");
  g_nccl.CommRegister = (decltype(g_nccl.CommRegister))dlsym(h, "ncclCommRegister");
  g_nccl.CommDeregister = (decltype(g_nccl.CommDeregister))dlsym(h, "ncclCommDeregister");
  g_nccl.CommGetAsyncError = (decltype(g_nccl.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
  g_nccl.CommAbort = (decltype(g_nccl.CommAbort))dlsym(h, "ncclCommAbort");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy;
  if (!g_nccl.ok) set_error("libnccl.so.2 lacks required symbols");
  return g_nccl.ok;
}

fbspca_status nccl_fail(ncclResult_t r, const char* where) {
  set_error(std::string(where) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
  return FBSPCA_ERR_NCCL;
}

// Errors NCCL raised asynchronously on a communicator (a peer died, a network failure): polled after every
// collective this library enqueues and by fbspca_comm_wait.
fbspca_status nccl_async_check(ncclComm_t comm, const char* where) {
  if (!g_nccl.CommGetAsyncError) return FBSPCA_OK;
  ncclResult_t st = ncclSuccess;
  ncclResult_t r = g_nccl.CommGetAsyncError(comm, &st);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
  if (st != ncclSuccess && st != ncclInProgress) return nccl_fail(st, where);
  return FBSPCA_OK;
}

// The plans' NCCL-visible partial buffers (SURVEY 8(e) Level 1): allocated with ncclMemAlloc and registered with
// the communicator on first use, so K5's chunk reduction writes straight into the buffer the in-place all-reduce
// reads (no staging copy).  Keyed by (plan, comm); released by fbspca_destroy or fbspca_comm_destroy, whichever
// comes first.
struct RegBuf { void* ptr = nullptr; void* handle = nullptr; size_t bytes = 0; };
std::mutex g_reg_mu;
std::map<std::pair<Plan*, void*>, RegBuf> g_reg;

void release_regbuf(std::pair<Plan*, void*> key, RegBuf& b) {
  if (b.handle && g_nccl.CommDeregister) g_nccl.CommDeregister((ncclComm_t)key.second, b.handle);
  if (b.ptr) { if (g_nccl.MemFree) g_nccl.MemFree(b.ptr); else cudaFree(b.ptr); }
  b = RegBuf{};
}

// Partial buffer for (plan, comm): registered if this NCCL supports it, else the plan's own buffer.
fbspca_status registered_partial(Plan& P, void* comm, double** out) {
  *out = P.d_partial;
  if (!comm || !g_nccl.MemAlloc || !g_nccl.CommRegister) return FBSPCA_OK;
  std::lock_guard<std::mutex> lk(g_reg_mu);
  RegBuf& b = g_reg[{&P, comm}];
  const size_t bytes = (size_t)(P.blk_off[P.k_max + 1] + P.p[0] + 1) * sizeof(double);
  if (!b.ptr) {
    ncclResult_t r = g_nccl.MemAlloc(&b.ptr, bytes);
    if (r != ncclSuccess) { b = RegBuf{}; return nccl_fail(r, "ncclMemAlloc"); }
    r = g_nccl.CommRegister((ncclComm_t)comm, b.ptr, bytes, &b.handle);
    if (r != ncclSuccess) { g_nccl.MemFree(b.ptr); b = RegBuf{}; return nccl_fail(r, "ncclCommRegister"); }
    b.bytes = bytes;
  }
  *out = static_cast<double*>(b.ptr);
  return FBSPCA_OK;
}

void release_plan_regbufs(Plan* P) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (auto it = g_reg.begin(); it != g_reg.end();) {
    if (it->first.first == P) { release_regbuf(it->first, it->second); it = g_reg.erase(it); }
    else ++it;
  }
}

void release_comm_regbufs(void* comm) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (auto it = g_reg.begin(); it != g_reg.end();) {
    if (it->first.second == comm) { release_regbuf(it->first, it->second); it = g_reg.erase(it); }
    else ++it;
  }
}

fbspca_status upload_plan(Plan& P) {
  DeviceGuard g(P.device);
  cudaDeviceProp prop;
  FB_CUDA(cudaGetDeviceProperties(&prop, P.device), "cudaGetDeviceProperties");
  if (prop.major < 10) { set_error("fbspca requires an sm_100 (Blackwell) device"); return FBSPCA_ERR_CONFIG; }
  P.num_sms = prop.multiProcessorCount;
  if (P.polar_smem > (int)prop.sharedMemPerBlockOptin) {
    set_error("polar kernel shared memory exceeds the device opt-in limit"); return FBSPCA_ERR_CONFIG;
  }
  P.polar_grid = P.num_sms;
  const bool f32 = P.dt == FBSPCA_F32;
  const size_t rsz = f32 ? 4 : 8, csz = 2 * rsz;
  const int nk = P.k_max + 1;
  const int64_t ncoef = P.coef_off[nk];
  if (f32) {
    auto tab = cast_vec<float>(P.table);
    // rings sampled at every s_j-th angle (plan.cpp): the angular quadrature weight 2 pi / (n_theta / s_j) is the
    // table's 2 pi / n_theta times s_j, a power of two -- folded in exactly here (K4's fp32 tables only)
    for (int64_t row = 0; row < ncoef; ++row)
      for (int j = 0; j < P.n_xi; ++j) tab[row * P.n_xi + j] *= float(P.ring_s[j]);
    FB_CUDA(upload(&P.d_table, tab.data(), tab.size()), "upload table");
    std::vector<float> hi(tab.size()), lo(tab.size());
    for (size_t i = 0; i < tab.size(); ++i) {          // tf32 round-to-nearest (ties away), as cvt.rna.tf32
      uint32_t b;
      std::memcpy(&b, &tab[i], 4);
      b = (b + 0x1000u) & ~0x1FFFu;
      std::memcpy(&hi[i], &b, 4);
      lo[i] = tab[i] - hi[i];
    }
    FB_CUDA(upload((void**)&P.d_table_hi, hi.data(), hi.size()), "upload table hi");
    FB_CUDA(upload((void**)&P.d_table_lo, lo.data(), lo.size()), "upload table lo");
    const char* k4 = getenv("FBSPCA_K4");
    P.use_tc = !(k4 && std::string(k4) == "simt");
    auto dp = cast_vec<float>(P.deapod);
    FB_CUDA(upload(&P.d_deapod, dp.data(), dp.size()), "upload deapod");
    auto tm = twiddles<float2, float>(P.M);
    FB_CUDA(upload(&P.d_tw_M, tm.data(), tm.size()), "upload twiddles");
    auto tt = twiddles<float2, float>(P.n_theta);
    FB_CUDA(upload(&P.d_tw_theta, tt.data(), tt.size()), "upload twiddles");
  } else {
    FB_CUDA(upload(&P.d_table, P.table.data(), P.table.size()), "upload table");
    FB_CUDA(upload(&P.d_deapod, P.deapod.data(), P.deapod.size()), "upload deapod");
    auto tm = twiddles<double2, double>(P.M);
    FB_CUDA(upload(&P.d_tw_M, tm.data(), tm.size()), "upload twiddles");
    auto tt = twiddles<double2, double>(P.n_theta);
    FB_CUDA(upload(&P.d_tw_theta, tt.data(), tt.size()), "upload twiddles");
  }
  FB_CUDA(upload((void**)&P.d_rbasis, P.rbasis.data(), P.rbasis.size()), "upload radial basis");
  FB_CUDA(upload((void**)&P.d_rho, P.rho.data(), P.rho.size()), "upload rho");
  FB_CUDA(upload((void**)&P.d_cs, P.cs.data(), P.cs.size()), "upload cs");
  FB_CUDA(upload((void**)&P.d_nodes, P.nodes.data(), P.nodes.size()), "upload nodes");
  FB_CUDA(upload((void**)&P.d_kj0, P.kj0.data(), P.kj0.size()), "upload kj0");
  FB_CUDA(upload((void**)&P.d_ring_s, P.ring_s.data(), P.ring_s.size()), "upload ring strides");
  FB_CUDA(upload((void**)&P.d_noderec, P.noderec.data(), P.noderec.size()), "upload node records");
  FB_CUDA(upload((void**)&P.d_dnoderec, P.dnoderec.data(), P.dnoderec.size()), "upload double node records");
  PolarParams& pp = P.pp;
  pp.xscratch_stride = (int64_t)P.L * pp.ncols_x;
  pp.pscratch_stride = (int64_t)P.n_xi * pp.half;
  pp.ghat_kstride = 2 * P.max_batch * (int64_t)P.n_xi;
  FB_CUDA(cudaStreamCreateWithFlags(&P.side, cudaStreamNonBlocking), "side stream");
  FB_CUDA(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming), "fork event");
  FB_CUDA(cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming), "join event");
  FB_CUDA(cudaMalloc(&P.d_xscratch, (size_t)P.polar_grid * pp.xscratch_stride * csz), "alloc xscratch");
  FB_CUDA(cudaMalloc(&P.d_pscratch, (size_t)P.polar_grid * pp.pscratch_stride * csz), "alloc pscratch");
  FB_CUDA(cudaMalloc(&P.d_ghat, (size_t)nk * P.max_batch * 2 * P.n_xi * rsz), "alloc ghat");
  const int64_t npart = P.blk_off[nk] + P.p[0] + 1;
  FB_CUDA(cudaMalloc((void**)&P.d_partial, npart * sizeof(double)), "alloc partial");
  FB_CUDA(cudaMalloc((void**)&P.d_cov_scratch, (size_t)kCovMaxChunks * npart * sizeof(double)), "alloc cov scratch");
  FB_CUDA(cudaMalloc((void**)&P.d_cov_scratch0, (size_t)kCovMaxSub0 * (P.blk_off[1] + P.p[0] + 1) * sizeof(double)),
          "alloc cov scratch0");
  FB_CUDA(upload((void**)&P.d_p, P.p.data(), P.p.size()), "upload p");
  FB_CUDA(upload((void**)&P.d_coef_off, P.coef_off.data(), P.coef_off.size()), "upload coef_off");
  FB_CUDA(upload((void**)&P.d_blk_off, P.blk_off.data(), P.blk_off.size()), "upload blk_off");
  FB_CUDA(upload((void**)&P.d_evec_off, P.evec_off.data(), P.evec_off.size()), "upload evec_off");
  FB_CUDA(cudaMalloc((void**)&P.d_eig_work, (size_t)2 * P.evec_off[nk] * sizeof(double) + 16), "alloc eig work");
  FB_CUDA(cudaMalloc((void**)&P.d_eig_sweeps, nk * sizeof(int)), "alloc eig sweeps");
  (void)ncoef;
  pp.deapod = P.d_deapod; pp.tw_M = P.d_tw_M; pp.tw_theta = P.d_tw_theta;
  pp.rho = P.d_rho; pp.cs = P.d_cs; pp.nodes = P.d_nodes; pp.kj0 = P.d_kj0; pp.ring_s = P.d_ring_s;
  pp.noderec = reinterpret_cast<const int4*>(P.d_noderec);
  pp.dnoderec = reinterpret_cast<const int4*>(P.d_dnoderec);
  pp.xscratch = P.d_xscratch; pp.pscratch = P.d_pscratch;
  FB_CUDA(upload((void**)&P.d_pp, &pp, 1), "upload polar params");
  return FBSPCA_OK;
}

void free_plan(Plan& P) {
  if (P.device < 0) return;
  DeviceGuard g(P.device);
  void* ptrs[] = {P.d_table, P.d_deapod, P.d_tw_M, P.d_tw_theta, P.d_rho, P.d_cs, P.d_nodes, P.d_xscratch,
                  P.d_pscratch, P.d_ghat, P.d_partial, P.d_p, P.d_coef_off, P.d_blk_off, P.d_evec_off,
                  P.d_eig_work, P.d_eig_sweeps, P.d_coef_k, P.d_pp, P.d_cov_scratch, P.d_cov_scratch0, P.d_table_hi, P.d_table_lo, P.d_rbasis,
                  P.d_synth_rho, P.d_synth_pidx, P.d_synth_pir, P.d_synth_pcs, P.d_synth_grp,
                  P.d_noderec, P.d_dnoderec, P.d_kj0, P.d_ring_s};
  for (void* p : ptrs) if (p) cudaFree(p);
  for (cudaEvent_t e : P.event_pool) cudaEventDestroy(e);
  P.event_pool.clear();
  P.tevents.clear();
  for (auto& g : P.graphs) if (g.exec) cudaGraphExecDestroy(g.exec);
  P.graphs.clear();
  if (P.ev_fork) cudaEventDestroy(P.ev_fork);
  if (P.ev_join) cudaEventDestroy(P.ev_join);
  if (P.side) cudaStreamDestroy(P.side);
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

fbspca_status check_compute_plan(fbspca_plan_t h) {
  if (!h) { set_error("null plan"); return FBSPCA_ERR_ARG; }
  if (reinterpret_cast<Plan*>(h)->device < 0) { set_error("host-only plan (device = -1) cannot compute"); return FBSPCA_ERR_ARG; }
  return FBSPCA_OK;
}

}  // namespace
}  // namespace fbspca

using namespace fbspca;

extern "C" {

struct fbspca_plan_s : public fbspca::Plan {};

const char* fbspca_last_error(void) { return g_err.c_str(); }
#ifndef FBSPCA_SRC_HASH
#define FBSPCA_SRC_HASH "unknown"
#endif
const char* fbspca_version(void) { return "fbspca-b200 0.2 (sm_100a) src " FBSPCA_SRC_HASH; }

fbspca_status fbspca_plan(int L, double c, double R, double eps, fbspca_dtype dt, int device, int64_t max_batch,
                          fbspca_plan_t* out) {
  if (!out) { set_error("out is null"); return FBSPCA_ERR_ARG; }
  *out = nullptr;
  if (dt != FBSPCA_F32 && dt != FBSPCA_F64) { set_error("bad dtype"); return FBSPCA_ERR_ARG; }
  auto* P = new fbspca_plan_s();
  P->L = L; P->c = c; P->R = R; P->dt = dt; P->device = device;
  P->eps = eps > 0 ? eps : (dt == FBSPCA_F32 ? 1e-5 : 1e-12);
  P->max_batch = max_batch > 0 ? max_batch : 4096;
  fbspca_status st = build_host_plan(*P);
  if (st == FBSPCA_OK && device >= 0) st = upload_plan(*P);
  if (st != FBSPCA_OK) { free_plan(*P); delete P; return st; }
  *out = P;
  return FBSPCA_OK;
}

fbspca_status fbspca_plan_info(fbspca_plan_t h, int* n_xi, int* n_theta, int* k_max, const int** p_k,
                               const int64_t** coef_off, const int64_t** blk_off, const int64_t** evec_off) {
  if (!h) { set_error("null plan"); return FBSPCA_ERR_ARG; }
  if (n_xi) *n_xi = h->n_xi;
  if (n_theta) *n_theta = h->n_theta;
  if (k_max) *k_max = h->k_max;
  if (p_k) *p_k = h->p.data();
  if (coef_off) *coef_off = h->coef_off.data();
  if (blk_off) *blk_off = h->blk_off.data();
  if (evec_off) *evec_off = h->evec_off.data();
  return FBSPCA_OK;
}

fbspca_status fbspca_plan_detail(fbspca_plan_t h, int* M, int* w, double* beta, int* n_phase, int* smem_bytes,
                                 const double** zeros, const double** xi, const double** wq) {
  if (!h) { set_error("null plan"); return FBSPCA_ERR_ARG; }
  if (M) *M = h->M;
  if (w) *w = h->w;
  if (beta) *beta = h->beta;
  if (n_phase) *n_phase = h->pp.n_phase;
  if (smem_bytes) *smem_bytes = h->polar_smem;
  if (zeros) *zeros = h->zeros.data();
  if (xi) *xi = h->xi.data();
  if (wq) *wq = h->wq.data();
  return FBSPCA_OK;
}

fbspca_status fbspca_plan_rings(fbspca_plan_t h, int* ring_stride, int* k_first_ring) {
  if (!h) { set_error("null plan"); return FBSPCA_ERR_ARG; }
  if (ring_stride) std::copy(h->ring_s.begin(), h->ring_s.end(), ring_stride);
  if (k_first_ring) std::copy(h->kj0.begin(), h->kj0.end(), k_first_ring);
  return FBSPCA_OK;
}

fbspca_status fbspca_expand(fbspca_plan_t h, const void* d_images, int64_t n, void* d_coeffs, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  const size_t rsz = P.dt == FBSPCA_F32 ? 4 : 8;
  if (!d_images || !d_coeffs || n < 1) { set_error("expand: null pointer or n < 1"); return FBSPCA_ERR_ARG; }
  if (!aligned(d_images, rsz) || !aligned(d_coeffs, 2 * rsz)) { set_error("expand: misaligned pointer"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t img_elems = (int64_t)P.L * P.L;
  for (int64_t b0 = 0; b0 < n; b0 += P.max_batch) {
    const int64_t nb = std::min<int64_t>(P.max_batch, n - b0);
    const char* imgs = (const char*)d_images + b0 * img_elems * rsz;
    {
      TimedRegion t(P, T_POLAR, s);
      FB_CUDA(launch_polar(P, imgs, nb, img_elems, s), "polar kernel");
    }
    {
      TimedRegion t(P, T_RADIAL, s);
      // tensor-core K4 takes p_0 <= 256 (its B tiles); larger bases (c R > ~80) run the SIMT kernel
      if (P.dt == FBSPCA_F32 && P.use_tc && P.n_xi % 4 == 0 && ((P.p[0] + 15) & ~15) <= 256)
        FB_CUDA(launch_radial_tma(P, nb, b0, n, d_coeffs, s), "radial tma kernel");
      else FB_CUDA(launch_radial(P, nb, b0, n, d_coeffs, s), "radial kernel");
    }
  }
  return FBSPCA_OK;
}

static fbspca_status cov_accumulate(fbspca_plan_t h, const void* d_coeffs, int64_t n_local, double* d_partial,
                                    fbspca_stream_t stream, bool zero) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_coeffs || !d_partial || n_local < 1) { set_error("covariance: null pointer or n_local < 1"); return FBSPCA_ERR_ARG; }
  const size_t rsz = P.dt == FBSPCA_F32 ? 4 : 8;
  if (!aligned(d_coeffs, 2 * rsz) || !aligned(d_partial, 8)) { set_error("covariance: misaligned pointer"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npart = P.blk_off[P.k_max + 1] + P.p[0] + 1;
  if (zero) FB_CUDA(cudaMemsetAsync(d_partial, 0, npart * sizeof(double), s), "memset partial");
  // images per launch: 16 split-K chunks (tensor path: 16 x 4096 = kCovBatchTc by default)
  const int64_t B = cov_uses_tc(P, n_local) ? int64_t(cov_tma_chunk()) * kCovMaxChunks : kCovBatch;
  TimedRegion t(P, T_COV, s);
  for (int64_t i0 = 0; i0 < n_local; i0 += B) {
    const int64_t nb = std::min<int64_t>(B, n_local - i0);
    FB_CUDA(launch_cov_accum(P, d_coeffs, n_local, i0, nb, d_partial, s), "cov kernel");
  }
  return FBSPCA_OK;
}

fbspca_status fbspca_covariance_partial(fbspca_plan_t h, const void* d_coeffs, int64_t n_local, double* d_partial,
                                        fbspca_stream_t stream) {
  return cov_accumulate(h, d_coeffs, n_local, d_partial, stream, true);
}

fbspca_status fbspca_covariance_accumulate(fbspca_plan_t h, const void* d_coeffs, int64_t n_local, double* d_partial,
                                           fbspca_stream_t stream) {
  return cov_accumulate(h, d_coeffs, n_local, d_partial, stream, false);
}

fbspca_status fbspca_allreduce_partial(fbspca_plan_t h, double* d_partial, void* nccl_comm, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  if (!d_partial) { set_error("allreduce: null pointer"); return FBSPCA_ERR_ARG; }
  if (!nccl_comm) return FBSPCA_OK;
  Plan& P = *h;
  if (!nccl_load()) return FBSPCA_ERR_NCCL;
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npart = P.blk_off[P.k_max + 1] + P.p[0] + 1;
  {
    TimedRegion t(P, T_ALLREDUCE, s);
    ncclResult_t r = g_nccl.AllReduce(d_partial, d_partial, (size_t)npart, ncclFloat64, ncclSum, (ncclComm_t)nccl_comm, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  }
  return nccl_async_check((ncclComm_t)nccl_comm, "ncclAllReduce (async)");
}

fbspca_status fbspca_covariance_finalize(fbspca_plan_t h, const double* d_partial, double* d_blocks, double* d_mean,
                                         fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_partial || !d_blocks || !d_mean) { set_error("finalize: null pointer"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  TimedRegion t(P, T_FINALIZE, s);
  FB_CUDA(launch_cov_finalize(P, d_partial, d_blocks, d_mean, s), "finalize kernel");
  return FBSPCA_OK;
}

fbspca_status fbspca_covariance(fbspca_plan_t h, const void* d_coeffs, int64_t n_local, int64_t n_total,
                                void* nccl_comm, double* d_blocks, double* d_mean, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (n_total < n_local) { set_error("n_total < n_local"); return FBSPCA_ERR_ARG; }
  if (!nccl_comm && n_total != n_local) { set_error("n_total != n_local without a communicator"); return FBSPCA_ERR_ARG; }
  double* part = P.d_partial;
  if (nccl_comm) {
    if (!nccl_load()) return FBSPCA_ERR_NCCL;
    DeviceGuard g(P.device);
    st = registered_partial(P, nccl_comm, &part);       // K5 writes straight into the all-reduce buffer
    if (st != FBSPCA_OK) return st;
  }
  st = fbspca_covariance_partial(h, d_coeffs, n_local, part, stream);
  if (st != FBSPCA_OK) return st;
  st = fbspca_allreduce_partial(h, part, nccl_comm, stream);
  if (st != FBSPCA_OK) return st;
  return fbspca_covariance_finalize(h, part, d_blocks, d_mean, stream);
}

fbspca_status fbspca_step(fbspca_plan_t h, const void* d_images, int64_t n_local, int64_t n_total, void* nccl_comm,
                          void* d_coeffs, double* d_blocks, double* d_mean, int use_graph, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  cudaStream_t s = (cudaStream_t)stream;
  auto eager = [&]() -> fbspca_status {
    fbspca_status r = fbspca_expand(h, d_images, n_local, d_coeffs, stream);
    if (r != FBSPCA_OK) return r;
    return fbspca_covariance(h, d_coeffs, n_local, n_total, nccl_comm, d_blocks, d_mean, stream);
  };
  if (!use_graph) return eager();
  if (!s) { set_error("step: graph capture needs a non-default stream"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  Plan::GraphEntry* ge = nullptr;
  for (auto& e : P.graphs)
    if (e.images == d_images && e.n_local == n_local && e.n_total == n_total && e.comm == nccl_comm &&
        e.coeffs == d_coeffs && e.blocks == d_blocks && e.mean == d_mean && e.stream == s) { ge = &e; break; }
  if (!ge) {
    P.graphs.push_back({d_images, n_local, n_total, nccl_comm, d_coeffs, d_blocks, d_mean, s, 0, nullptr});
    ge = &P.graphs.back();
  }
  if (ge->uses++ == 0) return eager();       // first call: eager (kernel attributes, NCCL registration happen here)
  if (!ge->exec) {                           // second call: capture the same launches into one graph
    FB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed), "begin capture");
    fbspca_status r = eager();
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (r != FBSPCA_OK) { if (graph) cudaGraphDestroy(graph); return r; }
    if (ce != cudaSuccess) return cuda_fail(ce, "end capture");
    ce = cudaGraphInstantiate(&ge->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) { ge->exec = nullptr; return cuda_fail(ce, "graph instantiate"); }
  }
  FB_CUDA(cudaGraphLaunch(ge->exec, s), "graph launch");
  if (nccl_comm) return nccl_async_check((ncclComm_t)nccl_comm, "graph all-reduce (async)");
  return FBSPCA_OK;
}

fbspca_status fbspca_eig(fbspca_plan_t h, const double* d_blocks, double* d_evals, double* d_evecs,
                         fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_blocks || !d_evals || !d_evecs) { set_error("eig: null pointer"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  {
    TimedRegion t(P, T_EIG, s);
    FB_CUDA(launch_eig(P, d_blocks, d_evals, d_evecs, s), "eig kernel");
  }
  std::vector<int> sweeps(P.k_max + 1);
  FB_CUDA(cudaMemcpyAsync(sweeps.data(), P.d_eig_sweeps, sweeps.size() * sizeof(int), cudaMemcpyDeviceToHost, s),
          "eig sweeps");
  FB_CUDA(cudaStreamSynchronize(s), "eig sync");
  for (int k = 0; k <= P.k_max; ++k)
    if (sweeps[k] >= 30) {
      set_error("Jacobi did not converge within 30 sweeps for block k = " + std::to_string(k));
      return FBSPCA_ERR_NUMERIC;
    }
  return FBSPCA_OK;
}

fbspca_status fbspca_svd(fbspca_plan_t h, const void* d_coeffs, int64_t n, double* d_mean, double* d_evals,
                         double* d_evecs, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_coeffs || !d_evals || !d_evecs || n < 1) { set_error("svd: bad argument"); return FBSPCA_ERR_ARG; }
  if (!aligned(d_coeffs, P.dt == FBSPCA_F32 ? 8 : 16) || !aligned(d_evals, 8) || !aligned(d_evecs, 8) ||
      (d_mean && !aligned(d_mean, 8))) { set_error("svd: misaligned pointer"); return FBSPCA_ERR_ARG; }
  if (P.p[0] > kSvdMaxP) { set_error("svd: p_0 above the kernel's bound"); return FBSPCA_ERR_CONFIG; }
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ncoef = P.coef_off[P.k_max + 1];
  const size_t bytes = (size_t)(2 * n * ncoef + P.evec_off[P.k_max + 1]) * sizeof(double);
  double* work = nullptr;
  FB_CUDA(cudaMallocAsync(&work, bytes, s), "svd workspace");
  cudaError_t e;
  {
    TimedRegion t(P, T_EIG, s);
    e = launch_svd(P, d_coeffs, n, work, d_mean, d_evals, d_evecs, s);
  }
  cudaFreeAsync(work, s);
  FB_CUDA(e, "svd kernel");
  std::vector<int> sweeps(P.k_max + 1);
  FB_CUDA(cudaMemcpyAsync(sweeps.data(), P.d_eig_sweeps, sweeps.size() * sizeof(int), cudaMemcpyDeviceToHost, s),
          "svd sweeps");
  FB_CUDA(cudaStreamSynchronize(s), "svd sync");
  for (int k = 0; k <= P.k_max; ++k)
    if (sweeps[k] >= kSvdMaxSweeps) {
      set_error("one-sided Jacobi did not converge within " + std::to_string(kSvdMaxSweeps) + " sweeps for block k = " +
                std::to_string(k));
      return FBSPCA_ERR_NUMERIC;
    }
  return FBSPCA_OK;
}

fbspca_status fbspca_radial_eigenfunctions(fbspca_plan_t h, const double* d_evecs, double* d_f,
                                           fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_evecs || !d_f) { set_error("radial_eigenfunctions: null pointer"); return FBSPCA_ERR_ARG; }
  if (!aligned(d_evecs, 8) || !aligned(d_f, 8)) { set_error("radial_eigenfunctions: misaligned pointer"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  FB_CUDA(launch_radial_eigfun(P, d_evecs, d_f, (cudaStream_t)stream), "radial eigenfunction kernel");
  return FBSPCA_OK;
}

fbspca_status fbspca_synthesize(fbspca_plan_t h, const void* d_coeffs, int64_t n, void* d_images,
                                fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  const size_t rsz = P.dt == FBSPCA_F32 ? 4 : 8;
  if (!d_coeffs || !d_images || n < 1) { set_error("synthesize: null pointer or n < 1"); return FBSPCA_ERR_ARG; }
  if (!aligned(d_coeffs, 2 * rsz) || !aligned(d_images, rsz)) { set_error("synthesize: misaligned pointer"); return FBSPCA_ERR_ARG; }
  if (n > 65535) { set_error("synthesize: n > 65535 per call"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  FB_CUDA(launch_synthesize(P, d_coeffs, n, d_images, (cudaStream_t)stream), "synthesis kernel");
  return FBSPCA_OK;
}

fbspca_status fbspca_backproject(fbspca_plan_t h, const void* d_c, int64_t n, const double* d_mean,
                                 const double* d_evecs, void* d_coeffs_out, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_c || !d_mean || !d_evecs || !d_coeffs_out || n < 1) { set_error("backproject: bad argument"); return FBSPCA_ERR_ARG; }
  if (d_c == d_coeffs_out) { set_error("backproject: output aliases input"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  FB_CUDA(launch_backproject(P, d_c, n, d_mean, d_evecs, d_coeffs_out, (cudaStream_t)stream), "backproject kernel");
  return FBSPCA_OK;
}

fbspca_status fbspca_project(fbspca_plan_t h, const void* d_coeffs, int64_t n, const double* d_mean,
                             const double* d_evals, const double* d_evecs, double sigma2, int mode, int64_t n_total,
                             void* d_out, fbspca_stream_t stream) {
  fbspca_status st = check_compute_plan(h);
  if (st != FBSPCA_OK) return st;
  Plan& P = *h;
  if (!d_coeffs || !d_mean || !d_evals || !d_evecs || !d_out || n < 1) { set_error("project: bad argument"); return FBSPCA_ERR_ARG; }
  if (mode < 0 || mode > 2 || n_total < 1 || !(sigma2 >= 0)) { set_error("project: bad mode/sigma2/n_total"); return FBSPCA_ERR_ARG; }
  if (d_out == d_coeffs) { set_error("project: d_out aliases d_coeffs"); return FBSPCA_ERR_ARG; }
  DeviceGuard g(P.device);
  cudaStream_t s = (cudaStream_t)stream;
  TimedRegion t(P, T_PROJECT, s);
  FB_CUDA(launch_project(P, d_coeffs, n, d_mean, d_evals, d_evecs, sigma2, mode, n_total, d_out, s), "project kernel");
  return FBSPCA_OK;
}

fbspca_status fbspca_estimate_params(int L, fbspca_dtype dt, int device, const void* d_images, int64_t n,
                                     double fraction, double* sigma2, double* R, double* c) {
  if (!d_images || !sigma2 || !R || !c) { set_error("estimate_params: null pointer"); return FBSPCA_ERR_ARG; }
  if (L < 16 || n < 2 || !(fraction > 0 && fraction <= 1) || (dt != FBSPCA_F32 && dt != FBSPCA_F64)) {
    set_error("estimate_params: need L >= 16, n >= 2, 0 < fraction <= 1"); return FBSPCA_ERR_ARG;
  }
  DeviceGuard g(device);
  double out[3];
  fbspca_status st = estimate_params(L, dt, device, d_images, n, fraction, out);
  *sigma2 = out[0]; *R = out[1]; *c = out[2];
  return st;
}

fbspca_status fbspca_nccl_unique_id(void* out) {
  if (!out) { set_error("null out"); return FBSPCA_ERR_ARG; }
  if (!nccl_load()) return FBSPCA_ERR_NCCL;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return FBSPCA_OK;
}

fbspca_status fbspca_comm_init(const void* uid, int nranks, int rank, void** comm_out) {
  if (!uid || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("comm_init: bad argument"); return FBSPCA_ERR_ARG; }
  if (!nccl_load()) return FBSPCA_ERR_NCCL;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm;
  ncclResult_t r = g_nccl.CommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm_out = comm;
  return FBSPCA_OK;
}

fbspca_status fbspca_comm_wait(void* comm, fbspca_stream_t stream, double timeout_s) {
  if (!comm) { set_error("comm_wait: null communicator"); return FBSPCA_ERR_ARG; }
  if (!nccl_load()) return FBSPCA_ERR_NCCL;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    fbspca_status st = nccl_async_check((ncclComm_t)comm, "NCCL (async)");
    if (st != FBSPCA_OK) {
      if (g_nccl.CommAbort) g_nccl.CommAbort((ncclComm_t)comm);
      return st;
    }
    cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
    if (q == cudaSuccess) return FBSPCA_OK;
    if (q != cudaErrorNotReady) return cuda_fail(q, "comm_wait: stream");
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s > 0 && el > timeout_s) {
      if (g_nccl.CommAbort) g_nccl.CommAbort((ncclComm_t)comm);
      set_error("comm_wait: stream not done after " + std::to_string(timeout_s) + " s; communicator aborted");
      return FBSPCA_ERR_NCCL;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
}

fbspca_status fbspca_comm_destroy(void* comm) {
  if (!comm) return FBSPCA_OK;
  if (!nccl_load()) return FBSPCA_ERR_NCCL;
  release_comm_regbufs(comm);
  ncclResult_t r = g_nccl.CommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return FBSPCA_OK;
}

fbspca_status fbspca_set_timing(fbspca_plan_t h, int enabled) {
  if (!h) { set_error("null plan"); return FBSPCA_ERR_ARG; }
  h->timing = enabled != 0;
  return FBSPCA_OK;
}

fbspca_status fbspca_get_timing(fbspca_plan_t h, int* count, const char* const** names, const float** ms) {
  if (!h) { set_error("null plan"); return FBSPCA_ERR_ARG; }
  Plan& P = *h;
  P.tms.assign(2 * T_NKINDS, 0.f);
  for (auto& ev : P.tevents) {
    float t = 0;
    cudaEventSynchronize(ev.second.second);
    cudaEventElapsedTime(&t, ev.second.first, ev.second.second);
    P.tms[ev.first] += t;
    P.tms[T_NKINDS + ev.first] += 1.f;
  }
  P.tevents.clear();
  P.tname_ptrs.assign(kTimingNames, kTimingNames + T_NKINDS);
  if (count) *count = T_NKINDS;
  if (names) *names = P.tname_ptrs.data();
  if (ms) *ms = P.tms.data();        // ms[0..N) totals, ms[N..2N) launch-region counts
  return FBSPCA_OK;
}

void fbspca_destroy(fbspca_plan_t h) {
  if (!h) return;
  release_plan_regbufs(h);
  free_plan(*h);
  delete h;
}

}  // extern "C"
