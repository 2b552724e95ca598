// kernels_tc.cu -- K4 radial quadrature (Eq. (a)) on the sm_100a tensor cores.
//
// Per angular frequency k the quadrature is a dense contraction
//     D[row][q] = sum_j ghat[k][row][j] * T_k[q][j],   row = 2 b + (re|im), j < n_xi, q < p_k,
// issued as tcgen05.mma.cta_group::1.kind::tf32 with M = 128 rows, N = p_k rounded up to 16, K = n_xi in
// chunks of 32.  Precision (3xTF32): ghat = a_hi + a_lo and T = t_hi + t_lo with *_hi = tf32(rna) and
// *_lo = x - x_hi (exact in fp32); D = a_hi t_hi + a_hi t_lo + a_lo t_hi accumulates in fp32 in TMEM
// (relative error ~2^-21, far below the 1e-4 coefficient tolerance; single TF32 would give ~5e-4).
// The table split is done once on the host; ghat is split while it is staged into shared memory.
//
// Shared-memory operand layout: canonical K-major SWIZZLE_NONE ("interleave") -- core matrices of
// 8 rows x 16 bytes stored contiguously; SBO = 128 B between 8-row groups, LBO = (rows/8) * 128 B
// between the two 16-byte K halves of one MMA.  One elected thread issues the MMAs and commits them to
// an mbarrier per stage; the 128 threads load / split the next chunk meanwhile (2-stage pipeline).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace fbspca {

namespace {

constexpr int TC_M = 128;     // rows per CTA (64 images x re/im)
constexpr int TC_KC = 32;     // K elements per pipeline chunk of the covariance kernel (4 MMAs of K = 8)
constexpr int RK_KC = 16;     // K elements per pipeline chunk of the radial kernel (2 MMAs; 48 KB smem -> 4 CTAs/SM)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;                       // descriptor version (sm_100)
  return d;                                     // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// byte offset of element (row, kk) (kk < 32) inside a K-major interleaved tile of `rows` rows
__device__ __forceinline__ uint32_t il_off(int row, int c16, int rows) {
  return uint32_t(c16) * uint32_t(rows / 8) * 128u + uint32_t(row >> 3) * 128u + uint32_t(row & 7) * 16u;
}

}  // namespace

__global__ void __launch_bounds__(128, 1)
radial_tc_kernel(const float* __restrict__ ghat, const float* __restrict__ t_hi, const float* __restrict__ t_lo,
                 const int* __restrict__ p, const int64_t* __restrict__ coef_off, int nb, int n_xi, int64_t i0,
                 int64_t ld, int tmem_cols, float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int k = blockIdx.y;
  const int pk = p[k];
  const int N = (pk + 15) & ~15;                 // MMA N (multiple of 16 for M = 128)
  const int rows = 2 * nb;
  const int r0 = blockIdx.x * TC_M;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NMAX = tmem_cols;                    // B tiles sized for the largest N of the plan
  const uint32_t a_bytes = TC_M * RK_KC * 4, b_bytes = uint32_t(NMAX) * RK_KC * 4;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = *tmem_slot;

  const float* A = ghat + (int64_t)k * rows * n_xi;
  const float* Bh = t_hi + coef_off[k] * n_xi;
  const float* Bl = t_lo + coef_off[k] * n_xi;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(TC_M >> 4) << 24);
  const int nchunks = (n_xi + RK_KC - 1) / RK_KC;

  // A chunk: 128 rows x 16 fp32 -> hi / lo tiles.  Item idx = tid + 128 u (u < 4): a warp covers 8
  // consecutive rows x 4 sixteen-byte chunks, so each 8-lane group stores one contiguous 128-B core-matrix
  // row block (conflict-free) and each row is read as one 64-B run.  Chunk c+1 is loaded into registers
  // before chunk c is split and stored (two chunks of loads in flight per thread).
  auto load_a = [&](int cc, float4* dst) {
    const int jb = cc * RK_KC;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 128 * u, w = idx >> 5, ln = idx & 31;
      const int row = w * 8 + (ln & 7), c16 = ln >> 3;
      const int r = r0 + row, j = jb + 4 * c16;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < rows && cc < nchunks) {
        const float* src = A + (int64_t)r * n_xi + j;
        if (j + 3 < n_xi) v = __ldg(reinterpret_cast<const float4*>(src));
        else {
          if (j < n_xi) v.x = src[0];
          if (j + 1 < n_xi) v.y = src[1];
          if (j + 2 < n_xi) v.z = src[2];
        }
      }
      dst[u] = v;
    }
  };
  float4 va[4], vn[4];
  load_a(0, va);
  for (int c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    unsigned char* st = sm + s * stage_bytes;
    const int j0 = c * RK_KC;
    load_a(c + 1, vn);                                        // prefetch the next chunk
    if (c >= 2) mbar_wait(&bars[s], ((c - 2) >> 1) & 1);     // MMAs of chunk c-2 released this stage
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 128 * u, w = idx >> 5, ln = idx & 31;
      const int row = w * 8 + (ln & 7), c16 = ln >> 3;
      const float4 v = va[u];
      const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
      const float4 lo = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      const uint32_t off = il_off(row, c16, TC_M);
      *reinterpret_cast<float4*>(st + off) = h;
      *reinterpret_cast<float4*>(st + a_bytes + off) = lo;
    }
    // B chunk: N rows (q) x 16 (pre-split on the host)
    for (int idx = tid; idx < N * 4; idx += 128) {
      const int w = idx >> 5, ln = idx & 31;         // same conflict-free mapping: 8 rows x 4 chunks per warp
      const int q = w * 8 + (ln & 7), c16 = ln >> 3;
      const int j = j0 + 4 * c16;
      float4 h = make_float4(0.f, 0.f, 0.f, 0.f), lo = h;
      if (q < pk) {
        const float* sh = Bh + (int64_t)q * n_xi + j;
        const float* sl = Bl + (int64_t)q * n_xi + j;
        if (j + 3 < n_xi) {
          h = *reinterpret_cast<const float4*>(sh);
          lo = *reinterpret_cast<const float4*>(sl);
        } else {
          if (j < n_xi) { h.x = sh[0]; lo.x = sl[0]; }
          if (j + 1 < n_xi) { h.y = sh[1]; lo.y = sl[1]; }
          if (j + 2 < n_xi) { h.z = sh[2]; lo.z = sl[2]; }
        }
      }
      const uint32_t off = il_off(q, c16, N);
      *reinterpret_cast<float4*>(st + 2 * a_bytes + off) = h;
      *reinterpret_cast<float4*>(st + 2 * a_bytes + b_bytes + off) = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t base = smem_u32(st);
        const uint32_t lbo_a = (TC_M / 8) * 128, lbo_b = uint32_t(N / 8) * 128;
#pragma unroll
        for (int s4 = 0; s4 < RK_KC / 8; ++s4) {
          const uint32_t ko_a = uint32_t(2 * s4) * lbo_a, ko_b = uint32_t(2 * s4) * lbo_b;
          const uint64_t ah = make_desc(base + ko_a, lbo_a, 128);
          const uint64_t al = make_desc(base + a_bytes + ko_a, lbo_a, 128);
          const uint64_t bh = make_desc(base + 2 * a_bytes + ko_b, lbo_b, 128);
          const uint64_t bl = make_desc(base + 2 * a_bytes + b_bytes + ko_b, lbo_b, 128);
          mma_tf32(tmem_d, ah, bh, idesc, (c | s4) ? 1u : 0u);
          mma_tf32(tmem_d, ah, bl, idesc, 1u);
          mma_tf32(tmem_d, al, bh, idesc, 1u);
        }
        mma_commit(&bars[s]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) va[u] = vn[u];
  }
  // the last commit tracks every MMA issued before it
  mbar_wait(&bars[(nchunks - 1) & 1], ((nchunks - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w owns TMEM lanes 32w..32w+31 = rows r0 + 32w + lane
  const int row = r0 + 32 * warp + lane;
  const int64_t base = coef_off[k];
  for (int q0 = 0; q0 < N; q0 += 16) {
    float v[16];
    tmem_ld16(tmem_d + (uint32_t(32 * warp) << 16) + uint32_t(q0), v);
    if (row < rows) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int q = q0 + i;
        if (q < pk) out[(base + q) * 2 * ld + 2 * i0 + row] = (k == 0 && (row & 1)) ? 0.f : v[i];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(tmem_cols));
}

int radial_tc_smem(int nmax) {
  const int a_bytes = TC_M * RK_KC * 4, b_bytes = nmax * RK_KC * 4;
  return 2 * (2 * a_bytes + 2 * b_bytes) + 64;
}

int radial_tc_cols(int pmax) {
  const int n = (pmax + 15) & ~15;
  int c = 32;
  while (c < n) c <<= 1;
  return c;
}

cudaError_t launch_radial_tc(const Plan& P, int64_t nb, int64_t i0, int64_t ld, void* d_coeffs, cudaStream_t s) {
  const int cols = radial_tc_cols(P.p[0]);
  const int smem = radial_tc_smem(cols);
  static int configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(radial_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid((unsigned)((2 * nb + TC_M - 1) / TC_M), (unsigned)(P.k_max + 1));
  radial_tc_kernel<<<grid, 128, smem, s>>>((const float*)P.d_ghat, P.d_table_hi, P.d_table_lo,
                                          P.d_p, P.d_coef_off, (int)nb, P.n_xi, i0, ld, cols, (float*)d_coeffs);
  return cudaGetLastError();
}

}  // namespace fbspca

// ---------------------------------------------------------------- K5 on tcgen05 (Eqs. (ck), (ck_0))
// CTA (k, chunk): S = A A^T over the chunk's kCovChunk images (2 kCovChunk real columns, re/im interleaved),
// A = block k (p_k rows x columns, K-major).  Both MMA operands come from the same shared tile (rows padded
// to R = roundup16(p_k) <= 256; M = 128 per tile, two M-tiles when R > 128).  3xTF32 products accumulate in
// fp32 in TMEM over the chunk; the upper triangle is stored as fp64 into scratch[chunk] (the fixed-order
// reduction over chunks is cov_reduce_kernel).  k = 0 also accumulates s_0 = sum_i a_{0,i} in fp64.
namespace fbspca {

__global__ void __launch_bounds__(128, 1)
cov_tc_kernel(const float* __restrict__ coeffs, const int* __restrict__ p, const int64_t* __restrict__ coef_off,
              const int64_t* __restrict__ blk_off, int64_t ld, int64_t i0, int64_t nb, int k_max, int tmem_cols,
              int tile_rows, double* __restrict__ scratch, int64_t scratch_stride) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int k = blockIdx.x + 1;                                  // k = 0 runs on the fp64 SIMT path (F9)
  const int pk = p[k];
  const int R = (pk + 15) & ~15;
  const int nmt = R > 128 ? 2 : 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t img0 = i0 + (int64_t)blockIdx.y * kCovChunk;
  const int64_t cnb = min((int64_t)kCovChunk, i0 + nb - img0);
  const int ncols = int(2 * cnb);
  const uint32_t tile_bytes = uint32_t(tile_rows) * TC_KC * 4;  // sized for the largest R of k >= 1
  const uint32_t stage_bytes = 2 * tile_bytes;                   // hi + lo
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = *tmem_slot;
  const float* A = coeffs + coef_off[k] * 2 * ld + 2 * img0;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(R >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  const int nchunks = (ncols + TC_KC - 1) / TC_KC;
  const uint32_t lbo = uint32_t(tile_rows / 8) * 128;           // tile laid out with tile_rows >= 128 rows

  for (int c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    unsigned char* st = sm + s * stage_bytes;
    if (c >= 2) mbar_wait(&bars[s], ((c - 2) >> 1) & 1);
    const int j0 = c * TC_KC;
    const int items = R * 8;
    for (int idx = tid; idx < items; idx += 128) {
      const int w = idx >> 5, ln = idx & 31;
      const int row = (w >> 1) * 8 + (ln & 7), c16 = (w & 1) * 4 + (ln >> 3);
      const int j = j0 + 4 * c16;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < pk) {
        const float* src = A + (int64_t)row * 2 * ld + j;
        if (j + 3 < ncols) v = __ldg(reinterpret_cast<const float4*>(src));
        else {
          if (j < ncols) v.x = src[0];
          if (j + 1 < ncols) v.y = src[1];
          if (j + 2 < ncols) v.z = src[2];
        }
      }
      const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
      const float4 lo = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      const uint32_t off = il_off(row, c16, tile_rows);
      *reinterpret_cast<float4*>(st + off) = h;
      *reinterpret_cast<float4*>(st + tile_bytes + off) = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t base = smem_u32(st);
#pragma unroll
        for (int s4 = 0; s4 < TC_KC / 8; ++s4) {
          const uint32_t ko = uint32_t(2 * s4) * lbo;
          const uint64_t bh = make_desc(base + ko, lbo, 128);
          const uint64_t bl = make_desc(base + tile_bytes + ko, lbo, 128);
          for (int mt = 0; mt < nmt; ++mt) {
            const uint32_t mo = uint32_t(mt) * 16u * 128u;          // 128 rows further
            const uint64_t ah = make_desc(base + ko + mo, lbo, 128);
            const uint64_t al = make_desc(base + tile_bytes + ko + mo, lbo, 128);
            const uint32_t d = tmem_d + uint32_t(mt * 256);
            mma_tf32(d, ah, bh, idesc, (c | s4) ? 1u : 0u);
            mma_tf32(d, ah, bl, idesc, 1u);
            mma_tf32(d, al, bh, idesc, 1u);
          }
        }
        mma_commit(&bars[s]);
      }
      __syncwarp();
    }
  }
  mbar_wait(&bars[(nchunks - 1) & 1], ((nchunks - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  double* dst = scratch + (int64_t)blockIdx.y * scratch_stride + blk_off[k];
  for (int mt = 0; mt < nmt; ++mt) {
    const int q = mt * 128 + 32 * warp + lane;
    for (int q0 = 0; q0 < R; q0 += 16) {
      float v[16];
      tmem_ld16(tmem_d + uint32_t(mt * 256) + (uint32_t(32 * warp) << 16) + uint32_t(q0), v);
      if (q < pk) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int qq = q0 + i;
          if (qq >= q && qq < pk) dst[(int64_t)q * pk - (int64_t)q * (q - 1) / 2 + (qq - q)] = double(v[i]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(tmem_cols));
}

cudaError_t launch_cov_tc(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb, cudaStream_t s) {
  if (P.k_max < 1) return cudaSuccess;
  const int R = (P.p[1] + 15) & ~15;                  // largest p_k over k >= 1
  if (R > 256) return cudaErrorInvalidValue;
  const int cols = R > 128 ? 512 : radial_tc_cols(P.p[1]);
  const int TR = R > 128 ? 256 : 128;                  // the M = 128 A operand reads 128 rows
  const int smem = 2 * (2 * TR * TC_KC * 4) + 64;
  static int configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(cov_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int nchunk = (int)((nb + kCovChunk - 1) / kCovChunk);
  const int64_t total = P.blk_off[P.k_max + 1] + P.p[0] + 1;
  dim3 grid((unsigned)P.k_max, (unsigned)nchunk);
  cov_tc_kernel<<<grid, 128, smem, s>>>((const float*)d_coeffs, P.d_p, P.d_coef_off, P.d_blk_off, ld, i0, nb, P.k_max,
                                        cols, TR, P.d_cov_scratch, total);
  return cudaGetLastError();
}

}  // namespace fbspca
