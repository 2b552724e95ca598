// kernels_tma.cu -- the two dense contractions of the path on the sm_100a tensor cores, fed by TMA:
//
//   K4 radial quadrature, Eq. (a):  D[row][q] = sum_j ghat[k][row][j] T_k[q][j]      (row = 2 b + re|im)
//   K5 covariance, Eqs. (ck):   S_k[q][q'] = sum_c A_k[q][c] A_k[q'][c]           (k >= 1; c = re|im
//                                                                                               columns of images)
// Both are persistent, warp-specialised kernels (160 + 32 threads): warp 4 issues TMA loads (cp.async.bulk.tensor,
// 128-B swizzle, K-major) of 32-wide K chunks into an NS-stage ring; warps 0-3 write each chunk's 3xTF32 low
// part into the same stage and drain TMEM; warp 5 issues tcgen05.mma.kind::tf32 into one of two TMEM
// accumulators (so the drain of one overlaps the MMAs of the next).
//
// Measured on B200 (tools/micro/mma_latency.cu): a kind::tf32 MMA with M = 128 costs max(64, N/2) cycles,
// i.e. the instruction count, not N, is the cost below N = 128.  So the operands are concatenated along N:
//   K4: B = [T_hi ; T_lo] (N = 2 b):   D = x_raw [T_hi;T_lo]^T + x_lo [T_hi;T_lo]^T   -> 2 MMAs per K step
//   K5: B = [x_raw ; x_lo] (N = 2 b):  D = x_raw [x_raw;x_lo]^T,  S = D_11 + D_12 + D_12^T   -> 1 MMA per K step
//
// Precision (3xTF32): kind::tf32 reads only the top 19 bits of an fp32 operand (measured: truncation,
// tools/micro/tf32_trunc.cu), so the raw fp32 tile IS the high part hi = trunc19(x) and only lo = x - hi
// (exact in fp32, |lo| < 2^-10 |x|) is materialised, elementwise in the same swizzled layout.
//   D = x_raw y_hi + x_raw y_lo + x_lo y_hi  (y = table, pre-split on the host, K4)
//   S = x_raw x_raw + x_raw x_lo + x_lo x_raw  (K5)
// dropped terms are ~2^-20 relative; accumulation is fp32 in TMEM.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace fbspca {
namespace {

constexpr int KC = 32;                       // fp32 elements per K chunk = one 128-B swizzle row
constexpr int ROWB = KC * 4;                 // 128 bytes

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major SWIZZLE_128B UMMA shared-memory descriptor: 8-row atoms of 128-B rows, atoms 1024 B apart (SBO).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;                    // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;            // SBO
  d |= uint64_t(1) << 46;                    // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                    // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = su32(b);
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}\n"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
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
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ float4 lo_part(float4 x) {
  auto lo = [](float v) { return v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); };
  return make_float4(lo(x.x), lo(x.y), lo(x.z), lo(x.w));
}

// lo tile of `bytes` bytes (multiple of 2048), 128 threads, 16-B granules (layout-agnostic: elementwise)
__device__ __forceinline__ void make_lo(const unsigned char* src, unsigned char* dst, int bytes, int tid) {
  const uint32_t s = su32(src), d = su32(dst);
  const int n = bytes >> 4;
  // four granules in flight per thread (one load / store pair at a time left every load's latency exposed)
  for (int i0 = tid; i0 < n; i0 += 4 * 128) {
    float4 x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = min(i0 + j * 128, n - 1);
      asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x[j].x), "=f"(x[j].y), "=f"(x[j].z), "=f"(x[j].w)
          : "r"(s + 16 * i) : "memory");
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i0 + j * 128 < n) {
        const float4 y = lo_part(x[j]);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(d + 16 * (i0 + j * 128)), "f"(y.x), "f"(y.y),
                     "f"(y.z), "f"(y.w) : "memory");
      }
    }
  }
}

__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

}  // namespace

// Tensor maps of one 2-D fp32 array with box rows 16, 32, 64, 128, 256 (TMA requests are few and large:
// a stage of R rows is one request with the smallest box >= R).
struct MapSet { CUtensorMap m[5]; };
__device__ __forceinline__ int box_idx(int rows) { return rows <= 16 ? 0 : rows <= 32 ? 1 : rows <= 64 ? 2 : rows <= 128 ? 3 : 4; }

// ---------------------------------------------------------------- shared pieces of the two kernels
namespace {
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ int pow2_cols(int c) { int t = 32; while (t < c) t <<= 1; return t; }
}  // namespace

// ---------------------------------------------------------------- K4
// Work item = (k, row tile of 128 rows of the batch); items are dealt round-robin to the persistent CTAs.
// Stage = A chunk (128 rows x 32 j, 16 KB, TMA) + B = [T_hi (b rows) ; T_lo (b rows)], b = the smallest TMA box
// >= roundup16(p_k); the lo part of A goes to a separate 2-deep ring (so more A is in flight per SM).
// b <= 128: 2 MMAs of N = 2b per K step, D[q] + D[b + q]; b = 256 (p_k > 128): 3 MMAs of N = b
// (x_raw T_hi, x_raw T_lo, x_lo T_hi).  Warps: 0-3 lo parts, 4 TMA, 5 MMA, 6-9 epilogue (TMEM lane quarter w % 4).
struct K4Args {
  int k_max, n_xi, nrt, rows, nkc, stages, bmax;   // bmax = largest box b of the plan
  const int* kj0;                                   // per k: first ring of the sum (chunks start there; plan.cpp)
  int64_t ghat_krows;                               // ghat rows per k (2 max_batch)
  int64_t i0, ld;
  const int* p;
  const int64_t* coef_off;
  float* out;
};

__global__ void __launch_bounds__(320, 1)
radial_tma_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ MapSet tm_bh,
                  const __grid_constant__ MapSet tm_bl, const K4Args args) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  // 1024-B aligned base by pointer arithmetic on the shared array (keeps the shared address space for the compiler)
  unsigned char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  const int NS = args.stages;
  const uint32_t a_bytes = 128 * ROWB, b_bytes = uint32_t(args.bmax) * ROWB;
  const uint32_t stage_bytes = a_bytes + 2 * b_bytes;               // A, T_hi, T_lo
  unsigned char* lo_ring = sm + NS * stage_bytes;                   // 2 x a_bytes
  uint64_t* full = reinterpret_cast<uint64_t*>(lo_ring + 2 * a_bytes);
  uint64_t* empty = full + NS;
  uint64_t* loready = empty + NS;                                   // 2
  uint64_t* lofree = loready + 2;                                   // 2
  uint64_t* accfull = lofree + 2;                                   // 2
  uint64_t* accempty = accfull + 2;                                 // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int acc_cols = args.bmax <= 128 ? 2 * args.bmax : args.bmax;
  const int tcols = pow2_cols(2 * acc_cols);

  if (warp == 0) tmem_alloc(tmem_slot, tcols);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) {
      bar_init(&loready[a], 128); bar_init(&lofree[a], 1); bar_init(&accfull[a], 1); bar_init(&accempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int n_items = (args.k_max + 1) * args.nrt;

  if (warp == 4) {                                                  // ---- TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_a);
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int k = item / args.nrt, rt = item - k * args.nrt;
        const int bi = box_idx((args.p[k] + 15) & ~15), b = 16 << bi;
        const int arow = int(k * args.ghat_krows) + rt * 128;
        const int brow = int(args.coef_off[k]);
        const int x0 = args.kj0[k], nkc = (args.n_xi - x0 + KC - 1) / KC;   // columns >= n_xi: TMA zero fill
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % NS;
          bar_wait(&empty[s], ((it / NS) & 1) ^ 1);
          unsigned char* st = sm + s * stage_bytes;
          bar_expect_tx(&full[s], a_bytes + 2u * uint32_t(b) * ROWB);
          tma_2d(st, &tm_a, x0 + kc * KC, arow, &full[s]);
          tma_2d(st + a_bytes, &tm_bh.m[bi], x0 + kc * KC, brow, &full[s]);
          tma_2d(st + a_bytes + b * ROWB, &tm_bl.m[bi], x0 + kc * KC, brow, &full[s]);
        }
      }
    }
    return;
  }
  if (warp == 5) {                                                  // ---- MMA issuer
    if (lane == 0) {
      int it = 0, t = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
        const int k = item / args.nrt;
        const int b = 16 << box_idx((args.p[k] + 15) & ~15);
        const bool cat = b <= 128;
        const uint32_t idesc = idesc_tf32(128, cat ? 2 * b : b);
        const int a = t & 1;
        const uint32_t d = tmem + uint32_t(a * acc_cols);
        bar_wait(&accempty[a], ((t >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int nkc = (args.n_xi - args.kj0[k] + KC - 1) / KC;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % NS, l = it & 1;
          bar_wait(&full[s], (it / NS) & 1);
          bar_wait(&loready[l], (it >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t xa = su32(sm + s * stage_bytes), bh = xa + a_bytes, bl = bh + b * ROWB;
          const uint32_t xl = su32(lo_ring + l * a_bytes);
#pragma unroll
          for (int s4 = 0; s4 < KC / 8; ++s4) {
            const uint32_t ko = uint32_t(s4) * 32u;                 // 8 tf32 = 32 B along the swizzled row
            const uint32_t acc0 = (kc | s4) ? 1u : 0u;
            if (cat) {
              mma_tf32(d, desc_sw128(xa + ko), desc_sw128(bh + ko), idesc, acc0);
              mma_tf32(d, desc_sw128(xl + ko), desc_sw128(bh + ko), idesc, 1u);
            } else {
              mma_tf32(d, desc_sw128(xa + ko), desc_sw128(bh + ko), idesc, acc0);
              mma_tf32(d, desc_sw128(xa + ko), desc_sw128(bl + ko), idesc, 1u);
              mma_tf32(d, desc_sw128(xl + ko), desc_sw128(bh + ko), idesc, 1u);
            }
          }
          mma_commit(&empty[s]);
          mma_commit(&lofree[l]);
        }
        mma_commit(&accfull[a]);
      }
    }
    return;
  }
  if (warp >= 6) {                                                  // ---- epilogue: TMEM lanes 32 (w % 4) ..
    const int wq = warp & 3;
    int t = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
      const int k = item / args.nrt, rt = item - k * args.nrt;
      const int pk = args.p[k];
      const int b = 16 << box_idx((pk + 15) & ~15);
      const bool cat = b <= 128;
      const int a = t & 1;
      bar_wait(&accfull[a], (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = rt * 128 + 32 * wq + lane;
      const int64_t base = args.coef_off[k];
      float* o = args.out + 2 * args.i0 + row + base * 2 * args.ld;
      const uint32_t tbase = tmem + (uint32_t(32 * wq) << 16) + uint32_t(a * acc_cols);
      const bool zero = (k == 0 && (row & 1));
      for (int q0 = 0; q0 < pk; q0 += 16) {
        float v[16];
        tmem_ld16(tbase + uint32_t(q0), v);
        if (cat) {
          float w[16];
          tmem_ld16(tbase + uint32_t(b + q0), w);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += w[i];
        }
        if (row < args.rows) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (q0 + i < pk) __stcs(o + (int64_t)(q0 + i) * 2 * args.ld, zero ? 0.f : v[i]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      bar_arrive(&accempty[a]);
    }
    named_sync(2, 256);                                             // TMEM reads done before the dealloc
    return;
  }
  // ---- warps 0-3: lo parts of every chunk into the 2-deep lo ring
  int it = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int nkc = (args.n_xi - args.kj0[item / args.nrt] + KC - 1) / KC;
    for (int kc = 0; kc < nkc; ++kc, ++it) {
      const int s = it % NS, l = it & 1;
      bar_wait(&full[s], (it / NS) & 1);
      bar_wait(&lofree[l], ((it >> 1) & 1) ^ 1);
      make_lo(sm + s * stage_bytes, lo_ring + l * a_bytes, a_bytes, tid);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(&loready[l]);
    }
  }
  named_sync(2, 256);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

// ---------------------------------------------------------------- K5 (k >= 1)
// Work item = (k, chunk of `chunk` images = 2 chunk columns).  Chunk tile = [x_raw (b rows, TMA) ; x_lo (b rows,
// written by warps 0-3)], b = the smallest TMA box >= roundup16(p_k) (<= 128); one MMA per K step with
// A = tile rows 0..127 (rows >= b: ignored outputs) and B = the whole tile (N = 2b):
//   D[q][c] = sum x_raw[q] x_raw[c] (c < b),  D[q][b + c] = sum x_raw[q] x_lo[c]
//   S[q][q'] = X[q][q'] + Y[q][q'] + Y[q'][q],  X = D[:, :b] (symmetric), Y = D[:, b:].
// A stage holds CK consecutive K chunks whose TMA boxes are issued back to back, so each coefficient row is
// read as CK x 128 contiguous bytes at once (the rows of block k are 2 n floats apart: DRAM page locality).
// A drain group of `drain` images accumulates in one of two TMEM accumulators (fp32 accumulation never runs
// longer than 2 drain = 256 terms); warps 0-3 drain it into fp32 registers, thread q keeping
//   acc[c] = sum Y[q][c] (c > q),  X[q][q] + 2 Y[q][q] (c = q),  X[q][c] + Y[q][c] (c < q),
// so that S[q][q'] = acc_q[q'] + acc_q'[q] (q < q'), S[q][q] = acc_q[q].  The item's S goes to scratch[chunk] as the
// fp64 upper triangle (combined through shared memory); cov_reduce_kernel adds the chunks in fixed order.
constexpr int K5_CK = 4;
#ifndef FBSPCA_K5_TH
#define FBSPCA_K5_TH 32
#endif
template <int RR> constexpr int K5_TH = RR < FBSPCA_K5_TH ? RR : FBSPCA_K5_TH;   // epilogue transpose pass width
struct K5Args {
  int k_max, nchunk, chunk, drain, stages, rmax, ck;              // ck: K chunks per stage (<= K5_CK)
  int k_lo;                                                       // first k of this launch (k_lo..k_max)
  int64_t i0, nb, ld;
  const int* p;
  const int64_t* coef_off;
  const int64_t* blk_off;
  double* scratch;
  int64_t scratch_stride;
};

// K-chunk stacking (RR <= 64): a 128-row tile holds G = 128 / (2 b) K-chunks of block k, [x; lo] each, so ONE MMA
// (M = N = 128) covers G chunks: D = tile tile^T, of which the G diagonal 2b x 2b blocks are the wanted
// [x; lo] [x; lo]^T of their chunks (the off-diagonal blocks pair different images and are never read).  Small p_k
// no longer costs a full 64-cycle M = 128 MMA per 32 image-columns.  Warp w drains its rows' diagonal block
// (group (32 w) / (2 b): uniform per warp); the G groups are summed through shared memory in the epilogue.
template <int RR>   // register accumulators per thread (= largest box b of k >= 1)
__global__ void __launch_bounds__(192, RR <= 64 ? 2 : 1)
cov_tma_kernel(const __grid_constant__ MapSet tm_a, const K5Args args) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  // 1024-B aligned base by pointer arithmetic on the shared array (keeps the shared address space for the compiler)
  unsigned char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  const int CK = args.ck;
  const int NS = args.stages;
  constexpr int TROWS = RR <= 64 ? 128 : 2 * RR;                   // tile rows (the M = 128 A operand reads 128)
  constexpr int AW = TROWS;                                         // accumulator columns (N of a stacked tile)
  const uint32_t tile_bytes = uint32_t(TROWS) * ROWB;
  const uint32_t stage_bytes = CK * tile_bytes;
  constexpr int TH = K5_TH<RR>;                                     // epilogue transpose: column passes of TH
  float* tr = reinterpret_cast<float*>(sm + NS * stage_bytes);      // RR x (TH + 1)
  uint64_t* full = reinterpret_cast<uint64_t*>(tr + RR * (TH + 1));
  uint64_t* loready = full + NS;
  uint64_t* empty = loready + NS;
  uint64_t* accfull = empty + NS;                                   // 2
  uint64_t* accempty = accfull + 2;                                 // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tcols = pow2_cols(2 * AW);                              // two accumulators

  if (warp == 0) tmem_alloc(tmem_slot, tcols);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { bar_init(&full[s], 1); bar_init(&loready[s], 128); bar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { bar_init(&accfull[a], 1); bar_init(&accempty[a], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int n_items = (args.k_max - args.k_lo + 1) * args.nchunk;
  // per item: b (box rows), G (chunks per tile), nkc (K chunks), ntile, nst (stages), spg (stages per drain group)
  struct Geo { int k, ch, b, G, nkc, ntile, nst, spg; };
  auto item_geom = [&](int item) {
    Geo e;
    e.k = args.k_lo + item / args.nchunk; e.ch = item - (e.k - args.k_lo) * args.nchunk;
    const int64_t img0 = args.i0 + int64_t(e.ch) * args.chunk;
    const int ncols = int(2 * min(int64_t(args.chunk), args.i0 + args.nb - img0));
    e.nkc = (ncols + KC - 1) / KC;
    e.b = 16 << box_idx((args.p[e.k] + 15) & ~15);
    e.G = RR <= 64 ? TROWS / (2 * e.b) : 1;
    e.ntile = (e.nkc + e.G - 1) / e.G;
    e.nst = (e.ntile + CK - 1) / CK;
    e.spg = max(1, (2 * args.drain) / (KC * CK * e.G));
    return e;
  };

  if (warp == 4) {                                                  // ---- TMA producer
    if (lane == 0) {
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const Geo e = item_geom(item);
        const int bi = box_idx(e.b);
        const int col0 = int(2 * (args.i0 + int64_t(e.ch) * args.chunk));
        const int row0 = int(args.coef_off[e.k]);
        for (int si = 0; si < e.nst; ++si, ++it) {
          const int s = it % NS, nt = min(CK, e.ntile - si * CK);
          const int kc0 = si * CK * e.G, nkc_here = min(nt * e.G, e.nkc - kc0);
          bar_wait(&empty[s], ((it / NS) & 1) ^ 1);
          bar_expect_tx(&full[s], uint32_t(nkc_here) * uint32_t(e.b) * ROWB);
          for (int u = 0; u < nkc_here; ++u)                        // chunk kc0 + u -> tile u / G, group u % G
            tma_2d(sm + s * stage_bytes + (u / e.G) * tile_bytes + (u % e.G) * 2 * e.b * ROWB, &tm_a.m[bi],
                   col0 + (kc0 + u) * KC, row0, &full[s]);
        }
      }
    }
    return;
  }
  if (warp == 5) {                                                  // ---- MMA issuer
    if (lane == 0) {
      int it = 0, g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const Geo e = item_geom(item);
        const uint32_t idesc = idesc_tf32(128, e.G * 2 * e.b);
        for (int si = 0; si < e.nst; ++si, ++it) {
          const bool first = (si % e.spg) == 0;
          const bool last = (si % e.spg) == e.spg - 1 || si == e.nst - 1;
          const int a = g & 1;
          const uint32_t d = tmem + uint32_t(a * AW);
          if (first) {
            bar_wait(&accempty[a], ((g >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          const int s = it % NS, nt = min(CK, e.ntile - si * CK);
          bar_wait(&loready[s], (it / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          for (int c = 0; c < nt; ++c) {
            const uint32_t x = su32(sm + s * stage_bytes + c * tile_bytes);
#pragma unroll
            for (int s4 = 0; s4 < KC / 8; ++s4) {
              const uint32_t ko = uint32_t(s4) * 32u;
              mma_tf32(d, desc_sw128(x + ko), desc_sw128(x + ko), idesc, (!first || c || s4) ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          if (last) { mma_commit(&accfull[a]); ++g; }
        }
      }
    }
    return;
  }
  // ---- warps 0-3
  const int q = 32 * warp + lane;
  int it = 0, g = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const Geo e = item_geom(item);
    const int k = e.k, ch = e.ch, b = e.b;
    const int pk = args.p[k];
    const int gw = RR <= 64 ? (32 * warp) / (2 * b) : 0;   // this warp's diagonal block (uniform per warp)
    const int qq = q - 2 * b * gw;                         // row within the block (< b: an x row)
    float acc[RR];
#pragma unroll
    for (int i = 0; i < RR; ++i) acc[i] = 0.f;
    auto drain = [&](int gg) {
      const int a = gg & 1;
      bar_wait(&accfull[a], (gg >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tb = tmem + (uint32_t(32 * warp) << 16) + uint32_t(a * AW + 2 * b * gw);
      // 16 columns of X and Y in flight per wait (b is a power of two >= 16; few registers: 2 CTAs per SM)
#pragma unroll
      for (int c1 = 0; c1 < RR; c1 += 16) {
        if (c1 < b) {
          uint32_t xr[16], yr[16];
          tmem_ld16_nowait(tb + uint32_t(c1), xr);
          tmem_ld16_nowait(tb + uint32_t(b + c1), yr);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = c1 + i;
            const float xv = __uint_as_float(xr[i]), yv = __uint_as_float(yr[i]);
            acc[c] += c > qq ? yv : c == qq ? xv + 2.f * yv : xv + yv;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      bar_arrive(&accempty[a]);
    };
    int pending = -1;
    for (int si = 0; si < e.nst; ++si, ++it) {
      const int s = it % NS, nt = min(CK, e.ntile - si * CK);
      const int kc0 = si * CK * e.G, nkc_here = min(nt * e.G, e.nkc - kc0);
      unsigned char* st = sm + s * stage_bytes;
      bar_wait(&full[s], (it / NS) & 1);
      if (nkc_here < nt * e.G) {                             // ragged end of the item: chunks not loaded, zero them
        for (int u = nkc_here; u < nt * e.G; ++u) {
          unsigned char* xu = st + (u / e.G) * tile_bytes + (u % e.G) * 2 * b * ROWB;
          for (int i = tid; i < b * KC; i += 128) reinterpret_cast<float*>(xu)[i] = 0.f;
        }
        named_sync(1, 128);
      }
      {
        // lo parts of all chunks of the stage as one flat loop, four 16-byte granules in flight per thread
        // (the chunk-by-chunk loop with volatile loads waited on every granule: shared latency bound)
        const int lg_per = 3 + box_idx(b) + 4;                 // log2(8 b): granules per chunk (b rows x 128 B)
        const int lg_g = 31 - __clz(e.G);
        const int ntot = (nt * e.G) << lg_per;
        const uint32_t sbase = su32(st);
        for (int f0 = tid; f0 < ntot; f0 += 4 * 128) {
          float4 x[4];
          uint32_t ad[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int f = min(f0 + j * 128, ntot - 1);
            const int u = f >> lg_per, i = f & ((1 << lg_per) - 1);
            ad[j] = sbase + uint32_t((u >> lg_g) * tile_bytes + (u & (e.G - 1)) * 2 * b * ROWB + 16 * i);
            asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x[j].x), "=f"(x[j].y), "=f"(x[j].z), "=f"(x[j].w)
                : "r"(ad[j]) : "memory");
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (f0 + j * 128 < ntot) {
              const float4 y = lo_part(x[j]);
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ad[j] + uint32_t(b * ROWB)), "f"(y.x),
                           "f"(y.y), "f"(y.z), "f"(y.w) : "memory");
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(&loready[s]);
      const bool last = (si % e.spg) == e.spg - 1 || si == e.nst - 1;
      if (last) {                                            // drain the previous group while this one runs
        if (pending >= 0) drain(pending);
        pending = g++;
      }
    }
    drain(pending);
    // S = acc_q[q'] + acc_q'[q] (summing the G stacked groups) as the fp64 upper triangle, through shared memory in
    // column passes of TH (tr holds A[r][h0 .. h0 + TH) of every row r, A = the group-summed acc rows: a third of the
    // full RR x (RR + 1) transpose, so a 2-CTA RR = 64 CTA fits three 32 KB stages).  Element (r, c), r < c: written
    // as double(A[c][r]) in r's pass when c lies in a later pass, += double(A[r][c]) in c's pass (the same fp64 sum
    // as in one pass; bar.sync orders the CTA's global accesses); both in one pass: written at once.
    double* dst = args.scratch + int64_t(ch) * args.scratch_stride + args.blk_off[k];
#pragma unroll
    for (int h0 = 0; h0 < RR; h0 += TH) {
      if (h0 < b) {
        for (int gg = 0; gg < e.G; ++gg) {
          named_sync(1, 128);
          if (gw == gg && qq < b) {
#pragma unroll
            for (int c = 0; c < TH; ++c) {
              if (gg == 0) tr[qq * (TH + 1) + c] = acc[h0 + c];
              else tr[qq * (TH + 1) + c] += acc[h0 + c];
            }
          }
        }
        named_sync(1, 128);
        const int h1 = h0 + TH;
        for (int r = warp; r < min(pk, h1); r += 4) {        // row r of the packed upper triangle: warp-wide
          double* drow = dst + (int64_t)r * pk - (int64_t)r * (r - 1) / 2;
          const bool rin = r >= h0;
          for (int c = max(r, h0) + lane; c < pk; c += 32) {
            const bool cin = c < h1;                           // c >= h0 here
            if (rin && cin)
              drow[c - r] = c == r ? double(tr[r * (TH + 1) + (r - h0)])
                                   : double(tr[r * (TH + 1) + (c - h0)]) + double(tr[c * (TH + 1) + (r - h0)]);
            else if (rin)                                      // c in a later pass: A[c][r] now
              drow[c - r] = double(tr[c * (TH + 1) + (r - h0)]);
            else if (cin)                                      // r in an earlier pass: + A[r][c]
              drow[c - r] += double(tr[r * (TH + 1) + (c - h0)]);
          }
        }
      }
    }
  }
  named_sync(1, 128);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

// ---------------------------------------------------------------- K5, blocks with 128 < p_k <= 256 (C5, T3)
// S_k in 128 x 128 output blocks (m, n) in {(0,0), (0,1), (1,1)} of the row halves x_0 = rows 0..127, x_1 = rows
// 128..255 (rows >= p_k: the next block's rows or TMA zero fill, outputs ignored).  Item = (k, chunk, block).
// Stage = one 32-column K chunk: [x_0; lo_0; x_1; lo_1] (512 rows; a diagonal item uses the first 256).
//   diagonal (m = n): D = x_m [x_m; lo_m]^T (N = 256): S = X + Y + Y^T as in cov_tma_kernel;
//   off-diagonal:     D = x_0 [x_1; lo_1]^T (N = 256) plus lo_0 x_1^T accumulated into D[:, 0:128] (N = 128):
//                     S_01 = D[:, 0:128] + D[:, 128:256]  (= x0 x1' + lo0 x1' + x0 lo1', the 3xTF32 terms).
// Two 256-column TMEM accumulators (double-buffered drains every `drain` images), one CTA per SM.
__global__ void __launch_bounds__(192, 1)
cov_tma_big_kernel(const __grid_constant__ CUtensorMap tm_a, const K5Args args) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  constexpr int RR = 128;
  const int NS = args.stages;
  constexpr uint32_t half_bytes = 128u * ROWB;                     // 128 rows of one K chunk
  constexpr uint32_t stage_bytes = 4u * half_bytes;                // x_0, lo_0, x_1, lo_1
  float* tr = reinterpret_cast<float*>(sm + NS * stage_bytes);      // 128 x 129 epilogue transpose
  uint64_t* full = reinterpret_cast<uint64_t*>(tr + RR * (RR + 1));
  uint64_t* loready = full + NS;
  uint64_t* empty = loready + NS;
  uint64_t* accfull = empty + NS;                                   // 2
  uint64_t* accempty = accfull + 2;                                 // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int tcols = 512;                                        // two accumulators of 256 columns
  if (warp == 0) tmem_alloc(tmem_slot, tcols);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { bar_init(&full[s], 1); bar_init(&loready[s], 128); bar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { bar_init(&accfull[a], 1); bar_init(&accempty[a], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int nk = args.k_max - args.k_lo + 1;
  const int n_items = nk * args.nchunk * 3;
  const int kc_per_group = max(1, (2 * args.drain) / KC);          // K chunks per drain group
  auto item_geom = [&](int item, int& k, int& ch, int& blk, int& nkc) {
    blk = item % 3;
    const int r = item / 3;
    k = args.k_lo + r / args.nchunk; ch = r - (k - args.k_lo) * args.nchunk;
    const int64_t img0 = args.i0 + int64_t(ch) * args.chunk;
    const int ncols = int(2 * min(int64_t(args.chunk), args.i0 + args.nb - img0));
    nkc = (ncols + KC - 1) / KC;
  };

  if (warp == 4) {                                                  // ---- TMA producer
    if (lane == 0) {
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int k, ch, blk, nkc;
        item_geom(item, k, ch, blk, nkc);
        const int col0 = int(2 * (args.i0 + int64_t(ch) * args.chunk));
        const int row0 = int(args.coef_off[k]);
        const int m = blk == 2 ? 1 : 0;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % NS;
          bar_wait(&empty[s], ((it / NS) & 1) ^ 1);
          unsigned char* st = sm + s * stage_bytes;
          if (blk == 1) {
            bar_expect_tx(&full[s], 2u * half_bytes);
            tma_2d(st, &tm_a, col0 + kc * KC, row0, &full[s]);
            tma_2d(st + 2 * half_bytes, &tm_a, col0 + kc * KC, row0 + 128, &full[s]);
          } else {
            bar_expect_tx(&full[s], half_bytes);
            tma_2d(st, &tm_a, col0 + kc * KC, row0 + 128 * m, &full[s]);
          }
        }
      }
    }
    return;
  }
  if (warp == 5) {                                                  // ---- MMA issuer
    if (lane == 0) {
      const uint32_t id256 = idesc_tf32(128, 256), id128 = idesc_tf32(128, 128);
      int it = 0, g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int k, ch, blk, nkc;
        item_geom(item, k, ch, blk, nkc);
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const bool first = (kc % kc_per_group) == 0;
          const bool last = (kc % kc_per_group) == kc_per_group - 1 || kc == nkc - 1;
          const int a = g & 1;
          const uint32_t d = tmem + uint32_t(a * 256);
          if (first) {
            bar_wait(&accempty[a], ((g >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          const int s = it % NS;
          bar_wait(&loready[s], (it / NS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t x0 = su32(sm + s * stage_bytes);
#pragma unroll
          for (int s4 = 0; s4 < KC / 8; ++s4) {
            const uint32_t ko = uint32_t(s4) * 32u;
            const uint32_t acc = (!first || s4) ? 1u : 0u;
            if (blk == 1) {
              const uint32_t x1 = x0 + 2 * half_bytes;
              mma_tf32(d, desc_sw128(x0 + ko), desc_sw128(x1 + ko), id256, acc);              // x0 [x1; lo1]^T
              mma_tf32(d, desc_sw128(x0 + half_bytes + ko), desc_sw128(x1 + ko), id128, 1u);  // + lo0 x1^T
            } else {
              mma_tf32(d, desc_sw128(x0 + ko), desc_sw128(x0 + ko), id256, acc);              // x_m [x_m; lo_m]^T
            }
          }
          mma_commit(&empty[s]);
          if (last) { mma_commit(&accfull[a]); ++g; }
        }
      }
    }
    return;
  }
  // ---- warps 0-3: lo parts, drains, epilogue (thread q = row of the 128 x 128 output block)
  const int q = 32 * warp + lane;
  int it = 0, g = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    int k, ch, blk, nkc;
    item_geom(item, k, ch, blk, nkc);
    const int pk = args.p[k];
    float acc[RR];
#pragma unroll
    for (int i = 0; i < RR; ++i) acc[i] = 0.f;
    auto drain = [&](int gg) {
      const int a = gg & 1;
      bar_wait(&accfull[a], (gg >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tb = tmem + (uint32_t(32 * warp) << 16) + uint32_t(a * 256);
#pragma unroll
      for (int c1 = 0; c1 < RR; c1 += 16) {
        uint32_t xr[16], yr[16];
        tmem_ld16_nowait(tb + uint32_t(c1), xr);
        tmem_ld16_nowait(tb + uint32_t(128 + c1), yr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = c1 + i;
          const float xv = __uint_as_float(xr[i]), yv = __uint_as_float(yr[i]);
          if (blk == 1) acc[c] += xv + yv;
          else acc[c] += c > q ? yv : c == q ? xv + 2.f * yv : xv + yv;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      bar_arrive(&accempty[a]);
    };
    int pending = -1;
    for (int kc = 0; kc < nkc; ++kc, ++it) {
      const int s = it % NS;
      unsigned char* st = sm + s * stage_bytes;
      bar_wait(&full[s], (it / NS) & 1);
      make_lo(st, st + half_bytes, half_bytes, tid);
      if (blk == 1) make_lo(st + 2 * half_bytes, st + 3 * half_bytes, half_bytes, tid);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(&loready[s]);
      const bool last = (kc % kc_per_group) == kc_per_group - 1 || kc == nkc - 1;
      if (last) {
        if (pending >= 0) drain(pending);
        pending = g++;
      }
    }
    drain(pending);
    named_sync(1, 128);
#pragma unroll
    for (int c = 0; c < RR; ++c) tr[q * (RR + 1) + c] = acc[c];
    named_sync(1, 128);
    double* dst = args.scratch + int64_t(ch) * args.scratch_stride + args.blk_off[k];
    const int m = blk == 2 ? 1 : 0, n = blk >= 1 ? 1 : 0;
    for (int r = warp; r < 128; r += 4) {                   // packed upper-triangle rows of S_k inside the block
      const int qr = 128 * m + r;
      if (qr >= pk) break;
      double* drow = dst + (int64_t)qr * pk - (int64_t)qr * (qr - 1) / 2 - qr;        // drow[col]
      const int c0 = blk == 1 ? 0 : r;
      for (int c = c0 + lane; c < 128 && 128 * n + c < pk; c += 32) {
        const int qc = 128 * n + c;
        drow[qc] = blk == 1 ? double(tr[r * (RR + 1) + c])
                            : (c == r ? double(tr[r * (RR + 1) + r]) : double(tr[r * (RR + 1) + c]) + double(tr[c * (RR + 1) + r]));
      }
    }
    named_sync(1, 128);
  }
  named_sync(1, 128);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

// ---------------------------------------------------------------- host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 row-major [rows][cols] (row stride ld_elems), box = 32 columns x box_rows rows, 128-B swizzle
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld_elems, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld_elems * 4)};
  cuuint32_t box[2] = {cuuint32_t(KC), cuuint32_t(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_radial_tma(const Plan& P, int64_t nb, int64_t i0, int64_t ld, void* d_coeffs, cudaStream_t s) {
  const int nk = P.k_max + 1;
  const int bmax = (P.p[0] + 15) & ~15;
  if (bmax > 256 || P.n_xi % 4) return cudaErrorInvalidValue;
  CUtensorMap ta;
  MapSet tbh, tbl;
  const int64_t krows = 2 * P.max_batch;
  if (!make_map(&ta, P.d_ghat, nk * krows, P.n_xi, P.n_xi, 128)) return cudaErrorInvalidValue;
  for (int i = 0; i < 5; ++i)
    if (!make_map(&tbh.m[i], P.d_table_hi, P.coef_off[nk], P.n_xi, P.n_xi, 16 << i) ||
        !make_map(&tbl.m[i], P.d_table_lo, P.coef_off[nk], P.n_xi, P.n_xi, 16 << i))
      return cudaErrorInvalidValue;
  K4Args a;
  a.k_max = P.k_max; a.n_xi = P.n_xi; a.rows = int(2 * nb); a.nrt = (a.rows + 127) / 128;
  a.nkc = (P.n_xi + KC - 1) / KC; a.bmax = bmax; a.ghat_krows = krows; a.i0 = i0; a.ld = ld;
  a.p = P.d_p; a.coef_off = P.d_coef_off; a.out = reinterpret_cast<float*>(d_coeffs); a.kj0 = P.d_kj0;
  const int bbox = bmax <= 16 ? 16 : bmax <= 32 ? 32 : bmax <= 64 ? 64 : bmax <= 128 ? 128 : 256;
  a.bmax = bbox;                                           // B tiles sized for the largest box
  const int stage = 128 * ROWB + 2 * bbox * ROWB;
  const int fixed = 2 * 128 * ROWB + 1024 + 256;
  // two CTAs per SM when each still gets >= 2 stages (two independent TMA / MMA pipelines per SM; measured at C3:
  // 4.43 ms vs 5.46 ms with one CTA of 6 stages)
  const char* env = getenv("FBSPCA_K4_CTAS");
  const int per_sm = env ? std::max(1, std::min(2, atoi(env))) : ((113 * 1024 - fixed) / stage >= 2 ? 2 : 1);
  const int budget = (per_sm == 2 ? 113 : 227) * 1024;
  a.stages = std::max(2, std::min(8, (budget - fixed) / stage));
  const int smem = a.stages * stage + fixed;
  cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(radial_tma_kernel), smem);
  if (e != cudaSuccess) return e;
  const int items = nk * a.nrt;
  const int grid = std::min(items, per_sm * P.num_sms);
  radial_tma_kernel<<<grid, 320, smem, s>>>(ta, tbh, tbl, a);
  return cudaGetLastError();
}

template <int RR>
static cudaError_t launch_cov_tma_t(const Plan& P, const MapSet& ta, K5Args& a, cudaStream_t s) {
  const int fixed = RR * (K5_TH<RR> + 1) * 4 + 1024 + 256;
  const char* env = getenv("FBSPCA_K5_CTAS");
  const int per_sm = env ? std::max(1, std::min(2, atoi(env))) : (RR <= 64 ? 2 : 1);   // RR = 128: 255 registers
  const int budget = (per_sm == 2 ? 113 : 227) * 1024;
  a.ck = K5_CK;                                            // fewer chunks per stage when a tile is 32 KB
  if (const char* e = getenv("FBSPCA_K5_CK")) a.ck = std::max(1, std::min(8, atoi(e)));   // A/B knob
  while (a.ck > 1 && 2 * a.ck * std::max(128, 2 * RR) * ROWB > budget - fixed) a.ck /= 2;
  const int stage = a.ck * std::max(128, 2 * RR) * ROWB;
  a.stages = std::max(2, std::min(8, (budget - fixed) / stage));
  const int smem = a.stages * stage + fixed;
  cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(cov_tma_kernel<RR>), smem);
  if (e != cudaSuccess) return e;
  const int items = (a.k_max - a.k_lo + 1) * a.nchunk;
  const int grid = std::min(items, per_sm * P.num_sms);
  cov_tma_kernel<RR><<<grid, 192, smem, s>>>(ta, a);
  return cudaGetLastError();
}

// images per tensor-core split-K chunk: kCovChunk x FBSPCA_K5_CHUNKS (1, 2 or 4; default 4: A/B on B200, C3 K5 2.53 ->
// 2.35 ms -- fewer per-item epilogues; partial-sum error unchanged at 1.8e-6).  TMEM drains every `drain` images into
// fp32 registers, so a chunk's register sums add chunk / drain drained groups (32 at the default)
int cov_tma_chunk() {
  static const int m = [] {
    const char* e = getenv("FBSPCA_K5_CHUNKS");
    const int v = e ? atoi(e) : 4;
    return (v == 1 || v == 2) ? v : 4;
  }();
  static_assert(kCovChunk * 4 <= kCovChunkTc, "tensor-core chunk");
  return kCovChunk * m;
}

// k >= 1 of the batch [i0, i0 + nb) into scratch[chunk] (chunks of cov_tma_chunk() images); k = 0 is not touched.
cudaError_t launch_cov_tma(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb, cudaStream_t s) {
  if (P.k_max < 1) return cudaSuccess;
  if (((P.p[1] + 15) & ~15) > 256) return cudaErrorInvalidValue;   // p_k > 256: not on this path
  // k in [1, kb]: 128 < p_k <= 256 (big-block kernel); k in (kb, k_max]: p_k <= 128 (p_k is non-increasing in k)
  int kb = 0;
  while (kb + 1 <= P.k_max && P.p[kb + 1] > 128) ++kb;
  MapSet ta;
  for (int i = 0; i < 4; ++i)
    if (!make_map(&ta.m[i], d_coeffs, P.coef_off[P.k_max + 1], 2 * ld, 2 * ld, 16 << i)) return cudaErrorInvalidValue;
  K5Args a;
  const int chunk = cov_tma_chunk();
  a.k_max = P.k_max; a.k_lo = kb + 1; a.chunk = chunk; a.nchunk = int((nb + chunk - 1) / chunk);
  a.drain = 128; a.i0 = i0; a.nb = nb; a.ld = ld; a.p = P.d_p; a.coef_off = P.d_coef_off; a.blk_off = P.d_blk_off;
  if (const char* e = getenv("FBSPCA_K5_DRAIN")) a.drain = std::max(16, std::min(512, atoi(e)));   // A/B knob
  a.scratch = P.d_cov_scratch; a.scratch_stride = P.blk_off[P.k_max + 1] + P.p[0] + 1;
  if (kb > 0) {
    K5Args b = a;
    b.k_lo = 1; b.k_max = kb; b.rmax = 256; b.ck = 1;
    const int stage = 4 * 128 * ROWB;
    const int fixed = 128 * 129 * 4 + 1024 + 256;
    b.stages = std::max(2, std::min(4, (227 * 1024 - fixed) / stage));
    const int smem = b.stages * stage + fixed;
    cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(cov_tma_big_kernel), smem);
    if (e != cudaSuccess) return e;
    const int grid = std::min(kb * b.nchunk * 3, P.num_sms);
    cov_tma_big_kernel<<<grid, 192, smem, s>>>(ta.m[3], b);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (kb == P.k_max) return cudaSuccess;
  }
  const int rmax = (P.p[kb + 1] + 15) & ~15;
  a.rmax = rmax;
  if (rmax <= 16) return launch_cov_tma_t<16>(P, ta, a, s);
  if (rmax <= 32) return launch_cov_tma_t<32>(P, ta, a, s);
  if (rmax <= 64) return launch_cov_tma_t<64>(P, ta, a, s);
  return launch_cov_tma_t<128>(P, ta, a, s);
}

// ---------------------------------------------------------------- K5, k = 0 (CUDA cores, fp64)
// Uncentred second moment of the real parts (Im a_0 = 0, Q8; mean^2/var ~ 10 -> fp64, reading F9), plus
// s_0 = sum_i a_{0,i} and the image count, for chunk blockIdx.y into scratch[chunk]; tiles of 64 x 64
// (blockIdx.x enumerates tq <= tqq), each thread 4 x 8 entries.
__global__ void __launch_bounds__(128)
cov_k0_kernel(const float* __restrict__ A0, int pk, int64_t ld, int64_t i0, int64_t nb, int chunk,
              int64_t blk0, int64_t s0_off, double* __restrict__ scratch, int64_t scratch_stride) {
  constexpr int BK = 32, TS = 65;
  __shared__ double S1[BK * TS], S2[BK * TS];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int nt = (pk + 63) / 64;
  int pair = blockIdx.x, tq = 0;
  while (tq < nt && pair >= nt - tq) { pair -= nt - tq; ++tq; }
  if (tq >= nt) return;
  const int tqq = tq + pair;
  const int64_t img0 = i0 + int64_t(blockIdx.y) * chunk;
  const int cnb = int(min(int64_t(chunk), i0 + nb - img0));
  const int64_t ld2 = 2 * ld;
  double* part = scratch + int64_t(blockIdx.y) * scratch_stride;
  const int qa = tq * 64, qb = tqq * 64;
  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  for (int cb = 0; cb < cnb; cb += BK) {
    __syncthreads();
    for (int e = tid; e < 64 * BK; e += 128) {
      const int rr = e / BK, cc = e - rr * BK;
      const int c = cb + cc;
      const int q1 = qa + rr, q2 = qb + rr;
      S1[cc * TS + rr] = (q1 < pk && c < cnb) ? double(__ldg(A0 + (int64_t)q1 * ld2 + 2 * (img0 + c))) : 0.0;
      S2[cc * TS + rr] = (q2 < pk && c < cnb) ? double(__ldg(A0 + (int64_t)q2 * ld2 + 2 * (img0 + c))) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = S1[kk * TS + tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = S2[kk * TS + ty + 8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
  double* dst = part + blk0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = qa + tx + 16 * i, qq = qb + ty + 8 * j;
      if (q < pk && qq < pk && q <= qq) dst[(int64_t)q * pk - (int64_t)q * (q - 1) / 2 + (qq - q)] = acc[i][j];
    }
  if (blockIdx.x == 0) {
    double* s0 = part + s0_off;
    for (int q = tid; q < pk; q += 128) {
      double s = 0;
      const float* row = A0 + (int64_t)q * ld2 + 2 * img0;
      for (int c = 0; c < cnb; ++c) s += double(__ldg(row + 2 * c));
      s0[q] = s;
    }
    if (tid == 0) s0[pk] = double(cnb);
  }
}

// scratch0[sub] = [packed k = 0 block | s_0 | count] per kCovChunk0 images
cudaError_t launch_cov_k0(const Plan& P, const void* d_coeffs, int64_t ld, int64_t i0, int64_t nb, cudaStream_t s) {
  const int nt = (P.p[0] + 63) / 64;
  dim3 grid((unsigned)(nt * (nt + 1) / 2), (unsigned)((nb + kCovChunk0 - 1) / kCovChunk0));
  const int64_t stride = P.blk_off[1] + P.p[0] + 1;
  cov_k0_kernel<<<grid, 128, 0, s>>>(reinterpret_cast<const float*>(d_coeffs) + P.coef_off[0] * 2 * ld, P.p[0], ld, i0,
                                     nb, kCovChunk0, 0, P.blk_off[1], P.d_cov_scratch0, stride);
  return cudaGetLastError();
}

}  // namespace fbspca
