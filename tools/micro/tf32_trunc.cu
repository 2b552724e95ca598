// Does tcgen05.mma kind::tf32 truncate or round the low 13 mantissa bits of an fp32 operand?
// D[128 x 16] = A[128 x 8] * B[16 x 8]^T with A[r][k] = x_r (k = 0 only, rest 0), B[n][k] = 1 (k = 0 only).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= uint64_t((saddr >> 4) & 0x3FFF); d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32; d |= uint64_t(1) << 46; return d; }
__device__ __forceinline__ uint32_t il_off(int row, int c16, int rows) {
  return uint32_t(c16) * uint32_t(rows / 8) * 128u + uint32_t(row >> 3) * 128u + uint32_t(row & 7) * 16u; }
__global__ void k(const float* x, float* out) {
  __shared__ __align__(1024) unsigned char sm[128 * 32 + 16 * 32 + 64];
  uint64_t* bar = (uint64_t*)(sm + 128 * 32 + 16 * 32);
  uint32_t* slot = (uint32_t*)(bar + 1);
  int tid = threadIdx.x, warp = tid >> 5;
  float* A = (float*)sm; float* B = (float*)(sm + 128 * 32);
  for (int i = tid; i < (128 * 32 + 16 * 32) / 4; i += 128) ((float*)sm)[i] = 0.f;
  __syncthreads();
  // element (row, kk): byte il_off(row, kk/4, rows) + 4*(kk%4)
  *(float*)((char*)A + il_off(tid, 0, 128)) = x[tid];
  if (tid < 16) *(float*)((char*)B + il_off(tid, 0, 16)) = 1.f;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(slot)));
                   asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = *slot;
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(16 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    uint64_t da = make_desc(smem_u32(A), 16 * 128, 128), db = make_desc(smem_u32(B), 2 * 128, 128);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done) asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(done) : "r"(smem_u32(bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm + (uint32_t(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[tid] = __uint_as_float(r);
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  float hx[128], ho[128]; float *dx, *dout;
  for (int i = 0; i < 128; ++i) { uint32_t b = 0x3f800000u | ((uint32_t(i) * 2654435761u) >> 9); if (i & 1) b |= 0x80000000u; memcpy(&hx[i], &b, 4); }
  cudaMalloc(&dx, 512); cudaMalloc(&dout, 512);
  cudaMemcpy(dx, hx, 512, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dx, dout);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(ho, dout, 512, cudaMemcpyDeviceToHost);
  int tr = 0, rn = 0, other = 0;
  for (int i = 0; i < 128; ++i) {
    uint32_t b; memcpy(&b, &hx[i], 4);
    uint32_t t = b & ~0x1FFFu; float ft; memcpy(&ft, &t, 4);
    uint32_t r2 = (b + 0x1000u) & ~0x1FFFu; float fr; memcpy(&fr, &r2, 4);
    if (ho[i] == ft && ft != fr) ++tr; else if (ho[i] == fr && ft != fr) ++rn; else if (ft != fr) ++other;
  }
  printf("err=%s truncate=%d round=%d other=%d  sample x=%.9g out=%.9g\n", cudaGetErrorString(e), tr, rn, other, hx[3], ho[3]);
  return 0;
}
