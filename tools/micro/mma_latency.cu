// Latency of tcgen05.mma kind::tf32 (M=128, N, K=8, SS operands, SWIZZLE_128B) from issue to the
// tcgen05.commit mbarrier arrive, for a burst of n MMAs; one CTA, one thread issues.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0; d |= uint64_t((saddr >> 4) & 0x3FFF); d |= uint64_t(1) << 16; d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46; d |= uint64_t(2) << 61; return d; }
__global__ void k(int N, int nmma, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~uintptr_t(1023));
  uint64_t* bar = (uint64_t*)(sm + 64 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 1);
  int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += 128) ((float*)sm)[i] = 1.0f;
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
                   asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = *slot;
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    for (int rep = 0; rep < 4; ++rep) {
      long long t0 = clock64();
      for (int i = 0; i < nmma; ++i) {
        uint64_t da = desc_sw128(su32(sm) + (i & 3) * 32), db = desc_sw128(su32(sm + 32768) + (i & 3) * 32);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(i));
      }
      long long t1 = clock64();
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
      uint32_t done = 0;
      while (!done) asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(done) : "r"(su32(bar)), "r"(rep & 1) : "memory");
      long long t2 = clock64();
      if (rep == 3) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  int Ns[] = {16, 64, 128, 256}; int ns[] = {1, 3, 12, 48, 192};
  for (int N : Ns) for (int n : ns) {
    k<<<1, 128, 70 * 1024>>>(N, n, d); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d nmma=%3d issue %6lld cyc  issue->commit-arrive %6lld cyc  (%.1f cyc/mma) %s\n", N, n, h[0], h[1], double(h[1]) / n, cudaGetErrorString(e));
  }
}
