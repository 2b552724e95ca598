// FP32 FMA issue throughput on sm_100a: scalar FFMA (3 registers) vs packed fma.rn.f32x2 (FFMA2).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__global__ void scalar(float* out, int iters, long long* cyc) {
  float a[8], b = threadIdx.x * 1e-7f, c = 1.0000001f + threadIdx.x * 1e-12f;
  for (int i = 0; i < 8; ++i) a[i] = i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], c, b);
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void packed(float* out, int iters, long long* cyc) {
  unsigned long long a[4], b = pk(threadIdx.x * 1e-7f, 1e-7f), c = pk(1.0000001f + threadIdx.x * 1e-12f, 1.0000001f);
  for (int i = 0; i < 4; ++i) a[i] = pk(2 * i, 2 * i + 1);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(c), "l"(b));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 4; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); s += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; long long h;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
  const int iters = 4096;
  for (int thr : {128, 256, 512, 1024}) {
    scalar<<<148, thr>>>(o, iters, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double fs = double(thr) * iters * 8 / h;
    packed<<<148, thr>>>(o, iters, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double fp = double(thr) * iters * 8 / h;
    printf("threads/SM %4d: scalar FFMA %.1f FMA/clk/SM, packed f32x2 %.1f FMA/clk/SM\n", thr, fs, fp);
  }
}
