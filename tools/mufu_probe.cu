#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__global__ void k(float* out, int iters, int mode) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -1.0f * (threadIdx.x + i) * 1e-3f;
  long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  } else if (mode == 1) {
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) h[i] = 0x3c003c00u;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
    for (int i = 0; i < 8; ++i) a[i] = (float)h[i];
  } else if (mode == 2) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
  } else {
    double b[8];
    for (int i = 0; i < 8; ++i) b[i] = a[i];
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(b[i]));
    for (int i = 0; i < 8; ++i) a[i] = (float)b[i];
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 1024 * 4 * 4);
  for (int mode = 0; mode < 4; ++mode) for (int threads : {128, 512, 1024}) {
    int iters = 1000;
    k<<<148, threads>>>(d, iters, mode); cudaDeviceSynchronize();
    k<<<148, threads>>>(d, iters, mode); cudaDeviceSynchronize();
    float cyc; cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 8 * (mode == 1 ? 2 : 1);
    printf("mode %d (%s) threads %4d: %.1f ops/clk/SM\n", mode, mode == 0 ? "ex2.f32" : mode == 1 ? "ex2.f16x2 (elems)" : mode == 2 ? "ffma" : "dfma", threads, ops / cyc);
  }
}
