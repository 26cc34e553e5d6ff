// Which warps of a 640-thread CTA share an SM sub-partition?  Run a DFMA chain loop on a
// chosen subset of warps (one CTA per SM) and time it; also print %warpid per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(unsigned mask, int iters, double* out, int* wid) {
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) {
    int x;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(x));
    wid[w] = x;
  }
  if (!((mask >> w) & 1)) return;
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* out;
  int* wid;
  cudaMalloc(&out, 8);
  cudaMalloc(&wid, 64 * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 150000);
  const int iters = 20000;
  struct { const char* name; unsigned mask; } sets[] = {
      {"w4", 1u << 4}, {"w4,5,6,7", 0xF0u}, {"w4,8,12,16", (1u << 4) | (1u << 8) | (1u << 12) | (1u << 16)},
      {"w4,5", 0x30u}, {"w4,6", 0x50u}, {"w4,8", 0x110u}, {"w4,12", (1u << 4) | (1u << 12)},
      {"w4..19", 0xFFFF0u}, {"w0..3", 0xFu}, {"w0,4", 0x11u}, {"w4,9,14,19", (1u<<4)|(1u<<9)|(1u<<14)|(1u<<19)}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& s : sets) {
    probe<<<sms, 640, 150000>>>(s.mask, 100, out, wid);
    cudaEventRecord(e0);
    probe<<<sms, 640, 150000>>>(s.mask, iters, out, wid);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const int nw = __builtin_popcount(s.mask);
    const double fma = (double)sms * nw * 32 * 16 * iters;
    printf("%-12s warps=%2d  %.3f ms  %.2f T DFMA/s  per-warp-time ratio %.2f\n", s.name, nw, ms, fma / ms / 1e9,
           ms / (iters * 16 * 2.0 / 1.965e6));
  }
  int h[20];
  cudaMemcpy(h, wid, 80, cudaMemcpyDeviceToHost);
  printf("warpid:");
  for (int i = 0; i < 20; ++i) printf(" %d", h[i]);
  printf("\n");
  return 0;
}
