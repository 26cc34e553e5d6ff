// Launch-gap probe: back-to-back launches of a kernel that spins ~100 us, for several
// (CTAs/SM, threads, dynamic smem, registers) shapes; reports event time per launch minus
// the spin time, i.e. the per-launch overhead outside CTA execution.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long ns, unsigned long long* rec) {
  extern __shared__ double sm[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while ((long long)(t - t0) < ns);
  if (threadIdx.x == 0) { sm[0] = t; if (t == 0) rec[blockIdx.x] = t0; }
}
__global__ void __launch_bounds__(160, 4) spin96(long long ns, unsigned long long* rec) {
  extern __shared__ double sm[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while ((long long)(t - t0) < ns);
  if (threadIdx.x == 0) { sm[0] = t; if (t == 0) rec[blockIdx.x] = t0; }
}
int main() {
  unsigned long long* rec; cudaMalloc(&rec, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct C { int grid, threads; size_t smem; } cs[] = {{592, 160, 53 * 1024}, {296, 288, 94 * 1024}, {592, 160, 8 * 1024},
                                                      {148, 160, 53 * 1024}, {1184, 160, 20 * 1024}, {592, 160, 0}};
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (auto c : cs) {
    for (int i = 0; i < 3; ++i) spin<<<c.grid, c.threads, c.smem>>>(100000, rec);
    cudaDeviceSynchronize();
    const int K = 20;
    cudaEventRecord(a);
    for (int i = 0; i < K; ++i) spin<<<c.grid, c.threads, c.smem>>>(100000, rec);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %5d threads %4d smem %6zu: %.2f us/launch (spin 100 us)  %s\n", c.grid, c.threads, c.smem, ms / K * 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
