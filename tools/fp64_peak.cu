// FP64 FMA peak microbenchmark (sm_100a). Measures sustained DFMA throughput
// with independent chains per thread; result is the roofline denominator for
// the direct packed-convolution kernels (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}
template <int CH>
double sweep(double* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000 * 8 / CH;
  double best_rate = 0;
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      if (tpb * bps > 2048 || tpb * CH > 16384) continue;   // register file: 2 regs per chain
      int grid = sms * bps;
      dfma_loop<CH><<<grid, tpb>>>(out, 100, 0.999999, 1e-7);
      cudaDeviceSynchronize();
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_loop<CH><<<grid, tpb>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      double fma = (double)grid * tpb * CH * iters;
      printf("chains=%d tpb=%d bps=%d: %.2f TFMA/s = %.2f TFLOP/s (%.3f ms)\n", CH, tpb, bps, fma / best / 1e9,
             2 * fma / best / 1e9, best);
      if (fma / best / 1e9 > best_rate) best_rate = fma / best / 1e9;
    }
  }
  return best_rate;
}

template <int CH>
void sustained(double* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000 * 8 / CH;
  int grid = sms * 2, tpb = 512, n = 0;
  float total = 0;
  cudaEventRecord(e0);
  while (total < 3000.f) {
    for (int k = 0; k < 10; ++k) dfma_loop<CH><<<grid, tpb>>>(out, iters, 0.999999, 1e-7);
    n += 10;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&total, e0, e1);
  }
  double fma = (double)grid * tpb * CH * iters * n;
  printf("sustained (chains=%d) %.1f ms: %.2f TFMA/s = %.2f TFLOP/s\n", CH, total, fma / total / 1e9,
         2 * fma / total / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double r8 = sweep<8>(out, sms), r16 = sweep<16>(out, sms), r32 = sweep<32>(out, sms);
  printf("best burst: 8 chains %.2f, 16 chains %.2f, 32 chains %.2f TFMA/s\n", r8, r16, r32);
  if (r16 >= r32) sustained<16>(out, sms); else sustained<32>(out, sms);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
