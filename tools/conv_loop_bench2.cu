// Inner-loop calibration for the persistent kernel's padded-layout core (conv_group_padded):
// FP64 FMA rate vs tile T and resident warps per SM, data in shared memory only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1201_3018_b200/csrc/pc_device.cuh"
using namespace pc;

template <int T>
__global__ void __maxnreg__(96) loop_kernel(int K_pad, int rows, int groups, int reps, double* out) {
  extern __shared__ double sm[];
  double* kr = sm;
  double* xs = sm + K_pad;
  for (int i = threadIdx.x; i < (T + 1) * rows; i += blockDim.x) xs[i] = 1.0 + 1e-9 * i;
  for (int i = threadIdx.x; i < K_pad; i += blockDim.x) kr[i] = 1e-3 * (i % 7);
  __syncthreads();
  double tot = 0;
  for (int rep = 0; rep < reps; ++rep)
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
      double acc[T];
      conv_group_padded<T>(smem_u32(xs) + 8u * (T + 1) * g, smem_u32(kr), K_pad, acc);
#pragma unroll
      for (int i = 0; i < T; ++i) tot += acc[i];
    }
  if (tot == 123.456) out[threadIdx.x] = tot;
}

template <int T>
void run(int threads, int ctas_per_sm, int K, double* dout, int sms) {
  const int K_pad = (K + T - 1) / T * T;
  const int groups = threads;
  const int rows = groups + K_pad / T + 2;
  const size_t smem = (size_t)((T + 1) * rows + K_pad) * 8;
  auto kfn = loop_kernel<T>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem);
  if (occ < ctas_per_sm) { printf("T=%d threads=%d: occ %d < %d\n", T, threads, occ, ctas_per_sm); return; }
  const int reps = 20, grid = sms * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kfn<<<grid, threads, smem>>>(K_pad, rows, groups, 2, dout);
  cudaEventRecord(a);
  kfn<<<grid, threads, smem>>>(K_pad, rows, groups, reps, dout);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fma = (double)grid * groups * T * K_pad * reps;
  printf("T=%2d threads=%3d ctas/SM=%d warps/SM=%2d K=%d: %.2f TFMA/s (%.1f%% of 17.0)\n", T, threads, ctas_per_sm,
         ctas_per_sm * threads / 32, K, fma / ms / 1e9, 100 * fma / ms / 1e9 / 17.0);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout;
  cudaMalloc(&dout, 8192 * 8);
  for (int c : {1, 2, 3, 4, 5}) run<14>(128, c, 513, dout, sms);
  for (int c : {1, 2, 3, 4}) run<16>(128, c, 513, dout, sms);
  for (int c : {1, 2, 4}) run<12>(128, c, 513, dout, sms);
  for (int c : {2, 4}) run<14>(64, c, 513, dout, sms);
  return 0;
}
