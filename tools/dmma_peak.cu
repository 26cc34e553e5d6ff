// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) peak microbenchmark for sm_100a, next to the
// DFMA rate of tools/fp64_peak.cu: is the FP64 MMA pipe a higher roof for the packed core?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void dmma_loop(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9 + i;
  double av = a + threadIdx.x * 1e-12, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(acc[i][0], acc[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// DMMA fed from shared memory the way a Toeplitz convolution core would be: per k-step each
// lane loads one A double (signal, row-shifted per step) and, every MT tiles, one B double.
template <int MT>
__global__ void dmma_smem(double* out, int iters) {
  __shared__ double sx[4096 + 64];
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 4096 + 64; i += blockDim.x) sx[i] = (i & 255) * 0.5;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = (i & 127) * 0.25;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = lane >> 2, col = lane & 3;
  double acc[MT][2];
#pragma unroll
  for (int t = 0; t < MT; ++t) acc[t][0] = acc[t][1] = 0;
  const double* xb = sx + (warp & 7) * 256 + row * 8 + col;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int j = 0; j < 64; ++j) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const double b = sh[(j * 8 + ks * 4 + col) * 8 + row & 1023];
#pragma unroll
        for (int t = 0; t < MT; ++t) dmma(acc[t][0], acc[t][1], xb[(t * 8 + j) * 8 + ks * 4], b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < MT; ++t) s += acc[t][0] + acc[t][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

template <int CH>
void sweep(double* out, int sms) {
  const int iters = 4000 * 8 / CH;
  for (int tpb : {128, 256, 512, 1024}) {
    for (int bps : {1, 2}) {
      if (tpb * bps > 2048 || tpb * CH * 4 > 65536 - tpb * 16) continue;
      const int grid = sms * bps;
      float ms = best_ms([&] { dmma_loop<CH><<<grid, tpb>>>(out, iters, 0.999999, 1e-7); });
      double fma = (double)grid * (tpb / 32) * CH * iters * 256;
      printf("dmma chains=%d tpb=%d bps=%d: %.2f TFMA/s = %.2f TFLOP/s\n", CH, tpb, bps, fma / ms / 1e9,
             2 * fma / ms / 1e9);
    }
  }
}

template <int MT>
void sweep_smem(double* out, int sms) {
  const int iters = 400;
  for (int tpb : {128, 256, 384, 512}) {
    const int grid = sms * (tpb <= 256 ? 2 : 1);
    float ms = best_ms([&] { dmma_smem<MT><<<grid, tpb>>>(out, iters); });
    double fma = (double)grid * (tpb / 32) * iters * 64 * 2 * MT * 256;
    printf("smem-fed MT=%d tpb=%d grid=%d: %.2f TFMA/s = %.2f TFLOP/s\n", MT, tpb, grid, fma / ms / 1e9,
           2 * fma / ms / 1e9);
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sweep<1>(out, sms);
  sweep<2>(out, sms);
  sweep<4>(out, sms);
  sweep<8>(out, sms);
  sweep_smem<1>(out, sms);
  sweep_smem<2>(out, sms);
  sweep_smem<4>(out, sms);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
