// Microbenchmark of the direct-convolution inner loop variants on shared memory
// (no companding/packing): measures FP64 FMA/s of the core alone, to find the design
// that approaches the FP64 roofline before wiring it into pc_kernels.cu.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double c_taps[8192];

template <int T, int TAPSRC, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) loop_kernel(const double* __restrict__ ktaps, int K_pad, int rows, int groups,
                                                       int reps, double* out) {
  extern __shared__ double sm[];
  double* xs = sm;
  double* kr = sm + T * rows;
  for (int i = threadIdx.x; i < T * rows; i += blockDim.x) xs[i] = 1.0 + 1e-9 * i;
  for (int i = threadIdx.x; i < K_pad; i += blockDim.x) kr[i] = ktaps[i];
  __syncthreads();
  double tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
      double acc[T], win[T];
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = 0.0;
#pragma unroll
      for (int c = 0; c < T - 1; ++c) win[c] = xs[c * rows + g];
      const double* xcol = xs + g;
      for (int j0 = 0; j0 < K_pad; j0 += T) {
        const int r0 = j0 / T;
        double kk[T];
        if (TAPSRC == 0) {
#pragma unroll
          for (int u = 0; u < T; u += 2) {
            const double2 k2 = *reinterpret_cast<const double2*>(kr + j0 + u);
            kk[u] = k2.x;
            kk[u + 1] = k2.y;
          }
        } else {
#pragma unroll
          for (int u = 0; u < T; ++u) kk[u] = c_taps[j0 + u];
        }
#pragma unroll
        for (int u = 0; u < T; ++u) {
          win[(T - 1 + u) % T] = xcol[((T - 1 + u) % T) * rows + r0 + (T - 1 + u) / T];
#pragma unroll
          for (int i = 0; i < T; ++i) acc[i] = fma(win[(i + u) % T], kk[u], acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < T; ++i) tot += acc[i];
    }
  }
  if (tot == 123.456) out[threadIdx.x] = tot;
}

template <int T, int TAPSRC, int MAXT = 1024>
void run(int threads, int K, double* dk, double* dout, int sms) {
  const int K_pad = (K + T - 1) / T * T;
  const int groups = threads;   // one group per thread
  const int rows = groups + K_pad / T + 2;
  const size_t smem = (size_t)(T * rows + K_pad) * 8;
  auto kfn = loop_kernel<T, TAPSRC, MAXT>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem);
  const int reps = 20;
  const int grid = sms * occ;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kfn<<<grid, threads, smem>>>(dk, K_pad, rows, groups, 2, dout);
  cudaEventRecord(a);
  kfn<<<grid, threads, smem>>>(dk, K_pad, rows, groups, reps, dout);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fma = (double)grid * groups * T * K_pad * reps;
  printf("T=%2d taps=%s threads=%4d K=%4d occ=%d warps/SM=%2d: %.2f TFMA/s (%.1f%% of 17.0)  err=%s\n", T,
         TAPSRC ? "const" : "smem ", threads, K, occ, occ * threads / 32, fma / ms / 1e9, 100 * fma / ms / 1e9 / 17.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *dk, *dout;
  cudaMalloc(&dk, 8192 * 8);
  cudaMalloc(&dout, 8192 * 8);
  cudaMemset(dk, 0, 8192 * 8);
  double h[8192];
  for (int i = 0; i < 8192; ++i) h[i] = 1e-3 * (i % 7);
  cudaMemcpyToSymbol(c_taps, h, sizeof(h));
  cudaMemcpy(dk, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int K : {513, 257}) {
    for (int th : {128, 224, 256, 448, 512, 1024}) {
      run<8, 0>(th, K, dk, dout, sms);
      run<8, 1>(th, K, dk, dout, sms);
    }
    for (int th : {128, 256, 512}) {
      run<16, 0, 512>(th, K, dk, dout, sms);
      run<16, 1, 512>(th, K, dk, dout, sms);
      run<8, 0, 512>(th, K, dk, dout, sms);
      run<4, 0>(th, K, dk, dout, sms);
    }
  }
  return 0;
}
