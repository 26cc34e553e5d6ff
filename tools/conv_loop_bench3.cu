// Core-loop variants at low occupancy (1 warp per SMSP) and full occupancy: the dependent
// FMA distance of the sliding-window loop decides how much one warp can issue.
//   V0: conv_chunk_padded as in pc_tiled.cu (compiler-scheduled)
//   V1: the same with every FMA an `asm volatile` fma.rn.f64 (program order kept: tap-major,
//       so acc[i] is re-used only T FMAs later)
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1201_3018_b200/csrc/pc_device.cuh"
using namespace pc;

__device__ __forceinline__ double vfma(double a, double b, double c) {
  double d;
  asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c));
  return d;
}

template <int T, int V>
__device__ __forceinline__ void core(uint32_t xs_row, uint32_t kr_addr, int n_taps, double (&acc)[T]) {
  double win[T];
#pragma unroll
  for (int c = 0; c < T - 1; ++c) win[c] = lds64(xs_row + 8u * c);
  uint32_t xa = xs_row, ka = kr_addr;
  for (int j0 = 0; j0 < n_taps; j0 += T, xa += 8u * (T + 1), ka += 8u * T) {
    double kk[T];
#pragma unroll
    for (int u = 0; u < T; u += 2) {
      const double2 k2 = lds128(ka + 8u * u);
      kk[u] = k2.x;
      kk[u + 1] = k2.y;
    }
#pragma unroll
    for (int u = 0; u < T; ++u) {
      win[(T - 1 + u) % T] = lds64(xa + 8u * (((T - 1 + u) / T) * (T + 1) + (T - 1 + u) % T));
#pragma unroll
      for (int i = 0; i < T; ++i) {
        if (V == 0) acc[i] = fma(win[(i + u) % T], kk[u], acc[i]);
        else acc[i] = vfma(win[(i + u) % T], kk[u], acc[i]);
      }
    }
  }
}


// V2: the T new words of iteration j0+T are loaded at the start of iteration j0 (a full
// iteration of latency cover), taps one pair ahead; registers: acc T + window T + next T.
template <int T>
__device__ __forceinline__ void core_v2(uint32_t xs_row, uint32_t kr_addr, int n_taps, double (&acc)[T]) {
  double win[T], nxt[T];
#pragma unroll
  for (int c = 0; c < T - 1; ++c) win[c] = lds64(xs_row + 8u * c);
  // new words of iteration 0: x[T-1+u]
#pragma unroll
  for (int u = 0; u < T; ++u) nxt[u] = lds64(xs_row + 8u * (((T - 1 + u) / T) * (T + 1) + (T - 1 + u) % T));
  uint32_t xa = xs_row, ka = kr_addr;
  double2 kp = lds128(ka);
  for (int j0 = 0; j0 < n_taps; j0 += T, xa += 8u * (T + 1), ka += 8u * T) {
    double cur[T];
#pragma unroll
    for (int u = 0; u < T; ++u) cur[u] = nxt[u];
    if (j0 + T < n_taps) {
#pragma unroll
      for (int u = 0; u < T; ++u)
        nxt[u] = lds64(xa + 8u * (T + 1) + 8u * (((T - 1 + u) / T) * (T + 1) + (T - 1 + u) % T));
    }
#pragma unroll
    for (int u = 0; u < T; ++u) {
      const double k = (u & 1) ? kp.y : kp.x;
      if (u & 1) kp = lds128(ka + 8u * (u + 1));     // next pair (the last one reads the next iteration's)
      win[(T - 1 + u) % T] = cur[u];
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = fma(win[(i + u) % T], k, acc[i]);
    }
  }
}

template <int T, int V, int NREG>
__global__ void __maxnreg__(NREG) loop_kernel(int K_pad, int rows, int groups, int reps, double* out) {
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
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = 0.0;
      if (V == 2) core_v2<T>(smem_u32(xs) + 8u * (T + 1) * g, smem_u32(kr), K_pad, acc);
      else core<T, V>(smem_u32(xs) + 8u * (T + 1) * g, smem_u32(kr), K_pad, acc);
#pragma unroll
      for (int i = 0; i < T; ++i) tot += acc[i];
    }
  if (tot == 123.456) out[threadIdx.x] = tot;
}

template <int T, int V, int NREG>
void run(int threads, int K, double* dout, int sms) {
  const int K_pad = (K + T - 1) / T * T;
  const int groups = threads;
  const int rows = groups + K_pad / T + 2;
  const size_t smem = (size_t)((T + 1) * rows + K_pad) * 8;
  auto kfn = loop_kernel<T, V, NREG>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  const int reps = 20, grid = sms;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kfn<<<grid, threads, 120000>>>(K_pad, rows, groups, 2, dout);
  cudaEventRecord(a);
  kfn<<<grid, threads, 120000>>>(K_pad, rows, groups, reps, dout);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fma = (double)grid * groups * T * K_pad * reps;
  printf("V%d T=%2d nreg=%3d warps/SMSP=%d K=%d: %.2f T DFMA/s (%.1f%% of 18.6 nominal)\n", V, T, NREG, threads / 128,
         K_pad, fma / ms / 1e9, 100 * fma / ms / 1e9 / 18.6);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout;
  cudaMalloc(&dout, 8192 * 8);
  for (int th : {128, 256, 384, 512}) {
    run<14, 0, 128>(th, 513, dout, sms);
    run<14, 2, 128>(th, 513, dout, sms);
    run<16, 0, 128>(th, 513, dout, sms);
    run<16, 2, 128>(th, 513, dout, sms);
  }
  return 0;
}
