// Does a DMMA-saturated SM slow down a co-resident memory-bound warp?  One CTA per SM, 512
// threads: warps 0-3 ("producers") run batches of 16 independent 16-byte global loads
// followed by integer (or FP64) max work; warps 4-15 ("consumers") run one of
//   0: nothing        1: DMMA from registers   2: DMMA fed by LDS.64 (the tiled core's mix)
//   3: DFMA chains    4: DMMA from registers, 1 of the 3 consumer warps per SMSP only
// and we report the producers' cycles per batch (clock64) next to the consumers' work rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_interference tools/dmma_interference.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(512, 1)
probe(const double2* __restrict__ src, long long n2, int batches, int mode, int fp64_prod, volatile int* stop,
      unsigned long long* out) {
  __shared__ double sx[6144];
  for (int i = threadIdx.x; i < 6144; i += 512) sx[i] = (i & 255) * 0.5;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) {
    unsigned long long m = 0;
    double md = 0.0;
    long long base = ((long long)blockIdx.x * 4 + warp) * 4096;
    const long long t0 = clock64();
    for (int b = 0; b < batches; ++b) {
      double2 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldg(src + ((base + u * 32 + lane) % n2));
      if (fp64_prod) {
#pragma unroll
        for (int u = 0; u < 16; ++u) md = fmax(md, fmax(fabs(v[u].x), fabs(v[u].y)));
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const unsigned long long a = (unsigned long long)__double_as_longlong(v[u].x) & 0x7fffffffffffffffull;
          const unsigned long long c = (unsigned long long)__double_as_longlong(v[u].y) & 0x7fffffffffffffffull;
          m = a > m ? a : m;
          m = c > m ? c : m;
        }
      }
      base += 16 * 32 * 148 * 4;
    }
    const long long t1 = clock64();
    if (lane == 0) {
      out[(blockIdx.x * 4 + warp) * 2] = t1 - t0;
      out[(blockIdx.x * 4 + warp) * 2 + 1] = m + (md > 1e300 ? 1 : 0);
    }
    __syncwarp();
    if (threadIdx.x == 0) *stop = 1;   // consumers run until the producers are done
    return;
  }
  if (mode == 0) return;
  if (mode == 4 && warp >= 8) return;
  if ((mode == 5 || mode >= 6) && warp >= 12) return;
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = i;
  double a = lane * 1e-3, bb = 0.5;
  unsigned long long work = 0;
  const int r = lane >> 2, k = lane & 3;
  while (*stop == 0) {
    for (int it = 0; it < 64; ++it) {
      if (mode == 1 || mode == 4 || mode == 5) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, bb);
      } else if (mode >= 6) {                      // 2 warps/SMSP, a short sleep after every 8 DMMAs
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, bb);
        __nanosleep(mode == 6 ? 20 : (mode == 7 ? 60 : 150));
      } else if (mode == 2) {
        const double* xb = sx + (warp & 3) * 1024 + r * 20 + k + (it & 7) * 20;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          double av[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) av[t] = xb[t * 160 + 4 * s];
          const double bv = sx[4096 + ((it * 16 + 4 * s + k - r + 64) & 1023)];
#pragma unroll
          for (int t = 0; t < 4; ++t) dmma(acc[2 * t + s][0], acc[2 * t + s][1], av[t], bv);
        }
      } else {
#pragma unroll
        for (int rep = 0; rep < 8; ++rep)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i][0] = fma(acc[i][0], a, bb);
      }
    }
    work += 64;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = work;
  if (lane == 0 && warp == 4) atomicAdd(&out[148 * 4 * 2 + 1], work);   // DMMA batches of warp 4 per CTA
}

int main() {
  const long long n2 = 1LL << 23;   // 128 MB of double2
  double2* src;
  cudaMalloc(&src, n2 * sizeof(double2));
  cudaMemset(src, 0, n2 * sizeof(double2));
  int* stop;
  cudaMalloc(&stop, 4);
  unsigned long long* out;
  cudaMalloc(&out, (148 * 4 * 2 + 2) * 8);
  unsigned long long h[148 * 4 * 2 + 2];
  const char* names[] = {"no consumers", "DMMA (registers), 3 warps/SMSP", "DMMA + LDS.64 (core mix)",
                         "DFMA chains, 3 warps/SMSP", "DMMA (registers), 1 warp/SMSP",
                         "DMMA (registers), 2 warps/SMSP", "2 warps/SMSP, sleep 20 ns / 8 DMMA",
                         "2 warps/SMSP, sleep 60 ns / 8 DMMA", "2 warps/SMSP, sleep 150 ns / 8 DMMA"};
  for (int fp : {0, 1})
    for (int mode = 0; mode < 9; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(stop, 0, 4);
        cudaMemset(out + 148 * 4 * 2, 0, 16);
        probe<<<148, 512>>>(src, n2, 64, mode, fp, stop, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double tot = 0;
      for (int i = 0; i < 148 * 4; ++i) tot += (double)h[2 * i];
      printf("producer max %s | consumers: %-36s: %.0f cycles per batch of 16 x LDG.128 (+ %s max); "
             "warp-4 DMMA per producer batch-time: %.2f\n",
             fp ? "FP64" : "int ", names[mode], tot / (148 * 4) / 64, fp ? "FP64" : "integer",
             (double)h[148 * 4 * 2 + 1] * 64 * 8 / 148 / (tot / (148 * 4)) * 16);
    }
  return 0;
}
