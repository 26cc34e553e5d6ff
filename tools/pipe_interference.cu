// Which instruction classes of a "producer" warp slow down next to DMMA-issuing warps on the same
// SM sub-partition?  One CTA per SM, 512 threads: warps 0-3 (one per SMSP) run N iterations of a
// kernel of independent chains of one instruction class; warps 4-15 run, per mode,
//   0: nothing   1: DMMA from registers, 2 warps per SMSP   2: the same, 3 warps per SMSP
//   3: DFMA chains, 3 warps per SMSP   4: DMMA from registers, 1 warp per SMSP
// and we report the producers' cycles per iteration (clock64).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pipe_interference tools/pipe_interference.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1201_3018_b200/csrc/pc_intfp.cuh"

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int KIND>
__device__ __forceinline__ unsigned long long prod_iter(double (&d)[8], float (&f)[8], unsigned (&u)[8],
                                                        unsigned long long (&l)[8], const double* sx, int it) {
  if (KIND == 0) {                      // FP64 multiply-add chains
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = fma(d[i], 1.0000001, 1e-9);
  } else if (KIND == 1) {               // FP32 FMA chains
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], 1.0000001f, 1e-9f);
  } else if (KIND == 2) {               // 32-bit integer add / logic
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = (u[i] + 0x9e3779b9u) ^ (u[i] >> 3);
  } else if (KIND == 3) {               // 32-bit IMAD
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = u[i] * 2654435761u + 12345u;
  } else if (KIND == 4) {               // 64-bit multiply
#pragma unroll
    for (int i = 0; i < 8; ++i) l[i] = l[i] * 0x9e3779b97f4a7c15ull + 1;
  } else if (KIND == 5) {               // shared-memory loads
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] += sx[(threadIdx.x * 8 + i * 256 + it * 8) & 4095];
  } else if (KIND == 6) {               // the FP32 fast companding of 8 samples
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float y = __fmul_rn(f[i], 437.25f);
      const float r = __fadd_rn(y, 12582912.0f);
      const float dd = __fsub_rn(y, __fsub_rn(r, 12582912.0f));
      u[i] += (__float_as_int(r) - 0x4B400000) + (fabsf(dd) > 0.4995f ? 1u : 0u);
      f[i] = __int_as_float((u[i] & 0x7fffff) | 0x3f000000);
    }
  } else if (KIND == 7) {               // FP64 companding (round(c x)) of 8 samples
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = round(__dmul_rn(d[i], 437.25)) * 1e-3 + 0.25;
  } else if (KIND == 9) {               // shared-memory 16-byte loads
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double2 v = reinterpret_cast<const double2*>(sx)[(threadIdx.x * 4 + i * 128 + it * 4) & 2047];
      d[i] += v.x + v.y;
    }
  } else if (KIND == 10) {              // shared-memory 16-byte stores (independent)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      reinterpret_cast<double2*>(const_cast<double*>(sx))[((threadIdx.x & 127) * 4 + i * 512 + it * 4) & 2047] =
          make_double2(d[i], (double)u[i]);
  } else if (KIND == 11) {              // FP32 min/max + compare + select
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      f[i] = fmaxf(fabsf(f[i] - 0.25f), fabsf(f[i] + 0.125f)) * 0.999f;
      u[i] += f[i] > 0.3f ? 1u : 0u;
    }
  } else if (KIND == 12) {              // 64-bit shifts / selects (the integer packing's word assembly)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int sh = (int)(u[i] & 31u);
      l[i] = ((l[i] << sh) | (l[i] >> (64 - sh - 1))) ^ (l[i] >> 7);
      u[i] += (unsigned)(l[i] >> 40);
    }
  } else if (KIND == 8) {               // exact integer companding of 8 samples
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      long long n;
      bool z;
      pc::ifp::compand_int(0x407b540000000000ull, l[i], n, z);
      l[i] = (l[i] ^ (unsigned long long)n) & 0x3fefffffffffffffull | 0x3fe0000000000000ull;
    }
  }
  return 0;
}

template <int KIND>
__global__ void __launch_bounds__(512, 1) probe(int iters, int mode, volatile int* stop, unsigned long long* out) {
  __shared__ __align__(16) double sx[4096];
  for (int i = threadIdx.x; i < 4096; i += 512) sx[i] = (i & 255) * 0.5;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) {
    double d[8];
    float f[8];
    unsigned u[8];
    unsigned long long l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      d[i] = 0.5 + i * 0.01 + lane * 1e-4;
      f[i] = 0.5f + i * 0.01f;
      u[i] = i * 77 + lane;
      l[i] = 0x3fe0000000000000ull + i * 12345 + lane;
    }
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) prod_iter<KIND>(d, f, u, l, sx, it);
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i] + f[i] + u[i] + (double)l[i];
    if (lane == 0) out[blockIdx.x * 4 + warp] = t1 - t0;
    if (s == 1.2345) out[0] = 0;
    __syncwarp();
    if (threadIdx.x == 0) *stop = 1;
    return;
  }
  if (mode == 0) return;
  if (mode == 1 && warp >= 12) return;           // 2 consumer warps per SMSP
  if (mode == 4 && warp >= 8) return;            // 1 consumer warp per SMSP
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = i;
  double a = lane * 1e-3, bb = 0.5;
  while (*stop == 0) {
    for (int it = 0; it < 64; ++it) {
      if (mode <= 2 || mode == 4) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, bb);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][0] = fma(acc[i][0], a, bb);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = 1;
}

template <int KIND>
void run(const char* name, int iters, int* stop, unsigned long long* out) {
  const char* modes[] = {"alone", "2 DMMA warps/SMSP", "3 DMMA warps/SMSP", "3 DFMA warps/SMSP", "1 DMMA warp/SMSP"};
  unsigned long long h[148 * 4];
  for (int mode = 0; mode < 5; ++mode) {
    double best = 1e30;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(stop, 0, 4);
      probe<KIND><<<148, 512>>>(iters, mode, stop, out);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error\n");
        return;
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double tot = 0;
      for (int i = 0; i < 148 * 4; ++i) tot += (double)h[i];
      best = tot / (148 * 4) / iters < best ? tot / (148 * 4) / iters : best;
    }
    printf("%-34s | %-20s: %8.1f cycles per iteration (8 independent ops)\n", name, modes[mode], best);
  }
}

int main() {
  int* stop;
  cudaMalloc(&stop, 4);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 4 * 8);
  run<0>("FP64 DFMA", 4096, stop, out);
  run<1>("FP32 FFMA", 4096, stop, out);
  run<2>("INT32 IADD/LOP", 4096, stop, out);
  run<3>("INT32 IMAD", 4096, stop, out);
  run<4>("INT64 multiply", 4096, stop, out);
  run<5>("LDS.64", 4096, stop, out);
  run<6>("FP32 fast companding", 4096, stop, out);
  run<7>("FP64 companding round(c x)", 4096, stop, out);
  run<8>("exact integer companding", 1024, stop, out);
  run<9>("LDS.128", 4096, stop, out);
  run<10>("STS.128", 4096, stop, out);
  run<11>("FP32 min/max/compare", 4096, stop, out);
  run<12>("64-bit shifts", 4096, stop, out);
  return 0;
}
