// Cost of one job's companding + packing (pack_window, raw block in shared memory, cfg2 asym2
// geometry: 4096-sample block, 513 taps, T = 16, pitch 20) by the four producer warps of the
// persistent kernel, with 0 / 1 / 2 DMMA-issuing warps per SM sub-partition alongside, for the
// FP64 form and the integer/FP32 form (ModeP::alu_pack).  Reports cycles per job (clock64).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/pack_probe tools/pack_probe.cu
#include "../paper_1201_3018_b200/csrc/pc_tiled.cu"

namespace pc {
__device__ __forceinline__ void dmma_p(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(512, 1) pack_probe(Geo g, ModeP mp, int alu, int mode, int jobs, volatile int* stop,
                                                     unsigned long long* out) {
  extern __shared__ __align__(16) double sm[];
  double* raw = sm;                                  // 4096 samples
  double* xs = sm + 4096;                            // stage
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += 512) {
    const unsigned h = (unsigned)i * 2654435761u;
    raw[i] = ((double)(h >> 8) / 16777216.0 - 0.5) * 1.7;
  }
  __syncthreads();
  const Blk b = block_info<PACK_ASYM2>(g, mp.K, 1);
  const int rows_s = (b.M_out + mp.K - 1 + 15) / 16 + 1;
  if (warp < 4) {
    const double c_s = 511.0 / 0.85;
    const long long t0 = clock64();
    for (int j = 0; j < jobs; ++j) {
      pack_window<PACK_ASYM2, 16, 1, 20, true>(g, b, mp, raw, 4096, c_s, 0, rows_s, xs, threadIdx.x, 128, alu != 0);
      named_bar(8, 128);
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 4 + warp] = (unsigned long long)(t1 - t0);
    named_bar(8, 128);
    if (threadIdx.x == 0) *stop = 1;
    return;
  }
  if (mode == 0) return;
  if (mode == 1 && warp >= 8) return;
  if (mode == 2 && warp >= 12) return;
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = i;
  const double a = lane * 1e-3, bb = 0.5;
  while (*stop == 0) {
    for (int it = 0; it < 64; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma_p(acc[i][0], acc[i][1], a, bb);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = 1;
}
}  // namespace pc

int main() {
  using namespace pc;
  Geo g{};
  g.L = 1 << 22;
  g.N = 512;
  g.Np = 513;
  g.W_block = 4096;
  g.W = 4096 - 513 - 1;
  g.P = (g.L + g.W - 1) / g.W;
  g.mode = 0;
  ModeP mp{};
  mp.Q = 511.0;
  mp.b = 21;
  mp.eps = 1.0 / (double)(1 << 21);
  mp.eps_inv = (double)(1 << 21);
  mp.pow2 = 1;
  mp.exact_pack = 1;
  mp.K = 513;
  int* stop;
  cudaMalloc(&stop, 4);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 4 * 8);
  const int smem = (4096 + 3200) * 8;
  cudaFuncSetAttribute(pack_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* modes[] = {"alone", "1 DMMA warp/SMSP", "2 DMMA warps/SMSP"};
  unsigned long long h[148 * 4];
  for (int alu = 0; alu < 2; ++alu)
    for (int mode = 0; mode < 3; ++mode) {
      mp.alu_pack = alu;
      cudaMemset(stop, 0, 4);
      pack_probe<<<148, 512, smem>>>(g, mp, alu, mode, 16, stop, out);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        return 1;
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double tot = 0;
      for (int i = 0; i < 148 * 4; ++i) tot += (double)h[i];
      printf("pack_window %-22s | %-18s: %8.0f cycles per job (%.2f us at 1.965 GHz)\n",
             alu ? "integer/FP32 (alu)" : "FP64", modes[mode], tot / (148 * 4) / 16, tot / (148 * 4) / 16 / 1965.0);
    }
  return 0;
}
