// Standalone rate of the tiled kernel's DMMA core loop (conv_chunk_mma from pc_tiled.cu) with
// 1..3 warps per SM sub-partition, each warp on its own 32-group part of a 16-row-pitch-20
// window in shared memory, 528 taps (cfg2 asym2), NMT = 4.  Reports DMMA-pipe utilisation.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1201_3018_b200/csrc \
//        -o tools/mma_core_bench tools/mma_core_bench.cu
#include "pc_tiled.cu"

namespace pc {
// variants of conv_chunk_mma: UNR = jj unroll, NTM = issue order n-tile-major, NOLD = no loads in the loop
template <int NMT, int PT, int UNR, int NTM, int NOLD>
__device__ __forceinline__ void core_v(uint32_t xs_row, uint32_t kc_addr, int jj_n, double (&fr)[4][2][2], int lane) {
  const int r = lane >> 2, k = lane & 3;
  uint32_t xa = xs_row + 8u * (uint32_t)(r * PT + k);
  uint32_t ka = kc_addr + 8u * (uint32_t)(k - r) - 64u;
  double b[6], bn[4], a[NMT], an[NMT];
#pragma unroll
  for (int f = 0; f < 6; ++f) b[f] = lds64(ka + 32u * f);
#pragma unroll
  for (int mt = 0; mt < NMT; ++mt) a[mt] = lds64(xa + 8u * (8 * mt * PT));
#pragma unroll UNR
  for (int jj = 0; jj < jj_n; ++jj, xa += 8u * PT, ka += 128u) {
    const bool more = jj + 1 < jj_n;
    if (more && !NOLD) {
#pragma unroll
      for (int f = 0; f < 4; ++f) bn[f] = lds64(ka + 128u + 32u * (f + 2));
    } else {
#pragma unroll
      for (int f = 0; f < 4; ++f) bn[f] = b[f + 2];
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if ((s < 3 || more) && !NOLD) {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt)
          an[mt] = lds64(xa + 8u * (8 * mt * PT) + (s < 3 ? 32u * (s + 1) : 8u * PT));
      } else {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) an[mt] = a[(mt + 1) % NMT];
      }
      if (NTM) {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) dmma884(fr[mt][0], a[mt], b[s + 2]);
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) dmma884(fr[mt][1], a[mt], b[s]);
      } else {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) {
          dmma884(fr[mt][0], a[mt], b[s + 2]);
          dmma884(fr[mt][1], a[mt], b[s]);
        }
      }
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) a[mt] = an[mt];
    }
    b[0] = b[4];
    b[1] = b[5];
#pragma unroll
    for (int f = 0; f < 4; ++f) b[f + 2] = bn[f];
  }
}

// Two independent jj streams (taps split in halves) interleaved k-step by k-step: 16 accumulator
// chains per warp instead of 8, so one warp can cover the DMMA latency.
template <int NMT, int PT, int NOLD>
__device__ __forceinline__ void core_dual(uint32_t xs_row, uint32_t kc_addr, int jj_n, double (&fr)[4][2][2],
                                          double (&fq)[4][2][2], int lane) {
  const int r = lane >> 2, k = lane & 3;
  const int h = jj_n / 2;
  uint32_t xa = xs_row + 8u * (uint32_t)(r * PT + k);
  uint32_t ka = kc_addr + 8u * (uint32_t)(k - r) - 64u;
  uint32_t xb = xa + 8u * PT * h, kb = ka + 128u * h;
  double b[6], bn[4], a[NMT], an[NMT], c[6], cn[4], d[NMT], dn[NMT];
#pragma unroll
  for (int f = 0; f < 6; ++f) { b[f] = lds64(ka + 32u * f); c[f] = lds64(kb + 32u * f); }
#pragma unroll
  for (int mt = 0; mt < NMT; ++mt) { a[mt] = lds64(xa + 8u * (8 * mt * PT)); d[mt] = lds64(xb + 8u * (8 * mt * PT)); }
#pragma unroll 1
  for (int jj = 0; jj < h; ++jj, xa += 8u * PT, ka += 128u, xb += 8u * PT, kb += 128u) {
    if (!NOLD) {
#pragma unroll
      for (int f = 0; f < 4; ++f) { bn[f] = lds64(ka + 128u + 32u * (f + 2)); cn[f] = lds64(kb + 128u + 32u * (f + 2)); }
    } else {
#pragma unroll
      for (int f = 0; f < 4; ++f) { bn[f] = b[f + 2]; cn[f] = c[f + 2]; }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (!NOLD) {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) {
          an[mt] = lds64(xa + 8u * (8 * mt * PT) + (s < 3 ? 32u * (s + 1) : 8u * PT));
          dn[mt] = lds64(xb + 8u * (8 * mt * PT) + (s < 3 ? 32u * (s + 1) : 8u * PT));
        }
      } else {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) { an[mt] = a[(mt + 1) % NMT]; dn[mt] = d[(mt + 1) % NMT]; }
      }
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) {
        dmma884(fr[mt][0], a[mt], b[s + 2]);
        dmma884(fq[mt][0], d[mt], c[s + 2]);
        dmma884(fr[mt][1], a[mt], b[s]);
        dmma884(fq[mt][1], d[mt], c[s]);
      }
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) { a[mt] = an[mt]; d[mt] = dn[mt]; }
    }
    b[0] = b[4]; b[1] = b[5]; c[0] = c[4]; c[1] = c[5];
#pragma unroll
    for (int f = 0; f < 4; ++f) { b[f + 2] = bn[f]; c[f + 2] = cn[f]; }
  }
}

template <int V>
__global__ void __launch_bounds__(512, 1) core_bench(int reps, int jj_n, double* out) {
  extern __shared__ __align__(128) double sm[];
  constexpr int PT = 20;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* taps = sm;                                 // 16 + 528 + 16
  double* win = sm + 576;                            // per warp-slot (4): (32 + 34) rows of pitch 20
  for (int i = threadIdx.x; i < 576 + 4 * 66 * PT; i += blockDim.x) sm[i] = (i % 61) * 0.25 - 7.0;
  __syncthreads();
  double fr[4][2][2], fq[4][2][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int q = 0; q < 4; ++q) fr[mt][q >> 1][q & 1] = fq[mt][q >> 1][q & 1] = 0.0;
  const uint32_t xrow = smem_u32(win + (warp & 3) * 66 * PT);
  for (int r = 0; r < reps; ++r) {
    if (V == 0) conv_chunk_mma<4, PT>(xrow, smem_u32(taps + 16), jj_n, fr, lane);
    if (V == 1) core_v<4, PT, 2, 0, 0>(xrow, smem_u32(taps + 16), jj_n, fr, lane);
    if (V == 2) core_v<4, PT, 1, 1, 0>(xrow, smem_u32(taps + 16), jj_n, fr, lane);
    if (V == 3) core_v<4, PT, 2, 1, 0>(xrow, smem_u32(taps + 16), jj_n, fr, lane);
    if (V == 4) core_v<4, PT, 1, 0, 1>(xrow, smem_u32(taps + 16), jj_n, fr, lane);
    if (V == 5) core_v<2, PT, 2, 1, 0>(xrow, smem_u32(taps + 16), jj_n, fr, lane);
    if (V == 6) core_dual<4, PT, 0>(xrow, smem_u32(taps + 16), jj_n, fr, fq, lane);
    if (V == 7) core_dual<4, PT, 1>(xrow, smem_u32(taps + 16), jj_n, fr, fq, lane);
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int q = 0; q < 4; ++q) fr[mt][q >> 1][q & 1] += fq[mt][q >> 1][q & 1];
  double s = 0;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int q = 0; q < 4; ++q) s += fr[mt][q >> 1][q & 1];
  if (s == 1.2345) out[threadIdx.x] = s;
}
}  // namespace pc

int main() {
  double* out;
  cudaMalloc(&out, 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (576 + 4 * 66 * 20) * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int jj_n = 34, reps = 200;
  auto kern = [&](int v) {
    void (*f)(int, int, double*) = v == 0 ? pc::core_bench<0> : v == 1 ? pc::core_bench<1> : v == 2 ? pc::core_bench<2>
                                 : v == 3 ? pc::core_bench<3> : v == 4 ? pc::core_bench<4> : v == 5 ? pc::core_bench<5>
                                 : v == 6 ? pc::core_bench<6> : pc::core_bench<7>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return f;
  };
  const char* vn[] = {"pc_tiled conv_chunk_mma", "jj unroll 2", "n-tile-major order", "unroll 2 + n-tile-major",
                      "no loads (ceiling)", "NMT=2 unroll2 ntm", "dual jj streams", "dual streams no loads"};
  for (int v = 0; v < 8; ++v)
  for (int wps : {1, 2}) {
    const int threads = 128 * wps;
    auto f = kern(v);
    f<<<sms, threads, smem>>>(2, jj_n, out);
    cudaEventRecord(e0);
    f<<<sms, threads, smem>>>(reps, jj_n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma = (double)sms * 4 * wps * reps * (v >= 6 ? 2 * (jj_n / 2) : jj_n) * (v == 5 ? 16 : 32);
    printf("%-26s ", vn[v]);
    const double fma = dmma * 256;
    printf("warps/SMSP=%d: %.2f TFMA/s (%.1f%% of 18.56 DMMA peak), %.1f cycles per DMMA per SMSP at 1.965 GHz\n",
           wps, fma / ms / 1e9, 100.0 * fma / ms / 1e9 / 18.56, ms * 1e-3 * 1.965e9 / (dmma / sms / 4));
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
