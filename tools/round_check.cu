// Checks pc_device.cuh's round_away (PC_RND_ADD = 1: add-based round half away from zero) against
// the host's round() on exact ties, neighbours of ties, signed zeros, the 2^51 guard and 2^26
// hashed values.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -DPC_RND_ADD=1 -o tools/round_check tools/round_check.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1201_3018_b200/csrc/pc_device.cuh"
__global__ void rk(const double* x, double* y, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = pc::round_away(x[i]);
}
static uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull; z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
int main() {
  std::vector<double> h;
  const double specials[] = {0.0, -0.0, 0.5, -0.5, 0.49999999999999994, -0.49999999999999994, 1.5, 2.5, -2.5,
                             2251799813685247.5, 2251799813685248.0, 2251799813685248.5, -2251799813685247.5,
                             4503599627370495.5, 4503599627370497.0, 9007199254740993.0, 1e300, -1e300,
                             INFINITY, -INFINITY, 4.9e-324, -4.9e-324, 2.2250738585072014e-308};
  for (double s : specials) h.push_back(s);
  for (int k = 0; k < (1 << 20); ++k) {                    // ties and their neighbours at many magnitudes
    const double t = (double)(mix(k) % (1ull << (k % 50))) + 0.5;
    for (double s : {t, -t, std::nextafter(t, 0.0), std::nextafter(t, 1e308), -std::nextafter(t, 0.0), -std::nextafter(t, 1e308)})
      h.push_back(s);
  }
  for (uint64_t k = 0; k < (1ull << 26); ++k) {            // hashed bit patterns, exponents up to 2^60
    uint64_t b = mix(k ^ 0xabcdefull);
    const uint64_t e = 1023 - 30 + (b >> 58) % 90;
    b = (b & 0x800fffffffffffffull) | (e << 52);
    double v; std::memcpy(&v, &b, 8); h.push_back(v);
  }
  const size_t n = h.size();
  double *dx, *dy;
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8);
  cudaMemcpy(dx, h.data(), n * 8, cudaMemcpyHostToDevice);
  rk<<<1184, 256>>>(dx, dy, n);
  std::vector<double> g(n);
  if (cudaMemcpy(g.data(), dy, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) { printf("cuda error\n"); return 2; }
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) {
    const double r = std::round(h[i]);
    if (std::memcmp(&r, &g[i], 8) != 0 && ++bad <= 10) printf("mismatch x=%a host=%a gpu=%a\n", h[i], r, g[i]);
  }
  printf("round_check: %zu values, %zu mismatches (PC_RND_ADD=%d)\n", n, bad, PC_RND_ADD);
  return bad != 0;
}
