/*
 * conv_example.c -- the C ABI of include/packedconv.h used from plain C (no Python, no torch):
 * a cfg2-shaped packed convolution (asymmetric M = 2, 10-bit companding, L1 range, dyadic eps)
 * through host buffers, checked against a direct double-precision convolution on the host.
 *
 *   gcc -O2 -I include examples/conv_example.c -o conv_example \
 *       -L /usr/local/cuda/lib64 -lcudart \
 *       -L paper_1201_3018_b200 -lpackedconv -Wl,-rpath,$PWD/paper_1201_3018_b200 -lm
 *   ./conv_example            (needs a B200; prints the SNR against full precision)
 *
 * Exit status 0 when the packed result is within the expected SNR, non-zero otherwise.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "packedconv.h"

/* The library allocates device memory itself; the kernel taps must be on the device for
 * conv_plan_set_kernel, so this example gets a device buffer through the CUDA runtime API
 * (declared here to keep the example free of CUDA headers). */
extern int cudaMalloc(void** p, size_t n);
extern int cudaMemcpy(void* dst, const void* src, size_t n, int kind);
extern int cudaFree(void* p);

static double lcg(unsigned long long* x) {   /* uniform [-1, 1) */
  *x = *x * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(*x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

int main(void) {
  const int64_t L = 1 << 16;
  const int32_t N = 511, W_block = 4096;
  double* s = (double*)malloc(sizeof(double) * L);
  double* k = (double*)malloc(sizeof(double) * N);
  double* r = (double*)malloc(sizeof(double) * (L + N - 1));
  unsigned long long seed = 12345;
  for (int64_t i = 0; i < L; ++i) s[i] = 0.5 * sin(0.01 * (double)i) + 0.1 * lcg(&seed);
  for (int32_t i = 0; i < N; ++i) k[i] = lcg(&seed) / (1.0 + 0.05 * fabs((double)i - N / 2));

  conv_opts o;
  conv_opts_default(&o);
  o.rmax_rule = PC_RMAX_L1;
  conv_plan* plan = NULL;
  int rc = conv_plan_create(&plan, L, N, W_block, PC_MODE_CONV, PC_PACK_ASYM2, 511, &o);
  if (rc) {
    fprintf(stderr, "conv_plan_create: %s\n", conv_status_string(rc));
    return 2;
  }
  void* k_dev = NULL;
  if (cudaMalloc(&k_dev, sizeof(double) * N) || cudaMemcpy(k_dev, k, sizeof(double) * N, 1 /* H2D */)) {
    fprintf(stderr, "cuda allocation failed\n");
    return 2;
  }
  rc = conv_plan_set_kernel(plan, (const double*)k_dev, NULL);
  if (rc == PC_OK) rc = conv_execute_host(plan, s, r, NULL);
  if (rc) {
    fprintf(stderr, "packed convolution: %s\n", conv_status_string(rc));
    return 3;
  }
  conv_plan_info info;
  conv_plan_query(plan, &info);
  double sig = 0.0, err = 0.0;
  for (int64_t m = 0; m < L + N - 1; ++m) {   /* direct convolution, Eq. (1) */
    double y = 0.0;
    for (int32_t n = 0; n < N; ++n)
      if (m - n >= 0 && m - n < L) y += s[m - n] * k[n];
    sig += y * y;
    err += (y - r[m]) * (y - r[m]);
  }
  const double snr = 10.0 * log10(sig / err);
  printf("asym2 Q=511: R_max %lld, eps 2^-%d, SNR vs full precision %.2f dB\n", (long long)info.R_max, info.eps_b, snr);
  conv_plan_destroy(plan);
  cudaFree(k_dev);
  free(s);
  free(k);
  free(r);
  return snr > 40.0 ? 0 : 1;
}
