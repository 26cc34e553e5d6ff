// pc_fft.cu -- FFT overlap-save core (SURVEY §8(a) a5 for config 3; "any off-the-shelf
// core", P:127 frequency-domain FLOP model).  Hand-written FP64 FFT in shared memory; no cuFFT.
//
// One CTA per (signal, block, part) job.  The packed core words of the part's window (real,
// length 2N) are loaded as N complex points z[n] = x[2n] + i x[2n+1]; a radix-16 Stockham FFT
// (all 16 points of a butterfly in registers, read-all / sync / write-all passes, so no
// ping-pong buffer: N = 8192 complex fits in 139 KB with one pad element per 16) transforms
// them; the real-FFT split/merge is fused with the product by the precomputed spectrum H of
// the core taps (H[k], k = 0..N, of the 2N-point real transform); the inverse transform
// yields the circular convolution p = x (*) h, whose entries p[m + K - 1] are the core
// outputs out[m] = sum_j x[m + j] kr[j] (kr = reversed taps).  The outputs are approximate;
// rounding to digits (unpacking) makes them exact integers as long as the FFT error stays
// below half an LSB -- monitored: the largest last-digit residual is kept per plan.
//
// Twiddles come from tables rounded once from long-double values on the host (recurrences
// break exactness at cfg3 sizes).
#include <cooperative_groups.h>

#include "pc_device.cuh"
#include "pc_kernels.h"

namespace cg = cooperative_groups;


#ifndef PC_FFT_PEAK_U
#define PC_FFT_PEAK_U 8
#endif
#ifndef PC_FFT_PACK_UB
#define PC_FFT_PACK_UB 8
#endif
#ifndef PC_FFT_CARVEOUT
#define PC_FFT_CARVEOUT 60   // % of the unified L1/shared array as shared memory
#endif

namespace pc {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse): sign = -1 forward
__device__ __forceinline__ double2 mul_i(double2 a, int sign) {
  return sign < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

// padded shared-memory index: one pad element every 16 (bank-conflict-free strided writes)
__device__ __forceinline__ int pidx(int e) { return e + (e >> 4); }

template <int SIGN>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
  const double2 s13 = cadd(a1, a3), d13 = mul_i(csub(a1, a3), SIGN);
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}

// exp(SIGN * 2 pi i m / 16), m = 0..9, correctly rounded constants
template <int SIGN>
__device__ __forceinline__ double2 w16(int m) {
  const double c1 = 0.92387953251128673848, s1 = 0.38268343236508978178;   // cos/sin(pi/8)
  const double r2 = 0.70710678118654752440;                                // cos/sin(pi/4)
  double c, s;
  switch (m) {
    case 0: c = 1.0; s = 0.0; break;
    case 1: c = c1; s = s1; break;
    case 2: c = r2; s = r2; break;
    case 3: c = s1; s = c1; break;
    case 4: c = 0.0; s = 1.0; break;
    case 5: c = -s1; s = c1; break;
    case 6: c = -r2; s = r2; break;
    case 7: c = -c1; s = s1; break;
    case 8: c = -1.0; s = 0.0; break;
    default: c = -c1; s = -s1; break;   // 9
  }
  return make_double2(c, SIGN * s);
}

// In-register DFT of 16 points (radix 4 x 4): v[q] <- sum_p v[p] exp(SIGN 2 pi i p q / 16)
template <int SIGN>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
#pragma unroll
  for (int p2 = 0; p2 < 4; ++p2) dft4<SIGN>(v[p2], v[4 + p2], v[8 + p2], v[12 + p2]);
  // v[4*q1 + p2] now holds a[p2][q1]; twiddle by W16^(p2 q1)
#pragma unroll
  for (int p2 = 1; p2 < 4; ++p2)
#pragma unroll
    for (int q1 = 1; q1 < 4; ++q1) v[4 * q1 + p2] = cmul(v[4 * q1 + p2], w16<SIGN>(p2 * q1));
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1) dft4<SIGN>(v[4 * q1 + 0], v[4 * q1 + 1], v[4 * q1 + 2], v[4 * q1 + 3]);
  // v[4*q1 + q2] holds X[q1 + 4 q2]; reorder to natural
  double2 t[16];
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) t[q1 + 4 * q2] = v[4 * q1 + q2];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = t[i];
}

template <int SIGN, int R>
__device__ __forceinline__ void dft_small(double2* v) {
  if (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if (R == 4) {
    dft4<SIGN>(v[0], v[1], v[2], v[3]);
  } else {   // R == 8: radix 2 x 4
    // a[p2][q1] = DFT4 over p1 of v[2 p1 + p2]
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<SIGN>(e0, e1, e2, e3);
    dft4<SIGN>(o0, o1, o2, o3);
    const double r2 = 0.70710678118654752440;
    o1 = cmul(o1, make_double2(r2, SIGN * r2));
    o2 = mul_i(o2, SIGN);
    o3 = cmul(o3, make_double2(-r2, SIGN * r2));
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1);
    v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2);
    v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3);
    v[7] = csub(e3, o3);
  }
}

// Twiddle sources: a correctly rounded global table, or (conv kernel) a two-level table in
// shared memory: w^m = hi[m >> 6] * lo[m & 63] with lo[b] = w^b, hi[a] = w^(64a) copied from
// the correctly rounded table (hi[0] = lo[0] = 1 exactly, so m < 64 or 64 | m are exact; else
// one complex product, <= ~1.5 ulp).  Shared-memory reads replace L1/L2 table loads, which
// were half of a pass's time.
struct TwGlobal {
  const double2* tw;
  __device__ __forceinline__ double2 operator()(int m) const { return __ldg(tw + m); }
};
struct TwSmem2 {
  const double2* lo;   // lo[b + (b >> 3)] = w^b: one pad entry per 8 (the pass-2 / pass-3 index sets
  const double2* hi;   // 16 (p k mod 4) and p j mod 64 hit one bank group without it)
  __device__ __forceinline__ double2 operator()(int m) const {
    const int b = m & 63;
    return cmul(hi[m >> 6], lo[b + (b >> 3)]);
  }
};
// The real-FFT split/merge twiddle W_k = exp(-2 pi i k / 2N), k <= N, from the N-point table:
// even k = 2m is w^m; odd k = 2m + 1 is w^m * exp(-pi i / N) (one more product).  Replaces a
// global-table load per pair (the product phase was bound by its table loads).
struct TwHalf {
  TwSmem2 t;
  double2 c1;                                        // exp(-pi i / N), correctly rounded
  int N;
  __device__ __forceinline__ double2 operator()(int k) const {
    if (k >= N) return make_double2(-1.0, 0.0);       // k = N: exp(-pi i)
    const double2 w = t(k >> 1);
    return (k & 1) ? cmul(w, c1) : w;
  }
};

}  // namespace

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// One radix-16 Stockham pass (sub-transform length LS before the pass).
template <int N, int SIGN, int LS, class TW>
__device__ __forceinline__ void stockham16(double2* s, const TW& tw) {
  constexpr int NB = N / 16;
  const int j = threadIdx.x;
  const int k = j & (LS - 1);
  double2 v[16];
#ifndef PC_FFT_TW_AFTER
  double2 w[16];
  if (LS > 1) {                                 // twiddle loads in flight across the barrier
    const int step = k * (N / (LS * 16));
#pragma unroll
    for (int p = 1; p < 16; ++p) w[p] = tw(p * step);
  }
#endif
#pragma unroll
  for (int p = 0; p < 16; ++p) v[p] = s[pidx(j + p * NB)];
  __syncthreads();
  if (LS > 1) {
#ifdef PC_FFT_TW_AFTER
    double2 w[16];
    const int step = k * (N / (LS * 16));
#pragma unroll
    for (int p = 1; p < 16; ++p) w[p] = tw(p * step);
#endif
#pragma unroll
    for (int p = 1; p < 16; ++p) {
      double2 wp = w[p];
      if (SIGN > 0) wp.y = -wp.y;
      v[p] = cmul(v[p], wp);
    }
  }
  dft16<SIGN>(v);
  const int ob = (j - k) * 16 + k;
#pragma unroll
  for (int q = 0; q < 16; ++q) s[pidx(ob + q * LS)] = v[q];
  __syncthreads();
}

// Final Stockham pass of radix R in {2, 4, 8} (16/R butterflies per thread).
template <int N, int SIGN, int LS, int R, class TW>
__device__ __forceinline__ void stockham_last(double2* s, const TW& tw) {
  constexpr int NB = N / 16, NBT = 16 / R;
  double2 v[16];
#pragma unroll
  for (int bb = 0; bb < NBT; ++bb)
#pragma unroll
    for (int p = 0; p < R; ++p) v[bb * R + p] = s[pidx(threadIdx.x + bb * NB + p * (N / R))];
  __syncthreads();
#pragma unroll
  for (int bb = 0; bb < NBT; ++bb) {
    const int j = threadIdx.x + bb * NB;
    const int k = j & (LS - 1);
    const int step = k * (N / (LS * R));
#pragma unroll
    for (int p = 1; p < R; ++p) {
      double2 w = tw(p * step);
      if (SIGN > 0) w.y = -w.y;
      v[bb * R + p] = cmul(v[bb * R + p], w);
    }
    dft_small<SIGN, R>(v + bb * R);
  }
#pragma unroll
  for (int bb = 0; bb < NBT; ++bb) {
    const int j = threadIdx.x + bb * NB;
    const int k = j & (LS - 1);
    const int ob = (j - k) * R + k;
#pragma unroll
    for (int q = 0; q < R; ++q) s[pidx(ob + q * LS)] = v[bb * R + q];
  }
  __syncthreads();
}

// In-place N-point complex DFT of s (padded layout) with blockDim.x == N/16 threads.
// SIGN = -1 forward, +1 inverse (unscaled).  tw[m] = exp(-2 pi i m / N), m < N.
// N = 16^P * R, R in {1, 2, 4, 8}: P radix-16 passes then one radix-R pass.
template <int N, int SIGN, class TW>
__device__ void fft_smem(double2* s, const TW& tw) {
  constexpr int LG = ilog2(N);
  constexpr int P = LG / 4, R = 1 << (LG % 4);
  static_assert(P >= 1 && P <= 3, "N in 2^10 .. 2^13");
  stockham16<N, SIGN, 1, TW>(s, tw);
  if (P >= 2) stockham16<N, SIGN, (P >= 2 ? 16 : 1), TW>(s, tw);
  if (P >= 3) stockham16<N, SIGN, (P >= 3 ? 256 : 1), TW>(s, tw);
  constexpr int LSF = (P == 1) ? 16 : (P == 2 ? 256 : 4096);
  if (R > 1) stockham_last<N, SIGN, LSF, (R > 1 ? R : 2), TW>(s, tw);
}

// Real-FFT split + product by H + merge for the inverse (see header comment):
// on entry s = Z = FFT_N(z); on exit s = Z' such that IFFT_N(Z') (unscaled) gives
// N * p packed as p[2n] + i p[2n+1]; the 1/N is folded in here.
template <int N, class TW2>
__device__ void spectrum_product(double2* s, const double2* __restrict__ H, const TW2& tw2) {
  const double sc = 1.0 / (double)N;   // exact (power of two)
  if (threadIdx.x == 0) {
    const double2 z0 = s[pidx(0)];
    const double X0 = z0.x + z0.y, XN = z0.x - z0.y;   // X[0], X[N] (real)
    const double2 P0 = make_double2(X0 * H[0].x, X0 * H[0].y);
    const double2 PN = make_double2(XN * H[N].x, XN * H[N].y);
    // Z'[0] = (P0 + conj PN)/2 + i (P0 - conj PN)/2
    const double2 e = make_double2(0.5 * (P0.x + PN.x), 0.5 * (P0.y - PN.y));
    const double2 o = make_double2(0.5 * (P0.x - PN.x), 0.5 * (P0.y + PN.y));
    s[pidx(0)] = make_double2((e.x - o.y) * sc, (e.y + o.x) * sc);
  }
  // k = 1 .. N/2 in rounds of UK per thread, every table and shared load of a round issued
  // before any use (the loop is latency-bound otherwise)
  constexpr int UK = 4;
  for (int k0 = 1 + threadIdx.x; k0 <= N / 2; k0 += UK * blockDim.x) {
    double2 Zk[UK], Zkp[UK], Wk[UK], Wkp[UK], Hk[UK], Hkp[UK];
#pragma unroll
    for (int u = 0; u < UK; ++u) {
      const int k = k0 + u * blockDim.x;
      const int kk = (k <= N / 2) ? k : N / 2;       // clamp (results of clamped lanes unused)
      const int kp = N - kk;
      Zk[u] = s[pidx(kk)];
      Zkp[u] = s[pidx(kp)];
      Wk[u] = tw2(kk);                                // exp(-2 pi i k / 2N)
      Wkp[u] = make_double2(-Wk[u].x, Wk[u].y);       // exp(-2 pi i (N-k) / 2N) = -conj(W_k)
      Hk[u] = __ldg(H + kk);
      Hkp[u] = __ldg(H + kp);
    }
#pragma unroll
    for (int u = 0; u < UK; ++u) {
      const int k = k0 + u * blockDim.x;
      if (k > N / 2) break;
      const int kp = N - k;
      // E[k] = (Z[k] + conj Z[k'])/2,  O[k] = -i/2 (Z[k] - conj Z[k'])
      const double2 Ek = make_double2(0.5 * (Zk[u].x + Zkp[u].x), 0.5 * (Zk[u].y - Zkp[u].y));
      const double2 Ok = make_double2(0.5 * (Zk[u].y + Zkp[u].y), -0.5 * (Zk[u].x - Zkp[u].x));
      const double2 Ekp = cconj(Ek), Okp = cconj(Ok);
      const double2 Xk = cadd(Ek, cmul(Wk[u], Ok));
      const double2 Xkp = cadd(Ekp, cmul(Wkp[u], Okp));
      const double2 Pk = cmul(Xk, Hk[u]), Pkp = cmul(Xkp, Hkp[u]);
      // Z'[k] = (P[k] + conj P[k'])/2 + i conj(W_k) (P[k] - conj P[k'])/2
      auto merge = [&](double2 a, double2 b, double2 W) {
        const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        const double2 d = make_double2(0.5 * (a.x - b.x), 0.5 * (a.y + b.y));
        const double2 o = cmul(d, cconj(W));
        return make_double2((e.x - o.y) * sc, (e.y + o.x) * sc);
      };
      const double2 Zpk = merge(Pk, Pkp, Wk[u]);
      const double2 Zpkp = merge(Pkp, Pk, Wkp[u]);
      s[pidx(k)] = Zpk;
      if (kp != k) s[pidx(kp)] = Zpkp;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ kernel spectrum (a1, FFT core)
// H = 2N-point real DFT of h[n] = kr[K-1-n] (n < K), k = 0..N.
template <int N>
__global__ void __launch_bounds__(N / 16) pc_fft_spectrum(const double* __restrict__ kr, int K,
                                                          const double2* __restrict__ tw,
                                                          const double2* __restrict__ tw2, double2* __restrict__ H) {
  extern __shared__ __align__(16) double2 sm[];
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    const int a = 2 * n, b = 2 * n + 1;
    sm[pidx(n)] = make_double2(a < K ? kr[K - 1 - a] : 0.0, b < K ? kr[K - 1 - b] : 0.0);
  }
  __syncthreads();
  fft_smem<N, -1>(sm, TwGlobal{tw});
  for (int k = threadIdx.x; k <= N; k += blockDim.x) {
    const double2 Zk = sm[pidx(k % N)], Zkp = sm[pidx((N - k) % N)];
    const double2 E = make_double2(0.5 * (Zk.x + Zkp.x), 0.5 * (Zk.y - Zkp.y));
    const double2 O = make_double2(0.5 * (Zk.y + Zkp.y), -0.5 * (Zk.x - Zkp.x));
    H[k] = cadd(E, cmul(__ldg(tw2 + k), O));
  }
}

// ------------------------------------------------------------------ the FFT-core conv kernel
template <int PACK, int N>
#ifndef PC_FFT_MINB
#define PC_FFT_MINB 2   // CTAs per SM the N <= 4096 transform is compiled for (register cap)
#endif
__global__ void __launch_bounds__(N / 16, (N <= 4096 ? PC_FFT_MINB : 1)) pc_fft_conv_kernel(Geo g, Exec e, FftArgs f) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ double red[32];
  const ModeP& mp = e.mp[PACK];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long job = blockIdx.x;
  double2* tw_lo = sm + (N + N / 16);                               // w^b, b < 64 (padded: TwSmem2)
  double2* tw_hi = tw_lo + 72;                                      // w^(64 a), a < N / 64
  for (int i = tid; i < 64 + N / 64; i += nt) {
    if (i < 64) tw_lo[i + (i >> 3)] = __ldg(f.tw + i);
    else tw_hi[i - 64] = __ldg(f.tw + 64 * (i - 64));
  }
  const long long sig = job / e.jobs_per_sig;
  long long r0 = job % e.jobs_per_sig;
  long long w;
  int part;
  if (e.b0 == 0 && r0 < f.parts0) {
    w = 0;
    part = (int)r0;
  } else {
    if (e.b0 == 0) r0 -= f.parts0;
    w = e.b0 + (e.b0 == 0 ? 1 : 0) + r0 / f.parts1;
    part = (int)(r0 % f.parts1);
  }
  const Blk b = block_info<PACK>(g, mp.K, w);
  const double* gsrc = e.s + sig * e.s_stride + (b.g0 - e.s_off);
  const long long avail = g.L - b.g0;
  const int n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));

  // diagnostics (conv_execute_profile): per job {smid, t0, t_peak, t_packed, t_fwd, t_prod, t_inv, t_end}
  unsigned long long* ft = (e.dbg_timing && tid == 0 && blockIdx.x < 4096) ? e.dbg_timing + 8 * blockIdx.x : nullptr;
  auto stamp = [&](int i) {
    if (ft) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ft[i] = t;
    }
  };
  if (ft) {
    unsigned sm_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
    ft[0] = sm_;
  }
  stamp(1);
  // a2/a3: block peak and c_s (Eq. (2))
  double c_s = 1.0;
  if (PACK != PACK_FULL) {
    constexpr int U = PC_FFT_PEAK_U;              // loads in flight per thread
    double mu[U];
#pragma unroll
    for (int u = 0; u < U; ++u) mu[u] = 0.0;
    if ((reinterpret_cast<uintptr_t>(gsrc) & 15u) == 0) {
      const double2* g2 = reinterpret_cast<const double2*>(gsrc);
      const int n2 = n_valid / 2;
      for (int i0 = tid; i0 < n2; i0 += U * nt) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (i0 + u * nt < n2) ? __ldg(g2 + i0 + u * nt) : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < U; ++u) mu[u] = fmax(mu[u], fmax(fabs(v[u].x), fabs(v[u].y)));
      }
      if ((n_valid & 1) && tid == 0) mu[0] = fmax(mu[0], fabs(gsrc[n_valid - 1]));
    } else {
      for (int i0 = tid; i0 < n_valid; i0 += U * nt) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (i0 + u * nt < n_valid) ? __ldg(gsrc + i0 + u * nt) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) mu[u] = fmax(mu[u], fabs(v[u]));
      }
    }
    double m = mu[0];
#pragma unroll
    for (int u = 1; u < U; ++u) m = fmax(m, mu[u]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    double peak = 0.0;
    for (int wi = 0; wi < nt / 32; ++wi) peak = fmax(peak, red[wi]);
    c_s = (peak == 0.0) ? 1.0 : mp.Q / peak;
  }
  const double inv = dequant_scale(c_s, mp.c_k);
  stamp(2);
  // part window: core outputs [m_lo, m_hi); sym parts after the first also need word m_lo-1
  const int front = (PACK == PACK_SYM && part > 0) ? 1 : 0;
  const int m_lo = (part == 0) ? 0 : f.part0_out + (part - 1) * f.part_out;
  const int m_hi = min(b.M_out, m_lo + (part == 0 ? f.part0_out : f.part_out));
  const int cw0 = m_lo - front;                 // core word at window position 0
  auto sample = [&](int i) -> double { return (i < 0 || i >= n_valid) ? 0.0 : __ldg(gsrc + i); };
  auto word = [&](int cw) -> double {           // a4: the core's input word cw
    if (cw < 0 || cw >= b.xlen) return 0.0;
    if (PACK == PACK_SYM) {
      const int j = cw - b.pre;
      if (j < 0) return 0.0;
      return pack_sym(compand1(c_s, sample(2 * j)), compand1(c_s, sample(2 * j + 1)), mp.eps);
    } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
      constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
      const int base = b.o0 - (g.Np - 1) + cw;
      double v = compand1(c_s, sample(base + (M - 1) * b.S));
#pragma unroll
      for (int q = M - 2; q >= 0; --q) v = __dadd_rn(compand1(c_s, sample(base + q * b.S)), __dmul_rn(mp.eps, v));
      return v;
    }
    return sample(b.o0 - (g.Np - 1) + cw);
  };
  // window of 2N real words (outputs need cw0 .. cw0 + (m_hi-m_lo+front) + K - 2)
  const int wlen = (m_hi - m_lo + front) + mp.K - 1;
  // a3/a4 with every sample load of UB complex points issued before any use (latency-bound
  // otherwise); same arithmetic, in the oracle's order, as word().
  constexpr int MS = (PACK == PACK_ASYM3) ? 3 : 2;   // samples per word (full: 1, sym: 2)
  constexpr int UB = (PACK == PACK_ASYM3) ? 3 : PC_FFT_PACK_UB;
  for (int n0 = tid; n0 < N; n0 += UB * nt) {
    double xv[UB][2][MS];
#pragma unroll
    for (int u = 0; u < UB; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cw = cw0 + 2 * (n0 + u * nt) + h;
        const bool live = (n0 + u * nt < N) && (2 * (n0 + u * nt) + h < wlen) && cw >= 0 && cw < b.xlen;
#pragma unroll
        for (int q = 0; q < MS; ++q) {
          int idx;
          if (PACK == PACK_SYM) idx = 2 * (cw - b.pre) + q;
          else if (PACK == PACK_FULL) idx = b.o0 - (g.Np - 1) + cw;
          else idx = b.o0 - (g.Np - 1) + cw + q * b.S;
          const bool ok = live && (PACK != PACK_SYM || cw - b.pre >= 0) && (PACK != PACK_FULL || q == 0);
          xv[u][h][q] = ok ? sample(idx) : 0.0;
        }
      }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int n = n0 + u * nt;
      if (n >= N) break;
      double wv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cw = cw0 + 2 * n + h;
        const bool live = (2 * n + h < wlen) && cw >= 0 && cw < b.xlen && (PACK != PACK_SYM || cw - b.pre >= 0);
        double v;
        if (PACK == PACK_SYM) {
          v = pack_sym(compand1(c_s, xv[u][h][0]), compand1(c_s, xv[u][h][1]), mp.eps);
        } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
          constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
          v = compand1(c_s, xv[u][h][M - 1]);
#pragma unroll
          for (int q = M - 2; q >= 0; --q) v = __dadd_rn(compand1(c_s, xv[u][h][q]), __dmul_rn(mp.eps, v));
        } else {
          v = xv[u][h][0];
        }
        wv[h] = live ? v : 0.0;
      }
      sm[pidx(n)] = make_double2(wv[0], wv[1]);
    }
  }
  __syncthreads();
  stamp(3);
  const TwSmem2 tws{tw_lo, tw_hi};
  fft_smem<N, -1>(sm, tws);                                         // a5: forward
  stamp(4);
  spectrum_product<N>(sm, f.H, TwHalf{tws, __ldg(f.tw2 + 1), N});
  stamp(5);
  fft_smem<N, +1>(sm, tws);                                         // a5: inverse
  stamp(6);
  // p[q] = Re/Im of sm[q/2]; core output m (window-relative mw = m - cw0) = p[mw + K - 1]
  auto pval = [&](int q) -> double {
    const double2 z = sm[pidx(q >> 1)];
    return (q & 1) ? z.y : z.x;
  };
  const int K1 = mp.K - 1;
  double* __restrict__ r = e.r + sig * e.r_stride;
  const long long gbase = b.g0 + b.o0;
  const long long L_conv = g.L + g.N - 1;
  auto store = [&](int k, double val) {
    const long long gg = gbase + k;
    if (g.mode == 0) {
      if (gg < L_conv) r[gg - e.r_off] = val;
    } else {
      const long long j = gg - (g.N - 1);
      if (j >= 0 && j <= g.L - g.N) r[j - e.r_off] = val;
    }
  };
  double resid = 0.0;                                               // last-digit residual (LSB)
  if (PACK == PACK_SYM) {
    const int moff = (w == 0) ? 0 : 1;
    for (int m = m_lo + tid; m < m_hi; m += nt) {
      if (m < moff) continue;
      const double v = pval(m - cw0 + K1);
      const Digits3 d = decode_sym(v, mp.eps, mp.eps_inv, mp.pow2);
      const double rem = __dsub_rn(v, __dmul_rn(d.C, mp.eps_inv));
      resid = fmax(resid, fabs(__dmul_rn(__dsub_rn(rem, d.A), mp.eps_inv) - d.B));
      double Bp = 0.0;
      if (m >= 1) Bp = decode_sym(pval(m - 1 - cw0 + K1), mp.eps, mp.eps_inv, mp.pow2).B;
      const int k = 2 * (m - moff);
      store(k + 1, __dmul_rn(d.A, inv));
      store(k, __dmul_rn(d.C + Bp, inv));
    }
  } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
    constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
    for (int m = m_lo + tid; m < m_hi; m += nt) {
      double v = pval(m - cw0 + K1);
#pragma unroll
      for (int q = 0; q < M; ++q) {
        const double t = rint(v);
        if (q == M - 1) resid = fmax(resid, fabs(v - t));
        if (q < M - 1) v = __dmul_rn(__dsub_rn(v, t), mp.eps_inv);
        const int k = q * b.S + m;
        if (k < b.n_out) store(k, __dmul_rn(t, inv));
      }
    }
  } else {
    for (int m = m_lo + tid; m < m_hi; m += nt) store(m, pval(m - cw0 + K1));
  }
  if (PACK != PACK_FULL) {
    for (int o = 16; o > 0; o >>= 1) resid = fmax(resid, __shfl_xor_sync(0xffffffffu, resid, o));
    if ((tid & 31) == 0 && resid > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(f.resid), (unsigned long long)__double_as_longlong(resid));
    if ((tid & 31) == 0 && resid > 0.25 && e.status)    // the plan's host-mapped margin flag (conv_execute)
      *reinterpret_cast<volatile int*>(e.status + kStatusMargin) = 1;
  }
  stamp(7);
}

// ------------------------------------------------------------------ n = 32768 (full precision)
// The configured full-precision core of cfg3 (BASELINE.json configs[2]: the block's linear
// convolution through a 32768-point real transform, SURVEY §8(d) "G6").  Its 16384 complex
// points (256 KB) exceed one CTA's shared memory, so a 2-CTA cluster shares the work: the
// window's data occupy only the first 8192 complex points (16384 real words; the rest is zero
// padding), so Z[2k'+r] = FFT_8192(z[n] W^{nr})[k'] (W = exp(-2 pi i/16384)) -- CTA r computes
// parity class r with no exchange; the real-transform split pairs k with 16384-k, which has
// the same parity, so the spectrum product is local too; the inverse gives q_r = IFFT_8192 of
// each class and p[n] = q_0[n] + W^{-n} q_1[n], formed by CTA 0 reading CTA 1's shared memory
// (DSMEM).  Twiddles: tw[m] = W^m (m < 16384); the 8192-point passes use W^{2m}.
namespace {
constexpr int kN32 = 8192;                 // complex points per CTA
constexpr int kN32Full = 2 * kN32;         // complex points of the transform (real length 32768)

struct TwStride2 {                         // w_8192^m = W^{2m} from the 16384-entry table, two-level in smem
  const double2* lo;                       // lo[b] = W^{2b}, b < 64
  const double2* hi;                       // hi[a] = W^{128 a}, a < 128
  __device__ __forceinline__ double2 operator()(int m) const { return cmul(hi[m >> 6], lo[m & 63]); }
};

// Parity-class partner of local index k' (global k = 2k'+r): 16384 - k is 2k''+r.
__device__ __forceinline__ int partner32(int kl, int r) { return r == 0 ? ((kN32 - kl) & (kN32 - 1)) : (kN32 - 1 - kl); }
}  // namespace

__global__ void __launch_bounds__(kN32 / 16) pc_fft32k_spectrum(const double* __restrict__ kr, int K,
                                                              const double2* __restrict__ tw,
                                                              const double2* __restrict__ tw2,
                                                              double2* __restrict__ H) {
  extern __shared__ __align__(16) double2 sm[];
  const int r = blockIdx.x;                 // parity class
  double2* lo = sm + (kN32 + kN32 / 16);
  double2* hi = lo + 64;
  for (int i = threadIdx.x; i < 64 + kN32 / 64; i += blockDim.x)
    lo[i] = (i < 64) ? __ldg(tw + 2 * i) : __ldg(tw + 128 * (i - 64));
  for (int n = threadIdx.x; n < kN32; n += blockDim.x) {   // h[n] = kr[K-1-n]; z[n] W^{nr}
    const int a = 2 * n, b = 2 * n + 1;
    double2 z = make_double2(a < K ? kr[K - 1 - a] : 0.0, b < K ? kr[K - 1 - b] : 0.0);
    if (r) z = cmul(z, __ldg(tw + n));
    sm[pidx(n)] = z;
  }
  __syncthreads();
  fft_smem<kN32, -1>(sm, TwStride2{lo, hi});
  // X[k] = E[k] + W2^k O[k] for k = 2k'+r (k = 0 .. 16384; k = 16384 is class 0, k' = 8192 = 0)
  for (int kl = threadIdx.x; kl <= (r == 0 ? kN32 : kN32 - 1); kl += blockDim.x) {
    const int k = 2 * kl + r;
    const double2 Zk = sm[pidx(kl & (kN32 - 1))], Zkp = sm[pidx(partner32(kl & (kN32 - 1), r))];
    const double2 E = make_double2(0.5 * (Zk.x + Zkp.x), 0.5 * (Zk.y - Zkp.y));
    const double2 O = make_double2(0.5 * (Zk.y + Zkp.y), -0.5 * (Zk.x - Zkp.x));
    H[k] = cadd(E, cmul(__ldg(tw2 + k), O));
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kN32 / 16, 1)
    pc_fft32k_full_kernel(Geo g, Exec e, FftArgs f) {
  extern __shared__ __align__(16) double2 sm[];
  const ModeP& mp = e.mp[PACK_FULL];
  const int tid = threadIdx.x, nt = blockDim.x;
  const unsigned r = cg::this_cluster().block_rank();
  const long long job = blockIdx.x >> 1;
  const long long sig = job / e.jobs_per_sig;
  const long long w = e.b0 + job % e.jobs_per_sig;
  double2* lo = sm + (kN32 + kN32 / 16);
  double2* hi = lo + 64;
  for (int i = tid; i < 64 + kN32 / 64; i += nt) lo[i] = (i < 64) ? __ldg(f.tw + 2 * i) : __ldg(f.tw + 128 * (i - 64));
  const Blk b = block_info<PACK_FULL>(g, mp.K, w);
  const double* gsrc = e.s + sig * e.s_stride + (b.g0 - e.s_off);
  const long long avail = g.L - b.g0;
  const int n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  // window = core words [cw0, xlen): block 0 skips its N'-1 zero prefix, so every window holds
  // at most W_block = 16384 real words (the first 8192 complex points)
  const int cw0 = (w == 0) ? g.Np - 1 : 0;
  const int wlen = b.xlen - cw0;
  auto word = [&](int i) -> double {
    const int idx = b.o0 - (g.Np - 1) + cw0 + i;
    return (i < wlen && idx >= 0 && idx < n_valid) ? __ldg(gsrc + idx) : 0.0;
  };
  constexpr int UB = 8;
  for (int n0 = tid; n0 < kN32; n0 += UB * nt) {
    double2 z[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int n = n0 + u * nt;
      z[u] = (n < kN32) ? make_double2(word(2 * n), word(2 * n + 1)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int n = n0 + u * nt;
      if (n < kN32) sm[pidx(n)] = r ? cmul(z[u], __ldg(f.tw + n)) : z[u];
    }
  }
  __syncthreads();
  const TwStride2 tws{lo, hi};
  fft_smem<kN32, -1>(sm, tws);                                      // a5: Z[2k'+r]
  // spectrum product by H (real-transform split/merge), pairs (k, 16384-k) of this class
  const double sc = 1.0 / (double)kN32Full;
  if (r == 0 && tid == 0) {
    const double2 z0 = sm[pidx(0)];
    const double X0 = z0.x + z0.y, XN = z0.x - z0.y;
    const double2 H0 = __ldg(f.H), HN = __ldg(f.H + kN32Full);
    const double2 P0 = make_double2(X0 * H0.x, X0 * H0.y);
    const double2 PN = make_double2(XN * HN.x, XN * HN.y);
    const double2 ee = make_double2(0.5 * (P0.x + PN.x), 0.5 * (P0.y - PN.y));
    const double2 oo = make_double2(0.5 * (P0.x - PN.x), 0.5 * (P0.y + PN.y));
    sm[pidx(0)] = make_double2((ee.x - oo.y) * sc, (ee.y + oo.x) * sc);
  }
  const int klo = (r == 0) ? 1 : 0, khi = (r == 0) ? kN32 / 2 : kN32 / 2 - 1;   // k' <= partner
  for (int kl = klo + tid; kl <= khi; kl += nt) {
    const int kp_l = partner32(kl, r);
    const int k = 2 * kl + (int)r, kp = kN32Full - k;
    const double2 Zk = sm[pidx(kl)], Zkp = sm[pidx(kp_l)];
    const double2 Wk = __ldg(f.tw2 + k), Wkp = __ldg(f.tw2 + kp);
    const double2 Ek = make_double2(0.5 * (Zk.x + Zkp.x), 0.5 * (Zk.y - Zkp.y));
    const double2 Ok = make_double2(0.5 * (Zk.y + Zkp.y), -0.5 * (Zk.x - Zkp.x));
    const double2 Xk = cadd(Ek, cmul(Wk, Ok));
    const double2 Xkp = cadd(cconj(Ek), cmul(Wkp, cconj(Ok)));
    const double2 Pk = cmul(Xk, __ldg(f.H + k)), Pkp = cmul(Xkp, __ldg(f.H + kp));
    auto merge = [&](double2 a, double2 bb, double2 W) {
      const double2 ee = make_double2(0.5 * (a.x + bb.x), 0.5 * (a.y - bb.y));
      const double2 d = make_double2(0.5 * (a.x - bb.x), 0.5 * (a.y + bb.y));
      const double2 o = cmul(d, cconj(W));
      return make_double2((ee.x - o.y) * sc, (ee.y + o.x) * sc);
    };
    const double2 Zpk = merge(Pk, Pkp, Wk);
    const double2 Zpkp = merge(Pkp, Pk, Wkp);
    sm[pidx(kl)] = Zpk;
    if (kp_l != kl) sm[pidx(kp_l)] = Zpkp;
  }
  __syncthreads();
  fft_smem<kN32, +1>(sm, tws);                                      // q_r = IFFT_8192 (unscaled)
  cg::this_cluster().sync();                                        // both classes ready
  if (r == 0) {
    const double2* q1 = cg::this_cluster().map_shared_rank(sm, 1);   // CTA 1's q_1 (DSMEM)
    double* __restrict__ out = e.r + sig * e.r_stride;
    const long long gbase = b.g0 + b.o0;
    const long long L_conv = g.L + g.N - 1;
    const int K1 = mp.K - 1;
    for (int m = tid; m < b.M_out; m += nt) {
      const int q = m - cw0 + K1;                                   // p index of core output m
      const int n = q >> 1;
      const double2 a = sm[pidx(n)], c = q1[pidx(n)];
      const double2 p = cadd(a, cmul(c, cconj(__ldg(f.tw + n))));  // q_0 + W^{-n} q_1
      const double v = (q & 1) ? p.y : p.x;
      const long long gg = gbase + m;
      if (g.mode == 0) {
        if (m < b.n_out && gg < L_conv) out[gg - e.r_off] = v;
      } else {
        const long long j = gg - (g.N - 1);                         // valid lag (C17)
        if (m < b.n_out && j >= 0 && j <= g.L - g.N) out[j - e.r_off] = v;
      }
    }
  }
  cg::this_cluster().sync();                                        // CTA 1's shared memory stays valid
}

// ------------------------------------------------------------------ launchers
template <int N>
static cudaError_t launch_fft_N(int packing, const Geo& g, const Exec& e, const FftArgs& f, long long n_jobs,
                                cudaStream_t st) {
  const size_t smem = (size_t)(N + N / 16 + 72 + N / 64) * sizeof(double2);   // + two-level twiddles (lo padded)
  cudaError_t err = cudaSuccess;
  switch (packing) {
#define PC_FFT_CASE(PK)                                                                                  \
  case PK: {                                                                                             \
    auto kfn = pc_fft_conv_kernel<PK, N>;                                                               \
    static LaunchAttrCache cache; /* per device, under a lock */                                       \
    static std::once_flag carve;                                                                         \
    int dev_ = 0, sms_ = 0;                                                                              \
    if ((err = cudaGetDevice(&dev_)) != cudaSuccess) return err;                                         \
    if ((err = cache.ensure(kfn, dev_, smem, N / 16, &sms_)) != cudaSuccess) return err;                \
    /* leave the rest of the 256 KB unified array to L1: the spectrum tables stay cached */             \
    std::call_once(carve, [&] {                                                                          \
      cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, PC_FFT_CARVEOUT);       \
    });                                                                                                  \
    kfn<<<(unsigned)n_jobs, N / 16, smem, st>>>(g, e, f);                                              \
    break;                                                                                               \
  }
    PC_FFT_CASE(PACK_FULL)
    PC_FFT_CASE(PACK_SYM)
    PC_FFT_CASE(PACK_ASYM2)
    PC_FFT_CASE(PACK_ASYM3)
#undef PC_FFT_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_fft_conv(int packing, int N, const Geo& g, const Exec& e, const FftArgs& f, long long n_jobs,
                            cudaStream_t st) {
  if (n_jobs <= 0) return cudaSuccess;
  switch (N) {
    case 1024: return launch_fft_N<1024>(packing, g, e, f, n_jobs, st);
    case 2048: return launch_fft_N<2048>(packing, g, e, f, n_jobs, st);
    case 4096: return launch_fft_N<4096>(packing, g, e, f, n_jobs, st);
    case 8192: return launch_fft_N<8192>(packing, g, e, f, n_jobs, st);
    case 16384: {                                         // full precision only (2-CTA clusters)
      if (packing != PACK_FULL) return cudaErrorInvalidValue;
      const size_t smem = (size_t)(kN32 + kN32 / 16 + 64 + kN32 / 64) * sizeof(double2);
      static LaunchAttrCache cache;                       // per device, under a lock
      int dev = 0, sms = 0;
      cudaError_t err = cudaGetDevice(&dev);
      if (err == cudaSuccess) err = cache.ensure(pc_fft32k_full_kernel, dev, smem, kN32 / 16, &sms, false);
      if (err != cudaSuccess) return err;
      pc_fft32k_full_kernel<<<(unsigned)(2 * n_jobs), kN32 / 16, smem, st>>>(g, e, f);
      return cudaGetLastError();
    }
  }
  return cudaErrorInvalidValue;
}

template <int N>
static cudaError_t launch_spec_N(const double* kr, int K, const double2* tw, const double2* tw2, double2* H,
                                 cudaStream_t st) {
  const size_t smem = (size_t)(N + N / 16) * sizeof(double2);
  auto kfn = pc_fft_spectrum<N>;
  cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  kfn<<<1, N / 16, smem, st>>>(kr, K, tw, tw2, H);
  return cudaGetLastError();
}

cudaError_t launch_fft_spectrum(int N, const double* kr, int K, const double2* tw, const double2* tw2, double2* H,
                                cudaStream_t st) {
  switch (N) {
    case 1024: return launch_spec_N<1024>(kr, K, tw, tw2, H, st);
    case 2048: return launch_spec_N<2048>(kr, K, tw, tw2, H, st);
    case 4096: return launch_spec_N<4096>(kr, K, tw, tw2, H, st);
    case 8192: return launch_spec_N<8192>(kr, K, tw, tw2, H, st);
    case 16384: {
      const size_t smem = (size_t)(kN32 + kN32 / 16 + 64 + kN32 / 64) * sizeof(double2);
      cudaError_t err = cudaFuncSetAttribute(pc_fft32k_spectrum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err != cudaSuccess) return err;
      pc_fft32k_spectrum<<<2, kN32 / 16, smem, st>>>(kr, K, tw, tw2, H);
      return cudaGetLastError();
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace pc
