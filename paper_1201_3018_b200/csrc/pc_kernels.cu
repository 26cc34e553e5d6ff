// pc_kernels.cu -- sm_100a kernels of the packed overlap-save path (arXiv 1201.3018).
//
//   pc_kernel_prep      a1: kernel companding once: pad/reverse, ||k||_inf,
//                       c_k, k~ = [[c_k k]], ||k~||_1 (for the L1 R_max rule, C3)
//   pc_build_taps       a1: core taps, reversed: packed kernel Eq. (5) under C1 (sym),
//                       k~ (asym, Eq. (8)) or k (full precision)
//   pc_fused_kernel     a2-a7 (+a9 store mapping) in ONE kernel, one CTA per overlap-save
//                       block: TMA bulk copy of the block and the taps into shared memory,
//                       block peak (warp shuffles), companding (Eq. (2)), packing (Eq. (4)
//                       or (7)) into a conflict-free column layout, the direct FP64 core
//                       on packed words, unpacking (Eqs. (11)-(15), balanced form),
//                       inverse companding (Eq. (16)), overlap discard and placement
//                       (Eq. (17)).  FULL = the same kernel without the Tier-1.5 layer
//                       (the full-precision reference path on identical tiling).
//   pc_block_stats      a8: per-block peak and order-independent sigma (reading C12)
//   pc_adapt_decide     a8: per-block mode choice from Eq. (19)
//   pc_xcorr_max        a9: per-signal max and argmax of the valid lags (C17)
#include "pc_device.cuh"
#include "pc_kernels.h"

namespace pc {

// ------------------------------------------------------------------ a1: kernel preparation
// One kernel (query) per CTA: pad to N' (C13), reverse for xcorr (a9), ||k||_inf, c_k = K_q /
// ||k||_inf (all-zero -> 1), k~ = [[c_k k]] (Eq. (2)) and ||k~||_1.
__device__ __forceinline__ void kernel_prep_one(const double* __restrict__ k_in, int N, int Np, int reverse,
                                                double K_q, double* __restrict__ k_pad, double* __restrict__ k_int,
                                                double* __restrict__ scal /* [peak, c_k, l1] */, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double m = 0.0;
  for (int i = tid; i < Np; i += nt) {
    double v = 0.0;
    if (i < N) v = k_in[reverse ? (N - 1 - i) : i];   // xcorr: reverse then pad (a9)
    k_pad[i] = v;
    m = fmax(m, fabs(v));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  if (tid < 32) {
    m = (tid < (nt + 31) / 32) ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tid == 0) red[0] = m;
  }
  __syncthreads();
  const double peak = red[0];
  const double c_k = (peak == 0.0) ? 1.0 : K_q / peak;   // P:53; all-zero -> c = 1
  __syncthreads();
  double l1 = 0.0;                                        // sum of integers < 2^53: exact
  for (int i = tid; i < Np; i += nt) {
    const double q = compand1(c_k, k_pad[i]);
    k_int[i] = q;
    l1 += fabs(q);
  }
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if ((tid & 31) == 0) red[tid >> 5] = l1;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < (nt + 31) / 32; ++w) t += red[w];
    scal[0] = peak;
    scal[1] = c_k;
    scal[2] = t;
  }
}

__global__ void pc_kernel_prep(const double* __restrict__ k_in, int N, int Np, int reverse, double K_q,
                               double* __restrict__ k_pad, double* __restrict__ k_int,
                               double* __restrict__ scal /* [peak, c_k, l1] */) {
  __shared__ double red[32];
  kernel_prep_one(k_in, N, Np, reverse, K_q, k_pad, k_int, scal, red);
}

// Many kernels at once (conv_plan_set_kernels, NEXT-3): problem i = blockIdx.x.
__global__ void pc_kernel_prep_batch(const double* __restrict__ k_in, long long k_stride, int N, int Np, int reverse,
                                     double K_q, double* __restrict__ k_pad, double* __restrict__ k_int,
                                     long long pad_stride, double* __restrict__ scal /* [n][3] */) {
  __shared__ double red[32];
  const long long i = blockIdx.x;
  kernel_prep_one(k_in + i * k_stride, N, Np, reverse, K_q, k_pad + i * pad_stride, k_int + i * pad_stride,
                  scal + 3 * i, red);
}

__device__ __forceinline__ double core_tap(const double* __restrict__ k_pad, const double* __restrict__ k_int,
                                           int Np, int packing, double eps_inv, int K, int j) {
  if (j >= K) return 0.0;
  const int n = K - 1 - j;   // reversed: kr[j] = core tap K-1-j
  if (packing == PACK_SYM) {
    // Eq. (5) under reading C1: k_bar[n] = k~[2n+1] + eps^-1 k~[2n], k~[N'] = 0
    const double kev = k_int[2 * n];
    const double kod = (2 * n + 1 < Np) ? k_int[2 * n + 1] : 0.0;
    return __dadd_rn(kod, __dmul_rn(eps_inv, kev));
  }
  if (packing == PACK_FULL) return k_pad[n];
  return k_int[n];             // Eq. (8): asymmetric packing convolves with k~
}

__global__ void pc_build_taps(const double* __restrict__ k_pad, const double* __restrict__ k_int, int Np,
                              int packing, double eps_inv, int K, int K_pad, double* __restrict__ kr) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K_pad; j += gridDim.x * blockDim.x)
    kr[j] = core_tap(k_pad, k_int, Np, packing, eps_inv, K, j);
}

__global__ void pc_build_taps_batch(const double* __restrict__ k_pad, const double* __restrict__ k_int,
                                    long long pad_stride, int Np, int packing, double eps_inv, int K, int K_pad,
                                    double* __restrict__ kr, long long kr_stride) {
  const long long i = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K_pad; j += gridDim.x * blockDim.x)
    kr[i * kr_stride + j] = core_tap(k_pad + i * pad_stride, k_int + i * pad_stride, Np, packing, eps_inv, K, j);
}

// ------------------------------------------------------------------ fused per-block kernel
__device__ __forceinline__ double block_max_abs(const double* raw, int n, const double* __restrict__ gsrc,
                                                long long g_avail, bool staged, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double m = 0.0;
  if (staged) {
    for (int i = tid; i < n; i += nt) m = fmax(m, fabs(raw[i]));
  } else {
    for (int i = tid; i < n; i += nt) m = fmax(m, (i < g_avail) ? fabs(gsrc[i]) : 0.0);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __syncthreads();   // red may still be read by a previous use
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (nt + 31) / 32; ++w) r = fmax(r, red[w]);
  return r;
}

template <int PACK, int T>
__device__ __forceinline__ void fused_block(const Geo& g, const Exec& e, const ModeP& mp, long long sig,
                                            long long w, unsigned char* smem) {
  // shared memory: [header][raw W_block (stage_raw only)][xs T x rows][kr K_pad][Rs (loop path only)]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* red = reinterpret_cast<double*>(smem + 16);
  double* raw = reinterpret_cast<double*>(smem + kSmemHeader);
  double* xs = raw + (e.stage_raw ? g.W_block : 0);
  double* kr = xs + (size_t)T * mp.rows;
  // register path: one T-output group per thread, results re-staged in the xs region after
  // the core finished; loop path: groups > threads, results in a separate region.
  double* Rs = e.reg_path ? xs : (kr + mp.K_pad);

  const int tid = threadIdx.x, nt = blockDim.x;
  const double* __restrict__ s = e.s + sig * e.s_stride;   // s[i - s_off] = sample i
  double* __restrict__ r = e.r ? e.r + sig * e.r_stride : nullptr;
  const Blk b = block_info<PACK>(g, mp.K, w);
  const long long dbg_row = sig * g.P + w;

  // ---- TMA bulk copies: the core taps (always) and the raw block (stage_raw)
  const long long avail = g.L - b.g0;                       // samples of this block inside L
  const int n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  const double* gsrc = s + (b.g0 - e.s_off);
  const bool aligned = ((reinterpret_cast<uintptr_t>(gsrc) & 15u) == 0);
  const int n_bulk = (e.stage_raw && aligned) ? (n_valid & ~1) : 0;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_arrive_expect_tx(bar, (uint32_t)n_bulk * 8u + (uint32_t)mp.K_pad * 8u);
    if (n_bulk) bulk_g2s(raw, gsrc, (uint32_t)n_bulk * 8u, bar);
    bulk_g2s(kr, mp.kr, (uint32_t)mp.K_pad * 8u, bar);
  }
  if (e.stage_raw) {
    for (int i = n_bulk + tid; i < g.W_block; i += nt) raw[i] = (i < n_valid) ? gsrc[i] : 0.0;
    __syncthreads();          // barrier init visible before anyone waits on it
    mbar_wait(bar, 0);
  }
  auto sample = [&](int i) -> double {      // local sample i of the block (0 outside)
    if (i < 0 || i >= n_valid) return 0.0;
    return e.stage_raw ? raw[i] : __ldg(gsrc + i);
  };

  // ---- a2/a3: block peak (coalesced, warp shuffles) and companding factor (Eq. (2))
  double c_s = 1.0;
  if (PACK != PACK_FULL) {
    double m = 0.0;
    if (e.stage_raw) {
      for (int i = tid; i < n_valid; i += nt) m = fmax(m, fabs(raw[i]));
    } else if (aligned) {
      const double2* g2 = reinterpret_cast<const double2*>(gsrc);
      for (int i = tid; i < n_valid / 2; i += nt) {
        const double2 v = __ldg(g2 + i);
        m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
      }
      if ((n_valid & 1) && tid == 0) m = fmax(m, fabs(gsrc[n_valid - 1]));
    } else {
      for (int i = tid; i < n_valid; i += nt) m = fmax(m, fabs(__ldg(gsrc + i)));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    double peak = 0.0;
    for (int wi = 0; wi < (nt + 31) / 32; ++wi) peak = fmax(peak, red[wi]);
    c_s = (peak == 0.0) ? 1.0 : mp.Q / peak;
  }

  // ---- a4: companding + packing.  Thread row g builds the T consecutive core words
  // gT..gT+T-1 and writes them to xs[c * rows + g] (lane-consecutive: conflict-free).
  for (int gr = tid; gr < mp.rows; gr += nt) {
#pragma unroll
    for (int c = 0; c < T; ++c) {
      const int i = gr * T + c;
      double v = 0.0;
      if (i < b.xlen) {
        if (PACK == PACK_SYM) {
          const int j = i - b.pre;              // s_bar[j] (Eq. (4))
          if (j >= 0) v = pack_sym(compand1(c_s, sample(2 * j)), compand1(c_s, sample(2 * j + 1)), mp.eps);
        } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
          constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
          const int base = b.o0 - (g.Np - 1) + i;   // Eq. (7) under C8, Horner (oracle order)
          v = compand1(c_s, sample(base + (M - 1) * b.S));
#pragma unroll
          for (int q = M - 2; q >= 0; --q)
            v = __dadd_rn(compand1(c_s, sample(base + q * b.S)), __dmul_rn(mp.eps, v));
        } else {
          v = sample(b.o0 - (g.Np - 1) + i);
        }
      }
      xs[c * mp.rows + gr] = v;
    }
  }
  if (e.dbg_packed && PACK != PACK_FULL) {
    double* dp = e.dbg_packed + dbg_row * e.dbg_packed_stride;
    if (PACK == PACK_SYM) {
      for (int j = tid; j < g.W_block / 2; j += nt)
        dp[j] = pack_sym(compand1(c_s, sample(2 * j)), compand1(c_s, sample(2 * j + 1)), mp.eps);
    }
  }
  if (e.dbg_cs && tid == 0) e.dbg_cs[dbg_row] = c_s;
  __syncthreads();
  if (!e.stage_raw) mbar_wait(bar, 0);      // taps landed (overlapped with peak + packing)
  if (e.dbg_packed && PACK != PACK_SYM && PACK != PACK_FULL) {
    double* dp = e.dbg_packed + dbg_row * e.dbg_packed_stride;
    for (int i = tid; i < b.xlen; i += nt) dp[i] = xs[(i % T) * mp.rows + i / T];
  }

  // ---- a5: the Tier-2 core on packed words (hot loop)
  const int ngroups = (b.M_out + T - 1) / T;
  if (e.reg_path) {
    // Full precision: S lanes per group (S a power of two <= 32, each lane >= 2 tap rows of T):
    // lane sl sums one slice of the taps, a shuffle tree adds the slices.  Short blocks (cfg1:
    // 136 groups, 64 taps) are latency-bound and the slices shorten each thread's FMA chain
    // (full precision 4.8 -> 4.4 us at cfg1; the sum order changes within rounding).  Packed
    // plans measured 0.1-0.2 us slower with slices (the packing phases dominate there): S = 1.
    const int nrow = mp.K_pad / T;
    int S = 1;
    if (PACK == PACK_FULL)
      while (S < 32 && ngroups * 2 * S <= nt && nrow >= 4 * S) S *= 2;
    const int gi = tid / S, sl = tid & (S - 1);
    const int rps = (nrow + S - 1) / S;
    const int jb = min(sl * rps, nrow) * T, je = min((sl + 1) * rps, nrow) * T;
    double acc[T];
    const bool mine = gi < ngroups;
    if (mine) {
      conv_group_range<T>(xs, mp.rows, kr, jb, je, gi, acc);
    } else {
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = 0.0;
    }
    for (int o = 1; o < S; o <<= 1)
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    __syncthreads();                         // every warp done reading xs
    if (mine && sl == 0) {
#pragma unroll
      for (int i = 0; i < T; ++i) {
        const int m = gi * T + i;
        if (m < b.M_out) Rs[m] = acc[i];
      }
    }
  } else {
    for (int gi = tid; gi < ngroups; gi += nt) {
      double acc[T];
      conv_group<T>(xs, mp.rows, kr, mp.K_pad, gi, acc);
#pragma unroll
      for (int i = 0; i < T; ++i) {
        const int m = gi * T + i;
        if (m < b.M_out) Rs[m] = acc[i];
      }
    }
  }
  __syncthreads();
  if (e.dbg_rbar) {
    double* dr = e.dbg_rbar + dbg_row * e.dbg_rbar_stride;
    for (int m = tid; m < b.M_out; m += nt) dr[m] = Rs[m];
  }

  // ---- a6/a7: unpack, inverse-compand, discard and place (Eqs. (11)-(17))
  const double inv = dequant_scale(c_s, mp.c_k);   // Eq. (16)
  const long long gbase = b.g0 + b.o0;        // global index of kept output 0
  long long* dri = e.dbg_rint ? e.dbg_rint + dbg_row * e.dbg_rint_stride : nullptr;
  double resid = 0.0;                         // debug: worst last-digit residual of this thread
  auto store = [&](int k, double rint_v, double val) {
    if (dri) dri[k] = (long long)rint_v;
    if (!r) return;
    const long long gi = gbase + k;
    if (g.mode == 0) {
      if (gi < g.L + g.N - 1) r[gi - e.r_off] = val;
    } else {
      const long long j = gi - (g.N - 1);      // valid lag j = 0 .. L-N (C17)
      if (j >= 0 && j <= g.L - g.N) r[j - e.r_off] = val;
    }
  };
  if (PACK == PACK_SYM) {
    // kept output k: w=0 -> packed m = k/2; w>0 -> m = k/2 + 1 (the seeded m = W_start
    // word only supplies B).  r~[2m+1] = A[m]; r~[2m] = C[m] + B[m-1], B[-1] = 0 (w=0).
    const int moff = (w == 0) ? 0 : 1;
    const int npairs = b.n_out / 2;
    for (int p = tid; p < npairs; p += nt) {
      const int m = p + moff;
      const Digits3 d = decode_sym(Rs[m], mp.eps, mp.eps_inv, mp.pow2);
      if (e.dbg_resid) {                       // last digit B: distance from its integer (LSB)
        const double rem = __dsub_rn(Rs[m], __dmul_rn(d.C, mp.eps_inv));
        resid = fmax(resid, fabs(__dmul_rn(__dsub_rn(rem, d.A), mp.eps_inv) - d.B));
      }
      const double Bp = (m >= 1) ? decode_sym_B(Rs[m - 1], mp.eps, mp.eps_inv, mp.pow2) : 0.0;
      const double ev = d.C + Bp, od = d.A;
      store(2 * p, ev, __dmul_rn(ev, inv));
      store(2 * p + 1, od, __dmul_rn(od, inv));
    }
  } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
    constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
    for (int m = tid; m < b.S; m += nt) {
      double v = Rs[m];
#pragma unroll
      for (int q = 0; q < M; ++q) {          // balanced digits, most significant first (C9)
        const double t = rint(v);
        if (q == M - 1 && e.dbg_resid && q * b.S + m < b.n_out) resid = fmax(resid, fabs(v - t));
        if (q < M - 1) v = __dmul_rn(__dsub_rn(v, t), mp.eps_inv);
        const int k = q * b.S + m;
        if (k < b.n_out) store(k, t, __dmul_rn(t, inv));
      }
    }
  } else {
    for (int m = tid; m < b.n_out; m += nt) store(m, 0.0, Rs[m]);
  }
  if (e.dbg_resid) {
    for (int o = 16; o > 0; o >>= 1) resid = fmax(resid, __shfl_xor_sync(0xffffffffu, resid, o));
    if ((tid & 31) == 0 && resid > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(e.dbg_resid), (unsigned long long)__double_as_longlong(resid));
  }
}

// PACK >= 0: one packing for every block.  PACK < 0: per-block packing from e.dec_pack
// (conv_adapt_block; "switch between asymmetric, symmetric and no packing").
template <int PACK>
__global__ void __launch_bounds__(kMaxThreads, 1) pc_fused_kernel(Geo g, Exec e) {
  extern __shared__ __align__(128) unsigned char smem[];
  const long long job = blockIdx.x;
  const long long sig = job / e.nblk;
  const long long w = e.b0 + job % e.nblk;
  if (PACK >= 0) {
    fused_block<(PACK < 0 ? 0 : PACK), kT>(g, e, e.mp[PACK < 0 ? 0 : PACK], sig, w, smem);
  } else {
    switch (e.dec_pack[sig * g.P + w]) {
      case PACK_SYM: fused_block<PACK_SYM, kT>(g, e, e.mp[PACK_SYM], sig, w, smem); break;
      case PACK_ASYM2: fused_block<PACK_ASYM2, kT>(g, e, e.mp[PACK_ASYM2], sig, w, smem); break;
      case PACK_ASYM3: fused_block<PACK_ASYM3, kT>(g, e, e.mp[PACK_ASYM3], sig, w, smem); break;
      default: fused_block<PACK_FULL, kT>(g, e, e.mp[PACK_FULL], sig, w, smem); break;
    }
  }
}

// ------------------------------------------------------------------ a8: block statistics
// Per block: peak p and sigma from the second moment on the fixed grid z = [[x 2^20/p]]
// with an exact int64 sum (reading C12).
// One CTA per block.  The block's samples (up to kStatsU per thread) stay in registers across
// both passes -- the peak, then sum z^2 on the fixed 2^20 grid -- so the input is read from HBM
// once with every load in flight (the two-pass loop re-read it and was latency-bound:
// 46 us for 134 MB at L = 2^24); longer blocks fall back to the loop.
constexpr int kStatsThreads = 256, kStatsU = 16;
// s is the global sample base (s[i] = sample i; a shard passes its slice minus its offset);
// blocks b0 .. b0 + gridDim.x - 1.
__global__ void __launch_bounds__(kStatsThreads) pc_block_stats(Geo g, const double* __restrict__ s, long long b0,
                                                                double* __restrict__ sigma, double* __restrict__ peak_out) {
  __shared__ double red[32];
  __shared__ unsigned long long ired[32];
  const long long w = b0 + blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long g0 = (w == 0) ? 0 : w * (long long)g.W - 2;
  const long long avail = g.L - g0;
  const int n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  const double* src = s + g0;
  unsigned long long acc = 0;
  double p;
  if (n_valid <= kStatsU * kStatsThreads && nt == kStatsThreads) {
    double v[kStatsU];
    double m = 0.0;
#pragma unroll
    for (int u = 0; u < kStatsU; ++u) {
      const int i = tid + u * kStatsThreads;
      v[u] = (i < n_valid) ? __ldg(src + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kStatsU; ++u) m = fmax(m, fabs(v[u]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    p = 0.0;
    for (int wi = 0; wi < kStatsThreads / 32; ++wi) p = fmax(p, red[wi]);
    if (p != 0.0) {
      const double sc = 1048576.0 / p;
#pragma unroll
      for (int u = 0; u < kStatsU; ++u) {
        const long long z = (long long)round(__dmul_rn(v[u], sc));   // zeros beyond n_valid add 0
        acc += (unsigned long long)(z * z);
      }
    }
  } else {
    p = block_max_abs(nullptr, n_valid, src, n_valid, false, red);
    if (p != 0.0) {
      const double sc = 1048576.0 / p;
      for (int i = tid; i < n_valid; i += nt) {
        const long long z = (long long)round(__dmul_rn(src[i], sc));
        acc += (unsigned long long)(z * z);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) ired[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < (nt + 31) / 32; ++i) t += ired[i];
    const double m2 = __ddiv_rn((double)t, (double)g.W_block);
    sigma[w] = (p == 0.0) ? 0.0 : __ddiv_rn(__dmul_rn(p, __dsqrt_rn(m2)), 1048576.0);
    peak_out[w] = p;
  }
}

// Eqs. (18)-(19) linear form in the oracle's evaluation order (oracle.snr_linear).
__device__ __forceinline__ double snr_linear(double ss, double sk, double ps, double pk, double Sq, double Kq) {
  const double sq12 = 3.4641016151377544;   // sqrt(12) correctly rounded
  const double vs = __ddiv_rn(ps, __dmul_rn(Sq, sq12));
  const double vk = __ddiv_rn(pk, __dmul_rn(Kq, sq12));
  const double a = __dmul_rn(ss, vk), b = __dmul_rn(sk, vs), c = __dmul_rn(vk, vs);
  const double D = __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c));
  const double n = __dmul_rn(ss, sk);
  return __ddiv_rn(__dmul_rn(n, n), D);
}

__global__ void pc_adapt_decide(long long P, const double* __restrict__ sigma, const double* __restrict__ peak,
                                double sig_k, double peak_k, const int* __restrict__ cand, const int* __restrict__ qmode,
                                int ncand, double thr_lin, int* __restrict__ dec_pack, int* __restrict__ dec_q,
                                double* __restrict__ dec_snr) {
  const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (w >= P) return;
  int mode = PACK_FULL, q = 0;
  double lin = __longlong_as_double(0x7ff0000000000000LL);   // +inf
  const double ss = sigma[w];
  if (ss > 0.0) {
    for (int c = 0; c < ncand; ++c) {
      const int Qm = qmode[c];
      if (Qm < 1) continue;
      const double l = snr_linear(ss, sig_k, peak[w], peak_k, (double)Qm, (double)Qm);
      if (l >= thr_lin) { mode = cand[c]; q = Qm; lin = l; break; }
    }
  } else {
    mode = cand[0];
    q = qmode[0];
  }
  dec_pack[w] = mode;
  dec_q[w] = q;
  dec_snr[w] = lin;
}

// ------------------------------------------------------------------ a8: per-packing block lists
// Compacts the per-block decisions into one ascending block list per packing (FULL, SYM,
// ASYM2, ASYM3), so the tiled kernel can run each packing's blocks in its own launch.
// One CTA of 1024 threads, kListsPer consecutive blocks per thread per round (fewer rounds and
// barriers): per-thread counts, a warp scan of them, a scan over warp totals per packing.
constexpr int kListsPer = 4;
// Blocks b0 .. b0 + P - 1 (dec_pack indexed by block; list stride `stride`).
__global__ void __launch_bounds__(1024) pc_adapt_lists(long long P, long long b0, long long stride,
                                                       const int* __restrict__ dec_pack, int* __restrict__ lists,
                                                       int* __restrict__ counts) {
  __shared__ int woff[4][32];   // per round: warp counts, then their exclusive offsets
  __shared__ int base[4];       // list lengths before the round
  __shared__ int rtot[4];       // round totals
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < 4) base[tid] = 0;
  for (long long r0 = 0; r0 < P; r0 += 1024 * kListsPer) {
    int d[kListsPer], cnt[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < kListsPer; ++j) {
      const long long w = r0 + (long long)kListsPer * tid + j;
      d[j] = (w < P) ? dec_pack[b0 + w] : -1;
#pragma unroll
      for (int m = 0; m < 4; ++m) cnt[m] += (d[j] == m);
    }
    int excl[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {                   // exclusive prefix of this thread within its warp
      int x = cnt[m];
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      excl[m] = x - cnt[m];
      if (lane == 31) woff[m][wid] = x;
    }
    __syncthreads();
    if (wid < 4) {                                  // warp m scans packing m's 32 warp counts
      const int v = woff[wid][lane];
      int x = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      woff[wid][lane] = x - v;
      if (lane == 31) rtot[wid] = x;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kListsPer; ++j) {           // ascending: thread order, then j
      const int m = d[j];
      if (m >= 0) {
        int pos = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == m) pos = base[q] + woff[q][wid] + excl[q]++;
        lists[(size_t)m * stride + pos] = (int)(b0 + r0 + (long long)kListsPer * tid + j);
      }
    }
    __syncthreads();
    if (tid < 4) base[tid] += rtot[tid];
    __syncthreads();
  }
  if (tid < 4) counts[tid] = base[tid];
}

// ------------------------------------------------------------------ a9: xcorr score
// One CTA per signal: max over valid lags, lowest lag on ties (C17).
__global__ void pc_xcorr_max(const double* __restrict__ c, long long n_lags, long long stride,
                             double* __restrict__ score, long long* __restrict__ lag) {
  __shared__ double sv[32];
  __shared__ long long sj[32];
  const long long sig = blockIdx.x;
  const double* row = c + sig * stride;
  double best = -__longlong_as_double(0x7ff0000000000000LL);
  long long bj = 0x7fffffffffffffffLL;
  for (long long j = threadIdx.x; j < n_lags; j += blockDim.x) {
    const double v = row[j];
    if (v > best) { best = v; bj = j; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (ov > best || (ov == best && oj < bj)) { best = ov; bj = oj; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; sj[threadIdx.x >> 5] = bj; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int wi = 1; wi < (int)((blockDim.x + 31) / 32); ++wi)
      if (sv[wi] > best || (sv[wi] == best && sj[wi] < bj)) { best = sv[wi]; bj = sj[wi]; }
    score[sig] = best;
    lag[sig] = bj;
  }
}

// ------------------------------------------------------------------ a2 ahead of the tiled core
// One CTA per (signal, block): p_w = max |x| over the block's W_block samples (reading C7),
// every load in flight at once, integer max of the |x| bits (non-negative doubles order like
// their bit patterns).  Lets the persistent kernel's producers skip the peak pass, which ran 3-6x
// slower next to the DMMA warps (profiles/r01_dmma_interference.log).  Triggers dependent launches
// at entry: the tiled kernel's prologue overlaps it and its griddepcontrol.wait covers the peaks.
constexpr int kPeakThreads = 256, kPeakU = 8;
__global__ void __launch_bounds__(kPeakThreads) pc_block_peak(Geo g, const double* __restrict__ s, long long s_off,
                                                              long long s_stride, long long b0, long long nblk,
                                                              double* __restrict__ peak, long long peak_stride) {
  __shared__ unsigned long long ired[kPeakThreads / 32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long sig = blockIdx.x / nblk, w = b0 + blockIdx.x % nblk;
  const long long g0 = (w == 0) ? 0 : w * (long long)g.W - 2;
  const long long avail = g.L - g0;
  const int n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  const double* src = s + sig * s_stride + (g0 - s_off);
  const int tid = threadIdx.x;
  unsigned long long m = 0ull;
  if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    const int n2 = n_valid / 2;
    for (int i0 = tid; i0 < n2; i0 += kPeakU * kPeakThreads) {
      double2 v[kPeakU];
#pragma unroll
      for (int u = 0; u < kPeakU; ++u) {
        const int i = i0 + u * kPeakThreads;
        v[u] = (i < n2) ? __ldg(s2 + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kPeakU; ++u) {
        const unsigned long long a = (unsigned long long)__double_as_longlong(v[u].x) & 0x7fffffffffffffffull;
        const unsigned long long b = (unsigned long long)__double_as_longlong(v[u].y) & 0x7fffffffffffffffull;
        m = a > m ? a : m;
        m = b > m ? b : m;
      }
    }
    if ((n_valid & 1) && tid == 0) {
      const unsigned long long a = (unsigned long long)__double_as_longlong(src[n_valid - 1]) & 0x7fffffffffffffffull;
      m = a > m ? a : m;
    }
  } else {
    for (int i = tid; i < n_valid; i += kPeakThreads) {
      const unsigned long long a = (unsigned long long)__double_as_longlong(__ldg(src + i)) & 0x7fffffffffffffffull;
      m = a > m ? a : m;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if ((tid & 31) == 0) ired[tid >> 5] = m;
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < kPeakThreads / 32; ++i) m = ired[i] > m ? ired[i] : m;
    peak[sig * peak_stride + w] = __longlong_as_double((long long)m);
  }
}

// ------------------------------------------------------------------ database winner (a9)
// One CTA: the largest score, ties to the smallest index (reading C17), over candidates
// (score[i], lag[i], first + i) or the rows {score, lag, index} of cand.
__global__ void __launch_bounds__(1024) pc_best_match(const double* __restrict__ score, const long long* __restrict__ lag,
                                                      const double* __restrict__ cand, long long n, long long first,
                                                      double* __restrict__ best) {
  __shared__ double sv[32], sl[32], si[32];
  double bv = -__longlong_as_double(0x7ff0000000000000LL), bl = 0.0, bi = -1.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = cand ? cand[3 * i] : score[i];
    const double l = cand ? cand[3 * i + 1] : (double)lag[i];
    const double x = cand ? cand[3 * i + 2] : (double)(first + i);
    if (bi < 0.0 || v > bv || (v == bv && x < bi)) {
      bv = v;
      bl = l;
      bi = x;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o), ol = __shfl_xor_sync(0xffffffffu, bl, o),
                 oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi >= 0.0 && (bi < 0.0 || ov > bv || (ov == bv && oi < bi))) {
      bv = ov;
      bl = ol;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    sl[threadIdx.x >> 5] = bl;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (si[w] >= 0.0 && (bi < 0.0 || sv[w] > bv || (sv[w] == bv && si[w] < bi))) {
        bv = sv[w];
        bl = sl[w];
        bi = si[w];
      }
    best[0] = bv;
    best[1] = bl;
    best[2] = bi;
  }
}

// ------------------------------------------------------------------ backend validation input
// x[i] = +-1 with the sign from a counter-based hash (splitmix64 of seed + i): every companded
// sample is +-S_q, so every packed digit has full magnitude ("randomized worst-case packed
// operands").
__global__ void pc_fill_pm1(double* __restrict__ x, long long n, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + 0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    x[i] = (z >> 63) ? -1.0 : 1.0;
  }
}

// ------------------------------------------------------------------ host-side launchers
template <int PACK>
static cudaError_t launch_fused_t(const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                                  cudaStream_t st) {
  auto kfn = pc_fused_kernel<PACK>;
  // the >48 KB opt-in is a per-function attribute: raised once per device and size, under a lock
  static LaunchAttrCache cache;
  int dev = 0, sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err == cudaSuccess) err = cache.ensure(kfn, dev, smem, threads, &sms);
  if (err != cudaSuccess) return err;
  kfn<<<(unsigned)n_jobs, threads, smem, st>>>(g, e);
  return cudaGetLastError();
}

cudaError_t launch_fused(int packing, const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                         cudaStream_t st) {
  if (n_jobs <= 0) return cudaSuccess;
  switch (packing) {
    case PACK_FULL: return launch_fused_t<PACK_FULL>(g, e, n_jobs, threads, smem, st);
    case PACK_SYM: return launch_fused_t<PACK_SYM>(g, e, n_jobs, threads, smem, st);
    case PACK_ASYM2: return launch_fused_t<PACK_ASYM2>(g, e, n_jobs, threads, smem, st);
    case PACK_ASYM3: return launch_fused_t<PACK_ASYM3>(g, e, n_jobs, threads, smem, st);
    case -1: return launch_fused_t<-1>(g, e, n_jobs, threads, smem, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_kernel_prep(const double* k_in, int N, int Np, int reverse, double K_q, double* k_pad,
                               double* k_int, double* scal, cudaStream_t st) {
  pc_kernel_prep<<<1, 1024, 0, st>>>(k_in, N, Np, reverse, K_q, k_pad, k_int, scal);
  return cudaGetLastError();
}

cudaError_t launch_build_taps(const double* k_pad, const double* k_int, int Np, int packing, double eps_inv, int K,
                              int K_pad, double* kr, cudaStream_t st) {
  const int blocks = (K_pad + 255) / 256;
  pc_build_taps<<<blocks, 256, 0, st>>>(k_pad, k_int, Np, packing, eps_inv, K, K_pad, kr);
  return cudaGetLastError();
}

cudaError_t launch_block_stats(const Geo& g, const double* s, double* sigma, double* peak, cudaStream_t st,
                               long long b0, long long nb) {
  if (nb < 0) nb = g.P - b0;
  if (nb <= 0) return cudaSuccess;
  pc_block_stats<<<(unsigned)nb, kStatsThreads, 0, st>>>(g, s, b0, sigma, peak);
  return cudaGetLastError();
}

cudaError_t launch_adapt_decide(long long P, const double* sigma, const double* peak, double sig_k, double peak_k,
                                const int* cand, const int* qmode, int ncand, double thr, int* dp, int* dq, double* ds,
                                cudaStream_t st) {
  pc_adapt_decide<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(P, sigma, peak, sig_k, peak_k, cand, qmode, ncand,
                                                                 thr, dp, dq, ds);
  return cudaGetLastError();
}

cudaError_t launch_kernel_prep_batch(const double* k_in, long long k_stride, long long n, int N, int Np, int reverse,
                                     double K_q, double* k_pad, double* k_int, long long pad_stride, double* scal,
                                     cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pc_kernel_prep_batch<<<(unsigned)n, 256, 0, st>>>(k_in, k_stride, N, Np, reverse, K_q, k_pad, k_int, pad_stride,
                                                    scal);
  return cudaGetLastError();
}

cudaError_t launch_build_taps_batch(const double* k_pad, const double* k_int, long long pad_stride, int Np,
                                    int packing, double eps_inv, int K, int K_pad, double* kr, long long kr_stride,
                                    long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pc_build_taps_batch<<<dim3((unsigned)((K_pad + 255) / 256), (unsigned)n), 256, 0, st>>>(
      k_pad, k_int, pad_stride, Np, packing, eps_inv, K, K_pad, kr, kr_stride);
  return cudaGetLastError();
}

cudaError_t launch_adapt_lists(long long P, const int* dec_pack, int* lists, int* counts, cudaStream_t st,
                               long long b0, long long stride) {
  pc_adapt_lists<<<1, 1024, 0, st>>>(P, b0, stride < 0 ? P : stride, dec_pack, lists, counts);
  return cudaGetLastError();
}

// Per signal: the maximum of the warp partials of the fused xcorr epilogue, lowest lag on ties.
__global__ void pc_xcorr_reduce(const double* __restrict__ val, const long long* __restrict__ lag, long long n_part,
                                double* __restrict__ score, long long* __restrict__ best) {
  __shared__ double sv[32];
  __shared__ long long sj[32];
  const long long sig = blockIdx.x;
  double v = -__longlong_as_double(0x7ff0000000000000LL);
  long long j = -1;
  for (long long i = threadIdx.x; i < n_part; i += blockDim.x) {
    const double a = val[sig * n_part + i];
    const long long b = lag[sig * n_part + i];
    if (b >= 0 && (j < 0 || a > v || (a == v && b < j))) {
      v = a;
      j = b;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long oj = __shfl_xor_sync(0xffffffffu, j, o);
    if (oj >= 0 && (j < 0 || ov > v || (ov == v && oj < j))) {
      v = ov;
      j = oj;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = v;
    sj[threadIdx.x >> 5] = j;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sj[w] >= 0 && (j < 0 || sv[w] > v || (sv[w] == v && sj[w] < j))) {
        v = sv[w];
        j = sj[w];
      }
    score[sig] = v;
    best[sig] = j;
  }
}

cudaError_t launch_xcorr_reduce(const double* val, const long long* lag, long long n_signals, long long n_part,
                                double* score, long long* best, cudaStream_t st) {
  if (n_signals <= 0) return cudaSuccess;
  pc_xcorr_reduce<<<(unsigned)n_signals, 256, 0, st>>>(val, lag, n_part, score, best);
  return cudaGetLastError();
}

// Reductions of the single-point SNR calibration (reading C18), one CTA, fixed order:
// out[0] = sum ref^2, out[1] = sum (ref - x)^2 over n outputs, out[2] = sum_b (sigma_b sigma_k)^2,
// out[3] = sum_b D_b with D_b Eq. (19)'s noise terms at S_q = K_q = Q (the oracle's
// snr_linear operation order per block; the sums differ from NumPy's only in order).
__global__ void __launch_bounds__(1024) pc_snr_sums(const double* __restrict__ ref, const double* __restrict__ x,
                                                    long long n, const double* __restrict__ sigma,
                                                    const double* __restrict__ peak, long long P, double sig_k,
                                                    double peak_k, double Q, double* __restrict__ out) {
  __shared__ double red[4][32];
  const int tid = threadIdx.x;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (long long i = tid; i < n; i += blockDim.x) {
    const double r = ref[i], d = __dsub_rn(r, x[i]);
    s0 = __dadd_rn(s0, __dmul_rn(r, r));
    s1 = __dadd_rn(s1, __dmul_rn(d, d));
  }
  const double q12 = __dmul_rn(Q, 3.4641016151377544);   // Q sqrt(12), sqrt(12) correctly rounded
  for (long long b = tid; b < P; b += blockDim.x) {
    const double v_s = __ddiv_rn(peak[b], q12), v_k = __ddiv_rn(peak_k, q12);
    const double a = __dmul_rn(sigma[b], v_k), bb = __dmul_rn(sig_k, v_s), c = __dmul_rn(v_k, v_s);
    const double D = __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(bb, bb)), __dmul_rn(c, c));
    const double nn = __dmul_rn(sigma[b], sig_k);
    s2 = __dadd_rn(s2, __dmul_rn(nn, nn));
    s3 = __dadd_rn(s3, D);
  }
  double v[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    for (int o = 16; o > 0; o >>= 1) v[q] = __dadd_rn(v[q], __shfl_xor_sync(0xffffffffu, v[q], o));
    if ((tid & 31) == 0) red[q][tid >> 5] = v[q];
  }
  __syncthreads();
  if (tid < 4) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t = __dadd_rn(t, red[tid][w]);
    out[tid] = t;
  }
}

cudaError_t launch_snr_sums(const double* ref, const double* x, long long n, const double* sigma, const double* peak,
                            long long P, double sig_k, double peak_k, double Q, double* out, cudaStream_t st) {
  pc_snr_sums<<<1, 1024, 0, st>>>(ref, x, n, sigma, peak, P, sig_k, peak_k, Q, out);
  return cudaGetLastError();
}

cudaError_t launch_xcorr_max(const double* c, long long n_signals, long long n_lags, long long stride,
                             double* score, long long* lag, cudaStream_t st) {
  pc_xcorr_max<<<(unsigned)n_signals, 1024, 0, st>>>(c, n_lags, stride, score, lag);
  return cudaGetLastError();
}

cudaError_t launch_fill_pm1(double* x, long long n, unsigned long long seed, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pc_fill_pm1<<<592, 256, 0, st>>>(x, n, seed);
  return cudaGetLastError();
}

cudaError_t launch_best_match(const double* score, const long long* lag, const double* cand, long long n,
                              long long first_index, double* best, cudaStream_t st) {
  pc_best_match<<<1, 1024, 0, st>>>(score, lag, cand, n, first_index, best);
  return cudaGetLastError();
}

cudaError_t launch_block_peak(const Geo& g, const double* s, long long s_off, long long s_stride, long long b0,
                              long long nblk, long long n_sig, double* peak, long long peak_stride, cudaStream_t st) {
  if (nblk <= 0 || n_sig <= 0) return cudaSuccess;
  pc_block_peak<<<(unsigned)(nblk * n_sig), kPeakThreads, 0, st>>>(g, s, s_off, s_stride, b0, nblk, peak, peak_stride);
  return cudaGetLastError();
}

}  // namespace pc
