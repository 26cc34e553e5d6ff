// pc_device.cuh -- device-side building blocks of the sm_100a packed overlap-save path.
//
// Paper: Anam & Andreopoulos, arXiv 1201.3018 (PAPER.md, cited P:<line>).  Readings of the
// paper (C1..C17) are those of SURVEY.md §8(c), listed in DESIGN.md §3.
//
// Everything numeric here is written so that the device reproduces the CPU oracle bit for
// bit where the method is exact: companding is one IEEE multiply and a round-half-away
// (CUDA round()), packing is explicit non-contracted products and sums (__dmul_rn /
// __dadd_rn), and under the dyadic epsilon (C4) every packed product and partial sum is
// exact in binary64, so the FMA order of the convolution core cannot change a bit.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pc {

enum { PACK_FULL = 0, PACK_SYM = 1, PACK_ASYM2 = 2, PACK_ASYM3 = 3 };

// ------------------------------------------------------------------ geometry (Eq.(17))
struct Geo {
  long long L;        // input samples
  long long P;        // overlap-save blocks, ceil(L / W)
  int N, Np;          // kernel taps, N' (odd, C13)
  int W_block, W;     // block samples, outputs per block (W = W_block - N' - 1)
  int mode;           // 0 conv, 1 xcorr
};

// Per-block description.  Block 0 reads input [0, W_block) and keeps local outputs
// [0, W+N'-1); block w >= 1 reads [wW-2, wW-2+W_block) and keeps [N'+1, N'+1+W)
// placed at global N'-1+wW (Eq. (17); reading C7).
struct Blk {
  long long g0;   // global index of local sample 0
  int o0, n_out;  // first kept local output, number kept
  int M_out;      // outputs of the convolution core (packed words)
  int xlen;       // words of the core's input (M_out + K - 1)
  int pre;        // SYM: core word i is s_bar[i - pre]
  int S;          // ASYM: segment length ceil(n_out / M) (reading C8)
};

// K = taps of the convolution core (ceil(N'/2) for symmetric packing, N' otherwise).
template <int PACK>
__host__ __device__ inline Blk block_info(const Geo& g, int K, long long w) {
  Blk b;
  b.g0 = (w == 0) ? 0 : w * (long long)g.W - 2;
  b.o0 = (w == 0) ? 0 : g.Np + 1;
  b.n_out = (w == 0) ? g.W + g.Np - 1 : g.W;
  b.pre = 0;
  b.S = 0;
  if (PACK == PACK_SYM) {
    // Eq. (9)-(10): packed outputs W_start <= m < W_block/2, W_start = 0 (w=0) / K-1
    b.M_out = (w == 0) ? (g.W + g.Np - 1) / 2 : g.W / 2 + 1;
    b.pre = (w == 0) ? K - 1 : 0;
  } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
    const int M = (PACK == PACK_ASYM2) ? 2 : 3;
    b.S = (b.n_out + M - 1) / M;
    b.M_out = b.S;
  } else {
    b.M_out = b.n_out;
  }
  b.xlen = b.M_out + K - 1;
  return b;
}

// ------------------------------------------------------------------ TMA bulk copy (sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Named barrier among `count` threads (count a multiple of 32); id 0 is __syncthreads.
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
#ifndef PC_SUSPEND_HINT_NS
#define PC_SUSPEND_HINT_NS 1000u
#endif
constexpr uint32_t kSuspendHintNs = PC_SUSPEND_HINT_NS;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "PC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra PC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(kSuspendHintNs)   // suspend-time hint (ns): sleep instead of spinning
      : "memory");
}

// ------------------------------------------------------------------ companding / packing
// Eq. (2): x~ = [[c x]], round half away from zero (reading C5) = CUDA round().
// round() compiles to DADD.RZ(y, copysign(0.5, y)) + FRND.F64.TRUNC.  Two bit-identical
// alternatives are kept as compile-time experiments (tools/round_check.cu: 73.4 M operands, 0
// mismatches; all GPU parity tests green; both measured SLOWER in the persistent kernel,
// DESIGN.md 7.3, so the default stays round()):
//   PC_RND_ADD = 1: for |y| < 2^51, trunc(|y| + 0.5) by two toward-zero adds and one exact
//     subtraction of 2^52 (|y| + 0.5 rounded toward zero never reaches the next integer unless
//     the exact sum does; the ulp at 2^52 is 1), with y's sign (round(-0.3) = -0.0 too) -- no
//     conversion-unit instruction, two more FP64 ones;
//   PC_RND_ADD = 2: rint() (one FRND) unless y may be an exact tie (integer filter), then round()
//     -- one FP64 instruction fewer on the common path, the rare path predicated.
// Larger |y|, infinities and NaNs (integer test of the high word) take round().
#ifndef PC_RND_ADD
#define PC_RND_ADD 0
#endif
__device__ __forceinline__ double round_away(double y) {
#if PC_RND_ADD == 1
  const int hi = __double2hiint(y);
  if ((hi & 0x7fffffff) < 0x43200000) {              // |y| < 2^51
    const double kTwo52 = 4503599627370496.0;
    const double t = __dadd_rz(fabs(y), 0.5);
    const double r = __dsub_rn(__dadd_rz(t, kTwo52), kTwo52);
    return __hiloint2double((__double2hiint(r) & 0x7fffffff) | (hi & (int)0x80000000), __double2loint(r));
  }
#endif
#if PC_RND_ADD == 2
  // rint() (one FRND, round half to even) equals round() unless y is an exact tie n + 0.5; for
  // |y| < 2^27 a tie has at most 28 significant bits, so a nonzero low 24-bit field of the
  // significand rules it out (integer test); ties, larger |y|, infinities and NaNs take round().
  const unsigned hi2 = (unsigned)__double2hiint(y) & 0x7fffffffu;
  const bool maybe = ((unsigned)__double2loint(y) & 0xffffffu) == 0u || hi2 >= 0x41a00000u;
  if (!maybe) return rint(y);
#endif
  return round(y);
}
__device__ __forceinline__ double compand1(double c, double x) { return round_away(__dmul_rn(c, x)); }

// Eq. (4): s_bar = s~_even + eps * s~_odd (one product, one sum; oracle order).
__device__ __forceinline__ double pack_sym(double s0, double s1, double eps) {
  return __dadd_rn(s0, __dmul_rn(eps, s1));
}

// ------------------------------------------------------------------ unpacking
// Symmetric balanced three-digit decode (C6): r_bar = A + eps B + eps^-1 C.
// Round to nearest even for |x| < 2^51 with two FP64 adds (exact; equals rint()).  The
// decoders only see values far below that bound (|digit| <= R_max < 2^27), and no ties
// occur in a valid decode, so this is bit-identical to the oracle's np.rint.
__device__ __forceinline__ double rint_fast(double x) {
  const double kMagic = 6755399441055744.0;   // 1.5 * 2^52
  return __dsub_rn(__dadd_rn(x, kMagic), kMagic);
}

struct Digits3 {
  double A, B, C;
};
__device__ __forceinline__ double div_eps_inv(double v, double eps, double eps_inv, bool pow2) {
  // v / eps^-1: exact multiply by 2^-b under POW2 (bit-identical to the division).
  return pow2 ? __dmul_rn(v, eps) : __ddiv_rn(v, eps_inv);
}
__device__ __forceinline__ Digits3 decode_sym(double r, double eps, double eps_inv, bool pow2) {
  Digits3 d;
  d.C = rint_fast(div_eps_inv(r, eps, eps_inv, pow2));
  const double rem = __dsub_rn(r, __dmul_rn(d.C, eps_inv));
  d.A = rint_fast(rem);
  d.B = rint_fast(__dmul_rn(__dsub_rn(rem, d.A), eps_inv));
  return d;
}
__device__ __forceinline__ double decode_sym_B(double r, double eps, double eps_inv, bool pow2) {
  return decode_sym(r, eps, eps_inv, pow2).B;
}

// Inverse companding, Eq. (16): r = (c_s c_k)^-1 r~ with the inverse formed once
// per block (one product, one IEEE division; reading C11) and one multiply per output.
__device__ __forceinline__ double dequant_scale(double c_s, double c_k) {
  return __ddiv_rn(1.0, __dmul_rn(c_s, c_k));
}

// ------------------------------------------------------------------ convolution core
// Valid-mode correlation on shared memory:  out[m] = sum_{j<K} x[m + j] * kr[j]
// (kr = core taps reversed, so this is Eq. (9)/(8)/(1) on the core's words).
//
// x is stored "column-major by T": word i lives at xs[(i % T) * rows + i / T].  Thread
// group g owns outputs [gT, gT+T); at tap j it needs the one new word gT + T-1 + j, which
// for consecutive g is consecutive in shared memory (conflict-free, 2 wavefronts per warp
// for 8-byte loads), while the tap kr[j] is a warp-uniform broadcast.  The T-word window
// slides through registers with static indices after full unrolling: T FP64 FMAs per
// (1 x-load + 1/2 tap-load).  T = 8 keeps the FP64 pipe, not shared memory, the limit
// (SURVEY §7 "Direct-kernel operand bandwidth").
template <int T>
__device__ __forceinline__ void conv_group_range(const double* __restrict__ xs, int rows,
                                                 const double* __restrict__ kr, int j_begin, int j_end, int g,
                                                 double (&acc)[T]) {
  // taps [j_begin, j_end) (multiples of T) of the T outputs of group g: word gT + j of the
  // window sits at column (j % T), row g + j / T
  double win[T];
#pragma unroll
  for (int i = 0; i < T; ++i) acc[i] = 0.0;
  const double* xcol = xs + g;
#pragma unroll
  for (int c = 0; c < T - 1; ++c) win[c] = xcol[c * rows + j_begin / T];
  for (int j0 = j_begin; j0 < j_end; j0 += T) {
    const int r0 = j0 / T;
    double kk[T];
#pragma unroll
    for (int u = 0; u < T; u += 2) {
      const double2 k2 = *reinterpret_cast<const double2*>(kr + j0 + u);
      kk[u] = k2.x;
      kk[u + 1] = k2.y;
    }
#pragma unroll
    for (int u = 0; u < T; ++u) {
      // new word x[gT + j0 + T-1 + u] -> column (T-1+u) % T, row g + r0 + (T-1+u) / T
      win[(T - 1 + u) % T] = xcol[((T - 1 + u) % T) * rows + r0 + (T - 1 + u) / T];
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = fma(win[(i + u) % T], kk[u], acc[i]);
    }
  }
}
template <int T>
__device__ __forceinline__ void conv_group(const double* __restrict__ xs, int rows,
                                           const double* __restrict__ kr, int K_pad, int g,
                                           double (&acc)[T]) {
  conv_group_range<T>(xs, rows, kr, 0, K_pad, g, acc);
}

// Padded row-major layout (persistent kernel): word i of the core's input lives at
// xs[(i / T) * (T + 1) + i % T].  Thread group g reads rows g, g+1, ...; the odd row pitch
// T+1 makes lane-consecutive rows conflict-free (2 wavefronts per 8-byte warp load), and
// every load of the unrolled tap loop is the thread's row pointer plus an immediate.
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds128(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
template <int T>
__device__ __forceinline__ void conv_group_padded(uint32_t xs_row, uint32_t kr_addr, int K_pad, double (&acc)[T]) {
  double win[T];
#pragma unroll
  for (int i = 0; i < T; ++i) acc[i] = 0.0;
#pragma unroll
  for (int c = 0; c < T - 1; ++c) win[c] = lds64(xs_row + 8u * c);
  uint32_t xa = xs_row, ka = kr_addr;
  for (int j0 = 0; j0 < K_pad; j0 += T, xa += 8u * (T + 1), ka += 8u * T) {
    double kk[T];
#pragma unroll
    for (int u = 0; u < T; u += 2) {
      const double2 k2 = lds128(ka + 8u * u);
      kk[u] = k2.x;
      kk[u + 1] = k2.y;
    }
#pragma unroll
    for (int u = 0; u < T; ++u) {
      // new word x[gT + j0 + T-1 + u]: row +(T-1+u)/T, column (T-1+u)%T
      win[(T - 1 + u) % T] = lds64(xa + 8u * (((T - 1 + u) / T) * (T + 1) + (T - 1 + u) % T));
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = fma(win[(i + u) % T], kk[u], acc[i]);
    }
  }
}

}  // namespace pc
