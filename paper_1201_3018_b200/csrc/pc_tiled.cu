// pc_tiled.cu -- the production kernel of the packed overlap-save path (arXiv 1201.3018):
// one persistent CTA per SM, warp-specialized, (block, output-tile) jobs in per-SM queues.
//
// Job = (signal, overlap-save block w, tile t).  Tile t covers core outputs
// [t*G*T, (t+1)*G*T) of block w (G = 32 npart groups of T outputs; npart warp parts).  The
// core taps are processed in chunks of KC (one chunk, taps resident in shared memory, when
// they fit), so any kernel length runs: cfg2's 513 taps in one chunk, cfg3/cfg4's 4097/8193
// in several.
//
//   producer warps  a2-a4: job m is produced by warp m mod 4 -- block peak (coalesced loads
//                   + shuffles; reused across the tiles of one block), companding (Eq. (2)),
//                   packing (Eq. (4) / Eq. (7)) of the words one (tile, chunk) needs into a
//                   stage of the ring; non-resident tap chunks arrive by TMA bulk copy on the
//                   stage's mbarrier
//   consumer warps  a5: the core on one part of a job (accumulators live across chunks):
//                   MMA = 1, a Toeplitz product on the FP64 tensor cores (conv_chunk_mma; at
//                   most PC_CORE_SLOTS = 2 warps per SMSP in it at once, claim-ordered ticket),
//                   the part a balanced share of the tile's 8-group m-tiles; MMA = 0, the
//                   register-tiled FMA loop (conv_chunk_padded) on 32 groups of T outputs;
//                   a6-a7: unpacking, inverse companding and placement through per-warp
//                   staging rows, coalesced stores
//
// Stages are handed over with mbarriers (full: producer -> consumers, + TMA bytes; empty:
// the job's part warps -> producers) and stamped with their sequence number.  Warp parts are
// bound to SM sub-partitions (part k of the job sequence runs on SMSP k mod 4).  Symmetric
// packing needs B of the word before each warp's first group: that warp computes the one
// extra core output by a warp-split dot product (exact under the dyadic eps, reading C4).
#include <cstdio>

#include "pc_device.cuh"
#include "pc_intfp.cuh"
#include "pc_kernels.h"

#ifndef PC_QUEUE_MIN
#define PC_QUEUE_MIN 8    // jobs per SM queue at least (fewer queues than SMs below 8 jobs each)
#endif
#ifndef PC_NO_STEAL
#define PC_NO_STEAL 0     // diagnostics: 1 = no work stealing between SM queues
#endif
#ifndef PC_PROD_YIELD
#define PC_PROD_YIELD 0   // 1: one DMMA core slot on an SMSP while its producer packs (measured: asym2 +1%, full +14%)
#endif
#ifndef PC_DMMA_NAP
#define PC_DMMA_NAP 0     // ns a DMMA-core warp sleeps after each k-step (0: none)
#endif
#ifndef PC_VEC_PEAK
#define PC_VEC_PEAK 1     // raw-staged producers: block peak by 16-byte shared-memory loads
#endif
#ifndef PC_PAIR_PACK
#define PC_PAIR_PACK 1    // raw-staged producers, asymmetric packing: word pairs by 16-byte loads / stores
#endif
#ifndef PC_SPLIT_AHEAD
#define PC_SPLIT_AHEAD 2  // producer-SM mode: job claims ahead of the consumers' part claims
#endif
#ifndef PC_CORE_SLOTS
#define PC_CORE_SLOTS 2   // DMMA core: warps per SM sub-partition allowed in the core at once
#endif

namespace pc {

namespace {

struct TSmem {
  uint64_t bar_taps, full[kTiledMaxStages], empty[kTiledMaxStages];
  long long job[kTiledMaxStages];   // -1: sentinel (no more work)
  unsigned long long jpos[kTiledMaxStages];   // the job's position (pack_pos): sig << 40 | w << 8 | t
  long long seq[kTiledMaxStages];   // stage sequence number the slot holds
  double inv[kTiledMaxStages];      // (c_s c_k)^-1 of the stage's block (Eq. (16))
  int smsp_ctr[4];                  // consumer warp-job claim counters, one per SM sub-partition
  int core_serve[4];                // DMMA core: the claim whose warp may run its core on each SMSP
  int mseq_hi;                      // 1 + the highest job sequence any consumer warp has claimed a part of
  int prod_busy[4];                 // producer warp of SMSP s is companding/packing (DMMA core: one core slot)
  long long turn;                   // next job sequence to claim (claims happen in sequence order)
  long long fjob[16];               // pipeline fill: jobs of sequences 0 .. nf-1
  double fcs[16], finv[16];         // their c_s and (c_s c_k)^-1
  long long m_end;                  // first job sequence whose claim failed (-1: not yet)
  uint64_t rawbar[2];               // raw-staged producers: TMA arrival of raw slot k
  uint64_t pbar[4];                 // producer CTAs (producer-SM mode): TMA arrival of group g's raw block
  long long pjob[2];                // raw-staged producers: claimed job of sequence m (slot m & 1)
  double red[32];
  long long cyc[4];   // diagnostics (consumer thread 0): wait, core, unpack/store cycles; clock mark
};
static_assert(sizeof(TSmem) <= kTiledHeader, "header");

struct JobPos {
  long long sig, w;
  int t;
};

__device__ __forceinline__ unsigned long long pack_pos(const JobPos& p) {
  return ((unsigned long long)p.sig << 40) | ((unsigned long long)p.w << 8) | (unsigned long long)p.t;
}
__device__ __forceinline__ JobPos unpack_pos(unsigned long long v) {
  JobPos p;
  p.sig = (long long)(v >> 40);
  p.w = (long long)((v >> 8) & 0xffffffffull);
  p.t = (int)(v & 0xffull);
  return p;
}
// 64-bit quotient / remainder through the 32-bit divide when both operands fit (the usual
// case; a 64-bit division is a ~70-instruction subroutine, expensive for warps that share their
// sub-partition with DMMA-issuing warps)
__device__ __forceinline__ long long qdiv(long long a, long long b) {
  return (((unsigned long long)a | (unsigned long long)b) >> 31) == 0 ? (long long)((unsigned)a / (unsigned)b) : a / b;
}
__device__ __forceinline__ long long qmod(long long a, long long b) {
  return (((unsigned long long)a | (unsigned long long)b) >> 31) == 0 ? (long long)((unsigned)a % (unsigned)b) : a % b;
}
__device__ __forceinline__ JobPos job_pos(const Exec& e, long long job) {
  JobPos p;
  if (e.blk_list) {                                  // adaptive: this launch's blocks, ascending
    const bool first0 = e.blk_list[0] == 0;          // block 0 (tiles0 tiles) can only come first
    p.sig = 0;
    if (first0 && job < e.tiles0) {
      p.w = 0;
      p.t = (int)job;
      return p;
    }
    const long long r = first0 ? job - e.tiles0 : job;
    p.w = e.blk_list[(first0 ? 1 : 0) + qdiv(r, e.tiles1)];
    p.t = (int)qmod(r, e.tiles1);
    return p;
  }
  p.sig = qdiv(job, e.jobs_per_sig);
  long long r = job - p.sig * e.jobs_per_sig;
  if (e.b0 == 0) {                                   // block 0 (if in range) has tiles0 tiles
    if (r < e.tiles0) {
      p.w = 0;
      p.t = (int)r;
      return p;
    }
    r -= e.tiles0;
    p.w = 1 + qdiv(r, e.tiles1);
    p.t = (int)(r - (p.w - 1) * e.tiles1);
  } else {
    const long long q = qdiv(r, e.tiles1);
    p.w = e.b0 + q;
    p.t = (int)(r - q * e.tiles1);
  }
  return p;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- integer (ALU-pipe) forms of the producer's arithmetic (pc_intfp.cuh): while two warps of an
// SM sub-partition issue DMMAs, an FP64 instruction of any other warp there waits until they
// pause (3.6-9.5 us measured for the first one of a producer's job), so with ModeP::alu_pack the
// producer warps compute c_s, (c_s c_k)^-1, the companded samples and the packed words with
// integer instructions only -- the same bits as the FP64 forms (tests/test_intfp.py).  An
// operand outside the integer forms' domain (subnormal, overflow) takes the FP64 instruction.
// PC_DIV_ALU = 1: only the two per-block scalars c_s and (c_s c_k)^-1 of the steady-state producers
// (two IEEE divisions, ~40 dependent FP64 instructions that each wait for a pause of the DMMA
// warps) take the integer forms; companding and packing stay on the FP64 pipe.
// words per producer thread in flight in pack_window (x UWF; full precision: 8).  4 for symmetric and
// asym2 packing: half the unrolled body of 8 (the producers lose 22 % of their stall samples to
// instruction fetch, profiles/r02k_src/) at no loss of overlap -- cfg2 sym 72.3 -> 71.0 us, asym2
// 88.9 -> 88.6 us; 2 costs asym2 +1 us; asym3 at 2 instead of 4: no gain (profiles/r02l_uw/)
#ifndef PC_PACK_UW
#define PC_PACK_UW 4
#endif
#ifndef PC_PACK_UW3
#define PC_PACK_UW3 4
#endif
#ifndef PC_DIV_ALU
#define PC_DIV_ALU 0
#endif
__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(uint64_t u) { return __longlong_as_double((long long)u); }
// c_s = Q / peak (Eq. (2); all-zero block: 1), the IEEE quotient
__device__ __forceinline__ double cs_quot(const ModeP& mp, double peak, bool alu) {
  const uint64_t pb = dbits(peak);
  if ((pb << 1) == 0) return 1.0;                    // +-0 (bit test: no FP64 compare)
  uint64_t r;
  if (alu && ifp::ddiv_rn_pos(dbits(mp.Q), pb, r)) return bitsd(r);
  return mp.Q / peak;
}
// Eq. (16)'s (c_s c_k)^-1: one product, one IEEE division (reading C11)
__device__ __forceinline__ double inv_scale(const ModeP& mp, double c_s, double c_k, bool alu) {
  uint64_t p, r;
  if (alu && ifp::dmul_rn_pos(dbits(c_s), dbits(c_k), p) && ifp::ddiv_rn_pos(dbits(1.0), p, r)) return bitsd(r);
  return dequant_scale(c_s, c_k);
}
// One packed word of M companded samples x[0..M-1] (Eq. (7) Horner in the oracle's order; for
// symmetric packing M = 2, Eq. (4)): integer digits n_q = round(c_s x_q), word = N 2^-((M-1) b)
// with N = sum n_q 2^((M-1-q) b), exact under ModeP::exact_pack (alu_pack implies it).  The
// exact integer form (~100 instructions per sample); pack_word_fast below is the common path.
template <int M>
__device__ __noinline__ double pack_word_exact(const ModeP& mp, double c_s, double x0, double x1, double x2) {
  const double x[3] = {x0, x1, x2};
  long long N = 0;
  bool neg0 = true, ok = true;
#pragma unroll
  for (int q = 0; q < M; ++q) {
    long long n;
    bool z;
    ok = ifp::compand_int(dbits(c_s), dbits(x[q]), n, z) && ok;
    N = N * (1LL << mp.b) + n;
    neg0 = neg0 && z;
  }
  if (ok) return bitsd(ifp::i2d_scaled(N, (M - 1) * mp.b, neg0));
  double a = compand1(c_s, x[M - 1]);                // FP64 forms (operand outside the integer domain)
#pragma unroll
  for (int q = M - 2; q >= 0; --q) a = __dadd_rn(compand1(c_s, x[q]), __dmul_rn(mp.eps, a));
  return a;
}
// |x| truncated to a float (24 leading significand bits; 0 below 2^-126): relative error < 2^-23
__device__ __forceinline__ float f32_trunc_abs(double x) {
  const uint32_t ah = (uint32_t)__double2hiint(x) & 0x7fffffffu, lo = (uint32_t)__double2loint(x);
  const int t = (int)(ah - (896u << 20));              // exponent rebias 1023 -> 127
  return t < (1 << 20) ? 0.0f : __int_as_float((t << 3) | (int)(lo >> 29));
}
// Fast companding (FP32 + integer instructions): y = c_f |x| with c_f = c_s and |x| truncated to
// floats is within 2.5 * 2^-23 Q of c_s |x| (|x| <= the block peak, so c_s |x| <= Q); its nearest
// integer is round(RN(c_s x)) unless y lies within thr of a half-integer, where the word is
// recomputed exactly (pack_word_exact; about one sample in 1 / (2^-19 Q)).  Valid per job when
// Q <= 2^19 and c_s in [2^-100, 2^100] (floats normal, y < 2^22).
struct FastCs {
  float c, thr;   // c_f, ambiguity threshold 0.5 - Q 2^-20 (twice the error bound)
  bool ok;
};
__device__ __forceinline__ FastCs fast_cs(const ModeP& mp, double c_s, bool alu) {
  FastCs f;
  const int ec = (int)((dbits(c_s) >> 52) & 0x7ff);
  // (bit compares and truncations only: an FP64 compare or conversion would wait behind the DMMAs)
  f.ok = alu && dbits(mp.Q) <= 0x4120000000000000ull && ec >= 1023 - 100 && ec <= 1023 + 100;   // Q <= 2^19
  f.c = f32_trunc_abs(c_s);
  f.thr = __fsub_rn(0.5f, __fmul_rn(f32_trunc_abs(mp.Q), 9.5367431640625e-07f));   // 0.5 - Q 2^-20 (Q exact)
  return f;
}
template <int M>
__device__ __forceinline__ double pack_word_fast(const FastCs& f, const ModeP& mp, double c_s, const double (&x)[M]) {
  if (!f.ok) return pack_word_exact<M>(mp, c_s, x[0], x[1], M > 2 ? x[M - 1] : 0.0);
  long long N = 0;
  bool neg0 = true, amb = false;
#pragma unroll
  for (int q = 0; q < M; ++q) {
    const float y = __fmul_rn(f.c, f32_trunc_abs(x[q]));
    const float r = __fadd_rn(y, 12582912.0f);          // 1.5 * 2^23: round to nearest even
    const float d = __fsub_rn(y, __fsub_rn(r, 12582912.0f));
    amb = amb || fabsf(d) > f.thr;
    const int a = __float_as_int(r) - 0x4B400000;
    const bool neg = __double2hiint(x[q]) < 0;
    N = N * (1LL << mp.b) + (neg ? -a : a);
    neg0 = neg0 && neg && a == 0;
  }
  if (amb) return pack_word_exact<M>(mp, c_s, x[0], x[1], M > 2 ? x[M - 1] : 0.0);
  return bitsd(ifp::i2d_scaled(N, (M - 1) * mp.b, neg0));
}

// |x| as ordered integer bits (non-negative doubles order like their bit patterns).
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return a > b ? a : b; }

// One Horner step of Eqs. (4)/(7), lo + eps * hi, in the oracle's order (product, then sum); when
// every packed word is exact in FP64 (dyadic eps, ModeP::exact_pack) both roundings are exact and
// one FMA gives the same bits with one FP64 instruction fewer (the producers wait behind the DMMA
// warps for every FP64 instruction they issue).
__device__ __forceinline__ double horner_step(const ModeP& mp, double lo, double hi) {
  return mp.exact_pack ? fma(mp.eps, hi, lo) : __dadd_rn(lo, __dmul_rn(mp.eps, hi));
}

// a4 for one stage: core words [cw0, cw0 + rows_s*T) of block b into the padded row-major
// window xs[(i / T) * PT + i % T] (pitch PT = T + 1 for the FMA core, T + 4 for the DMMA core).  Word-major over the producer threads (coalesced
// loads), UW words per thread with every sample load issued before any use.
template <int PACK, int T, int UWF = 1, int PT = T + 1, bool SRC_SMEM = false, bool ALU = false>
__device__ __forceinline__ void pack_window(const Geo& g, const Blk& b, const ModeP& mp, const double* gsrc,
                                            int n_valid, double c_s, int cw0, int rows_s, double* xs, int ptid,
                                            int nprod, bool alu) {
  constexpr int UW = UWF * ((PACK == PACK_ASYM3) ? PC_PACK_UW3 : (PACK == PACK_FULL) ? 8 : PC_PACK_UW);   // words per thread in flight
  const int words = rows_s * T;
  auto sample = [&](int i) -> double {
    return (i < 0 || i >= n_valid) ? 0.0 : (SRC_SMEM ? gsrc[i] : __ldg(gsrc + i));
  };
  if (!ALU) alu = false;                             // (the integer forms are compiled only where asked)
  const FastCs fcs = fast_cs(mp, c_s, alu);
  // window words [ilo, ihi) whose core word is inside the block's input (cw in [pre, xlen)) and
  // whose samples are all inside the block's valid samples: there, no per-sample / per-word range
  // checks (the checks were a fifth of the producers' instructions)
  int ilo, ihi;
  {
    constexpr int MS = (PACK == PACK_ASYM3) ? 3 : 2;
    if (PACK == PACK_SYM) {
      ilo = max(0, b.pre - cw0);
      ihi = min(words, b.xlen - cw0);
      ihi = n_valid >= 2 ? min(ihi, ((n_valid - 2) >> 1) + b.pre - cw0 + 1) : 0;
    } else {
      const int base = b.o0 - (g.Np - 1) + cw0;
      const int span = (PACK == PACK_FULL) ? 0 : (MS - 1) * b.S;
      ilo = max(0, max(-cw0, -base));
      ihi = min(words, min(b.xlen - cw0, n_valid - base - span));
    }
  }
  // Raw block in shared memory, asymmetric packing, even pitch: the interior in word pairs
  // (2j, 2j + 1) -- one 16-byte load per sample stream where it is aligned and one 16-byte store
  // per pair (the producers' shared-memory instructions queue behind the DMMA warps' fragment
  // loads, so fewer, wider ones shorten every job's packing).  Same arithmetic per word.
  int wlo = 0, whi = 0;                              // words [wlo, whi) done by the pair loop (none by default)
  if constexpr (PC_PAIR_PACK && SRC_SMEM && (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) && PT % 2 == 0 && T % 2 == 0) {
    constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
    constexpr int UP = UW / 2;                       // pairs per thread in flight
    const double* src = gsrc + (b.o0 - (g.Np - 1) + cw0);
    const int plo = (ilo + 1) >> 1, phi = ihi >> 1;  // pairs wholly inside [ilo, ihi)
    if ((reinterpret_cast<uintptr_t>(xs) & 15u) == 0 && phi > plo) {
      bool al[M];
#pragma unroll
      for (int q = 0; q < M; ++q) al[q] = (reinterpret_cast<uintptr_t>(src + q * b.S) & 15u) == 0;
      wlo = 2 * plo;
      whi = 2 * phi;
      for (int j0 = plo + ptid; j0 < phi; j0 += UP * nprod) {
        double2 x[M][UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int j = min(j0 + u * nprod, phi - 1);   // clamped lanes recompute pair phi-1 (not stored)
#pragma unroll
          for (int q = 0; q < M; ++q) {
            const double* p2 = src + q * b.S + 2 * j;
            x[q][u] = al[q] ? *reinterpret_cast<const double2*>(p2) : make_double2(p2[0], p2[1]);
          }
        }
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int j = j0 + u * nprod;
          double lo, hi;
          if (alu) {
            double xl[M], xh[M];
#pragma unroll
            for (int q = 0; q < M; ++q) {
              xl[q] = x[q][u].x;
              xh[q] = x[q][u].y;
            }
            lo = pack_word_fast<M>(fcs, mp, c_s, xl);
            hi = pack_word_fast<M>(fcs, mp, c_s, xh);
          } else {
            lo = compand1(c_s, x[M - 1][u].x);           // Horner, oracle order
            hi = compand1(c_s, x[M - 1][u].y);
#pragma unroll
            for (int q = M - 2; q >= 0; --q) {
              lo = horner_step(mp, compand1(c_s, x[q][u].x), lo);
              hi = horner_step(mp, compand1(c_s, x[q][u].y), hi);
            }
          }
          if (j < phi) {
            const int i = 2 * j;
            *reinterpret_cast<double2*>(xs + (i / T) * PT + i % T) = make_double2(lo, hi);
          }
        }
      }
    }
  }
  for (int i0 = ptid; i0 < words; i0 += UW * nprod) {
    double v[UW];
    if (i0 >= wlo && i0 + (UW - 1) * nprod < whi) continue;   // done by the pair loop
    if (i0 >= ilo && i0 + (UW - 1) * nprod < ihi && (i0 + (UW - 1) * nprod < wlo || i0 >= whi)) {   // interior: unchecked
      if (PACK == PACK_SYM) {
        double x0[UW], x1[UW];
        if (PC_PAIR_PACK && SRC_SMEM && (reinterpret_cast<uintptr_t>(gsrc) & 15u) == 0) {   // one 16-byte load per word
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            const double2 x2 = reinterpret_cast<const double2*>(gsrc)[cw0 + i0 + u * nprod - b.pre];
            x0[u] = x2.x;
            x1[u] = x2.y;
          }
        } else {
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            const int j = cw0 + i0 + u * nprod - b.pre;
            x0[u] = SRC_SMEM ? gsrc[2 * j] : __ldg(gsrc + 2 * j);
            x1[u] = SRC_SMEM ? gsrc[2 * j + 1] : __ldg(gsrc + 2 * j + 1);
          }
        }
        if (alu) {
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            const double xx[2] = {x0[u], x1[u]};
            v[u] = pack_word_fast<2>(fcs, mp, c_s, xx);
          }
        } else {
#pragma unroll
          for (int u = 0; u < UW; ++u) v[u] = horner_step(mp, compand1(c_s, x0[u]), compand1(c_s, x1[u]));
        }
      } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
        constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
        double x[M][UW];
        const double* src = gsrc + (b.o0 - (g.Np - 1) + cw0 + i0);
#pragma unroll
        for (int u = 0; u < UW; ++u)
#pragma unroll
          for (int q = 0; q < M; ++q) x[q][u] = SRC_SMEM ? src[q * b.S + u * nprod] : __ldg(src + q * b.S + u * nprod);
        if (alu) {                                           // integer Horner (dyadic eps), same bits
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            double xx[M];
#pragma unroll
            for (int q = 0; q < M; ++q) xx[q] = x[q][u];
            v[u] = pack_word_fast<M>(fcs, mp, c_s, xx);
          }
        } else {
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            double a = compand1(c_s, x[M - 1][u]);         // Horner, oracle order
#pragma unroll
            for (int q = M - 2; q >= 0; --q) a = horner_step(mp, compand1(c_s, x[q][u]), a);
            v[u] = a;
          }
        }
      } else {
        const double* src = gsrc + (b.o0 - (g.Np - 1) + cw0 + i0);
#pragma unroll
        for (int u = 0; u < UW; ++u) v[u] = SRC_SMEM ? src[u * nprod] : __ldg(src + u * nprod);
      }
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int i = i0 + u * nprod;
        xs[(i / T) * PT + i % T] = v[u];
      }
      continue;
    }
    if (PACK == PACK_SYM) {
      double x0[UW], x1[UW];
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int j = cw0 + i0 + u * nprod - b.pre;      // s_bar[j] uses samples 2j, 2j+1 (Eq. (4))
        x0[u] = sample(2 * j);
        x1[u] = sample(2 * j + 1);
      }
      if (alu) {                                             // n = s~0 2^b + s~1, word = n 2^-b
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          const int cw = cw0 + i0 + u * nprod;
          const double xx[2] = {x0[u], x1[u]};
          v[u] = (cw >= b.pre && cw < b.xlen) ? pack_word_fast<2>(fcs, mp, c_s, xx) : 0.0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          const int cw = cw0 + i0 + u * nprod;
          v[u] = (cw >= b.pre && cw < b.xlen) ? horner_step(mp, compand1(c_s, x0[u]), compand1(c_s, x1[u])) : 0.0;
        }
      }
    } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
      constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
      double x[M][UW];
      const int base = b.o0 - (g.Np - 1) + cw0;          // Eq. (7) under C8
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int q = 0; q < M; ++q) x[q][u] = sample(base + q * b.S + i0 + u * nprod);
      if (alu) {                                             // integer Horner: n = sum s~_q 2^((M-1-q) b)
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          double xx[M];
#pragma unroll
          for (int q = 0; q < M; ++q) xx[q] = x[q][u];
          const int cw = cw0 + i0 + u * nprod;
          v[u] = (cw >= 0 && cw < b.xlen) ? pack_word_fast<M>(fcs, mp, c_s, xx) : 0.0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          double a = compand1(c_s, x[M - 1][u]);         // Horner, oracle order
#pragma unroll
          for (int q = M - 2; q >= 0; --q) a = horner_step(mp, compand1(c_s, x[q][u]), a);
          const int cw = cw0 + i0 + u * nprod;
          v[u] = (cw >= 0 && cw < b.xlen) ? a : 0.0;
        }
      }
    } else {
      const int base = b.o0 - (g.Np - 1) + cw0;
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int cw = cw0 + i0 + u * nprod;
        v[u] = (cw >= 0 && cw < b.xlen) ? sample(base + i0 + u * nprod) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int i = i0 + u * nprod;
      if (i < words && (i < wlo || i >= whi)) xs[(i / T) * PT + i % T] = v[u];
    }
  }
}

// a2/a3: block peak over the W_block samples (16 loads in flight per thread, shuffles),
// companding factor c_s = Q / peak (Eq. (2)).  All `nprod` threads call it.
template <int PACK>
__device__ __forceinline__ double block_cs(const ModeP& mp, const double* gsrc, int n_valid, double* red, int ptid,
                                           int nprod, int bar_id) {
  if (PACK == PACK_FULL) return 1.0;
  constexpr int U = 16;
  unsigned long long m[U];                             // max |x| as ordered bits (integer pipe)
#pragma unroll
  for (int u = 0; u < U; ++u) m[u] = 0ull;
  if ((reinterpret_cast<uintptr_t>(gsrc) & 15u) == 0) {
    const double2* g2 = reinterpret_cast<const double2*>(gsrc);
    const int n2 = n_valid / 2;
    for (int i0 = ptid; i0 < n2; i0 += U * nprod) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nprod;
        v[u] = (i < n2) ? __ldg(g2 + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) m[u] = umax64(m[u], umax64(abs_bits(v[u].x), abs_bits(v[u].y)));
    }
    if ((n_valid & 1) && ptid == 0) m[0] = umax64(m[0], abs_bits(gsrc[n_valid - 1]));
  } else {
    for (int i = ptid; i < n_valid; i += nprod) m[0] = umax64(m[0], abs_bits(__ldg(gsrc + i)));
  }
#pragma unroll
  for (int u = 1; u < U; ++u) m[0] = umax64(m[0], m[u]);
  for (int o = 16; o > 0; o >>= 1) m[0] = umax64(m[0], __shfl_xor_sync(0xffffffffu, m[0], o));
  if ((ptid & 31) == 0) red[ptid >> 5] = __longlong_as_double((long long)m[0]);
  named_bar(bar_id, nprod);
  double peak = 0.0;
  for (int wi = 0; wi < nprod / 32; ++wi) peak = fmax(peak, red[wi]);
  named_bar(bar_id, nprod);
  return cs_quot(mp, peak, false);   // (the pipeline fill: no DMMA warps yet, FP64 is fastest)
}

// PC_PACK_CALL = 1: the steady-state producers reach pack_window through a real call (one copy of
// its body per kernel, out of line of the producer loop) -- an instruction-cache experiment;
// 2: for asym3 packing only (the one packing it helped).
#ifndef PC_PACK_CALL
#define PC_PACK_CALL 2
#endif
template <int PACK, int T, int UWF, int PT, bool SRC_SMEM, bool ALU>
__device__ __noinline__ void pack_window_call(const Geo& g, const Blk& b, const ModeP& mp, const double* gsrc,
                                              int n_valid, double c_s, int cw0, int rows_s, double* xs, int ptid,
                                              int nprod, bool alu) {
  pack_window<PACK, T, UWF, PT, SRC_SMEM, ALU>(g, b, mp, gsrc, n_valid, c_s, cw0, rows_s, xs, ptid, nprod, alu);
}

// a2/a3 from the raw block in shared memory (raw-staged producers): the same max |x| (integer
// order of the absolute-value bits) and the same IEEE division as block_cs.
template <int PACK, bool ALU = false>
__device__ __forceinline__ double smem_cs(const ModeP& mp, const double* raw, int n_valid, double* red, int ptid,
                                          int nprod, int bar_id, unsigned long long* dg = nullptr) {
  if (PACK == PACK_FULL) return 1.0;
  // 16-byte loads, eight in flight per thread (the producer warps' shared-memory loads queue
  // behind the DMMA warps' fragment loads: the number of dependent load rounds sets the time)
#if !PC_VEC_PEAK
  constexpr int U = 4;
  unsigned long long m[U];
#pragma unroll
  for (int u = 0; u < U; ++u) m[u] = 0ull;
  for (int i0 = ptid; i0 < n_valid; i0 += U * nprod) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nprod;
      if (i < n_valid) m[u] = umax64(m[u], abs_bits(raw[i]));
    }
  }
#else
  constexpr int U = 8;
  unsigned long long m[U];
#pragma unroll
  for (int u = 0; u < U; ++u) m[u] = 0ull;
  const int h = (reinterpret_cast<uintptr_t>(raw) & 15u) ? 1 : 0;   // raw[h] is 16-byte aligned
  const double2* r2 = reinterpret_cast<const double2*>(raw + h);
  const int n2 = n_valid > h ? (n_valid - h) >> 1 : 0;
  for (int i0 = ptid; i0 < n2; i0 += U * nprod) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nprod;
      v[u] = (i < n2) ? r2[i] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) m[u] = umax64(m[u], umax64(abs_bits(v[u].x), abs_bits(v[u].y)));
  }
  if (ptid == 0 && h && n_valid > 0) m[0] = umax64(m[0], abs_bits(raw[0]));
  if (ptid == 1 % nprod && n_valid > h && ((n_valid - h) & 1)) m[0] = umax64(m[0], abs_bits(raw[n_valid - 1]));
#endif
#pragma unroll
  for (int u = 1; u < U; ++u) m[0] = umax64(m[0], m[u]);
  if (dg) dg[0] = gtimer();
  for (int o = 16; o > 0; o >>= 1) m[0] = umax64(m[0], __shfl_xor_sync(0xffffffffu, m[0], o));
  if ((ptid & 31) == 0) red[ptid >> 5] = __longlong_as_double((long long)m[0]);
  named_bar(bar_id, nprod);
  if (dg) dg[1] = gtimer();
  unsigned long long pb = 0ull;                       // integer max of the warps' bit patterns
  for (int wi = 0; wi < nprod / 32; ++wi) pb = umax64(pb, (unsigned long long)__double_as_longlong(red[wi]));
  const double peak = __longlong_as_double((long long)pb);
  return cs_quot(mp, peak, PC_DIV_ALU || (ALU && mp.alu_pack));
}

// c_s from a block peak computed ahead (pc_block_peak / pc_block_stats): the same IEEE division.
template <int PACK>
__device__ __forceinline__ double cs_from_peak(const ModeP& mp, double peak, bool alu) {
  if (PACK == PACK_FULL) return 1.0;
  return cs_quot(mp, peak, alu);
}

// The same for one warp (producer warps work on different jobs): shuffles only.
template <int PACK, bool ALU = false>
__device__ __forceinline__ double warp_cs(const ModeP& mp, const double* gsrc, int n_valid, int lane) {
  if (PACK == PACK_FULL) return 1.0;
  constexpr int U = 16;
  unsigned long long m[U];                             // max |x| as ordered bits (integer pipe)
#pragma unroll
  for (int u = 0; u < U; ++u) m[u] = 0ull;
  if ((reinterpret_cast<uintptr_t>(gsrc) & 15u) == 0) {
    const double2* g2 = reinterpret_cast<const double2*>(gsrc);
    const int n2 = n_valid / 2;
    for (int i0 = lane; i0 < n2; i0 += U * 32) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * 32;
        v[u] = (i < n2) ? __ldg(g2 + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) m[u] = umax64(m[u], umax64(abs_bits(v[u].x), abs_bits(v[u].y)));
    }
    if ((n_valid & 1) && lane == 0) m[0] = umax64(m[0], abs_bits(gsrc[n_valid - 1]));
  } else {
    for (int i = lane; i < n_valid; i += 32) m[0] = umax64(m[0], abs_bits(__ldg(gsrc + i)));
  }
#pragma unroll
  for (int u = 1; u < U; ++u) m[0] = umax64(m[0], m[u]);
  for (int o = 16; o > 0; o >>= 1) m[0] = umax64(m[0], __shfl_xor_sync(0xffffffffu, m[0], o));
  const double peak = __longlong_as_double((long long)m[0]);
  return cs_quot(mp, peak, ALU && mp.alu_pack);
}

__device__ __forceinline__ long long fdiv_floor(long long a, long long b) {
  const long long q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
__device__ __forceinline__ long long fdiv_ceil(long long a, long long b) { return -fdiv_floor(-a, b); }

__device__ __forceinline__ unsigned smid_() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// Watchdog waits: a wait that has not completed after 4 s (%globaltimer) is a scheduling fault.
// Release builds raise the plan's host-mapped watchdog flag (conv_execute then returns
// PC_E_WATCHDOG) and end the thread, so every other wait of the launch times out the same way
// and the launch finishes without a sticky context error; PC_DEBUG_TRAP builds print where the
// wait is stuck and trap.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(kSuspendHintNs)
      : "memory");
  return ok != 0;
}
constexpr unsigned long long kWatchdogNs = 4000000000ull;
__device__ __noinline__ void mbar_stuck(int* status, int where, long long n, int st, uint32_t phase) {
#ifdef PC_DEBUG_TRAP
  printf("pc_tiled_kernel: wait %d stuck (block %d thread %d seq %lld slot %d parity %u)\n", where,
         (int)blockIdx.x, (int)threadIdx.x, n, st, phase);
  __trap();
#else
#ifdef PC_DEBUG_PRINT
  printf("pc_tiled_kernel: wait %d stuck (block %d thread %d seq %lld slot %d parity %u)\n", where,
         (int)blockIdx.x, (int)threadIdx.x, n, st, phase);
#endif
  (void)n;
  (void)st;
  (void)phase;
  if (status) *reinterpret_cast<volatile int*>(status + kStatusWatchdog) = 1 + where;   // host-mapped
  __threadfence_system();
  asm volatile("exit;");
#endif
}
// spin-wait step with the same 4-s watchdog; the timer is read every 64th step only (the spin
// loops of waiting warps were ~13% of the kernel's issued instructions with a read per step,
// profiles/r02_ncu_cfg2_asym2.json), competing for issue with the DMMA warps
struct Spin {
  unsigned n = 0;
  unsigned long long t0 = 0;
};
__device__ __forceinline__ void spin_wd(int* status, Spin& sp, unsigned ns, int where, long long n, int st) {
  __nanosleep(ns);
  if ((++sp.n & 63u) == 0u) {
    const unsigned long long t = gtimer();
    if (sp.t0 == 0) sp.t0 = t;
    else if (t - sp.t0 > kWatchdogNs) mbar_stuck(status, where, n, st, 0u);
  }
}
__device__ __forceinline__ void mbar_wait_wd(int* status, uint64_t* bar, uint32_t phase, int where, long long n,
                                             int st) {
  unsigned long long t0 = 0;
  for (unsigned i = 1;; ++i) {
    if (mbar_try(bar, phase)) return;                 // (suspends up to kSuspendHintNs per try)
    if ((i & 63u) == 0u) {
      const unsigned long long t = gtimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > kWatchdogNs) mbar_stuck(status, where, n, st, phase);
    }
  }
}

// Diagnostics layout of Exec::dbg_timing (conv_execute_profile), CTA c:
//   [4c + 0..3]            smid, t_start, t_end (ns), jobs consumed
//   [kTimCyc + 4c + 0..3]  consumer warp 0: cycles waiting on `full`, in the core, in unpack/store; fill ns
//   [kTimTr + 16c + j]     t (ns) when job j's core finished (j < 16)
constexpr int kTimCyc = 4 * 148 * 32, kTimTr = 8 * 148 * 32;
//   [kTimW + ((c * 16 + w) * 16 + j) * 4 + 0..3]  consumer warp w, part j < 16: job sequence,
//                                                   t full-ready, t core done, t stored (ns)
//   [kTimP + ((c * 4 + w) * 16 + j) * 4 + 0..3]   producer warp w, job j < 16: job sequence,
//                                                   t turn, t claimed, t published (ns)
constexpr int kTimW = 24 * 148 * 32, kTimP = kTimW + 148 * 16 * 16 * 4;
// total: kTimP + 148 * 4 * 16 * 4 uint64 entries

// Job claim (one full warp).  Job queues balance the FP64 work across SMs: with nq queues
// (nq = nsm when every SM gets >= 8 jobs, fewer for small launches), queue q owns jobs
// [J q / nq, J (q+1) / nq) and CTA c serves queue c % nq (one CTA per SM, so per CTA is per
// SM; %smid is not dense on every part); a CTA whose queue is empty steals from the others
// (warp-parallel scan), so every job runs.  Returns -1 when no job is left anywhere.
__device__ __forceinline__ long long claim_job(const Exec& e, long long njobs, int lane) {
  unsigned* ctr = e.sm_ctr;
  const long long nq_ = njobs / PC_QUEUE_MIN;
  const int nq = (int)(nq_ < 1 ? 1 : (nq_ > e.nsm ? e.nsm : nq_));
  const int s = (int)(blockIdx.x % (unsigned)nq);
  long long job = -1;
  if (lane == 0) {
    const long long lo = qdiv(njobs * s, nq), hi = qdiv(njobs * (s + 1), nq);
    if (lo < hi) {
      const unsigned n = atomicAdd(ctr + s, 1u);
      if (lo + n < hi) job = lo + n;
    }
  }
  job = __shfl_sync(0xffffffffu, job, 0);
  if (job >= 0 || PC_NO_STEAL) return job;
  for (int base = 1; base < nq; base += 32) {
    const int t = (s + base + lane) % nq;
    const long long lo = qdiv(njobs * t, nq), hi = qdiv(njobs * (t + 1), nq);
    const bool has = (base + lane < nq) && lo + (long long)*(volatile unsigned*)(ctr + t) < hi;
    unsigned mask = __ballot_sync(0xffffffffu, has);
    while (mask) {
      const int l = __ffs(mask) - 1;
      long long got = -1;
      if (lane == l) {
        const unsigned n = atomicAdd(ctr + t, 1u);
        if (lo + n < hi) got = lo + n;
      }
      got = __shfl_sync(0xffffffffu, got, l);
      if (got >= 0) return got;
      mask &= mask - 1;
    }
  }
  return -1;
}

// Called once per CTA after its last claim: the last CTA of the launch resets the queues,
// so every launch (and every replay of a captured graph) starts from zero.
__device__ __forceinline__ void retire_cta(const Exec& e) {
  __threadfence();
  if (atomicAdd(e.sm_ctr + kCtrDone, 1u) == gridDim.x - 1) {
    for (int i = 0; i < e.nsm; ++i) e.sm_ctr[i] = 0u;
    e.sm_ctr[kCtrDone] = 0u;
    if (e.split_P > 0) {                             // producer-SM mode: counters, and the next launch's epoch
      e.sm_ctr[kCtrProd] = 0u;
      e.sm_ctr[kCtrCons] = 0u;
      atomicAdd(e.split_ctl, 1u);
    }
    __threadfence();
  }
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace

// Accumulating variant of the padded-layout core: acc += sum over n_taps of this chunk.
template <int T>
__device__ __forceinline__ void conv_chunk_padded(uint32_t xs_row, uint32_t kr_addr, int n_taps, double (&acc)[T]) {
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
      for (int i = 0; i < T; ++i) acc[i] = fma(win[(i + u) % T], kk[u], acc[i]);
    }
  }
}

// a5 on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): the warp's part (32 groups of 16
// core outputs) as a Toeplitz product.  With output m = 16 i + p (group i, phase p) and
// c = 4 s + k the word offset inside a 16-word row,
//     out[16 i + p] = sum_jj sum_c x[16 (i + jj) + c] * kr[16 jj + c - p]
// (every tap t = 16 jj + c - p of [0, K) appears once per output).  A (8 x 4, row-major):
// A[i][k] = x[16 (8 mt + i + jj) + 4 s + k], rows of the stage window of pitch 20 (each
// half-warp hits 16 distinct banks); B (4 x 8): F_d[k][n] = kr[d + k - n], d = 16 jj + 4 s -
// 8 nt, d in {16 jj - 8, ..., 16 jj + 12}: a window of six fragments per jj of which four are
// new.  The taps carry 16 zeros (or the neighbour chunk's taps) on both sides, so no lane
// predicates its loads.  One warp per SMSP keeps the DMMA pipe busy (tools/dmma_peak.cu).
// fr[mt][nt][h]: group 8 mt + lane / 4, phase 8 nt + 2 (lane % 4) + h.  Exact under the
// dyadic eps (C4): every product and partial sum is a representable integer multiple of 2^-b,
// so the tensor core's summation order cannot change a bit (section 2.4 of DESIGN.md).
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
// One jj step of conv_chunk_mma (the A/B fragments of the next k-step / jj are loaded first).
// EDGE: the first or last jj of a chunk, where fragment F_d (taps [d - 7, d + 3]; d = 16 jj + 4 s
// for n-tile 0, 16 jj + 4 s - 8 for n-tile 1) can lie wholly outside the chunk's nonzero taps
// [t_lo, t_hi): its DMMAs are skipped (warp-uniform); the steps in between carry no test.
template <int NMT, int PT, bool EDGE>
__device__ __forceinline__ void mma_jj_step(int jj, int jj_n, uint32_t xa, uint32_t ka, double (&fr)[4][2][2],
                                            double (&b)[6], double (&a)[NMT], int t_lo, int t_hi) {
  double bn[4], an[NMT];
  const bool more = jj + 1 < jj_n;
  if (more) {
#pragma unroll
    for (int f = 0; f < 4; ++f) bn[f] = lds64(ka + 128u + 32u * (f + 2));
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < 3 || more) {
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt)
        an[mt] = lds64(xa + 8u * (8 * mt * PT) + (s < 3 ? 32u * (s + 1) : 8u * PT));
    }
    bool z0 = false, z1 = false;
    if (EDGE) {
      const int d0 = 16 * jj + 4 * s, d1 = d0 - 8;
      z0 = d0 + 3 < t_lo || d0 - 7 >= t_hi;
      z1 = d1 + 3 < t_lo || d1 - 7 >= t_hi;
    }
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) {
      if (!z0) dmma884(fr[mt][0], a[mt], b[s + 2]);
      if (!z1) dmma884(fr[mt][1], a[mt], b[s]);
    }
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) a[mt] = an[mt];
    // optional nap after each k-step: in tools/dmma_interference.cu a 20-ns nap per 8 DMMAs
    // lets the SMSP's other warps issue at ~5% of the DMMA rate; in this kernel it cost 5-12%
    // (cfg2 asym2 103.7 / full 172.9 us), so off
    if (PC_DMMA_NAP > 0) __nanosleep(PC_DMMA_NAP);
  }
  b[0] = b[4];
  b[1] = b[5];
  if (more) {
#pragma unroll
    for (int f = 0; f < 4; ++f) b[f + 2] = bn[f];
  }
}

template <int NMT, int PT>
__device__ __forceinline__ void conv_chunk_mma(uint32_t xs_row, uint32_t kc_addr, int jj_n, double (&fr)[4][2][2],
                                               int lane, int t_lo = -(1 << 30), int t_hi = 1 << 30) {
  const int r = lane >> 2, k = lane & 3;
  uint32_t xa = xs_row + 8u * (uint32_t)(r * PT + k);
  uint32_t ka = kc_addr + 8u * (uint32_t)(k - r) - 64u;   // b[f] = kr[16 jj - 8 + 4 f + k - r]
  // Software-pipelined: the A fragments of the next k-step and the B fragments of the next jj
  // are loaded before the current DMMAs issue (one warp alone must keep the pipe fed).
  double b[6], a[NMT];
#pragma unroll
  for (int f = 0; f < 6; ++f) b[f] = lds64(ka + 32u * f);
#pragma unroll
  for (int mt = 0; mt < NMT; ++mt) a[mt] = lds64(xa + 8u * (8 * mt * PT));
  if (jj_n <= 0) return;
  mma_jj_step<NMT, PT, true>(0, jj_n, xa, ka, fr, b, a, t_lo, t_hi);      // first jj: peeled
#pragma unroll 1
  for (int jj = 1; jj < jj_n - 1; ++jj)
    mma_jj_step<NMT, PT, false>(jj, jj_n, xa + 8u * PT * jj, ka + 128u * jj, fr, b, a, t_lo, t_hi);
  if (jj_n > 1)                                                            // last jj: peeled
    mma_jj_step<NMT, PT, true>(jj_n - 1, jj_n, xa + 8u * PT * (jj_n - 1), ka + 128u * (jj_n - 1), fr, b, a, t_lo,
                               t_hi);
}

// VAR = 1: the variant instantiation with the producer-SM mode (conv_opts.prepack < 0) and the
// integer/FP32 producer arithmetic (pack_alu = 1) compiled in (DMMA-core plans); VAR = 0, the
// default, compiles neither (their code alone cost the default path 1.4-3.3 us at cfg2).
template <int PACK, int T, int MMA, int VAR = 0>
__global__ void __launch_bounds__(tiled_threads(MMA), 1) pc_tiled_kernel(Geo g, Exec e) {
  constexpr bool kVar = VAR != 0;
  constexpr int NCW = tiled_cons_warps(MMA);   // consumer warps
  extern __shared__ __align__(128) unsigned char smem[];
  TSmem* ps = reinterpret_cast<TSmem*>(smem);
  const ModeP& mp = e.mp[PACK];
  const int G = e.G;                       // groups per tile = 32 * npart
  const int npart = G >> 5;                // consumer warps per job (one 32-group part each)
  const int KC = e.KC;                     // taps per chunk (multiple of T)
  const int nch = e.nchunks;
  const int NS = e.nstages;
  const int front = (PACK == PACK_SYM) ? 1 : 0;   // one row before the tile: the extra word
  const int rows_s = e.rows_s;
  constexpr int PT = MMA ? T + 4 : T + 1;           // stage window pitch (conflict-free for the core)
  constexpr bool FRAG_EPI = MMA && PACK != PACK_SYM;  // epilogue from the DMMA fragments (no staging rows)
  constexpr int TH = MMA ? 16 : 0;                  // DMMA core: zero / neighbour taps on both sides
  const int stage_x = (PT * rows_s + 1) & ~1;       // doubles of a stage's word window (16B-aligned end)
  const int stage_words = stage_x + (e.taps_resident ? 0 : KC + 2 * TH);
  double* kr_res = reinterpret_cast<double*>(smem + kTiledHeader) + TH;     // resident taps
  double* stg = kr_res + (e.taps_resident ? mp.K_pad + TH : -TH);           // NS stages
  double* wout = stg + (size_t)NS * stage_words;                            // per consumer warp: 32 (T+1)
  double* raw_base = wout + (FRAG_EPI ? (size_t)0 : (size_t)NCW * 32 * (T + 1));   // raw slots (e.raw_slots)
  const int tid = threadIdx.x;
  const int nprod = kTiledProdWarps * 32;
  const bool split = kVar && e.split_P > 0;         // producer-SM mode (Exec::split_P)
  const int CP = split ? e.split_P : 0;             // CTAs [0, CP) produce, the others consume

  if (tid == 0) {
    mbar_init(&ps->bar_taps, 1);
    mbar_init(&ps->rawbar[0], 1);
    mbar_init(&ps->rawbar[1], 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&ps->full[i], 32);
      mbar_init(&ps->empty[i], npart);
      ps->seq[i] = -1;
    }
    for (int i = 0; i < 4; ++i) ps->smsp_ctr[i] = ps->core_serve[i] = ps->prod_busy[i] = 0;
    ps->mseq_hi = 0;
    ps->turn = 1;
    ps->m_end = -1;
    const uint32_t tb = e.taps_resident ? (uint32_t)(mp.K_pad + 2 * TH) * 8u : 0u;
    mbar_arrive_expect_tx(&ps->bar_taps, tb);
    if (tb) bulk_g2s(kr_res - TH, mp.kr - TH, tb, &ps->bar_taps);   // the tap buffers carry 16 leading zeros
  }
  // Programmatic dependent launch: the next launch may start once every CTA of this one has
  // passed griddepcontrol.wait (the trigger follows each wait below), i.e. once the launch before
  // this one has completed -- so the next launch's queue array (the one the launch before used,
  // reset by its last CTA) is free when it claims before its own wait.
  if (!e.blk_list && !split) {
    // While the previous launch drains: L2 prefetch of the input of the (likely) first four
    // jobs of this CTA's queue.  A hint only -- L2 is coherent, so even if the preceding
    // kernel writes the input, the loads after griddepcontrol.wait see its data.
    const long long nj = e.jobs_per_sig * e.nsig;
    const long long nq_ = nj / PC_QUEUE_MIN;
    const long long nq = nq_ < 1 ? 1 : (nq_ > (long long)gridDim.x ? (long long)gridDim.x : nq_);
    const long long q = blockIdx.x % nq, lo = nj * q / nq, hi = nj * (q + 1) / nq;
    for (long long jb = lo; jb < hi && jb < lo + kTiledFillMax; ++jb) {
      const JobPos jp = job_pos(e, jb);
      const Blk b = block_info<PACK>(g, mp.K, jp.w);
      const long long avail = g.L - b.g0;
      const int nv = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
      const double* src = e.s + jp.sig * e.s_stride + (b.g0 - e.s_off);
      for (int i = threadIdx.x * 16; i < nv; i += blockDim.x * 16)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src + i));
    }
  }
  // early_fill (host-checked: the preceding launch on this stream is not one that writes this
  // input): the pipeline fill below only reads the input and the plan's taps and claims from
  // this launch's own queue array, so it may overlap the preceding launch's tail; everything
  // that writes global memory comes after griddepcontrol.wait.
  auto dep_wait = [&]() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  };
  if (split || (!e.early_fill && !e.early_claim)) dep_wait();
  __syncthreads();
  if (e.dbg_timing && tid == 0) e.dbg_timing[kTimCyc + 4 * blockIdx.x + 2] = gtimer();   // t_start (stash)
  long long njobs = e.jobs_per_sig * e.nsig;
  if (e.blk_list) {                                  // adaptive: count written by pc_adapt_lists
    const long long nb = *e.blk_count;
    njobs = nb == 0 ? 0 : (e.blk_list[0] == 0 ? e.tiles0 + (nb - 1) * e.tiles1 : nb * e.tiles1);
    if (njobs == 0) {          // no block chose this packing: leave once the tap copy has landed
      mbar_wait_wd(e.status, &ps->bar_taps, 0, 4, 0, 0);   // (every CTA leaves: the queues stay untouched)
      return;
    }
  }

  // Locate a job's block and input.
  auto job_block = [&](long long job, JobPos& jp, Blk& b, const double*& gsrc, int& n_valid) {
    jp = job_pos(e, job);
    b = block_info<PACK>(g, mp.K, jp.w);
    gsrc = e.s + jp.sig * e.s_stride + (b.g0 - e.s_off);
    const long long avail = g.L - b.g0;
    n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  };
  // Hand stage `st` to the consumers (+ the tap chunk by TMA when not resident).
  auto publish = [&](long long n, int st, int c, long long job, double inv, int ptid, bool win_src = true) {
    const bool win = job >= 0 && e.pre_win && win_src;   // the stage image comes from pre_win by bulk copy
    if (ptid == 0) {
      ps->job[st] = job;
      if (job >= 0) ps->jpos[st] = pack_pos(job_pos(e, job));   // consumers skip the 64-bit divisions
      ps->inv[st] = win ? e.pre_inv[job] : inv;
      ps->seq[st] = n;
    }
    const bool taps = job >= 0 && !e.taps_resident;
    if ((taps || win) && ptid == 0) {
      const int nt = (c == nch - 1) ? mp.K_pad - c * KC : KC;
      double* xs = stg + (size_t)st * stage_words;
      mbar_arrive_expect_tx(&ps->full[st], (taps ? (uint32_t)(nt + 2 * TH) * 8u : 0u) + (win ? (uint32_t)stage_x * 8u : 0u));
      if (win) bulk_g2s(xs, e.pre_win + job * e.pre_stride, (uint32_t)stage_x * 8u, &ps->full[st]);
      if (taps) {
        const double* kr_job = e.kr_sig ? e.kr_sig + (job / e.jobs_per_sig) * e.kr_stride : mp.kr;
        bulk_g2s(xs + stage_x, kr_job + (size_t)c * KC - TH, (uint32_t)(nt + 2 * TH) * 8u, &ps->full[st]);
      }
    } else {
      mbar_arrive(&ps->full[st]);
    }
  };

  // Pipeline fill: the first nf jobs (up to the ring's stages and the CTA's share) are claimed in
  // parallel (before griddepcontrol.wait: only this launch's queue array is touched), then
  // companded and packed by all 16 warps in four groups of four warps.
  // (never more than a CTA's share of the launch: small launches spread over all CTAs)
  // Producer-SM mode: the consumer CTAs pack jobs [0, F) in their pipeline fills (job c' + q C for
  // consumer c' of C, fill slot q), the producer CTAs every later job, in order.
  const int nfs = min(kTiledFillMax, NS);
  const int CC = (int)gridDim.x - CP;                 // consumer CTAs
  const long long F = split ? min(njobs, (long long)nfs * CC) : 0;
  if (split && (int)blockIdx.x < CP) {
    // ============================ producer CTA (no DMMA warps on this SM) ============================
    // Four groups of four warps, one job each: the job's raw block by one TMA bulk copy into the
    // group's slot (the ring area is free here), the next round's block prefetched into L2, block
    // peak, companding and packing from shared memory (FP64: nothing here competes for the FP64
    // pipe) straight into the job's stage image at pre_win, its (c_s c_k)^-1 at pre_inv, then the
    // job's ready flag (release) for the consumer CTAs.
    const unsigned want = *reinterpret_cast<volatile unsigned*>(e.split_ctl) + 1u;
    const int gq = tid >> 7, gtid = tid & 127;
    const int rstride = (g.W_block + 3) & ~1;          // doubles per raw slot (head offset, even)
    const bool staged = (size_t)4 * rstride <= (size_t)NS * stage_words;
    double* raw = stg + (size_t)gq * rstride;
    if (tid < 4) mbar_init(&ps->pbar[tid], 1);        // the groups' raw-block barriers
    __syncthreads();
    uint32_t ph = 0;
    unsigned long long t_cta0 = 0;
    if (e.dbg_timing && tid == 0) t_cta0 = gtimer();
    for (int pj = 0;; ++pj) {
      // diagnostics: per group and job j < 16 {job | 1 << 62, t claimed, t raw block landed, t flagged}
      unsigned long long* prec = (e.dbg_timing && gtid == 0 && pj < 16)
                                     ? e.dbg_timing + kTimP + (((size_t)blockIdx.x * 4 + gq) * 16 + pj) * 4
                                     : nullptr;
      if (gtid == 0) ps->fjob[gq] = F + (long long)atomicAdd(e.sm_ctr + kCtrProd, 1u);
      named_bar(1 + gq, 128);
      const long long job = ps->fjob[gq];
      if (job >= njobs) break;
      if (prec) {
        prec[0] = (unsigned long long)job | (1ull << 62);
        prec[1] = gtimer();
      }
      JobPos jp;
      Blk b;
      const double* gsrc;
      int n_valid;
      job_block(job, jp, b, gsrc, n_valid);
      const int head = (reinterpret_cast<uintptr_t>(gsrc) & 15u) ? 1 : 0, mid = max(0, n_valid - head) & ~1;
      double* rp = raw + head;                         // rp[i] = block sample i, rp[head] 16-byte aligned
      if (staged && gtid == 0) {
        mbar_arrive_expect_tx(&ps->pbar[gq], (uint32_t)mid * 8u);
        if (mid > 0) bulk_g2s(rp + head, gsrc + head, (uint32_t)mid * 8u, &ps->pbar[gq]);
        const long long pj = job + 4LL * CP;           // the block this group's next round likely needs
        if (pj < njobs) {
          JobPos jq;
          Blk bq;
          const double* gq_src;
          int nq;
          job_block(pj, jq, bq, gq_src, nq);
          const uintptr_t a0 = reinterpret_cast<uintptr_t>(gq_src) & ~(uintptr_t)15;
          const uint32_t bytes = (uint32_t)(((reinterpret_cast<uintptr_t>(gq_src + nq) + 15) & ~(uintptr_t)15) - a0);
#ifndef PC_NO_SPLIT_PREFETCH
          if (nq > 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(bytes) : "memory");
#endif
        }
      }
      double cs;
      if (staged) {
        if (gtid == 0 && head && n_valid > 0) rp[0] = __ldg(gsrc);
        if (gtid == 1 && head + mid < n_valid) rp[n_valid - 1] = __ldg(gsrc + n_valid - 1);
        mbar_wait_wd(e.status, &ps->pbar[gq], ph, 10, job, gq);
        ph ^= 1u;
        named_bar(1 + gq, 128);                        // head / tail elements visible
        if (prec) prec[2] = gtimer();
        cs = e.blk_peak ? cs_from_peak<PACK>(mp, e.blk_peak[jp.sig * e.peak_stride + jp.w], false)
                        : smem_cs<PACK>(mp, rp, n_valid, ps->red + 8 * gq, gtid, 128, 1 + gq);
        // smem_cs's reduction reads red[] after one barrier: fence the next job's writes to it
        named_bar(1 + gq, 128);
      } else {
        cs = e.blk_peak ? cs_from_peak<PACK>(mp, e.blk_peak[jp.sig * e.peak_stride + jp.w], false)
                        : block_cs<PACK>(mp, gsrc, n_valid, ps->red + 8 * gq, gtid, 128, 1 + gq);
      }
      double* xw = const_cast<double*>(e.pre_win) + job * e.pre_stride;
      if (staged)
        pack_window<PACK, T, 1, PT, true>(g, b, mp, rp, n_valid, cs, jp.t * G * T - front * T, rows_s, xw, gtid, 128, false);
      else
        pack_window<PACK, T, 1, PT>(g, b, mp, gsrc, n_valid, cs, jp.t * G * T - front * T, rows_s, xw, gtid, 128, false);
      if (gtid == 0)
        const_cast<double*>(e.pre_inv)[job] = inv_scale(mp, cs, e.scal_sig ? e.scal_sig[3 * jp.sig + 1] : mp.c_k, false);
      // the group's stores, then one release by thread 0 (cumulative over the barrier); the
      // consumer's acquire + proxy fence orders them before its bulk copy
      named_bar(1 + gq, 128);                          // (also: the raw slot is free for the next copy)
      if (gtid == 0) st_release_u32(e.split_flags + job, want);
      if (prec) prec[3] = gtimer();
    }
    __syncthreads();
    if (tid == 0) {
      if (e.dbg_timing) {
        e.dbg_timing[4 * blockIdx.x + 0] = smid_();
        e.dbg_timing[4 * blockIdx.x + 1] = t_cta0;
        e.dbg_timing[4 * blockIdx.x + 2] = gtimer();
        e.dbg_timing[4 * blockIdx.x + 3] = 0;
      }
      retire_cta(e);
    }
    return;
  }
  const long long share = (njobs + gridDim.x - 1) / gridDim.x;
  const int nf = split ? nfs : e.pre_win ? 0 : (nch == 1) ? (int)min((long long)min(kTiledFillMax, NS), share < 1 ? 1 : share) : 1;
  const int lane_ = tid & 31, warp_ = tid >> 5;
  if (split) {
    if (tid < nf) {
      const long long j = (long long)(blockIdx.x - CP) + (long long)tid * CC;
      ps->fjob[tid] = j < F ? j : -1;
    }
  } else if (warp_ < nf) {
    const long long j = claim_job(e, njobs, lane_);
    if (lane_ == 0) ps->fjob[warp_] = j;
  }
  __syncthreads();
  if (tid == 0) {                                    // successful claims first: no holes before M_end
    int k = 0;
    for (int q = 0; q < nf; ++q)
      if (ps->fjob[q] >= 0) ps->fjob[k++] = ps->fjob[q];
    for (int q = k; q < nf; ++q) ps->fjob[q] = -1;
    ps->m_end = (k < nf && !split) ? k : -1;        // (split: later jobs come from the producer CTAs)
    ps->turn = nf;
  }
  __syncthreads();
  if (e.early_claim && !e.early_fill && !split) dep_wait();   // the fill reads the input: after the wait
  {
    constexpr int GW = (kTiledProdWarps + NCW) / kTiledFillJobs;   // warps per fill group
    const int gq = warp_ / GW, gtid = tid - gq * GW * 32;
    for (int f = gq; f < nf; f += 4) {
      const long long fj = ps->fjob[f];
      if (fj < 0) break;
      JobPos jp;
      Blk b;
      const double* gsrc;
      int n_valid;
      job_block(fj, jp, b, gsrc, n_valid);
      unsigned long long* frec = (e.dbg_timing && gtid == 0 && f < 4)
                                     ? e.dbg_timing + kTimP + (((size_t)blockIdx.x * 4 + f) * 16 + 15) * 4
                                     : nullptr;
      if (frec) frec[0] = gtimer();
      double* xs_f = stg + (size_t)((f * nch) % NS) * stage_words;
      const double cs = e.blk_peak ? cs_from_peak<PACK>(mp, e.blk_peak[jp.sig * e.peak_stride + jp.w], false)
                                   : block_cs<PACK>(mp, gsrc, n_valid, ps->red + 8 * gq, gtid, GW * 32, 1 + gq);
      if (frec) frec[1] = gtimer();
      pack_window<PACK, T, 1, PT>(g, b, mp, gsrc, n_valid, cs, jp.t * G * T - front * T, rows_s, xs_f, gtid,
                                  GW * 32, false);   // (no DMMA warps during the fill: FP64 is fastest)
      if (frec) frec[2] = gtimer();
      if (gtid == 0) {
        ps->fcs[f] = cs;
        ps->finv[f] = inv_scale(mp, cs, e.scal_sig ? e.scal_sig[3 * jp.sig + 1] : mp.c_k, false);
      }
    }
  }
  __syncthreads();
  if (e.early_fill) dep_wait();
  if (e.dbg_timing && tid == 0)
    e.dbg_timing[kTimCyc + 4 * blockIdx.x + 3] = gtimer() - e.dbg_timing[kTimCyc + 4 * blockIdx.x + 2];

  if (tid < nprod && split) {
    // ============== producer-SM mode: the consumer CTA's producer warps move stage images ==============
    // Warp 0 publishes the fill's jobs, then claims jobs F, F+1, .. in order from the launch-wide
    // counter, waits for each one's ready flag and bulk-copies its stage image into the ring.
    if (tid >= 32) return;
    const int lane = tid;
    const int n_sent = NCW / npart;
    const unsigned want = *reinterpret_cast<volatile unsigned*>(e.split_ctl) + 1u;
    long long m = 0;
    for (; m < nf; ++m) {
      const long long job = ps->fjob[m];
      if (job < 0) break;
      publish(m, (int)(m % NS), 0, job, ps->finv[m], lane, false);
    }
    for (;; ++m) {
      long long k = 0;
      if (lane == 0) {
        // claim a job only when the consumers hold parts of job m - PC_SPLIT_AHEAD: a CTA with a
        // free ring would otherwise claim its ring's worth of not-yet-produced jobs, in order,
        // while other CTAs run dry (head-of-line blocking)
        Spin sp;
        while (m >= (long long)*reinterpret_cast<volatile int*>(&ps->mseq_hi) + PC_SPLIT_AHEAD)
          spin_wd(e.status, sp, 64, 11, m, 0);
        k = (long long)atomicAdd(e.sm_ctr + kCtrCons, 1u);
      }
      k = __shfl_sync(0xffffffffu, k, 0);
      if (F + k >= njobs) break;
      const int st = (int)qmod(m, NS);
      if (m >= NS) mbar_wait_wd(e.status, &ps->empty[st], (uint32_t)((qdiv(m, NS) & 1) ^ 1), 1, m, st);
      if (lane == 0) {
        Spin sp;
        while (ld_acquire_u32(e.split_flags + F + k) != want) spin_wd(e.status, sp, 64, 9, m, st);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncwarp();
      publish(m, st, 0, F + k, 0.0, lane);
    }
    for (const long long me = m; m < me + n_sent; ++m) {   // sentinels, one per consumer warp
      const int st = (int)qmod(m, NS);
      if (m >= NS) mbar_wait_wd(e.status, &ps->empty[st], (uint32_t)((qdiv(m, NS) & 1) ^ 1), 1, m, st);
      publish(m, st, 0, -1, 0.0, lane);
    }
    if (lane == 0) retire_cta(e);
    return;
  }

  if (tid < nprod && e.raw_slots > 0) {
    // ====================== raw-staged producer warps ======================
    // The four producer warps work on one job at a time.  Its raw block arrives in shared
    // memory by one TMA bulk copy (issued a job ahead when two raw slots fit), so the peak,
    // companding and packing read shared memory: no per-lane global loads and their latency
    // next to the DMMA warps.  Single-chunk plans (nch == 1) without prepacked windows.
    // Same claims (sequence order, one warp), stages, sentinels and publish as below.  One warp
    // waits on each mbarrier (ring slot, raw slot) and releases the others through the named
    // barrier: with all four warps polling the ring slot's `empty` barrier, about one run in five
    // of the cfg2 bench stalled -- two warps past the slot's release, two still waiting on it
    // (4-s watchdog) -- and none in 26 runs since.
    const int ptid = tid, lane = tid & 31, pw = tid >> 5;
    constexpr int PB = 8;                             // named barrier of the producer warps
    const int RS = e.raw_slots;
    const int n_sent = NCW / npart;
    uint32_t rph = 0;                                 // bit k: parity of raw slot k's next wait
    long long cur_blk_w = -1;
    double c_s_w = 1.0, inv_w = 0.0;
    auto claim_seq = [&](long long m) -> long long {  // job of sequence m, -1: none left (M_end)
      if (pw == 0) {
        long long j = -1;
        if (*reinterpret_cast<volatile long long*>(&ps->m_end) < 0) {
          if (lane == 0 && e.lookahead > 0) {
            Spin sp;
            while (m >= (long long)*reinterpret_cast<volatile int*>(&ps->mseq_hi) + max(e.lookahead, RS))
              spin_wd(e.status, sp, 128, 6, m, 0);
          }
          __syncwarp();
          j = claim_job(e, njobs, lane);
          if (j < 0 && lane == 0) *reinterpret_cast<volatile long long*>(&ps->m_end) = m;
        }
        if (lane == 0) ps->pjob[m & 1] = j;
      }
      named_bar(PB, nprod);
      return *reinterpret_cast<volatile long long*>(&ps->pjob[m & 1]);
    };
    // raw slot layout: rp[i] = block sample i; rp[head] is 16-byte aligned (TMA), the head and an
    // odd tail element are loaded by threads (the copy never reads outside [gsrc, gsrc + n_valid))
    auto raw_geom = [&](const double* gs, int nv, int slot, int& head, int& mid) -> double* {
      head = (reinterpret_cast<uintptr_t>(gs) & 15u) ? 1 : 0;
      mid = max(0, nv - head) & ~1;
      return raw_base + (size_t)slot * e.raw_stride + head;
    };
    auto issue_raw = [&](long long job, int slot) {
      if (ptid == 0) {
        JobPos jp;
        Blk b;
        const double* gs;
        int nv, head, mid;
        job_block(job, jp, b, gs, nv);
        double* rp = raw_geom(gs, nv, slot, head, mid);
        mbar_arrive_expect_tx(&ps->rawbar[slot], (uint32_t)mid * 8u);
        if (mid > 0) bulk_g2s(rp + head, gs + head, (uint32_t)mid * 8u, &ps->rawbar[slot]);
      }
    };
    long long m = 0;
    for (; m < nf; ++m) {                             // the pipeline fill's jobs: publish
      const long long job = ps->fjob[m];
      if (job < 0) break;
      const JobPos jq = job_pos(e, job);
      cur_blk_w = jq.sig * g.P + jq.w;
      c_s_w = ps->fcs[m];
      inv_w = ps->finv[m];
      if (pw == 0) publish(m, (int)(m % NS), 0, job, inv_w, lane);
    }
    long long job = (m == nf) ? claim_seq(m) : -1;
    if (job >= 0 && RS == 2) issue_raw(job, (int)(m & 1));
    int pj = 0;
    for (;; ++pj) {
      unsigned long long* prec = (e.dbg_timing && ptid == 0 && pj < 16)
                                     ? e.dbg_timing + kTimP + (((size_t)blockIdx.x * 4 + 0) * 16 + pj) * 4
                                     : nullptr;
      if (prec) {
        prec[0] = (unsigned long long)m;
        prec[1] = gtimer();
      }
      if (job < 0) {                                  // sentinels: sequences m .. M_end + n_sent - 1
        const long long me = *reinterpret_cast<volatile long long*>(&ps->m_end);
        if (pw == 0)                                  // (warp 0 alone waits on the ring and publishes)
          for (; m < me + n_sent; ++m) {
            const int st = (int)qmod(m, NS);
            if (m >= NS) mbar_wait_wd(e.status, &ps->empty[st], (uint32_t)((qdiv(m, NS) & 1) ^ 1), 1, m, st);
            publish(m, st, 0, -1, 0.0, lane);
          }
        break;
      }
      long long nxt = -1;
      if (RS == 2) {                                  // the next job's raw block in flight during this one
        nxt = claim_seq(m + 1);
        if (nxt >= 0) issue_raw(nxt, (int)((m + 1) & 1));
      } else {
        issue_raw(job, 0);
      }
      if (prec) prec[2] = gtimer();
      const int slot = (RS == 2) ? (int)(m & 1) : 0;
      JobPos jp;
      Blk b;
      const double* gs;
      int nv, head, mid;
      job_block(job, jp, b, gs, nv);
      double* rp = raw_geom(gs, nv, slot, head, mid);
      if (ptid == 0 && head && nv > 0) rp[0] = __ldg(gs);
      if (ptid == 1 && head + mid < nv) rp[nv - 1] = __ldg(gs + nv - 1);
      if (pw == 0) mbar_wait_wd(e.status, &ps->rawbar[slot], (rph >> slot) & 1u, 8, m, slot);   // warp 0 waits,
      rph ^= 1u << slot;
      named_bar(PB, nprod);                           // the others here; head / tail elements visible
      unsigned long long t_rw = 0;
      if (prec) t_rw = gtimer();
      // diagnostics: the peak phase's steps (loads + local max, cross-warp reduction, division,
      // Eq. (16) scale) in producer warp 1's record slots (raw-staged producers use warp 0's only)
      unsigned long long* dgr = prec ? e.dbg_timing + kTimP + (((size_t)blockIdx.x * 4 + 1) * 16 + pj) * 4 : nullptr;
      const long long blk_id = jp.sig * g.P + jp.w;
      if (blk_id != cur_blk_w) {
        cur_blk_w = blk_id;
        c_s_w = e.blk_peak ? cs_from_peak<PACK>(mp, e.blk_peak[jp.sig * e.peak_stride + jp.w], kVar && mp.alu_pack)
                           : smem_cs<PACK, kVar>(mp, rp, nv, ps->red + 28, ptid, nprod, PB, dgr);   // a2/a3
        if (dgr) dgr[2] = gtimer();
        inv_w = inv_scale(mp, c_s_w, e.scal_sig ? e.scal_sig[3 * jp.sig + 1] : mp.c_k,
                          PC_DIV_ALU || (kVar && mp.alu_pack));   // Eq. (16)
        if (dgr) dgr[3] = gtimer();
      }
      unsigned long long t_pk = 0, t_sl = 0;
      if (prec) t_pk = gtimer();
      const int st = (int)qmod(m, NS);
      if (m >= NS) {                                  // the ring slot: warp 0 waits for its release
        if (pw == 0) mbar_wait_wd(e.status, &ps->empty[st], (uint32_t)((qdiv(m, NS) & 1) ^ 1), 1, m, st);
        named_bar(PB, nprod);
      }
      if (prec) t_sl = gtimer();
      if constexpr (PC_PACK_CALL == 1 || (PC_PACK_CALL == 2 && PACK == PACK_ASYM3))
        pack_window_call<PACK, T, 1, PT, true, kVar>(g, b, mp, rp, nv, c_s_w, jp.t * G * T - front * T, rows_s,
                                               stg + (size_t)st * stage_words, ptid, nprod, mp.alu_pack);
      else
        pack_window<PACK, T, 1, PT, true, kVar>(g, b, mp, rp, nv, c_s_w, jp.t * G * T - front * T, rows_s,
                                          stg + (size_t)st * stage_words, ptid, nprod, mp.alu_pack);   // a3/a4
      named_bar(PB, nprod);
      if (pw == 0) publish(m, st, 0, job, inv_w, lane);
      if (prec) {   // m | (claimed -> raw block landed) | (-> peak done) | (-> slot free), 16-bit fields of 16 ns
        prec[3] = gtimer();
        const unsigned long long d0 = min((t_rw - prec[2]) >> 4, 0xffffull), d1 = min((t_pk - t_rw) >> 4, 0xffffull),
                                 d2 = min((t_sl - t_pk) >> 4, 0xffffull);
        prec[0] = (unsigned long long)(m & 0xffff) | (d0 << 16) | (d1 << 32) | (d2 << 48);
      }
      ++m;
      job = (RS == 2) ? nxt : claim_seq(m);
    }
    if (tid == 0) retire_cta(e);
    return;
  }

  if (tid < nprod) {
    // ============================ producer warps ============================
    // Job sequence m (its chunk c is stage sequence n = m * nch + c, slot n % NS) is produced
    // by producer warp m % 4, so four jobs are companded and packed concurrently.  Claims are
    // taken in sequence order (a turn counter), so the first failed claim M_end ends the real
    // jobs; sequences M_end .. M_end + 16/npart - 1 are sentinels (job = -1), one for every
    // consumer warp.  A slot is refilled only after its previous sequence was published and
    // then released by the consumers.
    const int pw = tid >> 5, lane = tid & 31;
    const int n_sent = NCW / npart;
    long long cur_blk_w = -1;
    double c_s_w = 1.0, inv_w = 0.0;
    int pj = 0;
    for (long long m = pw;; m += kTiledProdWarps, ++pj) {
      unsigned long long* prec = (e.dbg_timing && lane == 0 && pj < 16)
                                     ? e.dbg_timing + kTimP + (((size_t)blockIdx.x * 4 + pw) * 16 + pj) * 4
                                     : nullptr;
      if (prec) {
        prec[0] = (unsigned long long)m;
        prec[1] = gtimer();
      }
      long long job;
      bool prepacked = false;
      if (m < nf) {
        job = ps->fjob[m];
        prepacked = job >= 0;
        if (prepacked) {
          const JobPos jq = job_pos(e, job);
          cur_blk_w = jq.sig * g.P + jq.w;
          c_s_w = ps->fcs[m];
          inv_w = ps->finv[m];
        }
      } else {
        long long j = -1;
        if (lane == 0) {
          Spin sp;
          while (*reinterpret_cast<volatile long long*>(&ps->turn) != m) spin_wd(e.status, sp, 256, 5, m, 0);
          // bounded claim-ahead: a job claimed long before any warp can start it is work other
          // SMs can no longer steal (the launch's tail)
          // (sentinel sequences, after the first failed claim, are never held back)
          if (e.lookahead > 0)
            while (*reinterpret_cast<volatile long long*>(&ps->m_end) < 0 &&
                   m >= (long long)*reinterpret_cast<volatile int*>(&ps->mseq_hi) + e.lookahead)
              spin_wd(e.status, sp, 128, 6, m, 0);
          const long long me = *reinterpret_cast<volatile long long*>(&ps->m_end);
          j = (me >= 0) ? -1 : 0;
        }
        j = __shfl_sync(0xffffffffu, j, 0);
        if (j == 0) j = claim_job(e, njobs, lane);
        if (lane == 0) {
          if (j < 0 && *reinterpret_cast<volatile long long*>(&ps->m_end) < 0)
            *reinterpret_cast<volatile long long*>(&ps->m_end) = m;
          __threadfence_block();
          *reinterpret_cast<volatile long long*>(&ps->turn) = m + 1;
        }
        job = j;
      }
      if (prec) prec[2] = gtimer();
      if (job < 0) {
        long long me = 0;
        if (lane == 0) me = *reinterpret_cast<volatile long long*>(&ps->m_end);
        me = __shfl_sync(0xffffffffu, me, 0);
        if (m >= me + n_sent) break;
      }
      JobPos jp;
      Blk b;
      const double* gsrc = nullptr;
      int n_valid = 0;
      if (job >= 0 && MMA && PC_PROD_YIELD && lane == 0 && !e.pre_win)
        *reinterpret_cast<volatile int*>(&ps->prod_busy[pw & 3]) = 1;
      if (job >= 0) {
        job_block(job, jp, b, gsrc, n_valid);
        const long long blk_id = jp.sig * g.P + jp.w;
        if (blk_id != cur_blk_w && !e.pre_win) {
          cur_blk_w = blk_id;
          c_s_w = e.blk_peak ? cs_from_peak<PACK>(mp, e.blk_peak[jp.sig * e.peak_stride + jp.w], kVar && mp.alu_pack)
                             : warp_cs<PACK, kVar>(mp, gsrc, n_valid, lane);   // a2/a3 (Eq. (2))
          inv_w = inv_scale(mp, c_s_w, e.scal_sig ? e.scal_sig[3 * jp.sig + 1] : mp.c_k, kVar && mp.alu_pack);   // Eq. (16)
        }
      }
      unsigned long long t_pk = 0, t_sl = 0;                 // diagnostics: peak done, slot free
      if (prec) t_pk = gtimer();
      for (int c = 0; c < nch; ++c) {
        const long long n = m * nch + c;
        const int st = (int)qmod(n, NS);
        if (n >= NS) {
          if (lane == 0)
          {
            Spin sp;
            while (*reinterpret_cast<volatile long long*>(&ps->seq[st]) != n - NS) spin_wd(e.status, sp, 256, 7, n, st);
          }
          __syncwarp();
          mbar_wait_wd(e.status, &ps->empty[st], (uint32_t)((qdiv(n, NS) & 1) ^ 1), 1, n, st);
        }
        if (prec && c == 0) t_sl = gtimer();
        if (job >= 0 && !(prepacked && c == 0) && !e.pre_win)
          pack_window<PACK, T, 2, PT, false, kVar>(g, b, mp, gsrc, n_valid, c_s_w, jp.t * G * T - front * T + c * KC, rows_s,
                               stg + (size_t)st * stage_words, lane, 32, mp.alu_pack);
        __syncwarp();
        publish(n, st, c, job, inv_w, lane);
      }
      if (MMA && PC_PROD_YIELD && lane == 0) *reinterpret_cast<volatile int*>(&ps->prod_busy[pw & 3]) = 0;
      if (prec) {
        prec[3] = gtimer();
        // m | 0 | (claimed -> peak done) | (peak done -> slot free), 16-bit fields of 16 ns
        const unsigned long long d1 = min((t_pk - prec[2]) >> 4, 0xffffull), d2 = min((t_sl - t_pk) >> 4, 0xffffull);
        prec[0] = (unsigned long long)(m & 0xffff) | (d1 << 32) | (d2 << 48);
      }
    }
    if (tid == 0) {
      // every producer warp has finished claiming once the turn passed all of them
      retire_cta(e);
    }
    return;
  }

  // ============================ consumer warps ============================
  // Warp-job k = (job sequence k / npart, part k % npart) runs on SMSP k % 4: the warps of
  // SMSP s claim k = 4 c + s in order from their own counter, so every job's parts spread
  // over the four schedulers and a finished warp takes the next part (no CTA-wide barrier).
  const int ctid = tid - nprod;
  const int cw = ctid >> 5, lane = tid & 31;
  const int smsp = (tid >> 5) & 3;
  double* wbuf = wout + (size_t)cw * 32 * (T + 1);
  mbar_wait_wd(e.status, &ps->bar_taps, 0, 4, 0, 0);
  // A consumer warp may claim work up to NCW / npart jobs ahead of the producer, i.e. more than
  // one ring lap: a parity wait could then see the slot's previous lap; the sequence number
  // stamped by the producer tells the two apart.
  auto wait_full = [&](long long n, int st) {
    for (Spin sp;;) {
      mbar_wait_wd(e.status, &ps->full[st], (uint32_t)(qdiv(n, NS) & 1), 2, n, st);
      if (*reinterpret_cast<volatile long long*>(&ps->seq[st]) == n) return;
      spin_wd(e.status, sp, 200, 3, n, st);
    }
  };
  int njob = 0;
#define PC_REC (e.dbg_timing != nullptr && ctid == 0)
  if (PC_REC) ps->cyc[0] = ps->cyc[1] = ps->cyc[2] = 0;
  for (;; ++njob) {
    int cl = 0;
    if (lane == 0) cl = atomicAdd(&ps->smsp_ctr[smsp], 1);
    cl = __shfl_sync(0xffffffffu, cl, 0);
    const long long k = 4LL * cl + smsp;
    const long long mseq = qdiv(k, npart);
    if (lane == 0 && (e.lookahead > 0 || e.split_P > 0)) atomicMax(&ps->mseq_hi, (int)(mseq + 1));
    // parts rotate over the SMSPs from job to job, so ragged last parts do not pile up on one
    const int part = (int)qmod(k - mseq * npart + mseq, npart);
    long long n = mseq * nch;
    int st = (int)qmod(n, NS);
    if (PC_REC) ps->cyc[3] = clock64();
    wait_full(n, st);
    const long long job = ps->job[st];
    if (PC_REC) {
      const long long c1 = clock64();
      ps->cyc[0] += c1 - ps->cyc[3];
      ps->cyc[3] = c1;
    }
    unsigned long long* wrec = (e.dbg_timing && lane == 0 && njob < 16)
                                   ? e.dbg_timing + kTimW + (((size_t)blockIdx.x * 16 + cw) * 16 + njob) * 4
                                   : nullptr;
    if (wrec) {
      wrec[0] = (unsigned long long)mseq;
      wrec[1] = gtimer();
    }
    if (job < 0) {                                           // sentinel: release its stages, stop
      for (int c = 0; c < nch; ++c, ++n) {
        st = (int)qmod(n, NS);
        if (c > 0) wait_full(n, st);
        __syncwarp();
        if (lane == 0) mbar_arrive(&ps->empty[st]);
      }
      break;
    }
    const double inv = ps->inv[st];
    const JobPos jp = unpack_pos(ps->jpos[st]);
    const Blk b = block_info<PACK>(g, mp.K, jp.w);
    const int ngroups = (b.M_out + T - 1) / T;
    // FMA core: part p = groups [32 p, 32 p + 32) of the tile, one per lane.  DMMA core: the
    // tile's m-tiles (8 groups) are split evenly over the parts (e.g. 14 -> 3, 4, 3, 4).
    int pg0 = part * 32, pgn = 32;                           // the part's first group (in the tile), count
    if (MMA) {
      const int nmt_job = (min(G, ngroups - jp.t * G) + 7) >> 3;
      const int lo = part * nmt_job / npart, hi = (part + 1) * nmt_job / npart;
      pg0 = 8 * lo;
      pgn = 8 * (hi - lo);
    }
    const int gl = pg0 + lane;                               // this thread's group in the tile
    const int gi = jp.t * G + gl;                            // group index within the block
    const bool mine = gi < ngroups && lane < pgn;
    const int gi0 = jp.t * G + pg0;                          // the warp's first group
    const bool extra = (PACK == PACK_SYM) && gi0 > 0 && pgn > 0;   // needs B of the word before it
    double acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = 0.0;
    double fr[4][2][2];                                      // DMMA core: C fragments (see conv_chunk_mma)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int q = 0; q < 4; ++q) fr[mt][q >> 1][q & 1] = 0.0;
    // DMMA core: m-tiles (8 groups) of this part that hold outputs of the block (warp-uniform)
    const int n_mt = MMA ? min(pgn >> 3, max(0, (ngroups - gi0 + 7) >> 3)) : 0;
    double px = 0.0;                                         // sym: that word's core output (split)
    if (MMA) {
      // One core at a time per SM sub-partition, in claim order: a single warp with its 2 NMT
      // accumulator chains keeps the DMMA pipe busy, while every further warp queued on it
      // starves the SMSP's other warps (producers, epilogues) of issue -- measured 6-15x
      // slower loads and FP64 ops with three DMMA warps per SMSP, ~1.1x with one
      // (tools/dmma_interference.cu).
      if (lane == 0)
        // while the SMSP's producer warp packs, one core slot: a second queued DMMA warp would
        // slow its loads and FP64 ops 3x (tools/dmma_interference.cu)
        for (Spin sp;
             *reinterpret_cast<volatile int*>(&ps->core_serve[smsp]) +
                 (PC_PROD_YIELD && *reinterpret_cast<volatile int*>(&ps->prod_busy[smsp]) ? 1 : PC_CORE_SLOTS) <= cl;)
          spin_wd(e.status, sp, 128, 8, cl, smsp);
      if (wrec) wrec[0] |= ((gtimer() - wrec[1]) >> 4) << 32;   // diagnostics: token wait (16 ns units)
      __syncwarp();
    }
    for (int c = 0; c < nch; ++c, ++n) {
      st = (int)qmod(n, NS);
      if (c > 0) wait_full(n, st);
      const double* xs = stg + (size_t)st * stage_words;
      const double* kc = e.taps_resident ? kr_res + (size_t)c * KC : xs + stage_x + TH;
      const int nt = (c == nch - 1) ? mp.K_pad - c * KC : KC;
      if (MMA) {                                             // a5 on the tensor cores
        const uint32_t xrow = smem_u32(xs) + 8u * PT * (pg0 + front);
        // the last chunk ends where the taps end: jj covers taps [16 jj - 15, 16 jj + 15], so the
        // nonzero ones need jj < (K + 15) / 16 in all (one jj fewer than K_pad / 16 + 1 when
        // K = 1 mod 16, e.g. N' = 513, 4097: a whole jj of zero DMMAs saved)
        const int jj_n = (c == nch - 1) ? max(0, (mp.K + 30) / 16 - c * (KC / 16)) : KC / 16;
        switch (n_mt) {
          case 4: conv_chunk_mma<4, PT>(xrow, smem_u32(kc), jj_n, fr, lane, -c * KC, mp.K - c * KC); break;
          case 3: conv_chunk_mma<3, PT>(xrow, smem_u32(kc), jj_n, fr, lane, -c * KC, mp.K - c * KC); break;
          case 2: conv_chunk_mma<2, PT>(xrow, smem_u32(kc), jj_n, fr, lane, -c * KC, mp.K - c * KC); break;
          case 1: conv_chunk_mma<1, PT>(xrow, smem_u32(kc), jj_n, fr, lane, -c * KC, mp.K - c * KC); break;
          default: break;
        }
      } else if (mine) {
        conv_chunk_padded<T>(smem_u32(xs) + 8u * PT * (gl + front), smem_u32(kc), nt, acc);   // a5
      }
      if (extra) {
        const int i0 = pg0 * T + T - 1;                      // local word of core word gi0*T - 1
        for (int j = lane; j < nt; j += 32) {
          const int i = i0 + j;
          px = fma(xs[(i / T) * PT + i % T], kc[j], px);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps->empty[st]);
    }
    if (MMA && FRAG_EPI) {
      __syncwarp();
      if (lane == 0) atomicAdd(&ps->core_serve[smsp], 1);   // hand the DMMA pipe to the next claim
    } else if (MMA) {                                        // fragments -> group-major rows -> acc[T]
      __syncwarp();
      if (lane == 0) atomicAdd(&ps->core_serve[smsp], 1);   // hand the DMMA pipe to the next claim
      const int r = lane >> 2, k2 = 2 * (lane & 3);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2) {
          double* d = wbuf + (8 * mt + r) * (T + 1) + 8 * nt2 + k2;
          d[0] = fr[mt][nt2][0];
          d[1] = fr[mt][nt2][1];
        }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = wbuf[lane * (T + 1) + i];
      __syncwarp();
    }
    if (wrec) wrec[2] = gtimer();
    if (PC_REC) {
      const long long c1 = clock64();
      ps->cyc[1] += c1 - ps->cyc[3];
      ps->cyc[3] = c1;
      if (njob < 16) e.dbg_timing[kTimTr + 16 * blockIdx.x + njob] = gtimer();
    }
    // ---- a6/a7: unpack, inverse-compand, discard and place (Eqs. (11)-(17)).  Each warp
    // decodes into its own staging rows (pitch T+1, conflict-free) and writes them out in
    // order, 32 consecutive outputs per store; the valid outputs of a run are one contiguous
    // range, computed once (Eq. (17) placement, the L+N-1 trim, xcorr's valid lags).
    const long long gbase = b.g0 + b.o0;
    const long long goff = (g.mode == 0) ? 0 : (long long)(g.N - 1);     // xcorr: lag = gg - (N-1)
    const long long g_lo = goff, g_hi = (g.mode == 0) ? g.L + g.N - 1 : g.L;   // valid gg
    double* __restrict__ rsig = e.r + jp.sig * e.r_stride - e.r_off - goff;    // rsig[gg]
    const int mw = gi0 * T;                                  // first core output of the warp
    double* row = wbuf + lane * (T + 1);
    // fused xcorr score (a9): running max over this lane's valid lags, lowest lag on ties (C17)
    double sc_v = -__longlong_as_double(0x7ff0000000000000LL);   // -inf
    long long sc_j = -1;
    auto score_or_store = [&](double* dst, long long j, double v) {
      if (e.xc_val) {
        // dst + j is this signal's output slot r[lag - r_off] (placement of C17)
        const long long lagj = (long long)((dst + j) - (e.r + jp.sig * e.r_stride)) + e.r_off;
        if (v > sc_v) {
          sc_v = v;
          sc_j = lagj;
        }
      } else {
        *(dst + j) = v;
      }
    };
    auto flush = [&](double* dst, int step, long long jlo, long long jhi) {
      __syncwarp();
      if (jlo <= 0 && jhi >= 32 * T) {                      // the whole run is valid (most runs)
#pragma unroll
        for (int it = 0; it < T; ++it) {
          const int j = lane + 32 * it;
          score_or_store(dst, (long long)step * j, wbuf[(j / T) * (T + 1) + j % T]);
        }
      } else {
#pragma unroll
        for (int it = 0; it < T; ++it) {
          const int j = lane + 32 * it;
          if (j >= jlo && j < jhi) score_or_store(dst, (long long)step * j, wbuf[(j / T) * (T + 1) + j % T]);
        }
      }
      __syncwarp();
    };
    if (PACK == PACK_SYM) {
      const int moff = (jp.w == 0) ? 0 : 1;
      for (int o = 16; o > 0; o >>= 1) px += __shfl_xor_sync(0xffffffffu, px, o);
      double cb[T];
      if (!mp.paper_unpack) {
        const double Bw = extra ? decode_sym(px, mp.eps, mp.eps_inv, mp.pow2).B : 0.0;
        const double Blast = decode_sym(acc[T - 1], mp.eps, mp.eps_inv, mp.pow2).B;
        const double Bup = __shfl_up_sync(0xffffffffu, Blast, 1);
        double Bprev = (lane == 0) ? Bw : Bup;               // B of the word before the group
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const Digits3 d = decode_sym(acc[i], mp.eps, mp.eps_inv, mp.pow2);
          cb[i] = __dmul_rn(d.C + Bprev, inv);               // r~[2m] = C[m] + B[m-1] (Eqs. (12)-(14))
          acc[i] = __dmul_rn(d.A, inv);                      // r~[2m+1] = A[m] (Eq. (15))
          Bprev = d.B;
        }
      } else {
        // Literal Eqs. (11)-(15) (reading C6), the oracle's operation order:
        // u = r_bar + R_safe (11); side_eps[m] = eps^-1 (u[m-1] - floor u[m-1]) (12), R at the
        // block's first word; side_eps^-1 = floor(eps u) (13); even = floor(side_eps^-1 +
        // side_eps - 2R) (14); odd = floor(floor u - eps^-1 side_eps^-1 - R) (15).
        auto frac_side = [&](double r) {
          const double u = __dadd_rn(r, mp.R_safe);
          return __dmul_rn(mp.eps_inv, __dsub_rn(u, floor(u)));
        };
        const double se_w = extra ? frac_side(px) : mp.R;
        const double se_last = frac_side(acc[T - 1]);
        const double se_up = __shfl_up_sync(0xffffffffu, se_last, 1);
        double se = (lane == 0) ? se_w : se_up;
        const double twoR = __dmul_rn(2.0, mp.R);
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const double u = __dadd_rn(acc[i], mp.R_safe);
          const double fu = floor(u);
          const double sei = floor(__dmul_rn(mp.eps, u));
          cb[i] = __dmul_rn(floor(__dsub_rn(__dadd_rn(sei, se), twoR)), inv);
          acc[i] = __dmul_rn(floor(__dsub_rn(__dsub_rn(fu, __dmul_rn(mp.eps_inv, sei)), mp.R)), inv);
          se = __dmul_rn(mp.eps_inv, __dsub_rn(u, fu));
        }
      }
      // two rounds of 16 groups: rows (r~[2m], r~[2m+1], ...) of pitch 2T+1, one contiguous run
      constexpr int V2 = 2 * T;
      for (int h = 0; h < 2; ++h) {
        if ((lane >> 4) == h) {
          double* row2 = wbuf + (lane & 15) * (V2 + 1);
#pragma unroll
          for (int i = 0; i < T; ++i) {
            row2[2 * i] = cb[i];
            row2[2 * i + 1] = acc[i];
          }
        }
        __syncwarp();
        // output k = 2 (m - moff) + parity = k0 + j for j < 16 * 2T, gg = gbase + k
        const long long k0 = 2LL * ((long long)mw + 16 * h * T - moff);
        long long jlo = -k0, jhi = 2LL * b.M_out - 2LL * moff - k0;   // moff <= m < M_out
        jlo = max(jlo, g_lo - gbase - k0);
        jhi = min(jhi, g_hi - gbase - k0);
        jlo = max(jlo, 0LL);
        jhi = min(jhi, (long long)((min(pgn, 16 * h + 16) - 16 * h) * V2));   // the part's groups only
        double* dst = rsig + gbase + k0;
        if (jlo <= 0 && jhi >= 32 * T) {
#pragma unroll
          for (int it = 0; it < T; ++it) {
            const int j = lane + 32 * it;
            score_or_store(dst, j, wbuf[(j / V2) * (V2 + 1) + j % V2]);
          }
        } else {
#pragma unroll
          for (int it = 0; it < T; ++it) {
            const int j = lane + 32 * it;
            if (j >= jlo && j < jhi) score_or_store(dst, j, wbuf[(j / V2) * (V2 + 1) + j % V2]);
          }
        }
        __syncwarp();
      }
    } else if (FRAG_EPI) {
      // DMMA core, asymmetric / full: every digit is an elementwise function of its packed output
      // (balanced digits, C9), so decode straight from the accumulator fragments -- lane (g, t)
      // holds outputs (8 mt + g) T + 8 nt + 2 t + h of the warp's run -- and store them from there
      // (no shared-memory transpose or staging: the kernel's stages take that space)
      constexpr int M = (PACK == PACK_ASYM2) ? 2 : (PACK == PACK_ASYM3 ? 3 : 1);
      const int seg = (PACK == PACK_FULL) ? b.n_out : b.S;   // outputs per digit segment
      const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        const long long k0 = (long long)q * seg + mw;          // output k = k0 + j
        long long jhi = min((long long)seg - mw, (long long)b.n_out - k0);
        jhi = min(jhi, g_hi - gbase - k0);
        jhi = min(jhi, (long long)(pgn * T));
        const long long jlo = max(0LL, g_lo - gbase - k0);
        double* dst = rsig + gbase + k0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt2 = 0; nt2 < 2; ++nt2)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = (8 * mt + gq) * T + 8 * nt2 + 2 * tq + h;
              const double v = fr[mt][nt2][h];
              double o;
              if (PACK == PACK_FULL) {
                o = v;
              } else {
                const double t = rint_fast(v);
                o = __dmul_rn(t, inv);
                if (q < M - 1) fr[mt][nt2][h] = __dmul_rn(__dsub_rn(v, t), mp.eps_inv);
              }
              if (j >= jlo && j < jhi) score_or_store(dst, j, o);
            }
      }
    } else {
      constexpr int M = (PACK == PACK_ASYM2) ? 2 : (PACK == PACK_ASYM3 ? 3 : 1);
      const int seg = (PACK == PACK_FULL) ? b.n_out : b.S;   // outputs per digit segment
#pragma unroll 1
      for (int q = 0; q < M; ++q) {
#pragma unroll
        for (int i = 0; i < T; ++i) {
          if (PACK == PACK_FULL) {
            row[i] = acc[i];
          } else {                                           // balanced digits (C9)
            const double t = rint_fast(acc[i]);
            row[i] = __dmul_rn(t, inv);
            if (q < M - 1) acc[i] = __dmul_rn(__dsub_rn(acc[i], t), mp.eps_inv);
          }
        }
        const long long k0 = (long long)q * seg + mw;          // output k = k0 + j
        long long jhi = min((long long)seg - mw, (long long)b.n_out - k0);
        jhi = min(jhi, g_hi - gbase - k0);
        const long long jlo = max(0LL, g_lo - gbase - k0);
        flush(rsig + gbase + k0, 1, jlo, min(jhi, (long long)(pgn * T)));
      }
    }
    if (e.xc_val) {                                          // warp max, lowest lag on ties
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, sc_v, o);
        const long long oj = __shfl_xor_sync(0xffffffffu, sc_j, o);
        if (oj >= 0 && (sc_j < 0 || ov > sc_v || (ov == sc_v && oj < sc_j))) {
          sc_v = ov;
          sc_j = oj;
        }
      }
      if (lane == 0) {
        const long long slot = jp.sig * e.jobs_per_sig * npart + (job % e.jobs_per_sig) * npart + part;
        e.xc_val[slot] = sc_v;
        e.xc_lag[slot] = sc_j;
      }
    }
    if (wrec) wrec[3] = gtimer();
    if (PC_REC) ps->cyc[2] += clock64() - ps->cyc[3];
  }
  if (e.dbg_timing && lane == 0) atomicMax(e.dbg_timing + 4 * blockIdx.x + 2, gtimer());   // CTA end = last warp
  if (PC_REC) {
    unsigned long long* tim = e.dbg_timing;
    tim[4 * blockIdx.x + 0] = smid_();
    tim[4 * blockIdx.x + 1] = tim[kTimCyc + 4 * blockIdx.x + 2];   // t_start (stashed)
    tim[4 * blockIdx.x + 3] = njob;
    tim[kTimCyc + 4 * blockIdx.x + 0] = ps->cyc[0];
    tim[kTimCyc + 4 * blockIdx.x + 1] = ps->cyc[1];
    tim[kTimCyc + 4 * blockIdx.x + 2] = ps->cyc[2];
  }
#undef PC_REC
}

// ------------------------------------------------------------------ prepack (a2-a4 ahead)
// One CTA per job: the block's W_block samples are loaded once into shared memory (coalesced,
// every load in flight at once) while the block peak is reduced from them (integer max of |x|
// bits), c_s = Q / peak (Eq. (2)); the job's stage image -- exactly the words pack_window writes
// into a ring stage, pitch PT -- is then packed from shared memory into HBM (L2-resident for the
// tiled launch that follows), with (c_s c_k)^-1 (Eq. (16)).  The tiled kernel's producer warps
// then move each image with one bulk copy.
constexpr int kPrepackThreads = 512;
template <int PACK, int T, int PT>
__global__ void __launch_bounds__(kPrepackThreads) pc_prepack_kernel(Geo g, Exec e) {
  extern __shared__ __align__(16) double raw[];
  __shared__ unsigned long long ired[kPrepackThreads / 32];
  const ModeP& mp = e.mp[PACK];
  const long long job = blockIdx.x;
  const int tid = threadIdx.x;
  const JobPos jp = job_pos(e, job);
  const Blk b = block_info<PACK>(g, mp.K, jp.w);
  const double* gsrc = e.s + jp.sig * e.s_stride + (b.g0 - e.s_off);
  const long long avail = g.L - b.g0;
  const int n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int U = 8;
  unsigned long long m = 0ull;
  for (int i0 = tid; i0 < n_valid; i0 += U * kPrepackThreads) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kPrepackThreads;
      v[u] = (i < n_valid) ? __ldg(gsrc + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kPrepackThreads;
      if (i < n_valid) raw[i] = v[u];
      m = umax64(m, abs_bits(v[u]));
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = umax64(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) ired[tid >> 5] = m;
  __syncthreads();
  unsigned long long pm = 0ull;
#pragma unroll
  for (int w = 0; w < kPrepackThreads / 32; ++w) pm = umax64(pm, ired[w]);
  const double peak = __longlong_as_double((long long)pm);
  const double cs = (PACK == PACK_FULL || peak == 0.0) ? 1.0 : mp.Q / peak;   // Eq. (2)
  const int front = (PACK == PACK_SYM) ? 1 : 0;
  double* xs = const_cast<double*>(e.pre_win) + job * e.pre_stride;
  pack_window<PACK, T, 1, PT, true>(g, b, mp, raw, n_valid, cs, jp.t * e.G * T - front * T, e.rows_s, xs, tid,
                                    kPrepackThreads, false);
  if (tid == 0)
    const_cast<double*>(e.pre_inv)[job] = dequant_scale(cs, e.scal_sig ? e.scal_sig[3 * jp.sig + 1] : mp.c_k);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int PACK, int T, int PT>
static cudaError_t launch_prepack_t(const Geo& g, const Exec& e, long long n_jobs, cudaStream_t st) {
  auto kfn = pc_prepack_kernel<PACK, T, PT>;
  const size_t smem = (size_t)g.W_block * sizeof(double);
  static LaunchAttrCache cache;                      // per device, under a lock
  int dev = 0, sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err == cudaSuccess) err = cache.ensure(kfn, dev, smem, kPrepackThreads, &sms);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_jobs);
  cfg.blockDim = dim3(kPrepackThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, g, e);
}

template <int T, int PT>
static cudaError_t launch_prepack_T(int packing, const Geo& g, const Exec& e, long long n_jobs, cudaStream_t st) {
  switch (packing) {
    case PACK_SYM: return launch_prepack_t<PACK_SYM, T, PT>(g, e, n_jobs, st);
    case PACK_ASYM2: return launch_prepack_t<PACK_ASYM2, T, PT>(g, e, n_jobs, st);
    case PACK_ASYM3: return launch_prepack_t<PACK_ASYM3, T, PT>(g, e, n_jobs, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_prepack(int packing, int T, int mma, const Geo& g, const Exec& e, long long n_jobs, cudaStream_t st) {
  if (n_jobs <= 0) return cudaSuccess;
  if ((size_t)g.W_block * sizeof(double) > 200 * 1024) return cudaErrorInvalidValue;   // raw block in smem
  if (mma) return T == 16 ? launch_prepack_T<16, 20>(packing, g, e, n_jobs, st) : cudaErrorInvalidValue;
  switch (T) {
    case 12: return launch_prepack_T<12, 13>(packing, g, e, n_jobs, st);
    case 14: return launch_prepack_T<14, 15>(packing, g, e, n_jobs, st);
    case 16: return launch_prepack_T<16, 17>(packing, g, e, n_jobs, st);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ launcher
template <int PACK, int T, int MMA>
static cudaError_t launch_tiled_t(const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                                  cudaStream_t st, int* grid_out) {
  // the variant instantiation (VAR = 1) only for DMMA-core packed plans that ask for it
  constexpr bool kHasVar = MMA == 1 && PACK != PACK_FULL;
  const bool want_var = kHasVar && (e.split_P > 0 || e.mp[PACK].alu_pack);
  auto kfn = want_var ? pc_tiled_kernel<PACK, T, MMA, kHasVar ? 1 : 0> : pc_tiled_kernel<PACK, T, MMA, 0>;
  static LaunchAttrCache cache[2];                   // per kernel instantiation and device, under a lock
  int dev = 0, c_sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err == cudaSuccess) err = cache[want_var ? 1 : 0].ensure(kfn, dev, smem, threads, &c_sms);
  if (err != cudaSuccess) return err;
  if (c_sms > kCtrDone) return cudaErrorInvalidConfiguration;
  Exec ex = e;
  ex.nsm = c_sms;
  if (!want_var && ex.split_P > 0) {                 // producer-SM mode not compiled for this kernel: the
    ex.split_P = 0;                                  // fused producers (the FMA-core plans)
    ex.pre_win = nullptr;
    ex.pre_inv = nullptr;
  }
  long long grid = c_sms;                            // one persistent CTA per SM (smem >= half an SM)
  if (ex.split_P > 0) {                              // producer-SM mode: every SM, at most half of them producing
    if (ex.split_P > grid / 2) ex.split_P = (int)(grid / 2);
    if (ex.split_P < 1) {                            // (a single SM: the fused producers)
      ex.split_P = 0;
      ex.pre_win = nullptr;
      ex.pre_inv = nullptr;
    }
  } else if (grid > n_jobs) {
    grid = n_jobs;
  }
  *grid_out = (int)grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, g, ex);
}

template <int T, int MMA>
static cudaError_t launch_tiled_T(int packing, const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                                  cudaStream_t st, int* grid_out) {
  switch (packing) {
    case PACK_FULL: return launch_tiled_t<PACK_FULL, T, MMA>(g, e, n_jobs, threads, smem, st, grid_out);
    case PACK_SYM: return launch_tiled_t<PACK_SYM, T, MMA>(g, e, n_jobs, threads, smem, st, grid_out);
    case PACK_ASYM2: return launch_tiled_t<PACK_ASYM2, T, MMA>(g, e, n_jobs, threads, smem, st, grid_out);
    case PACK_ASYM3: return launch_tiled_t<PACK_ASYM3, T, MMA>(g, e, n_jobs, threads, smem, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tiled(int packing, int T, int mma, const Geo& g, const Exec& e, long long n_jobs, int threads,
                         size_t smem, cudaStream_t st, int* grid_out) {
  *grid_out = 0;
  if (n_jobs <= 0) return cudaSuccess;
  if (mma) return T == 16 ? launch_tiled_T<16, 1>(packing, g, e, n_jobs, threads, smem, st, grid_out)
                          : cudaErrorInvalidValue;
  switch (T) {
    case 12: return launch_tiled_T<12, 0>(packing, g, e, n_jobs, threads, smem, st, grid_out);
    case 14: return launch_tiled_T<14, 0>(packing, g, e, n_jobs, threads, smem, st, grid_out);
    case 16: return launch_tiled_T<16, 0>(packing, g, e, n_jobs, threads, smem, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pc
