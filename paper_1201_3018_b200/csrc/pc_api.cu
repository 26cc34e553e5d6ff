// pc_api.cu -- the C ABI of include/packedconv.h: plan geometry, kernel initialization,
// bound policy and launch orchestration.  All numeric work runs in pc_kernels.cu.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <utility>

#include <cuda_runtime.h>

#include "../../include/packedconv.h"
#include "pc_kernels.h"

using pc::Exec;
using pc::Geo;
using pc::ModeP;

namespace {

constexpr size_t kMaxSmem = 232448;      // 227 KB dynamic shared memory per CTA (sm_100)
constexpr long long kSmallCoreFma = 100000;   // per-block core FMAs below which the per-block kernel runs
constexpr size_t kSmemPerSM = 233472;    // 228 KB shared memory per SM

struct ModeState {
  int valid = 0;
  int Q = 0, K_q = 0;
  long long R = 0, bound = 0;
  int bound_ok = 0;
  double eps = 0, eps_inv = 0;
  int b = 0;
  double c_k = 1.0;
  double* kr = nullptr;
  int K = 0, K_pad = 0, rows = 0;      // per-block kernel layout (tile kT)
};

}  // namespace

struct conv_plan {
  long long L = 0, P = 0;
  int N = 0, Np = 0, W_block = 0, W = 0;
  int mode = 0, packing = 0, Q = 0, K_q = 0;
  conv_opts opts;
  int device = 0;
  int kernel_set = 0;
  double k_peak = 0, k_sigma = 0;
  ModeState ms[4];
  int qmode[4] = {0, 0, 0, 0};
  double* d_k_pad = nullptr;
  double* d_k_int = nullptr;
  double* d_scal = nullptr;
  // adaptive decisions (per block)
  int* d_dec_pack = nullptr;
  int* d_dec_q = nullptr;
  double* d_dec_snr = nullptr;
  double* d_sigma = nullptr;
  double* d_peak = nullptr;
  int* d_cand = nullptr;
  int* d_lists = nullptr;              // adaptive: per-packing ascending block lists [4][P]
  int* d_counts = nullptr;             // adaptive: their lengths [4]
  int adapt_ready = 0;
  long long adapt_b0 = 0, adapt_b1 = 0;  // the block range the decisions (and lists) cover
  // host end-to-end staging
  double* d_in = nullptr;
  double* d_out = nullptr;
  cudaStream_t st_h2d = nullptr, st_d2h = nullptr;   // conv_execute_host pipeline (plan-owned)
  // conv_plan_set_kernels / conv_xcorr_pairs (NEXT-3): one kernel per pair
  long long n_kernels = 0;
  double* d_pk_pad = nullptr;          // [n][N'] padded (reversed) kernels, then k~
  double* d_pk_int = nullptr;
  double* d_pk_scal = nullptr;         // [n][3] {peak, c_k, l1}
  double* d_pk_taps = nullptr;         // [n][K + 32] core taps, reversed
  double* d_xc_pval = nullptr;         // conv_xcorr_max fused: per warp-part partial max and its lag
  long long* d_xc_plag = nullptr;
  size_t xc_part_n = 0;
  cudaEvent_t ev_in[16] = {}, ev_done[16] = {}, ev_out = nullptr;
  // xcorr scratch
  double* d_xc = nullptr;
  size_t d_xc_bytes = 0;
  // persistent kernel job counter (monotonic; base tracked on the host)
  unsigned* d_counter = nullptr;        // tiled kernel: two arrays of per-SM job queues + done counter (zero between launches)
  int ctr_flip = 0;                     // the array the next non-adaptive tiled launch uses
  int cand_ok = 0;                      // adaptive: d_cand holds this kernel's candidate table
  double* d_pre = nullptr;              // prepacked stage images + per-job inverse scales (pc_prepack_kernel)
  long long pre_flags_jobs = -1;         // producer-SM mode: job count the ready flags were zeroed for
  long long pre_cap = 0;                // doubles allocated at d_pre
  // FFT core
  int fft_N = 0;                       // complex points (real transform length 2N)
  double2* d_tw = nullptr;             // exp(-2 pi i m / N)
  double2* d_tw2 = nullptr;            // exp(-2 pi i k / 2N), k <= N
  double2* d_H = nullptr;              // spectrum of the core taps, k <= N
  double* d_resid = nullptr;           // max last-digit residual (LSB)
  int backend_ok = -1;                 // FFT backend validation: 1 pass, 0 fail (WARN), -1 not run
  double backend_resid = 0.0, u_sys_cal = 0.0;
  // flags the kernels raise in host-mapped pinned memory (pc::kStatusMargin / kStatusWatchdog)
  int* h_status = nullptr;             // host view
  int* d_status = nullptr;             // device view of the same memory
  double* d_dbg_resid = nullptr;       // conv_execute_debug: max last-digit residual
  double* d_blkpeak = nullptr;         // block peaks ahead of the persistent kernel [n_sig][P]
  long long blkpeak_cap = 0;
};

namespace {

int n_digits(int p) { return p == PC_PACK_ASYM2 ? 2 : 3; }

// Reading C4: eps = 2^-b exact iff R(2^{2b}+2^b+1) < 2^53 (3 digits) / R(2^b+1) < 2^53.
bool pow2_exact(long long R, int digits) {
  if (R < 1) return true;
  const int b = 64 - __builtin_clzll((unsigned long long)(2 * R));
  if (b > 40) return false;
  unsigned __int128 span = digits == 3 ? (((unsigned __int128)1 << (2 * b)) + ((unsigned __int128)1 << b) + 1)
                                       : (((unsigned __int128)1 << b) + 1);
  return (unsigned __int128)R * span < ((unsigned __int128)1 << 53);
}
long long pow2_bound(int digits) {
  long long lo = 1, hi = 1LL << 40;
  while (lo < hi) {
    const long long mid = lo + (hi - lo + 1) / 2;
    if (pow2_exact(mid, digits)) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// Table 1 for the paper's eps; the dyadic exactness bound for POW2.
long long bound_for(int packing, int eps_rule) {
  if (eps_rule == PC_EPS_POW2) return pow2_bound(n_digits(packing));
  return packing == PC_PACK_ASYM2 ? 43165096LL : 97667LL;
}

int core_taps(const conv_plan* p, int packing) { return packing == PC_PACK_SYM ? (p->Np + 1) / 2 : p->Np; }

Geo make_geo(const conv_plan* p) {
  Geo g;
  g.L = p->L;
  g.P = p->P;
  g.N = p->N;
  g.Np = p->Np;
  g.W_block = p->W_block;
  g.W = p->W;
  g.mode = p->mode;
  return g;
}

template <int PACK>
void max_core_sizes(const Geo& g, int K, int* m_out_max, int* m_out_typ) {
  const pc::Blk b0 = pc::block_info<PACK>(g, K, 0);
  const pc::Blk b1 = pc::block_info<PACK>(g, K, 1);
  *m_out_max = b0.M_out > b1.M_out ? b0.M_out : b1.M_out;
  *m_out_typ = g.P > 1 ? b1.M_out : b0.M_out;
}
void core_sizes(const conv_plan* p, int packing, int* mmax, int* mtyp) {
  const Geo g = make_geo(p);
  const int K = core_taps(p, packing);
  switch (packing) {
    case PC_PACK_SYM: max_core_sizes<pc::PACK_SYM>(g, K, mmax, mtyp); break;
    case PC_PACK_ASYM2: max_core_sizes<pc::PACK_ASYM2>(g, K, mmax, mtyp); break;
    case PC_PACK_ASYM3: max_core_sizes<pc::PACK_ASYM3>(g, K, mmax, mtyp); break;
    default: max_core_sizes<pc::PACK_FULL>(g, K, mmax, mtyp); break;
  }
}

// Column layout of the core's input words for a tile of T outputs per thread: K padded to a
// multiple of T; rows >= groups + K_pad/T, rounded to 4 mod 16 so that lane-consecutive
// word stores (packing) hit every bank pair exactly twice.
void layout_for(int K, int mmax, int T, int* K_pad, int* rows) {
  *K_pad = (K + T - 1) / T * T;
  const int ngroups = (mmax + T - 1) / T;
  int r = ngroups + *K_pad / T + 1;
  r = (r + 11) / 16 * 16 + 4;
  *rows = r;
}
void set_core_layout(const conv_plan* p, int packing, ModeState* m) {
  int mmax, mtyp;
  core_sizes(p, packing, &mmax, &mtyp);
  m->K = core_taps(p, packing);
  layout_for(m->K, mmax, pc::kT, &m->K_pad, &m->rows);
}

// Launch shape of the fused kernel for the packings that may run in this plan.
// Threads: one T-output group per thread when the largest block has <= 1024 groups (the
// register path); otherwise 256 threads looping over groups with a separate result region.
// The raw block is TMA-staged in shared memory only when that does not lower the number
// of resident CTAs per SM (64 registers/thread cap from __launch_bounds__).
struct Shape {
  int threads;
  int stage_raw;
  int reg_path;
  size_t smem;
};
// Per-block kernel: threads per CTA at least (cfg1, 1024-sample blocks: one CTA per block on
// fewer CTAs than SMs, so each block's phases are latency-bound; 64 -> 256 threads measured asym2
// 9-bit 8.8 -> 5.7 us, full precision 4.8 -> 4.4 us with the tap slices of fused_block).
#ifndef PC_FUSED_TMIN
#define PC_FUSED_TMIN 256
#endif
#ifndef PC_FUSED_TMIN_FULL
#define PC_FUSED_TMIN_FULL 256
#endif
bool launch_shape(const conv_plan* p, const int* packs, int npacks, Shape* sh) {
  size_t core = 0;
  int mmax_all = 0, groups_max = 0;
  for (int i = 0; i < npacks; ++i) {
    const ModeState& m = p->ms[packs[i]];
    int mmax, mtyp;
    core_sizes(p, packs[i], &mmax, &mtyp);
    const size_t c = (size_t)pc::kT * m.rows * 8 + (size_t)m.K_pad * 8;
    if (c > core) core = c;
    if (mmax > mmax_all) mmax_all = mmax;
    const int gm = (mmax + pc::kT - 1) / pc::kT;
    if (gm > groups_max) groups_max = gm;
  }
  sh->reg_path = groups_max <= pc::kMaxThreads;
  int t = sh->reg_path ? (groups_max + 31) / 32 * 32 : 256;
  const int t_min = (p->packing == PC_PACK_FULL) ? PC_FUSED_TMIN_FULL : PC_FUSED_TMIN;
  if (t < t_min) t = t_min;
  sh->threads = t;
  const size_t base = pc::kSmemHeader + core + (sh->reg_path ? 0 : (size_t)mmax_all * 8 + 16);
  const size_t staged = base + (size_t)p->W_block * 8;
  const int by_regs = 65536 / (t * 64);
  auto ctas = [&](size_t sm) { return (int)(kSmemPerSM / (sm + 1024)); };
  int mode = p->opts.raw_staging;   // 0 auto, 1 force staging, 2 never stage
  bool stage = staged <= kMaxSmem && (mode == 1 || (mode == 0 && ctas(staged) >= (by_regs < ctas(base) ? by_regs : ctas(base))));
  if (stage) {
    sh->stage_raw = 1;
    sh->smem = staged;
  } else if (base <= kMaxSmem) {
    sh->stage_raw = 0;
    sh->smem = base;
  } else {
    return false;
  }
  return true;
}

// Tiled persistent kernel (pc_tiled.cu), one CTA per SM: choose the tile T and the parts per
// job (G = 32 * npart groups, npart in {1, 2, 4}) so that typical blocks' groups fill whole
// tiles; taps resident when <= 4096, else chunks of ~1024 taps (a multiple of T); as many
// stage-ring slots as shared memory holds (2..8) after the per-warp output staging rows.
struct TShape {
  int T, mma, threads, G, KC, nchunks, taps_resident, rows_s, K_pad, nstages;
  int raw_slots, raw_stride;   // raw-staged producers: raw block slots in smem (0: global loads)
  long long tiles0, tiles1;
  size_t smem;
};
bool tiled_shape(const conv_plan* p, int packing, TShape* sh, bool taps_per_signal = false) {
  int mmax, mtyp;
  core_sizes(p, packing, &mmax, &mtyp);
  const int K = core_taps(p, packing);
  const int force = p->opts.core_tile;
  // core: the FP64 tensor cores (DMMA, T = 16) unless the FMA core or another tile is forced;
  // auto keeps the FMA core for symmetric packing with a short core (about N/2 taps): there the
  // three-digit epilogue weighs as much as the core and the DMMA interference slows it (cfg2,
  // 257 taps: FMA 71.6 vs DMMA 75.6 us; 512 taps: within +-8% either way by geometry); from 768
  // taps on DMMA wins (1025: 429 vs 438 us, cfg4's 4097: 143.4 vs 160.0 ms); likewise asymmetric
  // M = 3 below 256 taps (129 taps: FMA 49.9
  // vs 55.1 us; 257: equal; 513: DMMA 82.6 vs 95); asym2 and full precision: DMMA at every length
  const int core = p->opts.core_variant;
  const bool long_core = packing == PC_PACK_SYM ? K >= 768 : (packing == PC_PACK_ASYM3 ? K >= 256 : true);
  sh->mma = (core == 2 || (core == 0 && long_core)) && (force == 0 || force == 16);
  double best = -1.0;
  for (int T : pc::kTPChoices) {
    if ((force == 12 || force == 14 || force == 16) && T != force) continue;
    if (sh->mma && T != 16) continue;
    const double speed = T == 16 ? 1.0 : (T == 14 ? 0.96 : 0.92);   // core-loop calibration (profiles)
    for (int npart : {4, 2, 1}) {
      if (p->opts.parts_per_job > 0 && npart != p->opts.parts_per_job) continue;   // diagnostics: force G
      const int G = 32 * npart;
      const long long groups = (mtyp + T - 1) / T;
      const long long tiles = (groups + G - 1) / G;
      // the DMMA core skips a part's m-tiles (8 groups) past the block's end
      const double util = sh->mma ? (double)groups / (double)((groups + 7) / 8 * 8)
                                  : (double)groups / (double)(tiles * G);
      // fewer parts per job: more jobs (ring slots, producer work) per resident warp
      const double score = util * speed * (npart == 4 ? 1.0 : (npart == 2 ? 0.9 : 0.75));
      if (score > best + 1e-9) {
        best = score;
        sh->T = T;
        sh->G = G;
      }
    }
  }
  const int T = sh->T;
  sh->K_pad = (K + T - 1) / T * T;
  sh->threads = pc::tiled_threads(sh->mma);
  const int KCmax = taps_per_signal ? 1024 : 4096;   // per-signal taps travel with every stage
  if (sh->K_pad <= KCmax && !taps_per_signal) {
    sh->taps_resident = 1;
    sh->nchunks = 1;
    sh->KC = sh->K_pad;
  } else {
    sh->taps_resident = 0;
    const int nch = (sh->K_pad + 1023) / 1024;
    sh->KC = ((sh->K_pad + nch - 1) / nch + T - 1) / T * T;
    sh->nchunks = (sh->K_pad + sh->KC - 1) / sh->KC;
  }
  const int front = packing == PC_PACK_SYM ? 1 : 0;
  sh->rows_s = front + sh->G + sh->KC / T;   // the window reads rows up to G-1 + KC/T (+front)
  const long long g0 = (mmax + T - 1) / T;         // block 0 has the most groups
  const long long g1 = (mtyp + T - 1) / T;
  sh->tiles0 = (g0 + sh->G - 1) / sh->G;
  sh->tiles1 = (g1 + sh->G - 1) / sh->G;
  const int PT = sh->mma ? T + 4 : T + 1, TH = sh->mma ? 16 : 0;   // as pc_tiled_kernel
  const size_t stage = (size_t)((PT * sh->rows_s + 1) & ~1) * 8 + (sh->taps_resident ? 0 : (size_t)(sh->KC + 2 * TH) * 8);
  // per-warp output staging rows: the FMA core and symmetric packing only (the DMMA core's
  // asymmetric / full epilogue decodes from its fragments, so those rows become ring stages)
  const bool staging = !sh->mma || packing == PC_PACK_SYM;
  size_t fixed = pc::kTiledHeader + (sh->taps_resident ? (size_t)(sh->K_pad + 2 * TH) * 8 : 0) +
                 (staging ? (size_t)pc::tiled_cons_warps(sh->mma) * 32 * (T + 1) * 8 : 0);
  if (fixed + 2 * stage > kMaxSmem) return false;
  // Raw-staged producers (single-chunk plans; opts.raw_staging 0 auto / 1 on / 2 off): the job's
  // raw block (W_block samples) arrives by one TMA bulk copy into a shared-memory slot, two slots
  // (the next job's copy in flight) when the ring keeps >= PC_RAW_MIN_STAGES stages, else one
  // (cfg2 asym2/sym: one slot and 7 stages measured 0.9-2% faster than two slots and 6).
#ifndef PC_RAW_PROD
#define PC_RAW_PROD 1
#endif
#ifndef PC_RAW_MIN_STAGES
#define PC_RAW_MIN_STAGES 7
#endif
  sh->raw_slots = 0;
  sh->raw_stride = 0;
  // (auto: asymmetric M = 2 and symmetric packing; measured at cfg2: asym2 93.2 -> 88.5 us, sym 73.8
  // -> 72.7, while asym3 80.0 vs 78.5 and full precision -- no peak, plain copies -- 158 vs 144 lose)
  if (PC_RAW_PROD && sh->nchunks == 1 && p->opts.raw_staging != 2 &&
      (packing == PC_PACK_ASYM2 || packing == PC_PACK_SYM || p->opts.raw_staging == 1)) {
    const size_t rs = (size_t)((p->W_block + 3) & ~1);   // doubles per slot (head offset, even)
    for (int k = 2; k >= 1; --k) {
      const size_t f2 = fixed + (size_t)k * rs * 8;
      const int nst = f2 + 2 * stage <= kMaxSmem ? (int)((kMaxSmem - f2) / stage) : 0;
      if (nst >= (p->opts.raw_staging == 1 ? 2 : PC_RAW_MIN_STAGES - (2 - k))) {
        sh->raw_slots = k;
        sh->raw_stride = (int)rs;
        fixed = f2;
        break;
      }
    }
  }
  sh->nstages = (int)((kMaxSmem - fixed) / stage);
  if (sh->nstages > pc::kTiledMaxStages) sh->nstages = pc::kTiledMaxStages;
  if (p->opts.stage_cap >= 2 && sh->nstages > p->opts.stage_cap) sh->nstages = p->opts.stage_cap;   // diagnostics
  sh->smem = fixed + (size_t)sh->nstages * stage;
  if (sh->smem < kMaxSmem / 2 + 4096) sh->smem = kMaxSmem / 2 + 4096;   // one CTA per SM
  return true;
}

// FFT core geometry: part sizes and counts for 2N real points.  A block's first part gives
// 2N - K + 1 outputs; later parts 2N - K (a symmetric part after the first also needs the
// word before it, for B of its first even output).
struct FShape {
  int part0_out, part_out;
  long long parts0, parts1;
};
bool fft_shape(const conv_plan* p, int packing, int N, FShape* f) {
  int mmax, mtyp;
  core_sizes(p, packing, &mmax, &mtyp);
  const int K = core_taps(p, packing);
  f->part0_out = 2 * N - K + 1;
  f->part_out = 2 * N - K;
  if (f->part_out < 1) return false;
  auto parts = [&](int M) -> long long {
    return M <= f->part0_out ? 1 : 1 + (M - f->part0_out + f->part_out - 1) / f->part_out;
  };
  int m0, m1;
  {
    const Geo g = make_geo(p);
    switch (packing) {
      case PC_PACK_SYM: m0 = pc::block_info<pc::PACK_SYM>(g, K, 0).M_out; m1 = pc::block_info<pc::PACK_SYM>(g, K, 1).M_out; break;
      case PC_PACK_ASYM2: m0 = pc::block_info<pc::PACK_ASYM2>(g, K, 0).M_out; m1 = pc::block_info<pc::PACK_ASYM2>(g, K, 1).M_out; break;
      case PC_PACK_ASYM3: m0 = pc::block_info<pc::PACK_ASYM3>(g, K, 0).M_out; m1 = pc::block_info<pc::PACK_ASYM3>(g, K, 1).M_out; break;
      default: m0 = pc::block_info<pc::PACK_FULL>(g, K, 0).M_out; m1 = pc::block_info<pc::PACK_FULL>(g, K, 1).M_out; break;
    }
  }
  f->parts0 = parts(m0);
  f->parts1 = parts(m1);
  return true;
}
// FFT size N (complex points, 1024..8192) minimizing the modelled time of a typical block:
// parts x (transform work N log2 N + the block's sample loads 3 W_block), divided by the
// CTAs an SM overlaps (1.4x effective for N <= 4096, two CTAs per SM; measured on cfg3).
int choose_fft_N(const conv_plan* p, int packing) {
  int mmax, mtyp;
  core_sizes(p, packing, &mmax, &mtyp);
  const int K = core_taps(p, packing);
  const int force = p->opts.fft_n;                  // complex points N (0 = cost model)
  if (force == 1024 || force == 2048 || force == 4096 || force == 8192) return 2 * force - K >= 1 ? force : 0;
  // 32768-point real transform of the whole block (cfg3's configured full-precision core):
  // full precision, windows of at most 16384 real words (2-CTA cluster kernel)
  if (force == 16384) return (packing == PC_PACK_FULL && p->W_block <= 16386) ? 16384 : 0;
  int best_N = 0;
  double best = 0.0;
  for (int N = 1024, lg = 10; N <= 8192; N *= 2, ++lg) {
    const int part_out = 2 * N - K;
    if (part_out < 1) continue;
    const long long parts = mtyp <= part_out + 1 ? 1 : 1 + (mtyp - (part_out + 1) + part_out - 1) / part_out;
    const double cost = (double)parts * ((double)N * lg + 3.0 * p->W_block) / (N <= 4096 ? 1.4 : 1.0);
    if (best_N == 0 || cost < best) {
      best = cost;
      best_N = N;
    }
  }
  return best_N;
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? PC_OK : PC_E_CUDA; }

void fill_modep(const ModeState& m, int packing, ModeP* mp) {
  mp->kr = m.kr;
  mp->Q = (double)m.Q;
  mp->c_k = m.c_k;
  mp->eps = m.eps;
  mp->eps_inv = m.eps_inv;
  mp->pow2 = m.b > 0;
  mp->b = m.b;
  // Packed words as integers n * 2^-((M-1) b): exact in FP64 iff |n| < 2^53, then the integer
  // Horner of the companded digits equals the FP64 one bit for bit (pc_tiled.cu, pack_window).
  const int M = packing == PC_PACK_ASYM3 ? 3 : 2;
  mp->alu_pack = packing != PC_PACK_FULL && m.b > 0 && (M - 1) * m.b <= 60 &&
                 (double)m.Q * (std::ldexp(1.0, (M - 1) * m.b) * 2.0) < std::ldexp(1.0, 53);
  mp->exact_pack = mp->alu_pack;   // (not cleared with alu_pack: the FMA form is the default)
  mp->K = m.K;
  mp->K_pad = m.K_pad;
  mp->rows = m.rows;
  mp->paper_unpack = 0;
  mp->R = (double)m.R;
  mp->R_safe = 0.0;
}

// The packings a plan's launches may use.
int plan_packs(const conv_plan* p, int* packs) {
  if (p->packing == PC_PACK_ADAPTIVE) {
    packs[0] = PC_PACK_SYM;
    packs[1] = PC_PACK_ASYM2;
    packs[2] = PC_PACK_FULL;
    return 3;
  }
  packs[0] = p->packing;
  return 1;
}

// Does a (non-debug) direct-core execute of this non-adaptive plan run the tiled kernel?
// (The per-block kernel serves small cores unless the tiled kernel is forced; see run_exec.)
bool small_core_plan(const conv_plan* p, const int* packs, int np) {
  for (int i = 0; i < np; ++i) {
    int mmax, mtyp;
    core_sizes(p, packs[i], &mmax, &mtyp);
    if ((long long)mtyp * core_taps(p, packs[i]) >= kSmallCoreFma) return false;
  }
  return true;
}
bool forced_tiled(const conv_plan* p) {
  return p->opts.core_tile != 0 || p->opts.parts_per_job != 0 || p->opts.unpack_form == PC_UNPACK_LITERAL;
}
bool uses_tiled(const conv_plan* p) {
  if (p->opts.core != PC_CORE_DIRECT || p->packing == PC_PACK_ADAPTIVE) return false;
  if (p->opts.exec != PC_EXEC_FUSED && p->opts.exec != PC_EXEC_TILED) return false;
  TShape ts;
  if (!tiled_shape(p, p->packing, &ts)) return false;
  if (p->opts.exec == PC_EXEC_TILED || forced_tiled(p)) return true;
  int packs[4];
  const int np = plan_packs(p, packs);
  Shape sh;
  return !(small_core_plan(p, packs, np) && launch_shape(p, packs, np, &sh));
}

// Tiled launches overlap (programmatic dependent launch): with opts.early_fill = 1 the next
// launch's pipeline fill may run before the preceding launch on the stream has finished as long
// as it does not read what that launch writes.  Opt-in: measured no faster at cfg2 (102.7 vs
// 102.1 us per step; the step is bound by each SM's own 8 jobs), and a foreign kernel with its
// own programmatic trigger between two of ours could not be seen by this check.  Per (device,
// stream): the output address range of the last tiled launch.  A kernel of anyone else in
// between has no programmatic trigger, so the tiled launch after it starts only once it has
// completed -- the stale record can only make this check conservative.
std::mutex g_streams_mu;
std::map<std::pair<int, cudaStream_t>, std::pair<uintptr_t, uintptr_t>> g_last_out;
bool early_fill_ok(const conv_plan* p, cudaStream_t st, uintptr_t in_lo, uintptr_t in_hi) {
  if (p->opts.early_fill != 1) return false;
  std::lock_guard<std::mutex> lk(g_streams_mu);
  auto it = g_last_out.find({p->device, st});
  return it == g_last_out.end() || in_hi <= it->second.first || it->second.second <= in_lo;
}
void record_out(int dev, cudaStream_t st, uintptr_t lo, uintptr_t hi) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  g_last_out[{dev, st}] = {lo, hi};
}

int run_exec(conv_plan* p, const double* s, long long s_off, long long s_stride, double* r, long long r_off,
              long long r_stride, long long b0, long long nblk, long long n_sig, Exec* dbg, cudaStream_t st,
              unsigned long long* timing = nullptr, int* grid_out = nullptr, double* xc_val = nullptr,
              long long* xc_lag = nullptr, bool pairs = false) {
  if (!p->kernel_set) return PC_E_STATE;
  if (p->packing == PC_PACK_ADAPTIVE &&
      (!p->adapt_ready || n_sig != 1 || b0 < p->adapt_b0 || b0 + nblk > p->adapt_b1))
    return PC_E_STATE;                                  // execute only blocks with decisions
  if (nblk <= 0 || n_sig <= 0) return PC_OK;
  int packs[4];
  const int np = plan_packs(p, packs);
  Shape sh;
  const bool per_block_ok = launch_shape(p, packs, np, &sh);
  Exec e;
  std::memset(&e, 0, sizeof(e));
  if (dbg) e = *dbg;
  e.s = s;
  e.s_off = s_off;
  e.s_stride = s_stride;
  e.r = r;
  e.r_off = r_off;
  e.r_stride = r_stride;
  e.b0 = b0;
  e.nblk = nblk;
  e.stage_raw = per_block_ok ? sh.stage_raw : 0;
  e.reg_path = per_block_ok ? sh.reg_path : 0;
  for (int i = 0; i < np; ++i) {
    fill_modep(p->ms[packs[i]], packs[i], &e.mp[packs[i]]);
    if (p->opts.pack_alu != 1) e.mp[packs[i]].alu_pack = 0;   // integer companding/packing only when asked (measured slower)
  }
  if (p->opts.unpack_form == PC_UNPACK_LITERAL) {   // literal Eqs. (11)-(15) (SYM, tiled kernel)
    pc::ModeP& ms = e.mp[PC_PACK_SYM];
    ms.paper_unpack = 1;
    ms.R_safe = ms.R * (ms.eps + 1.0 + ms.eps_inv) + p->opts.u_sys * ms.eps_inv;   // P:103, oracle order
  }
  e.dec_pack = p->packing == PC_PACK_ADAPTIVE ? p->d_dec_pack : nullptr;
  e.nsig = n_sig;
  e.status = p->d_status;
  const int launch_pack = p->packing == PC_PACK_ADAPTIVE ? -1 : p->packing;
  if (p->opts.core == PC_CORE_FFT) {
    if (dbg) return PC_E_CONFIG;                      // per-step dumps exist for the direct core
    FShape fs;
    if (!fft_shape(p, p->packing, p->fft_N, &fs)) return PC_E_CONFIG;
    pc::FftArgs f;
    f.tw = p->d_tw;
    f.tw2 = p->d_tw2;
    f.H = p->d_H;
    f.resid = p->d_resid;
    f.part0_out = fs.part0_out;
    f.part_out = fs.part_out;
    f.parts0 = fs.parts0;
    f.parts1 = fs.parts1;
    e.jobs_per_sig = (b0 == 0) ? fs.parts0 + (nblk - 1) * fs.parts1 : nblk * fs.parts1;
    e.dbg_timing = timing;
    if (grid_out) *grid_out = (int)(e.jobs_per_sig * n_sig);
    return cuda_status(pc::launch_fft_conv(p->packing, p->fft_N, make_geo(p), e, f, e.jobs_per_sig * n_sig, st));
  }
  TShape ts;
  // Small cores (cfg1: 1024-sample blocks, 65 taps): a job's core is shorter than the tiled
  // kernel's per-job pipeline latency, so one CTA per block (phases in sequence) is faster
  // (measured 2x at N = 64 for 65k..1M samples; the tiled kernel wins from N = 128 at 4096).
  const bool small_core = small_core_plan(p, packs, np);
  const bool forced = forced_tiled(p);                 // tile / parts forced, literal unpack: tiled
  if (!dbg && !xc_val && !pairs && small_core && !forced && per_block_ok && p->opts.exec == PC_EXEC_FUSED)
    return cuda_status(pc::launch_fused(launch_pack, make_geo(p), e, nblk * n_sig, sh.threads, sh.smem, st));
  const bool tiled_ok = p->opts.exec == PC_EXEC_FUSED || p->opts.exec == PC_EXEC_TILED;
  if (!dbg && p->packing == PC_PACK_ADAPTIVE && tiled_ok && n_sig == 1 && b0 == p->adapt_b0 &&
      b0 + nblk == p->adapt_b1 && p->d_lists) {
    // a8 -> a2..a7: one tiled launch per packing over its block list (pc_adapt_lists)
    TShape sh3[3];
    const int order[3] = {PC_PACK_ASYM2, PC_PACK_SYM, PC_PACK_FULL};
    bool ok = true;
    for (int i = 0; i < 3; ++i) ok = ok && p->ms[order[i]].valid && tiled_shape(p, order[i], &sh3[i]);
    if (ok) {
      for (int i = 0; i < 3; ++i) {
        const int pk = order[i];
        const TShape& t = sh3[i];
        Exec el = e;
        el.dec_pack = nullptr;
        el.blk_peak = p->d_peak;                        // a2 done by pc_block_stats (same max|x|)
        el.peak_stride = 0;
        el.early_fill = 0;
        el.blk_list = p->d_lists + (size_t)pk * p->P;
        el.blk_count = p->d_counts + pk;
        el.sm_ctr = p->d_counter;
        el.dbg_timing = timing;
        el.G = t.G;
        el.nstages = t.nstages;
        el.KC = t.KC;
        el.nchunks = t.nchunks;
        el.taps_resident = t.taps_resident;
        el.raw_slots = t.raw_slots;
        el.raw_stride = t.raw_stride;
        el.rows_s = t.rows_s;
        el.tiles0 = t.tiles0;
        el.tiles1 = t.tiles1;
        el.jobs_per_sig = (b0 == 0 ? t.tiles0 + (nblk - 1) * t.tiles1 : nblk * t.tiles1);   // upper bound: grid size
        el.mp[pk].K_pad = t.K_pad;
        int grid = 0;
        cudaError_t err = pc::launch_tiled(pk, t.T, t.mma, make_geo(p), el, el.jobs_per_sig, t.threads, t.smem, st, &grid);
        if (err != cudaSuccess) return PC_E_CUDA;
        record_out(p->device, st, (uintptr_t)(r - r_off - p->N), (uintptr_t)(r - r_off + p->L + 2 * p->N));
        if (grid_out) *grid_out = grid;
      }
      return PC_OK;
    }
  }
  if (!dbg && p->packing != PC_PACK_ADAPTIVE && (tiled_ok || pairs) && tiled_shape(p, p->packing, &ts, pairs)) {
    if (pairs) {
      e.kr_sig = p->d_pk_taps;
      e.kr_stride = ((long long)p->ms[p->packing].K + 33) & ~1LL;   // as conv_plan_set_kernels
      e.scal_sig = p->d_pk_scal;
    }
    e.sm_ctr = p->d_counter + (p->ctr_flip ? pc::kCtrDone + 1 : 0);   // alternate: see early_fill
    p->ctr_flip ^= 1;
    e.dbg_timing = timing;
    e.lookahead = p->opts.stage_cap < 0 ? -p->opts.stage_cap : 0;   // diagnostics
    e.xc_val = xc_val;
    e.xc_lag = xc_lag;
    e.G = ts.G;
    e.nstages = ts.nstages;
    e.KC = ts.KC;
    e.nchunks = ts.nchunks;
    e.taps_resident = ts.taps_resident;
    e.raw_slots = e.lookahead > 0 ? 0 : ts.raw_slots;   // (the claim-ahead diagnostics use the warp producers)
    e.raw_stride = ts.raw_stride;
    e.rows_s = ts.rows_s;
    e.tiles0 = ts.tiles0;
    e.tiles1 = ts.tiles1;
    e.jobs_per_sig = (b0 == 0) ? ts.tiles0 + (nblk - 1) * ts.tiles1 : nblk * ts.tiles1;
    e.mp[p->packing].K_pad = ts.K_pad;
    const long long njobs = e.jobs_per_sig * n_sig;
    // a2-a4 ahead of the DMMA-core launch (single-chunk packed plans, opts.prepack = 1): measured
    // slower than the fused producers at cfg2 (the separate pass costs ~26 us, the persistent
    // kernel's tail does not shrink), so off by default
    const bool split = ts.nchunks == 1 && p->packing != PC_PACK_FULL && p->opts.prepack < 0 && !pairs;
    if (ts.nchunks == 1 && p->packing != PC_PACK_FULL && (p->opts.prepack == 1 || split) &&
        (long long)p->W_block * 8 <= 200 * 1024) {
      const long long stride = ((long long)(ts.T + (ts.mma ? 4 : 1)) * ts.rows_s + 1) & ~1LL;   // stage_x of pc_tiled_kernel
      const long long nflag = (njobs + 1) / 2;        // doubles holding the u32 ready flags
      const long long need = njobs * stride + njobs + nflag;
      if (need > p->pre_cap) {
        cudaFree(p->d_pre);
        p->d_pre = nullptr;
        p->pre_cap = 0;
        if (cudaMalloc(&p->d_pre, sizeof(double) * need) != cudaSuccess) return PC_E_CUDA;
        if (cudaMemsetAsync(p->d_pre + njobs * stride + njobs, 0, sizeof(double) * nflag, st) != cudaSuccess)
          return PC_E_CUDA;
        p->pre_cap = need;
        p->pre_flags_jobs = njobs;
      }
      e.pre_win = p->d_pre;
      e.pre_stride = stride;
      e.pre_inv = p->d_pre + njobs * stride;
      if (split) {
        e.split_P = std::min(-p->opts.prepack, 64);
        e.split_flags = reinterpret_cast<unsigned*>(p->d_pre + njobs * stride + njobs);
        e.split_ctl = p->d_counter + 2 * (pc::kCtrDone + 1);
        if (p->pre_flags_jobs != njobs) {              // flag array re-laid for this job count: zero it and the epoch
          if (cudaMemsetAsync(e.split_flags, 0, sizeof(unsigned) * njobs, st) != cudaSuccess ||
              cudaMemsetAsync(e.split_ctl, 0, sizeof(unsigned), st) != cudaSuccess)
            return PC_E_CUDA;
          p->pre_flags_jobs = njobs;
        }
      } else {
        if (pc::launch_prepack(p->packing, ts.T, ts.mma, make_geo(p), e, njobs, st) != cudaSuccess) return PC_E_CUDA;
        e.raw_slots = 0;                               // the producers only move prepacked windows
      }
    }
    // a2 ahead (PC_PEAK_AHEAD builds): the block peaks of this launch's blocks in one bandwidth-bound
    // pass, so the producers only compand and pack (their peak pass runs 3-6x slower next to the
    // DMMA warps).  Peaks for free: adaptive plans (pc_block_stats), below.
#ifndef PC_PEAK_AHEAD
#define PC_PEAK_AHEAD 0   // measured: the extra pass costs more per step (cfg2 asym2 100.6 vs 95.1 us) than it
#endif                    // saves in the persistent kernel (89.3 vs 92.6 us); adaptive plans reuse pc_block_stats'
    if (PC_PEAK_AHEAD && p->packing != PC_PACK_FULL && !e.pre_win) {
      const long long need = n_sig * p->P;
      if (need > p->blkpeak_cap) {
        cudaFree(p->d_blkpeak);
        p->d_blkpeak = nullptr;
        p->blkpeak_cap = 0;
        if (cudaMalloc(&p->d_blkpeak, sizeof(double) * need) != cudaSuccess) return PC_E_CUDA;
        p->blkpeak_cap = need;
      }
      if (pc::launch_block_peak(make_geo(p), s, s_off, s_stride, b0, nblk, n_sig, p->d_blkpeak, p->P, st) !=
          cudaSuccess)
        return PC_E_CUDA;
      e.blk_peak = p->d_blkpeak;
      e.peak_stride = p->P;
    }
    // every address this launch may read as input / write as output (rows sig < n_sig)
    const uintptr_t in_lo = (uintptr_t)(s - s_off), in_hi = (uintptr_t)(s - s_off + (n_sig - 1) * s_stride + p->L);
    const uintptr_t out_lo = (uintptr_t)(r - r_off - p->N), out_hi = (uintptr_t)(r - r_off + (n_sig - 1) * r_stride + p->L + 2 * p->N);
    e.early_fill = !timing && !e.pre_win && !e.blk_peak && early_fill_ok(p, st, in_lo, in_hi);
    e.early_claim = 1;                                 // claims touch only this launch's queue array
    int grid = 0;
    cudaError_t err = pc::launch_tiled(p->packing, ts.T, ts.mma, make_geo(p), e, njobs, ts.threads, ts.smem, st, &grid);
    record_out(p->device, st, out_lo, out_hi);
    if (err != cudaSuccess) return PC_E_CUDA;
    if (grid_out) *grid_out = grid;
    return PC_OK;
  }
  if (pairs || xc_val) return PC_E_CONFIG;  // per-pair taps / fused scores exist only in the tiled kernel
  if (!per_block_ok) return PC_E_CONFIG;   // debug dumps / adaptive need the per-block kernel
  return cuda_status(pc::launch_fused(launch_pack, make_geo(p), e, nblk * n_sig, sh.threads, sh.smem, st));
}

// Status of an enqueue that succeeded: the sticky flags completed launches of the plan raised in
// host-mapped memory (read without synchronizing).
int plan_flags(const conv_plan* p, int rc) {
  if (rc != PC_OK || !p->h_status) return rc;
  if (reinterpret_cast<volatile int*>(p->h_status)[pc::kStatusWatchdog]) return PC_E_WATCHDOG;
  if (reinterpret_cast<volatile int*>(p->h_status)[pc::kStatusMargin]) return PC_W_UNPACK_MARGIN;
  return PC_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void conv_opts_default(conv_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->eps_rule = PC_EPS_POW2;
  o->rmax_rule = PC_RMAX_PAPER;
  o->bound_policy = PC_BOUND_STRICT;
  o->core = PC_CORE_DIRECT;
  o->exec = PC_EXEC_FUSED;
  o->K_q = 0;
  o->device = -1;
  o->u_sys = 3.1193e-11;
}

const char* conv_status_string(int s) {
  switch (s) {
    case PC_OK: return "ok";
    case PC_E_CONFIG: return "config error";
    case PC_E_BOUND: return "companding range exceeds the packing bound";
    case PC_E_BACKEND: return "backend validation failure";
    case PC_E_CUDA: return "CUDA error";
    case PC_W_UNPACK_MARGIN: return "unpack margin warning";
    case PC_E_STATE: return "invalid call order";
    case PC_E_WATCHDOG: return "kernel watchdog timeout (launch abandoned)";
  }
  return "unknown status";
}

int conv_plan_create(conv_plan** out, int64_t L, int32_t N, int32_t W_block, int32_t mode, int32_t packing,
                     int32_t Q, const conv_opts* opts) {
  if (!out) return PC_E_CONFIG;
  *out = nullptr;
  if (L < 1 || N < 1 || W_block < 4) return PC_E_CONFIG;
  if (mode != PC_MODE_CONV && mode != PC_MODE_XCORR) return PC_E_CONFIG;
  if (packing < PC_PACK_FULL || packing > PC_PACK_ADAPTIVE) return PC_E_CONFIG;
  if (packing != PC_PACK_FULL && packing != PC_PACK_ADAPTIVE && Q < 1) return PC_E_CONFIG;
  if (mode == PC_MODE_XCORR && L < N) return PC_E_CONFIG;
  conv_opts o;
  conv_opts_default(&o);
  if (opts) o = *opts;
  if (o.core != PC_CORE_DIRECT && o.core != PC_CORE_FFT) return PC_E_CONFIG;
  if (o.core == PC_CORE_FFT && packing == PC_PACK_ADAPTIVE) return PC_E_CONFIG;
  const int Np = (N % 2) ? N : N + 1;                 // P:45, C13
  const long long W = (long long)W_block - Np - 1;
  if (W < 2 || (W % 2) || W < 2LL * Np) return PC_E_CONFIG;
  int dev = o.device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) return PC_E_CUDA;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1 || dev >= ndev) return PC_E_CUDA;
  if (cudaSetDevice(dev) != cudaSuccess) return PC_E_CUDA;
  conv_plan* p = new (std::nothrow) conv_plan();
  if (!p) return PC_E_CUDA;
  p->L = L;
  p->N = N;
  p->Np = Np;
  p->W_block = W_block;
  p->W = (int)W;
  p->P = (L + W - 1) / W;                             // P = ceil(L / W)
  p->mode = mode;
  p->packing = packing;
  p->Q = Q;
  p->K_q = o.K_q > 0 ? o.K_q : Q;
  p->opts = o;
  p->device = dev;
  cudaError_t e = cudaSuccess;
  e = cudaMalloc(&p->d_k_pad, sizeof(double) * Np);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_k_int, sizeof(double) * Np);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_scal, sizeof(double) * 4);
  // two arrays of queue counters (alternating launches) + the producer-SM mode's epoch
  if (e == cudaSuccess) e = cudaMalloc(&p->d_counter, (2 * (pc::kCtrDone + 1) + 8) * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(p->d_counter, 0, (2 * (pc::kCtrDone + 1) + 8) * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaHostAlloc(&p->h_status, 4 * sizeof(int), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    std::memset(p->h_status, 0, 4 * sizeof(int));
    e = cudaHostGetDevicePointer(&p->d_status, p->h_status, 0);
  }
  if (e != cudaSuccess) {
    conv_plan_destroy(p);
    return PC_E_CUDA;
  }
  // shared-memory feasibility: the tiled kernel (production) or, for adaptive plans, the
  // per-block kernel (which also serves conv_execute_debug when it fits)
  int packs[4];
  const int np = plan_packs(p, packs);
  for (int i = 0; i < np; ++i) set_core_layout(p, packs[i], &p->ms[packs[i]]);
  Shape sh;
  TShape ts;
  bool ok;
  if (o.core == PC_CORE_FFT) {
    p->fft_N = choose_fft_N(p, packing);
    FShape fs;
    ok = p->fft_N > 0 && fft_shape(p, packing, p->fft_N, &fs);
    if (ok) {
      // twiddle tables, rounded once from long double (recurrences are too inexact)
      const int N = p->fft_N;
      double2* tw = (double2*)std::malloc(sizeof(double2) * N);
      double2* tw2 = (double2*)std::malloc(sizeof(double2) * (N + 1));
      const long double two_pi = 6.283185307179586476925286766559005768L;
      for (int m = 0; m < N; ++m) {
        const long double a = two_pi * (long double)m / (long double)N;
        tw[m] = make_double2((double)cosl(a), (double)(-sinl(a)));
      }
      for (int k = 0; k <= N; ++k) {
        const long double a = two_pi * (long double)k / (long double)(2 * N);
        tw2[k] = make_double2((double)cosl(a), (double)(-sinl(a)));
      }
      cudaError_t err = cudaMalloc(&p->d_tw, sizeof(double2) * N);
      if (err == cudaSuccess) err = cudaMalloc(&p->d_tw2, sizeof(double2) * (N + 1));
      if (err == cudaSuccess) err = cudaMalloc(&p->d_H, sizeof(double2) * (N + 1));
      if (err == cudaSuccess) err = cudaMalloc(&p->d_resid, sizeof(double));
      if (err == cudaSuccess) err = cudaMemcpy(p->d_tw, tw, sizeof(double2) * N, cudaMemcpyHostToDevice);
      if (err == cudaSuccess) err = cudaMemcpy(p->d_tw2, tw2, sizeof(double2) * (N + 1), cudaMemcpyHostToDevice);
      if (err == cudaSuccess) err = cudaMemset(p->d_resid, 0, sizeof(double));
      std::free(tw);
      std::free(tw2);
      if (err != cudaSuccess) {
        conv_plan_destroy(p);
        return PC_E_CUDA;
      }
    }
  } else {
    ok = (packing == PC_PACK_ADAPTIVE) ? launch_shape(p, packs, np, &sh) : tiled_shape(p, packing, &ts);
  }
  if (!ok) {
    conv_plan_destroy(p);
    return PC_E_CONFIG;
  }
  *out = p;
  return PC_OK;
}

void conv_plan_destroy(conv_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  for (auto& m : p->ms)
    if (m.kr) cudaFree(m.kr - 16);
  cudaFree(p->d_k_pad);
  cudaFree(p->d_k_int);
  cudaFree(p->d_scal);
  cudaFree(p->d_dec_pack);
  cudaFree(p->d_dec_q);
  cudaFree(p->d_dec_snr);
  cudaFree(p->d_lists);
  cudaFree(p->d_counts);
  cudaFree(p->d_sigma);
  cudaFree(p->d_peak);
  cudaFree(p->d_cand);
  cudaFree(p->d_in);
  cudaFree(p->d_out);
  cudaFree(p->d_xc_pval);
  cudaFree(p->d_xc_plag);
  cudaFree(p->d_pk_pad);
  cudaFree(p->d_pk_int);
  cudaFree(p->d_pk_scal);
  if (p->d_pk_taps) cudaFree(p->d_pk_taps - 16);
  for (int i = 0; i < 16; ++i) {
    if (p->ev_in[i]) cudaEventDestroy(p->ev_in[i]);
    if (p->ev_done[i]) cudaEventDestroy(p->ev_done[i]);
  }
  if (p->ev_out) cudaEventDestroy(p->ev_out);
  if (p->st_h2d) cudaStreamDestroy(p->st_h2d);
  if (p->st_d2h) cudaStreamDestroy(p->st_d2h);
  cudaFree(p->d_xc);
  cudaFree(p->d_counter);
  cudaFree(p->d_pre);
  cudaFree(p->d_tw);
  cudaFree(p->d_tw2);
  cudaFree(p->d_H);
  cudaFree(p->d_resid);
  cudaFree(p->d_dbg_resid);
  cudaFree(p->d_blkpeak);
  if (p->h_status) cudaFreeHost(p->h_status);
  delete p;
}

}  // extern "C"

namespace {

// Initialization of one packing at S_q = Q, K_q: k~, R_max, eps, bound, core taps.
int init_mode(conv_plan* p, int packing, int Q, int K_q, const double* k_dev, cudaStream_t st) {
  ModeState& m = p->ms[packing];
  set_core_layout(p, packing, &m);
  double scal[4] = {0, 0, 0, 0};
  cudaError_t e = pc::launch_kernel_prep(k_dev, p->N, p->Np, p->mode == PC_MODE_XCORR, (double)K_q, p->d_k_pad,
                                         p->d_k_int, p->d_scal, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(scal, p->d_scal, sizeof(double) * 3, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return PC_E_CUDA;
  p->k_peak = scal[0];
  m.Q = Q;
  m.K_q = K_q;
  if (packing == PC_PACK_FULL) {
    m.c_k = 1.0;
    m.R = 0;
    m.bound = 0;
    m.bound_ok = 1;
    m.eps = m.eps_inv = 0.0;
    m.b = 0;
  } else {
    m.c_k = scal[1];
    const long long l1 = (long long)scal[2];
    long long R = (p->opts.rmax_rule == PC_RMAX_L1) ? (long long)Q * l1 : (long long)p->Np * Q * (long long)K_q;
    if (R < 1) R = 1;
    m.R = R;
    if (p->opts.eps_rule == PC_EPS_PAPER) {
      m.eps_inv = 2.0 * (double)R;            // Eq. (6)
      m.eps = 1.0 / m.eps_inv;
      m.b = 0;
    } else if (p->opts.eps_rule == PC_EPS_RADIX) {
      m.eps_inv = 2.0 * (double)R + 1.0;      // reading C2
      m.eps = 1.0 / m.eps_inv;
      m.b = 0;
    } else {
      m.b = 64 - __builtin_clzll((unsigned long long)(2 * R));   // reading C4
      m.eps_inv = std::ldexp(1.0, m.b);
      m.eps = std::ldexp(1.0, -m.b);
    }
    m.bound = bound_for(packing, p->opts.eps_rule);
    m.bound_ok = R <= m.bound;
    if (!m.bound_ok && p->opts.bound_policy == PC_BOUND_STRICT) return PC_E_BOUND;
  }
  const int kr_len = m.K + 32;   // zero taps past K serve every tile padding (8..16)
  if (!m.kr) {                   // + 16 leading zeros (the DMMA core's Toeplitz fragments read kr[-15..])
    double* buf = nullptr;
    if (cudaMalloc(&buf, sizeof(double) * (kr_len + 16)) != cudaSuccess) return PC_E_CUDA;
    if (cudaMemsetAsync(buf, 0, sizeof(double) * 16, st) != cudaSuccess) return PC_E_CUDA;
    m.kr = buf + 16;
  }
  e = pc::launch_build_taps(p->d_k_pad, p->d_k_int, p->Np, packing, m.eps_inv, m.K, kr_len, m.kr, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return PC_E_CUDA;
  m.valid = 1;
  return PC_OK;
}

// R_max(Q) for the L1 rule needs k~ at each Q: evaluated with the prep kernel.
int l1_at(conv_plan* p, int Q, const double* k_dev, cudaStream_t st, long long* l1) {
  double scal[4];
  cudaError_t e = pc::launch_kernel_prep(k_dev, p->N, p->Np, p->mode == PC_MODE_XCORR, (double)Q, p->d_k_pad,
                                         p->d_k_int, p->d_scal, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(scal, p->d_scal, sizeof(double) * 3, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return PC_E_CUDA;
  *l1 = (long long)scal[2];
  return PC_OK;
}

// Largest tied Q = S_q = K_q whose R_max meets the packing's bound.
int max_q(conv_plan* p, int packing, const double* k_dev, cudaStream_t st, int* q_out) {
  const long long bound = bound_for(packing, p->opts.eps_rule);
  int lo = 0, hi = 1 << 15;
  while (lo < hi) {
    const int mid = lo + (hi - lo + 1) / 2;
    long long R;
    if (p->opts.rmax_rule == PC_RMAX_L1) {
      long long l1;
      int rc = l1_at(p, mid, k_dev, st, &l1);
      if (rc) return rc;
      R = (long long)mid * l1;
    } else {
      R = (long long)p->Np * mid * (long long)mid;
    }
    if (R <= bound) lo = mid; else hi = mid - 1;
  }
  *q_out = lo;
  return PC_OK;
}

// Backend validation of an FFT-core plan (P:103, P:153 u_sys): the plan's own
// FFT kernel on worst-case operand windows -- every sample +-1 with random signs, so every packed
// digit is +-S_q, convolved with the installed kernel k~ -- over the first blocks of the plan's
// geometry until `trials` jobs (transform windows) ran; the kernels' last-digit residual monitor
// gives the worst deviation d (LSB) from the exact integers.  u_sys_cal = 4 d x the unit of the
// last digit in the packed word (eps for symmetric and asym2, eps^2 for asym3).
int validate_fft_backend(conv_plan* p, cudaStream_t st) {
  FShape fs;
  if (!fft_shape(p, p->packing, p->fft_N, &fs)) return PC_E_CONFIG;
  const long long trials = p->opts.validate_trials > 0 ? p->opts.validate_trials : 128;
  long long nb = 1, jobs = fs.parts0;
  while (jobs < trials && nb < p->P) {
    ++nb;
    jobs += fs.parts1;
  }
  long long in_len = (nb - 1 == 0 ? 0 : (nb - 1) * (long long)p->W - 2) + p->W_block;
  if (in_len > p->L) in_len = p->L;
  const long long out_len = (long long)p->Np - 1 + nb * (long long)p->W + p->N;
  double *x = nullptr, *y = nullptr;
  cudaError_t e = cudaMalloc(&x, sizeof(double) * in_len);
  if (e == cudaSuccess) e = cudaMalloc(&y, sizeof(double) * out_len);
  if (e == cudaSuccess) e = pc::launch_fill_pm1(x, in_len, 0x5eed0000ull + (unsigned long long)p->Np, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p->d_resid, 0, sizeof(double), st);
  int rc = e == cudaSuccess ? PC_OK : PC_E_CUDA;
  if (!rc) rc = run_exec(p, x, 0, 0, y, 0, 0, 0, nb, 1, nullptr, st);
  double d = 0.0;
  if (!rc) {
    e = cudaMemcpyAsync(&d, p->d_resid, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_resid, 0, sizeof(double), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = PC_E_CUDA;
  }
  cudaFree(x);
  cudaFree(y);
  if (rc) return rc;
  reinterpret_cast<volatile int*>(p->h_status)[pc::kStatusMargin] = 0;   // the validation's own flag
  const ModeState& m = p->ms[p->packing];
  const int last = p->packing == PC_PACK_ASYM3 ? 2 : 1;                  // power of eps of the last digit
  p->backend_resid = d;
  p->u_sys_cal = 4.0 * d * std::pow(m.eps, (double)last);
  p->backend_ok = 4.0 * d <= 0.5 ? 1 : 0;
  return PC_OK;
}

}  // namespace

extern "C" {

int conv_plan_set_kernel(conv_plan* p, const double* k_dev, void* stream) {
  if (!p || !k_dev) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  p->kernel_set = 0;
  p->adapt_ready = 0;
  p->cand_ok = 0;
  int rc;
  if (p->packing == PC_PACK_ADAPTIVE) {
    const int cands[2] = {PC_PACK_SYM, PC_PACK_ASYM2};
    for (int c : cands) {
      int q;
      if ((rc = max_q(p, c, k_dev, st, &q))) return rc;
      p->qmode[c] = q;
      if (q >= 1) {
        if ((rc = init_mode(p, c, q, q, k_dev, st))) return rc;
      } else {
        p->ms[c].valid = 0;
      }
    }
    if ((rc = init_mode(p, PC_PACK_FULL, 0, 1, k_dev, st))) return rc;
    // sigma_k, ||k||_inf (reading C12), on the padded kernel
    Geo g;
    std::memset(&g, 0, sizeof(g));
    g.L = p->Np;
    g.P = 1;
    g.W_block = p->Np;
    g.W = p->Np;
    double* d_sk = nullptr;
    if (cudaMalloc(&d_sk, 2 * sizeof(double)) != cudaSuccess) return PC_E_CUDA;
    cudaError_t e = pc::launch_block_stats(g, p->d_k_pad, d_sk, d_sk + 1, st);
    double hk[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(hk, d_sk, sizeof(hk), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_sk);
    if (e != cudaSuccess) return PC_E_CUDA;
    p->k_sigma = hk[0];
    p->k_peak = hk[1];
  } else {
    if ((rc = init_mode(p, p->packing, p->Q, p->K_q, k_dev, st))) return rc;
    if (p->opts.core == PC_CORE_FFT) {
      const ModeState& m = p->ms[p->packing];
      cudaError_t e = pc::launch_fft_spectrum(p->fft_N, m.kr, m.K, p->d_tw, p->d_tw2, p->d_H, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return PC_E_CUDA;
      p->backend_ok = -1;
      p->backend_resid = p->u_sys_cal = 0.0;
      if (p->packing != PC_PACK_FULL) {                // validate the FFT regime
        p->kernel_set = 1;                             // (run_exec needs an installed kernel)
        rc = validate_fft_backend(p, st);
        p->kernel_set = 0;
        if (rc) return rc;
        if (!p->backend_ok && p->opts.bound_policy == PC_BOUND_STRICT) return PC_E_BACKEND;
      }
    }
  }
  p->kernel_set = 1;
  return PC_OK;
}

int conv_execute(conv_plan* p, const double* s, double* r, void* stream) {
  if (!p || !s || !r) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  return plan_flags(p, run_exec(p, s, 0, 0, r, 0, 0, 0, p->P, 1, nullptr, (cudaStream_t)stream));
}

int conv_execute_blocks(conv_plan* p, const double* s, int64_t s_offset, double* r, int64_t r_offset,
                        int64_t block_begin, int64_t block_end, void* stream) {
  if (!p || !s || !r) return PC_E_CONFIG;
  if (block_begin < 0 || block_end > p->P || block_begin > block_end) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  return plan_flags(p, run_exec(p, s, s_offset, 0, r, r_offset, 0, block_begin, block_end - block_begin, 1,
                                nullptr, (cudaStream_t)stream));
}

int conv_execute_batch(conv_plan* p, const double* s, int64_t n_signals, int64_t s_stride, double* r,
                       int64_t r_stride, void* stream) {
  if (!p || !s || !r || n_signals < 0) return PC_E_CONFIG;
  if (p->packing == PC_PACK_ADAPTIVE && n_signals > 1) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  return plan_flags(p, run_exec(p, s, 0, s_stride, r, 0, r_stride, 0, p->P, n_signals, nullptr, (cudaStream_t)stream));
}

int conv_execute_host(conv_plan* p, const double* s_host, double* r_host, void* stream) {
  if (!p) return PC_E_CONFIG;
  return conv_execute_host_blocks(p, s_host, 0, r_host, 0, 0, p->P, stream);
}

int conv_execute_host_blocks(conv_plan* p, const double* s_host, int64_t s_offset, double* r_host, int64_t r_offset,
                             int64_t B0, int64_t B1, void* stream) {
  if (!p || !s_host || !r_host) return PC_E_CONFIG;
  if (B0 < 0 || B1 > p->P || B0 > B1) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  if (B0 == B1) return PC_OK;
  if (p->packing == PC_PACK_ADAPTIVE && (B0 != 0 || B1 != p->P)) return PC_E_CONFIG;   // decisions: whole input
  cudaStream_t st = (cudaStream_t)stream;
  const long long L_out = p->mode == PC_MODE_XCORR ? p->L - p->N + 1 : p->L + p->N - 1;
  // device buffers addressed by global sample / output index (a shard uses its own range)
  if (!p->d_in && cudaMalloc(&p->d_in, sizeof(double) * p->L) != cudaSuccess) return PC_E_CUDA;
  if (!p->d_out && cudaMalloc(&p->d_out, sizeof(double) * L_out) != cudaSuccess) return PC_E_CUDA;
  // input read by blocks [B0, b1) and outputs written by them (reading C7, Eq. (17)), as
  // conv_shard_range
  const long long W = p->W, Wb = p->W_block, Np = p->Np;
  auto in_end_of = [&](long long b1) {
    const long long last = b1 - 1;
    const long long e = (last == 0 ? 0 : last * W - 2) + Wb;
    return e < p->L ? e : p->L;
  };
  auto out_end_of = [&](long long b1) {
    long long o = (b1 == p->P) ? p->L + p->N - 1 : Np - 1 + b1 * W;
    if (o > p->L + p->N - 1) o = p->L + p->N - 1;
    if (p->mode == PC_MODE_XCORR) {                                   // lag j = gg - (N-1)
      const long long lo = p->N - 1, hi = p->L;
      o = (o < lo ? lo : (o > hi ? hi : o)) - lo;
    }
    return o;
  };
  const long long in_begin = B0 == 0 ? 0 : B0 * W - 2;
  const long long out_begin = B0 == 0 ? 0 : out_end_of(B0);
  // Adaptive plans (decisions belong to one device input) and small ranges: one pass.
  // Chunk weights: small first and last ranges shorten the pipeline ramp (the first H2D and
  // the last D2H are not overlapped).  (Zero-copy was measured and dropped: the tiled kernel
  // reading pinned input over PCIe took 2.1 ms at cfg2 -- the peak and packing passes read each
  // sample twice over the link -- and storing outputs straight to pinned memory 1.07-1.36 ms,
  // against 1.04 ms for this copy pipeline; the link's duplex floor is 0.71 ms.)
  // (15 ranges 1:1:2:..:2:1:1 measured 0.98-1.00 ms at cfg2 against 1.04-1.05 for 1:2:4:4:4:4:4:2:1
  // and 1.01-1.02 for 16 equal ranges; round 2, another box: 1.04 ms against 1.03 for 1:2:3:3:2:1,
  // 1.03 for 1:3:3:1, 1.07 for 1:2:..:2:1 (8), 1.12 for 12 equal -- the copy engines' duplex floor
  // for the 64 MB is 0.71 ms, profiles/r02/pcie_e2e.log)
  static const int kW[] = {1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 1, 1};
  constexpr int kNW = (int)(sizeof(kW) / sizeof(kW[0]));
  static_assert(kNW <= 16, "event pairs");
  const int nchunk = (p->packing == PC_PACK_ADAPTIVE || B1 - B0 < 128) ? 1 : kNW;
  long long cum[17] = {0};
  for (int i = 0; i < kNW; ++i) cum[i + 1] = cum[i] + kW[i];
  const long long nb = B1 - B0;
  if (nchunk <= 1) {
    const long long i1 = in_end_of(B1), o1 = out_end_of(B1);
    if (cudaMemcpyAsync(p->d_in + in_begin, s_host + (in_begin - s_offset), sizeof(double) * (i1 - in_begin),
                        cudaMemcpyHostToDevice, st) != cudaSuccess)
      return PC_E_CUDA;
    int rc = run_exec(p, p->d_in, 0, 0, p->d_out, 0, 0, B0, nb, 1, nullptr, st);
    if (rc) return rc;
    if (o1 > out_begin && cudaMemcpyAsync(r_host + (out_begin - r_offset), p->d_out + out_begin,
                                          sizeof(double) * (o1 - out_begin), cudaMemcpyDeviceToHost,
                                          st) != cudaSuccess)
      return PC_E_CUDA;
    return plan_flags(p, cuda_status(cudaStreamSynchronize(st)));
  }
  // Pipeline over block ranges: the H2D of chunk c+1, the core of chunk c and the D2H of
  // chunk c-1 overlap (two copy engines + the SMs).  Each input sample and each output is
  // copied once; block ranges, halos and output ranges follow Eq. (17) (reading C7).
  if (!p->st_h2d) {
    if (cudaStreamCreateWithFlags(&p->st_h2d, cudaStreamNonBlocking) != cudaSuccess) return PC_E_CUDA;
    if (cudaStreamCreateWithFlags(&p->st_d2h, cudaStreamNonBlocking) != cudaSuccess) return PC_E_CUDA;
    for (int i = 0; i < 16; ++i) {
      if (cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming) != cudaSuccess) return PC_E_CUDA;
      if (cudaEventCreateWithFlags(&p->ev_done[i], cudaEventDisableTiming) != cudaSuccess) return PC_E_CUDA;
    }
    if (cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming) != cudaSuccess) return PC_E_CUDA;
  }
  cudaError_t e = cudaEventRecord(p->ev_out, st);                    // stream order before the call
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->st_h2d, p->ev_out, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->st_d2h, p->ev_out, 0);
  if (e != cudaSuccess) return PC_E_CUDA;
  long long in_done = in_begin, out_done = out_begin;
  for (int c = 0; c < nchunk; ++c) {
    const long long b0 = B0 + nb * cum[c] / cum[nchunk], b1 = B0 + nb * cum[c + 1] / cum[nchunk];
    if (b1 <= b0) continue;
    const long long in_end = in_end_of(b1), out_end = out_end_of(b1);
    if (in_end > in_done) {
      e = cudaMemcpyAsync(p->d_in + in_done, s_host + (in_done - s_offset), sizeof(double) * (in_end - in_done),
                          cudaMemcpyHostToDevice, p->st_h2d);
      if (e != cudaSuccess) return PC_E_CUDA;
      in_done = in_end;
    }
    if ((e = cudaEventRecord(p->ev_in[c], p->st_h2d)) != cudaSuccess) return PC_E_CUDA;
    if ((e = cudaStreamWaitEvent(st, p->ev_in[c], 0)) != cudaSuccess) return PC_E_CUDA;
    const int rc = run_exec(p, p->d_in, 0, 0, p->d_out, 0, 0, b0, b1 - b0, 1, nullptr, st);
    if (rc) return rc;
    if ((e = cudaEventRecord(p->ev_done[c], st)) != cudaSuccess) return PC_E_CUDA;
    if ((e = cudaStreamWaitEvent(p->st_d2h, p->ev_done[c], 0)) != cudaSuccess) return PC_E_CUDA;
    if (out_end > out_done) {
      e = cudaMemcpyAsync(r_host + (out_done - r_offset), p->d_out + out_done, sizeof(double) * (out_end - out_done),
                          cudaMemcpyDeviceToHost, p->st_d2h);
      if (e != cudaSuccess) return PC_E_CUDA;
      out_done = out_end;
    }
  }
  if (out_done != out_end_of(B1)) return PC_E_CONFIG;   // geometry bug guard
  if ((e = cudaEventRecord(p->ev_out, p->st_d2h)) != cudaSuccess) return PC_E_CUDA;
  if ((e = cudaStreamWaitEvent(st, p->ev_out, 0)) != cudaSuccess) return PC_E_CUDA;
  return plan_flags(p, cuda_status(cudaStreamSynchronize(st)));
}

int conv_execute_debug(conv_plan* p, const double* s, double* r, double* packed, double* rbar, int64_t* rint,
                       double* c_s, double* max_residual, void* stream) {
  if (!p || !s) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  if (max_residual) {
    if (!p->d_dbg_resid && cudaMalloc(&p->d_dbg_resid, sizeof(double)) != cudaSuccess) return PC_E_CUDA;
    if (cudaMemsetAsync(p->d_dbg_resid, 0, sizeof(double), st) != cudaSuccess) return PC_E_CUDA;
  }
  conv_plan_info info;
  conv_plan_query(p, &info);
  Exec d;
  std::memset(&d, 0, sizeof(d));
  d.dbg_packed = packed;
  d.dbg_packed_stride = info.packed_stride;
  d.dbg_rbar = rbar;
  d.dbg_rbar_stride = info.rbar_stride;
  d.dbg_rint = reinterpret_cast<long long*>(rint);
  d.dbg_rint_stride = info.rint_stride;
  d.dbg_cs = c_s;
  d.dbg_resid = max_residual ? p->d_dbg_resid : nullptr;
  const int rc = run_exec(p, s, 0, 0, r, 0, 0, 0, p->P, 1, &d, st);
  if (rc || !max_residual) return rc;
  if (cudaMemcpyAsync(max_residual, p->d_dbg_resid, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return PC_E_CUDA;
  return cuda_status(cudaStreamSynchronize(st));
}

int conv_plan_set_kernels(conv_plan* p, const double* q_dev, int64_t n, int64_t q_stride, void* stream) {
  if (!p || !q_dev || n < 1 || q_stride < p->N) return PC_E_CONFIG;
  if (p->packing == PC_PACK_ADAPTIVE || p->opts.core != PC_CORE_DIRECT) return PC_E_CONFIG;
  if (p->packing != PC_PACK_FULL && p->opts.rmax_rule != PC_RMAX_PAPER) return PC_E_CONFIG;   // pair-independent eps
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  // the packing state (R_max = N' S_q K_q, eps, bound, taps layout) from the first kernel
  int rc = conv_plan_set_kernel(p, q_dev, stream);
  if (rc) return rc;
  const ModeState& m = p->ms[p->packing];
  const long long Np = p->Np, kr_len = ((long long)m.K + 33) & ~1LL;   // rows 16-byte aligned (TMA)
  if (n > p->n_kernels) {
    cudaFree(p->d_pk_pad);
    cudaFree(p->d_pk_int);
    cudaFree(p->d_pk_scal);
    if (p->d_pk_taps) cudaFree(p->d_pk_taps - 16);
    p->d_pk_pad = p->d_pk_int = p->d_pk_scal = p->d_pk_taps = nullptr;
    p->n_kernels = 0;
    cudaError_t e = cudaMalloc(&p->d_pk_pad, sizeof(double) * n * Np);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_pk_int, sizeof(double) * n * Np);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_pk_scal, sizeof(double) * 3 * n);
    double* tb = nullptr;                            // + 16 leading zeros, as the plan's taps
    if (e == cudaSuccess) e = cudaMalloc(&tb, sizeof(double) * (n * kr_len + 16));
    if (e == cudaSuccess) e = cudaMemsetAsync(tb, 0, sizeof(double) * 16, st);
    if (e != cudaSuccess) return PC_E_CUDA;
    p->d_pk_taps = tb + 16;
  }
  p->n_kernels = n;
  cudaError_t e = pc::launch_kernel_prep_batch(q_dev, q_stride, n, p->N, p->Np, p->mode == PC_MODE_XCORR,
                                               (double)m.K_q, p->d_pk_pad, p->d_pk_int, Np, p->d_pk_scal, st);
  if (e == cudaSuccess)
    e = pc::launch_build_taps_batch(p->d_pk_pad, p->d_pk_int, Np, p->Np, p->packing, m.eps_inv, m.K, (int)kr_len,
                                    p->d_pk_taps, kr_len, n, st);
  return cuda_status(e);
}

int conv_xcorr_pairs(conv_plan* p, const double* x_dev, int64_t n, int64_t x_stride, double* score, int64_t* lag,
                     void* stream) {
  if (!p || !x_dev || !score || !lag || n < 0 || x_stride < p->L) return PC_E_CONFIG;
  if (p->mode != PC_MODE_XCORR || n > p->n_kernels) return n > p->n_kernels ? PC_E_STATE : PC_E_CONFIG;
  if (n == 0) return PC_OK;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  TShape ts;
  if (!tiled_shape(p, p->packing, &ts, true)) return PC_E_CONFIG;
  const long long jobs_per_sig = ts.tiles0 + (p->P - 1) * ts.tiles1;
  const long long n_part = jobs_per_sig * (ts.G / 32);
  const size_t need = (size_t)n * (size_t)n_part;
  if (need > p->xc_part_n) {
    cudaFree(p->d_xc_pval);
    cudaFree(p->d_xc_plag);
    p->d_xc_pval = nullptr;
    p->d_xc_plag = nullptr;
    p->xc_part_n = 0;
    if (cudaMalloc(&p->d_xc_pval, sizeof(double) * need) != cudaSuccess) return PC_E_CUDA;
    if (cudaMalloc(&p->d_xc_plag, sizeof(long long) * need) != cudaSuccess) return PC_E_CUDA;
    p->xc_part_n = need;
  }
  const long long n_lags = p->L - p->N + 1;
  int rc = run_exec(p, x_dev, 0, x_stride, p->d_xc_pval, 0, n_lags, 0, p->P, n, nullptr, st, nullptr, nullptr,
                    p->d_xc_pval, p->d_xc_plag, true);
  if (rc) return rc;
  return plan_flags(p, cuda_status(pc::launch_xcorr_reduce(p->d_xc_pval, p->d_xc_plag, n, n_part, score,
                                                           reinterpret_cast<long long*>(lag), st)));
}

int conv_xcorr_max(conv_plan* p, const double* db, int64_t n_signals, int64_t s_stride, double* score,
                   int64_t* lag, void* stream) {
  if (!p || !db || !score || !lag || n_signals < 0) return PC_E_CONFIG;
  if (p->mode != PC_MODE_XCORR || p->packing == PC_PACK_ADAPTIVE) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n_lags = p->L - p->N + 1;
  if (uses_tiled(p) && n_signals > 0) {
    // a9 fused: the tiled kernel's epilogue keeps each warp part's max over its
    // valid lags (lowest lag on ties) instead of storing the lags; one launch over all
    // signals, then a per-signal reduction of the partials.  No lag scratch.
    TShape ts;
    tiled_shape(p, p->packing, &ts);
    const long long jobs_per_sig = ts.tiles0 + (p->P - 1) * ts.tiles1;
    const long long n_part = jobs_per_sig * (ts.G / 32);
    const size_t need = (size_t)n_signals * (size_t)n_part;
    if (need > p->xc_part_n) {
      cudaFree(p->d_xc_pval);
      cudaFree(p->d_xc_plag);
      p->d_xc_pval = nullptr;
      p->d_xc_plag = nullptr;
      p->xc_part_n = 0;
      if (cudaMalloc(&p->d_xc_pval, sizeof(double) * need) != cudaSuccess) return PC_E_CUDA;
      if (cudaMalloc(&p->d_xc_plag, sizeof(long long) * need) != cudaSuccess) return PC_E_CUDA;
      p->xc_part_n = need;
    }
    int rc = run_exec(p, db, 0, s_stride, p->d_xc_pval, 0, n_lags, 0, p->P, n_signals, nullptr, st, nullptr,
                      nullptr, p->d_xc_pval, p->d_xc_plag);
    if (rc) return rc;
    cudaError_t e = pc::launch_xcorr_reduce(p->d_xc_pval, p->d_xc_plag, n_signals, n_part, score,
                                            reinterpret_cast<long long*>(lag), st);
    return plan_flags(p, cuda_status(e));
  }
  long long chunk = (1LL << 28) / n_lags;    // <= 2 GiB of lag scratch
  if (chunk < 1) chunk = 1;
  if (chunk > n_signals) chunk = n_signals;
  const size_t need = sizeof(double) * (size_t)chunk * (size_t)n_lags;
  if (need > p->d_xc_bytes) {
    cudaFree(p->d_xc);
    p->d_xc = nullptr;
    p->d_xc_bytes = 0;
    if (cudaMalloc(&p->d_xc, need) != cudaSuccess) return PC_E_CUDA;
    p->d_xc_bytes = need;
  }
  for (long long s0 = 0; s0 < n_signals; s0 += chunk) {
    const long long n = (n_signals - s0 < chunk) ? n_signals - s0 : chunk;
    int rc = run_exec(p, db + s0 * s_stride, 0, s_stride, p->d_xc, 0, n_lags, 0, p->P, n, nullptr, st);
    if (rc) return rc;
    cudaError_t e = pc::launch_xcorr_max(p->d_xc, n, n_lags, n_lags, score + s0,
                                         reinterpret_cast<long long*>(lag) + s0, st);
    if (e != cudaSuccess) return PC_E_CUDA;
  }
  return plan_flags(p, PC_OK);
}

int conv_snr_calibrate(conv_plan* p, const double* s, const double* k, int32_t Q, double* offset_db,
                       double* measured_db, double* model_db, void* stream) {
  if (!p || !s || !k || Q < 1) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  // any exact packing gives the same integer results at S_q = K_q = Q; the plan's own if packed
  const int pk = (p->packing == PC_PACK_SYM || p->packing == PC_PACK_ASYM3) ? p->packing : PC_PACK_ASYM2;
  conv_opts o = p->opts;
  o.core = PC_CORE_DIRECT;
  conv_plan *pq = nullptr, *pf = nullptr;
  double *d_ref = nullptr, *d_x = nullptr, *d_st = nullptr;
  const long long L_out = p->mode == PC_MODE_XCORR ? p->L - p->N + 1 : p->L + p->N - 1;
  const long long P = p->P;
  int rc = conv_plan_create(&pq, p->L, p->N, p->W_block, p->mode, pk, Q, &o);
  if (!rc) rc = conv_plan_create(&pf, p->L, p->N, p->W_block, p->mode, PC_PACK_FULL, 0, &o);
  if (!rc) rc = conv_plan_set_kernel(pq, k, stream);
  if (!rc) rc = conv_plan_set_kernel(pf, k, stream);
  if (!rc && (cudaMalloc(&d_ref, sizeof(double) * L_out) != cudaSuccess ||
              cudaMalloc(&d_x, sizeof(double) * L_out) != cudaSuccess ||
              cudaMalloc(&d_st, sizeof(double) * (2 * P + 2 + 4)) != cudaSuccess))
    rc = PC_E_CUDA;
  if (!rc) rc = conv_execute(pf, s, d_ref, stream);
  if (!rc) rc = conv_execute(pq, s, d_x, stream);
  double h[6] = {0, 0, 0, 0, 0, 0};
  if (!rc) {
    // sigma_s, peak per block and sigma_k, ||k||_inf (reading C12), then the sums
    Geo gk;
    std::memset(&gk, 0, sizeof(gk));
    gk.L = pq->Np;
    gk.P = 1;
    gk.W_block = pq->Np;
    gk.W = pq->Np;
    double* d_sk = d_st + 2 * P;
    cudaError_t e = pc::launch_block_stats(make_geo(pq), s, d_st, d_st + P, st);
    if (e == cudaSuccess) e = pc::launch_block_stats(gk, pq->d_k_pad, d_sk, d_sk + 1, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d_sk, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess)
      e = pc::launch_snr_sums(d_ref, d_x, L_out, d_st, d_st + P, P, h[0], h[1], (double)Q, d_sk + 2, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h + 2, d_sk + 2, 4 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = PC_E_CUDA;
  }
  cudaFree(d_ref);
  cudaFree(d_x);
  cudaFree(d_st);
  conv_plan_destroy(pq);
  conv_plan_destroy(pf);
  if (rc) return rc;
  const double meas = h[3] == 0.0 ? INFINITY : 10.0 * std::log10(h[2] / h[3]);
  const double model = 10.0 * std::log10(h[4] / h[5]);
  if (measured_db) *measured_db = meas;
  if (model_db) *model_db = model;
  if (offset_db) *offset_db = meas - model;
  return PC_OK;
}

int conv_adapt_block(conv_plan* p, const double* s, double snr_floor_db, double calib_offset_db,
                     conv_block_decision* out, void* stream) {
  if (!p) return PC_E_CONFIG;
  return conv_adapt_blocks(p, s, 0, 0, p->P, snr_floor_db, calib_offset_db, out, stream);
}

int conv_adapt_blocks(conv_plan* p, const double* s, int64_t s_offset, int64_t B0, int64_t B1, double snr_floor_db,
                      double calib_offset_db, conv_block_decision* out, void* stream) {
  if (!p || !s) return PC_E_CONFIG;
  if (p->packing != PC_PACK_ADAPTIVE) return PC_E_CONFIG;
  if (B0 < 0 || B1 > p->P || B0 > B1) return PC_E_CONFIG;
  if (!p->kernel_set) return PC_E_STATE;
  if (B0 == B1) return PC_OK;                          // an empty shard (more ranks than blocks)
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  const long long P = p->P, nb = B1 - B0;
  cudaError_t e = cudaSuccess;
  if (!p->d_dec_pack) {
    e = cudaMalloc(&p->d_dec_pack, sizeof(int) * P);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_dec_q, sizeof(int) * P);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_dec_snr, sizeof(double) * P);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_sigma, sizeof(double) * P);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_peak, sizeof(double) * P);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_cand, sizeof(int) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_lists, sizeof(int) * 4 * P);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_counts, sizeof(int) * 4);
    if (e != cudaSuccess) return PC_E_CUDA;
  }
  int hc[8] = {0};
  int nc = 0;
  const int cands[2] = {PC_PACK_SYM, PC_PACK_ASYM2};
  for (int c : cands) {
    hc[nc] = c;
    hc[4 + nc] = p->ms[c].valid ? p->qmode[c] : 0;
    ++nc;
  }
  // predicted_db >= floor  <=>  snr_lin >= 10^((floor - offset)/10)
  const double thr = std::pow(10.0, (snr_floor_db - calib_offset_db) / 10.0);
  // the candidate table changes only with the kernel: uploaded once (synchronously), so the
  // call is stream-ordered device work only and can be captured in a CUDA graph
  if (!p->cand_ok) {
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaMemcpy(p->d_cand, hc, sizeof(hc), cudaMemcpyHostToDevice) != cudaSuccess)
      return PC_E_CUDA;
    p->cand_ok = 1;
  }
  e = pc::launch_block_stats(make_geo(p), s - s_offset, p->d_sigma, p->d_peak, st, B0, nb);
  if (e == cudaSuccess)
    e = pc::launch_adapt_decide(nb, p->d_sigma + B0, p->d_peak + B0, p->k_sigma, p->k_peak, p->d_cand, p->d_cand + 4,
                                nc, thr, p->d_dec_pack + B0, p->d_dec_q + B0, p->d_dec_snr + B0, st);
  if (e == cudaSuccess) e = pc::launch_adapt_lists(nb, p->d_dec_pack, p->d_lists, p->d_counts, st, B0, P);
  if (e != cudaSuccess) return PC_E_CUDA;
  if (out) {
    int* hp = (int*)std::malloc(sizeof(int) * nb * 2);
    double* hs = (double*)std::malloc(sizeof(double) * nb);
    if (!hp || !hs) {
      std::free(hp);
      std::free(hs);
      return PC_E_CUDA;
    }
    e = cudaMemcpyAsync(hp, p->d_dec_pack + B0, sizeof(int) * nb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hp + nb, p->d_dec_q + B0, sizeof(int) * nb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs, p->d_dec_snr + B0, sizeof(double) * nb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
      for (long long w = 0; w < nb; ++w) {
        out[w].packing = hp[w];
        out[w].Q = hp[nb + w];
        out[w].snr_lin = hs[w];
      }
    }
    std::free(hp);
    std::free(hs);
    if (e != cudaSuccess) return PC_E_CUDA;
  }
  p->adapt_ready = 1;   // decisions live on the device: the next execute is stream-ordered
  p->adapt_b0 = B0;
  p->adapt_b1 = B1;
  return PC_OK;
}

int conv_plan_residual(conv_plan* p, double* resid_host, int32_t reset, void* stream) {
  if (!p || !resid_host) return PC_E_CONFIG;
  *resid_host = 0.0;
  if (!p->d_resid) return PC_OK;                     // direct core: exact, no residual
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(resid_host, p->d_resid, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && reset) e = cudaMemsetAsync(p->d_resid, 0, sizeof(double), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return PC_E_CUDA;
  if (reset) reinterpret_cast<volatile int*>(p->h_status)[pc::kStatusMargin] = 0;   // after the sync: no launch pending
  return *resid_host > 0.25 ? PC_W_UNPACK_MARGIN : PC_OK;
}

int conv_execute_profile(conv_plan* p, const double* s, double* r, uint64_t* rec, int32_t* grid_out, void* stream) {
  if (!p || !s || !r || !rec || !grid_out) return PC_E_CONFIG;
  if (cudaSetDevice(p->device) != cudaSuccess) return PC_E_CUDA;
  int grid = 0;
  const int rc = run_exec(p, s, 0, 0, r, 0, 0, 0, p->P, 1, nullptr, (cudaStream_t)stream,
                          reinterpret_cast<unsigned long long*>(rec), &grid);
  *grid_out = grid;
  return rc;
}

int conv_shard_range(int64_t L, int32_t N, int32_t W_block, int32_t mode, int32_t rank, int32_t world,
                     conv_shard* out) {
  if (!out || L < 1 || N < 1 || world < 1 || rank < 0 || rank >= world) return PC_E_CONFIG;
  if (mode == PC_MODE_XCORR && L < N) return PC_E_CONFIG;
  const long long Np = (N % 2) ? N : N + 1;
  const long long W = (long long)W_block - Np - 1;
  if (W < 2 || (W % 2) || W < 2 * Np) return PC_E_CONFIG;
  const long long P = (L + W - 1) / W;
  const long long b0 = P * rank / world, b1 = P * (rank + 1) / world;
  out->block_begin = b0;
  out->block_end = b1;
  if (b0 == b1) {
    out->in_begin = out->in_end = out->out_begin = out->out_end = 0;
    return PC_OK;
  }
  // block w reads [g0(w), g0(w) + W_block) with g0(0) = 0, g0(w) = wW - 2 (reading C7)
  const long long g_first = b0 == 0 ? 0 : b0 * W - 2;
  const long long g_last = (b1 - 1) == 0 ? 0 : (b1 - 1) * W - 2;
  out->in_begin = g_first < L ? g_first : L;
  out->in_end = (g_last + W_block) < L ? (g_last + W_block) : L;
  // block 0 keeps global [0, W+N'-1); block w >= 1 keeps [N'-1+wW, N'-1+(w+1)W) (Eq. (17))
  const long long L_conv = L + N - 1;
  long long o0 = b0 == 0 ? 0 : Np - 1 + b0 * W;
  long long o1 = Np - 1 + b1 * W;
  if (o1 > L_conv) o1 = L_conv;
  if (o0 > L_conv) o0 = L_conv;
  if (mode == PC_MODE_XCORR) {                        // lag j = global output - (N-1), 0..L-N
    const long long lo = N - 1, hi = L;               // valid global outputs [N-1, L)
    o0 = (o0 < lo ? lo : (o0 > hi ? hi : o0)) - lo;
    o1 = (o1 < lo ? lo : (o1 > hi ? hi : o1)) - lo;
  }
  out->out_begin = o0;
  out->out_end = o1;
  return PC_OK;
}

int conv_plan_query(const conv_plan* p, conv_plan_info* info) {
  if (!p || !info) return PC_E_CONFIG;
  std::memset(info, 0, sizeof(*info));
  info->L = p->L;
  info->L_out = p->mode == PC_MODE_XCORR ? p->L - p->N + 1 : p->L + p->N - 1;
  info->P = p->P;
  info->N = p->N;
  info->Np = p->Np;
  info->W_block = p->W_block;
  info->W = p->W;
  info->mode = p->mode;
  info->packing = p->packing;
  info->Q = p->Q;
  info->K_q = p->K_q;
  const int pk = p->packing == PC_PACK_ADAPTIVE ? PC_PACK_ASYM2 : p->packing;
  const ModeState& m = p->ms[pk];
  info->taps = core_taps(p, pk);
  info->kernel_set = p->kernel_set;
  info->R_max = m.R;
  info->bound = m.bound;
  info->bound_ok = m.bound_ok;
  info->eps_b = m.b;
  info->eps = m.eps;
  info->eps_inv = m.eps_inv;
  info->c_k = m.c_k;
  info->k_peak = p->k_peak;
  int mmax = 0, mtyp = 0, best = 0;
  for (int pkk = 0; pkk < 4; ++pkk) {
    core_sizes(p, pkk, &mmax, &mtyp);
    const int xl = mmax + core_taps(p, pkk) - 1;
    if (xl > best) best = xl;
  }
  info->packed_stride = best > p->W_block / 2 ? best : p->W_block / 2;
  core_sizes(p, pk, &mmax, &mtyp);
  int mm = 0;
  for (int pkk = 0; pkk < 4; ++pkk) {
    core_sizes(p, pkk, &mmax, &mtyp);
    if (mmax > mm) mm = mmax;
  }
  info->rbar_stride = mm;
  info->rint_stride = p->W + p->Np - 1;
  for (int i = 0; i < 4; ++i) info->q_mode[i] = p->qmode[i];
  TShape ts;
  info->core_tile = (p->packing != PC_PACK_ADAPTIVE && p->opts.core == PC_CORE_DIRECT && tiled_shape(p, pk, &ts)) ? ts.T : 0;
  info->fft_n = p->fft_N;
  info->core_mma = info->core_tile ? ts.mma : 0;
  info->backend_ok = p->backend_ok;
  info->backend_resid = p->backend_resid;
  info->u_sys_cal = p->u_sys_cal;
  info->device = p->device;
  info->exec_used = p->opts.core == PC_CORE_FFT ? -1 : (uses_tiled(p) ? PC_EXEC_TILED : PC_EXEC_PERBLOCK);
  return PC_OK;
}

int conv_best_match(const double* score, const int64_t* lag, const double* cand, int64_t n, int64_t first_index,
                    double* best, void* stream) {
  if (!best || n < 1 || (!cand && (!score || !lag))) return PC_E_CONFIG;
  return cuda_status(pc::launch_best_match(score, reinterpret_cast<const long long*>(lag), cand, n, first_index, best,
                                           (cudaStream_t)stream));
}

}  // extern "C"
