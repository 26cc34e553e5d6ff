/*
 * packedconv.h -- C ABI of the B200 (sm_100a) packed approximate overlap-save convolution.
 *
 * Implements the hot path of Anam & Andreopoulos, "Throughput Scaling Of Convolution For
 * Error-Tolerant Multimedia Applications" (arXiv 1201.3018; PAPER.md cited P:<line>):
 * per overlap-save block, uniform companding to integers (Eq. (2)), tight packing of
 * several integers into one binary64 word (symmetric Eqs. (4)-(5), or asymmetric
 * Eq. (7)), a direct FP64 convolution of the packed words (Eqs. (8)-(9)),
 * unpacking (Eqs. (11)-(15)), inverse companding (Eq. (16)) and output
 * placement (Eq. (17)).  Readings of the paper where it is ambiguous are listed in
 * DESIGN.md §3 (codes C1..C17).
 *
 * Conventions for every entry point
 *  - Pointers named *_dev are CUDA device pointers; *_host are host pointers (pinned
 *    memory recommended).  The caller owns every buffer passed in; the plan owns its own
 *    device memory (packed kernels, scratch) and frees it in conv_plan_destroy.
 *  - Device buffers of samples must be 16-byte aligned for the TMA bulk-copy path;
 *    misaligned buffers take a slower plain-load path with identical results.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *    execution entry points are stream-ordered and asynchronous unless stated.
 *  - One plan may be used by one stream at a time (it owns scratch state).
 *  - No exception or C++ type crosses this boundary.  Every int-returning call returns a
 *    PC_* status code; conv_status_string() names it.
 *  - There is no CPU fallback: without a CUDA device every call that would launch work
 *    returns PC_E_CUDA.
 */
#ifndef PACKEDCONV_H
#define PACKEDCONV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (SPEC.md S:522 exit codes 0/2/3/4, plus CUDA and margin) ---------- */
enum {
  PC_OK = 0,
  PC_E_CONFIG = 2,          /* invalid geometry / arguments ("config error")        */
  PC_E_BOUND = 3,           /* R_max exceeds the packing's bound under STRICT      */
  PC_E_BACKEND = 4,         /* backend validation failure: the FFT core's
                               worst-case last-digit error, x4, exceeds 0.5 LSB    */
  PC_E_CUDA = 5,            /* a CUDA runtime call failed / no device                     */
  PC_W_UNPACK_MARGIN = 6,   /* warning: digit residual exceeded 0.25 LSB (FFT core)        */
  PC_E_STATE = 7,           /* call order violated (e.g. execute before set_kernel)        */
  PC_E_WATCHDOG = 8         /* a persistent kernel's internal wait timed out (4 s) and the
                               launch abandoned its work: its outputs are invalid          */
};

/* ---- enumerations -------------------------------------------------------------------- */
enum { PC_MODE_CONV = 0, PC_MODE_XCORR = 1 };              /* P:31 Eq.(1); P:189 xcorr   */
enum { PC_PACK_FULL = 0, PC_PACK_SYM = 1, PC_PACK_ASYM2 = 2, PC_PACK_ASYM3 = 3,
       PC_PACK_ADAPTIVE = 4 };                             /* P:59 options (i)-(iii)      */
enum { PC_EPS_PAPER = 0, PC_EPS_RADIX = 1, PC_EPS_POW2 = 2 };   /* Eq.(6); C2; C4         */
enum { PC_RMAX_PAPER = 0, PC_RMAX_L1 = 1 };                /* Eq.(3); C3                  */
enum { PC_BOUND_STRICT = 0, PC_BOUND_WARN = 1 };
enum { PC_CORE_DIRECT = 0, PC_CORE_FFT = 1 };              /* Tier-2 core          */
/* Execution form: FUSED = automatic (the tiled kernel, or the per-block kernel when a
 * block's core is below 1e5 FMAs, where the tiled pipeline's per-job latency dominates);
 * TILED = always the persistent warp-specialized tiled kernel (producer warps compand and
 * pack jobs n+1.. while consumer warps run the core on job n); PERBLOCK = one CTA per
 * block, phases separated by barriers (also the form that serves conv_execute_debug). */
enum { PC_EXEC_FUSED = 0, PC_EXEC_PERBLOCK = 1, PC_EXEC_TILED = 2 };

/* Direct-core variants (conv_opts.core_variant).  AUTO = the FP64 tensor cores (DMMA,
 * mma.sync m8n8k4 f64, tile 16) except symmetric packing with < 768 core taps and asym3 with
 * < 256, which keep the FP64 FMA core (measured). */
enum { PC_CORE_AUTO = 0, PC_CORE_FMA = 1, PC_CORE_DMMA = 2 };
enum { PC_UNPACK_BALANCED = 0, PC_UNPACK_LITERAL = 1 };  /* C6; Eqs.(11)-(15) P:101-115    */

/* Plan options.  conv_opts_default() fills: eps_rule POW2, rmax_rule PAPER, bound_policy
 * STRICT, core DIRECT, exec FUSED, K_q 0 (= Q), device -1 (current), every tuning field 0
 * (automatic), u_sys 3.1193e-11.  Packed results are bit-identical under every tuning
 * setting and full precision is within 1e-12 (tested); the tuning fields exist for tests
 * and measurements. */
typedef struct conv_opts {
  int32_t eps_rule;         /* PC_EPS_*: Eq. (6), C2, C4                            */
  int32_t rmax_rule;        /* PC_RMAX_*: Eq. (3) or the attainable L1 range (C3)   */
  int32_t bound_policy;     /* PC_BOUND_*: refuse (STRICT) or flag (WARN) beyond the bound */
  int32_t core;             /* PC_CORE_DIRECT / PC_CORE_FFT                  */
  int32_t exec;             /* PC_EXEC_*                                                    */
  int32_t K_q;              /* kernel companding range; 0 means K_q = S_q = Q       */
  int32_t device;           /* CUDA device ordinal, -1 = current device                    */
  int32_t raw_staging;      /* raw block TMA-staged in shared memory (per-block kernel; the
                               persistent kernel's producers): 0 auto / 1 on / 2 off         */
  int32_t core_tile;        /* persistent direct core: outputs per thread, 0 auto / 12/14/16 */
  int32_t core_variant;     /* PC_CORE_AUTO / PC_CORE_FMA / PC_CORE_DMMA                    */
  int32_t parts_per_job;    /* persistent direct core: consumer warps per job, 0 auto / 1,2,4 */
  int32_t fft_n;            /* FFT core: complex points N, 0 auto / 1024..8192 (real transform
                               2N); 16384 = the 32768-point real transform of the whole block
                               (full precision, W_block <= 16386, 2-CTA clusters)          */
  int32_t unpack_form;      /* PC_UNPACK_BALANCED, or PC_UNPACK_LITERAL: the literal
                               Eqs. (11)-(15) with the u_sys guard (symmetric packing, direct
                               core; exact for R_max < 89,524, reading C6)                 */
  int32_t pack_alu;         /* persistent DMMA-core producers: 1 = c_s, (c_s c_k)^-1, companding and
                               packing with integer/FP32 ops, bit-identical to the FP64 ops
                               (dyadic eps, exact packed words; measured slower, DESIGN.md
                               §7.3); 0 or 2 = FP64 ops                                     */
  int32_t stage_cap;        /* >= 2: cap on the persistent kernel's stage-ring slots; < 0: the
                               producers claim job m only once consumers hold parts of
                               m + stage_cap; 0 automatic                                   */
  int32_t prepack;          /* 1: compand/pack in a prepack kernel ahead of the persistent
                               launch instead of its producer warps (single-chunk plans,
                               W_block <= 25,600); -P (P >= 1): producer-SM mode (DMMA-core
                               plans; else ignored) -- the persistent launch's first P CTAs (at most half of the SMs)
                               compand and pack jobs into stage images in HBM/L2 and flag
                               them, the other CTAs pack their pipeline fill and bulk-copy the
                               rest (measured slower); 0 in the producer warps */
  int32_t early_fill;       /* 1: a persistent launch's pipeline fill may overlap the tail of
                               the preceding launch on the stream when that launch does not
                               write this launch's input (host-checked against this library's
                               own launches; do not enable when a foreign kernel with its own
                               programmatic-launch trigger may write the input on the same
                               stream); 0 off (default)                                      */
  int32_t validate_trials;  /* FFT core: worst-case operand pairs of the backend validation
                               run by conv_plan_set_kernel, 0 = 128             */
  double u_sys;             /* P:153; used by the literal paper unpack form                */
} conv_opts;

/* Read-only plan description (conv_plan_query). */
typedef struct conv_plan_info {
  int64_t L;                /* input samples                                               */
  int64_t L_out;            /* output samples: L+N-1 (conv) or L-N+1 valid lags (xcorr)   */
  int64_t P;                /* overlap-save blocks, ceil(L/W)                        */
  int32_t N, Np;            /* kernel taps; N' = N or N+1 (odd)                       */
  int32_t W_block, W;       /* block samples; outputs per block W = W_block - N' - 1 */
  int32_t mode, packing;
  int32_t Q, K_q;           /* S_q and K_q                                           */
  int32_t taps;             /* taps of the convolution core: ceil(N'/2) (sym) or N'        */
  int32_t kernel_set;       /* 1 after conv_plan_set_kernel succeeded                      */
  int64_t R_max;            /* Eq. (3) or the L1 rule (C3)                                  */
  int64_t bound;            /* Table 1 bound (PAPER/RADIX eps) or dyadic bound (POW2)      */
  int32_t bound_ok;         /* R_max <= bound                                               */
  int32_t eps_b;            /* eps = 2^-eps_b under POW2, else 0                            */
  double eps, eps_inv;      /* packing coefficient (Eq. (6) / C2 / C4) and its inverse     */
  double c_k, k_peak;       /* kernel companding factor and ||k||_inf                */
  int64_t packed_stride;    /* per-block stride (words) of the debug packed-word dump      */
  int64_t rbar_stride;      /* per-block stride (words) of the debug packed-output dump    */
  int64_t rint_stride;      /* per-block stride of the debug integer dump (= W + N' - 1)   */
  int32_t q_mode[4];        /* ADAPTIVE: max Q per packing under its bound          */
  int32_t core_tile;        /* outputs per thread of the persistent core (12, 14 or 16)      */
  int32_t fft_n;            /* FFT core: complex points N (real transform length 2N), else 0 */
  int32_t core_mma;         /* 1: the tiled core runs on the FP64 tensor cores (DMMA), else 0  */
  int32_t backend_ok;       /* FFT core: 1 if the backend validation passed (4 x resid <= 0.5
                               LSB), 0 if it failed (WARN plans only), -1 not run           */
  double backend_resid;     /* FFT core: worst last-digit residual (LSB) of the validation  */
  double u_sys_cal;         /* FFT core: calibrated u_sys = 4 x that residual x the last
                               digit's unit (absolute); 0 for the exact direct core */
  int32_t device;           /* CUDA device ordinal the plan's memory lives on               */
  int32_t exec_used;        /* the kernel conv_execute runs: PC_EXEC_TILED (persistent direct
                               core), PC_EXEC_PERBLOCK (one CTA per block), -1 the FFT core   */
} conv_plan_info;

/* Per-block decision of conv_adapt_block. */
typedef struct conv_block_decision {
  int32_t packing;          /* PC_PACK_SYM / ASYM2 / ASYM3 / FULL                           */
  int32_t Q;                /* S_q = K_q used for the block (0 for FULL)                    */
  double snr_lin;           /* Eq. (19) linear prediction (inf for FULL)                    */
} conv_block_decision;

/* Block-range shard of one rank: blocks [block_begin, block_end), the
 * input samples it reads [in_begin, in_end) (its range plus the N'+1-sample overlap-save
 * halo, clipped to L) and the outputs it writes [out_begin, out_end) (conv: global output
 * index; xcorr: lag index).  Ranks' output ranges are disjoint and cover all outputs. */
typedef struct conv_shard {
  int64_t block_begin, block_end;
  int64_t in_begin, in_end;
  int64_t out_begin, out_end;
} conv_shard;

typedef struct conv_plan conv_plan;

void conv_opts_default(conv_opts* opts);

/* Create a plan for an L-sample input and an N-tap kernel in W_block-sample overlap-save
 * blocks.  mode: PC_MODE_*; packing: PC_PACK_*; Q = S_q >= 1 (ignored for
 * FULL).  Geometry: N' = N | 1; W = W_block - N' - 1 must be even and >= 2N'.
 * Returns PC_E_CONFIG on invalid arguments, PC_E_CUDA if no device. *out is NULL on error. */
int conv_plan_create(conv_plan** out, int64_t L, int32_t N, int32_t W_block, int32_t mode,
                     int32_t packing, int32_t Q, const conv_opts* opts);

/* Install the N-tap kernel (device pointer, N doubles).  Performs the paper's
 * Initialization on the device: pad to N' (C13), reverse for xcorr,
 * ||k||_inf, c_k = K_q/||k||_inf, k~ = [[c_k k]] (Eq. (2)), R_max (Eq. (3) / C3), eps
 * (Eq. (6) / C2 / C4), bound check (Table 1), packed kernel (Eq. (5) under C1, or
 * k~ for asymmetric, Eq. (8)).  Synchronizes `stream` (one-time plan cost).
 * Returns PC_E_BOUND under STRICT when R_max exceeds the bound (kernel not installed).
 * FFT-core plans of a packed mode then validate the backend: the plan's own
 * FFT kernel runs on validate_trials worst-case operand windows (every sample +-1, random signs,
 * so every packed digit is +-S_q; the installed kernel, companded to +-K_q) and its last-digit
 * residual monitor gives the worst deviation d (LSB) from the exact integers; u_sys_cal =
 * 4 d x the digit unit.  If 4 d > 0.5 LSB the regime (N', R_max, fft_n) is unsafe: PC_E_BACKEND
 * under STRICT (kernel not installed), recorded (backend_ok = 0) under WARN. */
int conv_plan_set_kernel(conv_plan* plan, const double* k_dev, void* stream);

/* Run the whole hot path on an L-sample device input, writing L_out device outputs:
 * r_out (Eq. (17)) for conv, or the valid cross-correlation lags c[j] = sum_n s[j+n] q[n],
 * 0 <= j <= L-N, for xcorr (C17).  s_dev and r_dev must not overlap.
 * Returns PC_OK, or (FFT core) PC_W_UNPACK_MARGIN when a completed launch of this plan saw a
 * last-digit residual above 0.25 LSB (the kernels raise a flag in host-mapped memory; it stays
 * raised until conv_plan_residual(reset = 1); the launch of this call is enqueued either way),
 * or PC_E_WATCHDOG when a completed launch of this plan abandoned its work (sticky likewise). */
int conv_execute(conv_plan* plan, const double* s_dev, double* r_dev, void* stream);

/* Same as conv_execute restricted to blocks [block_begin, block_end) -- the unit of
 * multi-GPU sharding.  s_dev holds global samples [s_offset, ...) (the
 * block range plus its N'+1-sample halo); r_dev receives global outputs [r_offset, ...).
 * Returns as conv_execute. */
int conv_execute_blocks(conv_plan* plan, const double* s_dev, int64_t s_offset, double* r_dev,
                        int64_t r_offset, int64_t block_begin, int64_t block_end, void* stream);

/* n_signals independent signals of L samples (row stride s_stride doubles) through the
 * same plan; outputs row stride r_stride doubles.  One launch over all blocks.  Returns as
 * conv_execute. */
int conv_execute_batch(conv_plan* plan, const double* s_dev, int64_t n_signals, int64_t s_stride,
                       double* r_dev, int64_t r_stride, void* stream);

/* End-to-end through host memory: copies s_host (L doubles) to the device, runs
 * conv_execute, copies L_out doubles back to r_host, and synchronizes `stream`.  Plans of
 * >= 128 blocks pipeline 15 block ranges over plan-owned copy streams (H2D of range
 * c+1, core of range c and D2H of range c-1 overlap); pinned host buffers are needed for
 * the copies to overlap.  Results are identical to conv_execute; returns as conv_execute (it
 * synchronizes, so the flags include this call's own launches). */
int conv_execute_host(conv_plan* plan, const double* s_host, double* r_host, void* stream);

/* conv_execute_host restricted to blocks [block_begin, block_end) (a rank's shard, SURVEY
 * §8(e)): s_host holds global samples [s_offset, ...) -- at least the shard's input range
 * conv_shard_range reports -- and r_host receives global outputs (conv) / lags (xcorr)
 * [r_offset, ...) of the shard's output range.  Same pipeline and return codes; adaptive plans
 * need the whole range (PC_E_CONFIG otherwise). */
int conv_execute_host_blocks(conv_plan* plan, const double* s_host, int64_t s_offset, double* r_host,
                             int64_t r_offset, int64_t block_begin, int64_t block_end, void* stream);

/* Database winner of the music-matching score (reading C17): over n candidates --
 * candidate i = (score_dev[i], lag_dev[i], first_index + i), or, if cand_dev is non-NULL, the
 * rows {score, lag, index} of cand_dev (n x 3 doubles, e.g. the all-gathered winners of every
 * rank) -- the largest score, ties to the smallest index.  Writes {score, lag, index} (3 doubles,
 * lag and index exact integers) to best_dev.  Device pointers, stream-ordered, one launch (no
 * plan needed). */
int conv_best_match(const double* score_dev, const int64_t* lag_dev, const double* cand_dev, int64_t n,
                    int64_t first_index, double* best_dev, void* stream);

/* Many (signal, kernel) pairs, one kernel each -- the MPEG-7 stereo-descriptor regime of §IV.C
 * (SURVEY NEXT-3): block b of one channel cross-correlated with block b of the other.
 * conv_plan_set_kernels companding each of the n kernels (q_dev: n rows of N doubles, row
 * stride q_stride; device) on its own (reading C5): per-kernel c_k, k~ and core taps,
 * with one R_max = N' S_q K_q for all (PAPER rule required for packed modes, so eps is
 * common; CONFIG otherwise).  It also performs conv_plan_set_kernel with row 0.  The plan's
 * mode, packing, Q and geometry apply to every pair.  Plan-owned memory: about
 * n (2 N' + K + 35) doubles.  Returns BOUND (STRICT) as conv_plan_set_kernel. */
int conv_plan_set_kernels(conv_plan* plan, const double* q_dev, int64_t n, int64_t q_stride, void* stream);

/* xcorr plans after conv_plan_set_kernels(n' >= n): pair i = signal row i of x_dev (L
 * doubles at x_dev + i*x_stride; device) with kernel i: score[i] = max over valid lags j of
 * c_i[j] = sum_n x_i[j+n] q_i[n], lag[i] = the lowest j attaining it (C17) (device arrays).
 * Always the tiled kernel with the fused score epilogue (tap chunks per stage).  Callers wanting
 * all 2N-1 lags of equal-length blocks pad x with N-1 zeros on each side.  STATE if n exceeds
 * the kernels set. */
int conv_xcorr_pairs(conv_plan* plan, const double* x_dev, int64_t n, int64_t x_stride, double* score,
                     int64_t* lag, void* stream);

/* xcorr plans only: per signal, the maximum of c[j] over valid lags and its argmax
 * (lowest j on ties; C17) -- the music-matching score.  On the tiled kernel the
 * score is fused into the epilogue (warp partials + a per-signal reduction; plan-owned
 * partials of n_signals x jobs x parts entries, no lag buffer); otherwise the lags go
 * through a plan-owned scratch of <= 2 GiB and are scanned. */
int conv_xcorr_max(conv_plan* plan, const double* db_dev, int64_t n_signals, int64_t s_stride,
                   double* score_dev, int64_t* lag_dev, void* stream);

/* Parity/debug run of the whole path that also dumps, per block w (row w of each array,
 * strides from conv_plan_info; any pointer may be NULL): packed words as the core sees
 * them (Eq. (4)/(7)), packed outputs (Eq. (9)/(8)), unpacked integers of the kept range
 * (Eqs. (12)-(15)), and c_s (Eq. (2)).  r_dev as in conv_execute (may be NULL).
 * max_residual_host (may be NULL): the largest distance of a decoded last digit from its
 * integer over all blocks (LSB; exactly 0 under the dyadic eps, C4); synchronizes `stream`
 * when non-NULL. */
int conv_execute_debug(conv_plan* plan, const double* s_dev, double* r_dev, double* packed_dev,
                       double* rbar_dev, int64_t* rint_dev, double* c_s_dev, double* max_residual_host,
                       void* stream);

/* SNR-constrained adaptation for ADAPTIVE plans: per block, the first
 * packing of {SYM, ASYM2} whose Eq. (19) prediction at its maximum Q under its bound
 * meets snr_floor_db - calib_offset_db, else FULL.  Decisions are installed for the next
 * conv_execute on the same input and copied to out_host (P entries) if non-NULL.
 * Synchronizes `stream` only when out_host is non-NULL (otherwise stream-ordered). */
int conv_adapt_block(conv_plan* plan, const double* s_dev, double snr_floor_db,
                     double calib_offset_db, conv_block_decision* out_host, void* stream);

/* conv_adapt_block on a rank's blocks [block_begin, block_end): s_dev holds global
 * samples [s_offset, ...) (the shard's input range); out_host receives block_end - block_begin
 * decisions.  The next conv_execute_blocks over exactly this range runs one persistent launch per
 * packing; executes of blocks outside the decided range return PC_E_STATE. */
int conv_adapt_blocks(conv_plan* plan, const double* s_dev, int64_t s_offset, int64_t block_begin,
                      int64_t block_end, double snr_floor_db, double calib_offset_db,
                      conv_block_decision* out_host, void* stream);

/* Single-point calibration of the Eq. (19) SNR model (Fig. 5: "calibrated via a single
 * measurement at the coarsest quantization (S_q = K_q = 8)"; reading C18).  Runs the plan's
 * geometry (L, N, W_block, mode, options) on s_dev (L samples, device) with kernel k_dev (N taps,
 * device) twice -- packed at S_q = K_q = Q (the plan's packing if SYM/ASYM3, else ASYM2; at Q = 8
 * every exact packing gives the same integers) and full precision -- and returns the measured
 * SNR over all outputs, the model's prediction sum_b (sigma_b sigma_k)^2 / sum_b D_b (per-block
 * Eq. (19) terms, P:222 statistics) and offset_db = measured - model, the calib_offset_db for
 * conv_adapt_block.  Temporary plans and buffers (2 L_out doubles) are created and freed inside;
 * synchronizes `stream`.  PC_E_CONFIG on invalid arguments, PC_E_BOUND if Q exceeds the packing's
 * bound under STRICT. */
int conv_snr_calibrate(conv_plan* plan, const double* s_dev, const double* k_dev, int32_t Q,
                       double* offset_db, double* measured_db, double* model_db, void* stream);

/* Diagnostics: conv_execute that records, when the tiled kernel or the FFT core runs, a
 * timeline into cta_records_dev (uint64, at least 24*148*32 + 148*16*16*4 + 148*4*16*4 entries,
 * zeroed by the caller): tiled kernel -- per CTA c {SM id, start / end %globaltimer (ns), jobs}
 * at [4c..4c+3], consumer-warp-0 cycle totals at [4*148*32 + 4c ..], per consumer warp and part
 * {job sequence, ready, core done, stored} and per producer warp and job {sequence, turn,
 * claimed, published} (layout in pc_tiled.cu, read by tools/tiled_timeline.py); FFT core -- per
 * job {SM id, start, peak, packed, forward, product, inverse, end} at [8 job ..] for the first
 * 4096 jobs (tools/fft_timeline.py).  *grid_out receives the CTA count (0 for the per-block
 * kernel, which records nothing). */
int conv_execute_profile(conv_plan* plan, const double* s_dev, double* r_dev, uint64_t* cta_records_dev,
                         int32_t* grid_out, void* stream);

/* Host-only (no device needed): the shard of `rank` among `world` ranks for a plan of the
 * same (L, N, W_block, mode): blocks [P*rank/world, P*(rank+1)/world).  PC_E_CONFIG on
 * invalid geometry. */
int conv_shard_range(int64_t L, int32_t N, int32_t W_block, int32_t mode, int32_t rank, int32_t world,
                     conv_shard* out);

/* FFT core (opts.core = PC_CORE_FFT): the packed words are convolved through a
 * hand-written FP64 FFT, so the packed outputs are approximate and exact integers are
 * recovered only while the error stays below half an LSB.  The kernels keep the largest
 * last-digit residual (in LSB) seen since the last reset; this call copies it to
 * *resid_host (synchronizes `stream`), resets it (and the margin flag conv_execute reports)
 * if `reset`, and returns PC_W_UNPACK_MARGIN if it exceeded 0.25 LSB (SURVEY §5 unpack-residual
 * monitor).  Direct-core plans are exact: *resid_host = 0, PC_OK. */
int conv_plan_residual(conv_plan* plan, double* resid_host, int32_t reset, void* stream);

int conv_plan_query(const conv_plan* plan, conv_plan_info* info);
void conv_plan_destroy(conv_plan* plan);
const char* conv_status_string(int status);

#ifdef __cplusplus
}
#endif
#endif /* PACKEDCONV_H */
